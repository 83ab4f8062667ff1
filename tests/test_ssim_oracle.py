"""SSIM and the photometric loss (loss.cpp:10-153): the C restatement
pinned bitwise to the reference's own ssim<float> / photometric_loss<float> (mode B), on rendered
images and edge shapes (images narrower than the 11-tap window, one channel)."""
import numpy as np
import pytest

from paper_2411_12788_b200 import scenes


def _pair(oracle, w=64, h=48):
    s = scenes.make_gaussians(2000, seed=2)
    cam = scenes.ring_camera(1, 8, width=w, height=h)
    a = oracle.render(s, cam)["color"]
    b = oracle.render(scenes.perturbed(s), cam)["color"]
    return a, b


def _bits(x):
    return np.asarray(x, np.float32).view(np.uint32)


def test_ssim_pinned(oracle, ref):
    a, b = _pair(oracle)
    v, g = oracle.ssim(a, b)
    rv, rg = ref.ssim(a, b)
    assert _bits(v) == _bits(rv) and np.array_equal(_bits(g), _bits(rg))
    assert 0.0 < v < 1.0 and np.abs(g).max() > 0
    # identical images: SSIM 1 (within float rounding) and a ~zero gradient
    v1, g1 = oracle.ssim(a, a)
    assert abs(v1 - 1.0) < 1e-5 and np.abs(g1).max() < 1e-6


@pytest.mark.parametrize("w,h,ch", [(7, 5, 3), (1, 30, 1), (40, 3, 2), (11, 11, 3)])
def test_ssim_small_shapes_pinned(oracle, ref, w, h, ch):
    rng = np.random.default_rng(w * 100 + h)
    a = rng.random((h, w, ch)).astype(np.float32)
    b = rng.random((h, w, ch)).astype(np.float32)
    v, g = oracle.ssim(a, b)
    rv, rg = ref.ssim(a, b)
    assert _bits(v) == _bits(rv) and np.array_equal(_bits(g), _bits(rg))


@pytest.mark.parametrize("lam", [0.0, 0.2, 1.0])
def test_photometric_loss_pinned(oracle, ref, lam):
    a, b = _pair(oracle)
    v, g = oracle.photometric_loss(a, b, lam)
    rv, rg = ref.photometric_loss(a, b, lam)
    assert _bits(v) == _bits(rv) and np.array_equal(_bits(g), _bits(rg))


def _ssim64(a, b):
    """loss.cpp's mean SSIM restated in float64 with scipy (zero-padded separable 11-tap blur)."""
    from scipy.ndimage import correlate1d
    d = np.arange(11) - 5.0
    k = np.exp(-d * d / 4.5)
    k /= k.sum()

    def blur(x):
        return correlate1d(correlate1d(x, k, axis=1, mode="constant"), k, axis=0, mode="constant")
    c1, c2 = 1e-4, 9e-4
    ma, mb = blur(a), blur(b)
    va, vb, cov = blur(a * a) - ma * ma, blur(b * b) - mb * mb, blur(a * b) - ma * mb
    s = ((2 * ma * mb + c1) * (2 * cov + c2)) / ((ma * ma + mb * mb + c1) * (va + vb + c2))
    return s.mean()


def test_ssim_gradient_finite_difference(oracle):
    """The analytic gradient (loss.cpp:105-131) against central differences of a float64 SSIM."""
    a, b = _pair(oracle, 24, 20)
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    v, g = oracle.ssim(a, b)
    assert abs(v - _ssim64(a64, b64)) < 1e-5
    rng = np.random.default_rng(0)
    for idx in rng.choice(a.size, 16, replace=False):
        e = np.zeros(a.size)
        e[idx] = 1e-4
        e = e.reshape(a.shape)
        fd = (_ssim64(a64 + e, b64) - _ssim64(a64 - e, b64)) / 2e-4
        gi = float(g.reshape(-1)[idx])
        assert abs(fd - gi) <= 1e-3 * np.abs(g).max() + 1e-3 * abs(fd), (idx, fd, gi)
