"""§8f (densification / simplification) oracle pinned to the reference build, on CPU.

The C restatement (oracle/splat_oracle.c) of quantile_threshold, build_masks, identify_critical,
aggressive_clone + apply_densify_plan and importance_prune against the reference's own functions
compiled in place (oracle/_ref, mode B: shared splat_expf / splat_logf): bit-exact selections,
masks, cloned parameters and moment sources."""
import numpy as np
import pytest

from paper_2411_12788_b200 import scenes
from paper_2411_12788_b200.capi import RasterConfig

CRITERIA = {"random": 0, "opacity": 1, "accum-weight": 2, "max-weight": 3}


@pytest.fixture(scope="module")
def scene():
    s = scenes.make_gaussians(3000, seed=11, log_scale_mean=np.log(0.03))
    cams = [scenes.ring_camera(k, 5, width=96, height=64) for k in range(5)]
    return s, cams


def _np_quantile(v, keep_q):  # quantile.hpp:16-28 restated with numpy, for the pin
    v = np.sort(np.asarray(v))
    h = (1.0 - keep_q) * (v.size - 1)
    lo = int(np.floor(h))
    hi = min(lo + 1, v.size - 1)
    return v.dtype.type(float(v[lo]) + (h - lo) * (float(v[hi]) - float(v[lo])))


def test_quantile_threshold(oracle):
    rng = np.random.default_rng(0)
    for n in (1, 2, 7, 1000):
        v = rng.random(n).astype(np.float32)
        for q in (0.01, 0.5, 0.99):
            tau, cnt = oracle.quantile_threshold(v, q)
            assert cnt == n and np.float32(tau) == _np_quantile(v, q)
            sel = (np.arange(n) % 3 == 0).astype(np.uint8)
            tau, cnt = oracle.quantile_threshold(v, q, sel)
            assert cnt == sel.sum() and np.float32(tau) == _np_quantile(v[sel.astype(bool)], q)
            d = v.astype(np.float64) * 3.0
            assert oracle.quantile_threshold(d, q)[0] == _np_quantile(d, q)
    with pytest.raises(RuntimeError):
        oracle.quantile_threshold(np.zeros(0, np.float32), 0.5)
    with pytest.raises(RuntimeError):
        oracle.quantile_threshold(np.ones(4, np.float32), 1.0)


def test_build_masks_pinned(oracle, ref, scene):
    s, cams = scene
    for q in (0.1, 0.5, 0.99):
        want = ref.build_masks(s, cams, q)
        for k, cam in enumerate(cams):
            imp = oracle.render(s, cam)["importance"]
            assert np.array_equal(oracle.visibility_mask(imp, q), want[k]), (q, k)
    # edge rules: nothing positive -> all zero; all positives equal -> every positive kept
    assert not oracle.visibility_mask(np.zeros(10, np.float32), 0.5).any()
    eq = np.array([0, 2, 2, 0, 2], np.float32)
    assert np.array_equal(oracle.visibility_mask(eq, 0.5), (eq > 0).astype(np.uint8))


@pytest.mark.parametrize("criterion", list(CRITERIA))
@pytest.mark.parametrize("keep_q", [0.05, 0.5, 0.95])
def test_identify_critical_pinned(oracle, ref, scene, criterion, keep_q):
    s, cams = scene
    c = CRITERIA[criterion]
    want, want_n = ref.identify_critical_views(s, cams, c, keep_q, seed=1234)
    best, cnt, summed = oracle.view_statistics(s, cams)
    rnd = ref.random_scores(1234, s.n)
    got, got_n = oracle.identify_critical(s, best, cnt, summed, c, keep_q, random=rnd)
    assert got_n == want_n and np.array_equal(got, want)
    assert want_n > 0 and want.sum() == want_n


def test_identify_critical_with_visibility_masks(oracle, ref, scene):
    s, cams = scene
    masks = ref.build_masks(s, cams, 0.7)
    want, want_n = ref.identify_critical_views(s, cams, CRITERIA["max-weight"], 0.5, masks=masks)
    best, cnt, summed = oracle.view_statistics(s, cams, masks=masks)
    got, got_n = oracle.identify_critical(s, best, cnt, summed, CRITERIA["max-weight"], 0.5)
    assert got_n == want_n and np.array_equal(got, want)


def test_float_keep_q_1001_candidates(oracle, ref):
    """visibility.cpp:23 / densify.cpp:63 narrow keep_q to float before the quantile: with 1001
    positives and keep_q = 0.99 the lower order statistic is 9 (float) rather than 10 (double)."""
    s = scenes.grid_gaussians(1001, seed=5)
    # eleven faint Gaussians ~25 % apart at the bottom of the order, so the two candidate order
    # statistics (9 vs 10) interpolate to visibly different thresholds
    s.opacity_logits[:11] = np.linspace(-5.0, -2.5, 11, dtype=np.float32)
    s.opacity_logits[11:] = np.abs(s.opacity_logits[11:]) + 0.5
    cam = scenes.fov_camera(256, 256, 60.0, (0.0, 0.0, -3.0))
    imp = oracle.render(s, cam)["importance"]
    assert int((imp > 0).sum()) == 1001
    want = ref.build_masks(s, [cam], 0.99)[0]
    got = oracle.visibility_mask(imp, 0.99)
    assert np.array_equal(got, want)
    v = np.sort(imp[imp > 0])
    assert want.sum() == int((imp > _np_quantile(v, float(np.float32(0.99)))).sum())
    assert want.sum() != int((imp > _np_quantile(v, 0.99)).sum())  # the narrowing matters here
    wc, wn = ref.identify_critical_views(s, [cam], CRITERIA["max-weight"], 0.99)
    best, cnt, summed = oracle.view_statistics(s, [cam])
    assert int((cnt > 0).sum()) == 1001
    gc, gn = oracle.identify_critical(s, best, cnt, summed, CRITERIA["max-weight"], 0.99)
    assert gn == wn and np.array_equal(gc, wc)


def test_aggressive_clone_pinned(oracle, ref, scene):
    s, _ = scene
    rng = np.random.default_rng(3)
    critical = (rng.random(s.n) < 0.3).astype(np.uint8)
    s2 = s.select(np.arange(s.n))
    s2.opacity_logits[:5] = [-30.0, 30.0, 0.0, -16.2, 16.2]  # tiny / saturated / mid opacities
    critical[:5] = 1
    got, gms = oracle.aggressive_clone(s2, critical)
    want, wms = ref.aggressive_clone(s2, critical)
    assert np.array_equal(gms, wms)
    for a, b, name in zip(got, want, ("centers", "log_scales", "rotations", "opacity_logits", "sh")):
        assert a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32)), name
    assert got[0].shape[0] > s.n  # clones were appended


def test_importance_prune_pinned(oracle, ref, scene):
    s, cams = scene
    _, _, summed = oracle.view_statistics(s, cams)
    for q in (0.1, 0.5, 0.9):
        assert np.array_equal(oracle.importance_prune(summed, q), ref.importance_prune(summed, q, s=s))
    flat = np.full(s.n, 2.5)  # keep-all edge rule
    assert np.array_equal(oracle.importance_prune(flat, 0.5), np.arange(s.n))
