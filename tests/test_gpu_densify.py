"""§8f on device (paper_2411_12788_b200/densify.py, csrc/densify.cu) vs the CPU oracle and the
reference build: quantiles, build_masks, identify_critical (all criteria), aggressive_clone +
apply_densify_plan, importance_prune, GaussianSet::select and OptimState::remap.  Selections,
masks, cloned parameters and moment sources are bit-exact for identical inputs."""
import numpy as np
import pytest
import torch

from helpers import assert_bitwise
from paper_2411_12788_b200 import densify as D
from paper_2411_12788_b200 import scenes
from paper_2411_12788_b200.rasterizer import DeviceGaussians, OptimState

pytestmark = pytest.mark.gpu
CRITERIA = {"random": 0, "opacity": 1, "accum-weight": 2, "max-weight": 3}


@pytest.fixture(scope="module")
def scene():
    s = scenes.make_gaussians(6000, seed=21, log_scale_mean=np.log(0.03))
    cams = [scenes.ring_camera(k, 6, width=160, height=112) for k in range(6)]
    return s, cams


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_quantile_threshold_matches_oracle(oracle):
    rng = np.random.default_rng(1)
    for n in (1, 5, 4096, 300_001):
        v = rng.random(n).astype(np.float32)
        sel = (rng.random(n) < 0.4).astype(np.uint8)
        sel[0] = 1
        for q in (0.01, 0.5, 0.99):
            assert D.quantile_threshold(_cuda(v), q) == oracle.quantile_threshold(v, q)
            assert D.quantile_threshold(_cuda(v), q, _cuda(sel)) == oracle.quantile_threshold(v, q, sel)
            d = v.astype(np.float64) * 7.0 - 1.0  # negatives too
            assert D.quantile_threshold(_cuda(d), q) == oracle.quantile_threshold(d, q)
    with pytest.raises(Exception):
        D.quantile_threshold(_cuda(np.zeros(4, np.float32)), 0.5, _cuda(np.zeros(4, np.uint8)))
    with pytest.raises(Exception):
        D.quantile_threshold(_cuda(np.ones(4, np.float32)), 0.0)


def test_float_keep_q_1001_candidates(oracle, ref):
    """keep_q is narrowed to float before the quantile (visibility.cpp:23, densify.cpp:63): 1001
    positives / candidates at keep_q = 0.99 take order statistic 9, not 10."""
    s = scenes.grid_gaussians(1001, seed=5)
    s.opacity_logits[:11] = np.linspace(-5.0, -2.5, 11, dtype=np.float32)
    s.opacity_logits[11:] = np.abs(s.opacity_logits[11:]) + 0.5
    cam = scenes.fov_camera(256, 256, 60.0, (0.0, 0.0, -3.0))
    want = ref.build_masks(s, [cam], 0.99)[0]
    assert_bitwise(D.build_masks(s, [cam], 0.99)[0].cpu().numpy(), want, "mask, 1001 positives")
    wc, wn = ref.identify_critical_views(s, [cam], CRITERIA["max-weight"], 0.99)
    gc, gn = D.identify_critical(s, [cam], "max-weight", 0.99)
    assert gn == wn
    assert_bitwise(gc.cpu().numpy(), wc, "critical, 1001 candidates")


def test_build_masks(oracle, ref, scene):
    s, cams = scene
    # the mask kernel on identical importances is bit-exact
    for k, cam in enumerate(cams[:3]):
        imp = oracle.render(s, cam)["importance"]
        got = torch.zeros(s.n, dtype=torch.uint8, device="cuda")
        from paper_2411_12788_b200.rasterizer import Context
        ctx = Context.default()
        ctx.bind_stream()
        ctx.check(ctx.lib.splat_visibility_mask(ctx.h, _cuda(imp).data_ptr(), s.n, 0.5, got.data_ptr()))
        assert_bitwise(got.cpu().numpy(), oracle.visibility_mask(imp, 0.5), f"view {k} mask kernel")
    # end to end: GPU importance sums are float atomics, so entries within rounding of tau may flip
    got = D.build_masks(s, cams, 0.5).cpu().numpy()
    want = ref.build_masks(s, cams, 0.5)
    diff = (got != want).sum()
    assert diff <= max(2, 1e-3 * want.size), f"{diff} mask entries differ"


@pytest.mark.parametrize("criterion", list(CRITERIA))
def test_identify_critical_selection_bit_exact(oracle, ref, scene, criterion):
    """Same per-view statistics in -> identical CriticalSelection out."""
    s, cams = scene
    best, cnt, summed = oracle.view_statistics(s, cams)
    rnd = ref.random_scores(77, s.n)
    want, want_n = oracle.identify_critical(s, best, cnt, summed, CRITERIA[criterion], 0.6, random=rnd)
    got, got_n = D.identify_critical(s, cams, criterion, 0.6, random_scores=_cuda(rnd),
                                     stats=(_cuda(best), _cuda(cnt), _cuda(summed)))
    assert got_n == want_n
    assert_bitwise(got.cpu().numpy(), want, f"{criterion} critical flags")


def test_identify_critical_end_to_end_maxweight(ref, scene):
    """MaxWeight from the GPU's own view statistics (max weights and argmax counts are exact)
    equals the reference's identify_critical, also with visibility masks."""
    s, cams = scene
    want, want_n = ref.identify_critical_views(s, cams, CRITERIA["max-weight"], 0.5)
    got, got_n = D.identify_critical(s, cams, "max-weight", 0.5)
    assert got_n == want_n
    assert_bitwise(got.cpu().numpy(), want, "max-weight critical flags")
    masks = ref.build_masks(s, cams, 0.7)
    want, want_n = ref.identify_critical_views(s, cams, CRITERIA["max-weight"], 0.5, masks=masks)
    got, got_n = D.identify_critical(s, cams, "max-weight", 0.5, masks=_cuda(masks))
    assert got_n == want_n
    assert_bitwise(got.cpu().numpy(), want, "masked max-weight critical flags")


def test_aggressive_clone_bit_exact(oracle, scene):
    s, _ = scene
    s2 = s.select(np.arange(s.n))
    s2.opacity_logits[:5] = [-30.0, 30.0, 0.0, -16.2, 16.2]
    crit = (np.random.default_rng(5).random(s.n) < 0.25).astype(np.uint8)
    crit[:5] = 1
    want, wms = oracle.aggressive_clone(s2, crit)
    grown, ms = D.aggressive_clone(DeviceGaussians.from_host(s2), _cuda(crit))
    assert grown.n == want[0].shape[0]
    assert_bitwise(ms.cpu().numpy(), wms, "moment_source")
    h = grown.to_host()
    for a, b, name in zip((h.centers, h.log_scales, h.rotations, h.opacity_logits, h.sh), want,
                          ("centers", "log_scales", "rotations", "opacity_logits", "sh")):
        assert_bitwise(a, b, f"cloned {name}")


def test_importance_prune_select_and_remap(oracle, scene):
    s, cams = scene
    _, _, summed = oracle.view_statistics(s, cams)
    ds = DeviceGaussians.from_host(s)
    kept_set, kept = D.importance_prune(ds, _cuda(summed), 0.4)
    want = oracle.importance_prune(summed, 0.4)
    assert_bitwise(kept.cpu().numpy(), want, "kept indices")
    assert_bitwise(kept_set.to_host().sh, s.sh[want], "selected rows")
    # OptimState::remap: moments follow their rows, -1 rows are zero
    opt = OptimState(n=s.n)
    opt.m.copy_(torch.arange(opt.m.numel(), dtype=torch.float32, device="cuda"))
    opt.v.copy_(-torch.arange(opt.v.numel(), dtype=torch.float32, device="cuda"))
    src = np.concatenate([want, [-1, 3]]).astype(np.int32)
    m_old = opt.m.cpu().numpy()
    D.remap(opt, _cuda(src))
    m_new = opt.m.cpu().numpy()
    n_old, n_new = s.n, src.size
    o_old = o_new = 0
    for w in (3, 3, 4, 1, 48):
        old = m_old[o_old:o_old + w * n_old].reshape(n_old, w)
        new = m_new[o_new:o_new + w * n_new].reshape(n_new, w)
        exp = np.where((src >= 0)[:, None], old[np.maximum(src, 0)], 0.0)
        assert_bitwise(new, exp.astype(np.float32), f"remapped moments width {w}")
        o_old += w * n_old
        o_new += w * n_new


def test_rng_draws_match_reference(ref):
    """splat_rng (std::mt19937 restated) draws the reference's Random scores and Fisher-Yates picks."""
    for seed in (0, 17):
        got = D.random_scores(D.Rng(seed), 5000).cpu().numpy()
        assert np.array_equal(got, ref.random_scores(seed, 5000))
    r = D.Rng(3)
    a = D.random_scores(r, 700).cpu().numpy()
    st = r.state()
    b = D.random_scores(r, 900).cpu().numpy()
    r2 = D.Rng(1)
    r2.set_state(st)
    assert np.array_equal(D.random_scores(r2, 900).cpu().numpy(), b)
    assert np.array_equal(np.concatenate([a, b]), ref.random_scores(3, 1600))
    from paper_2411_12788_b200.rasterizer import Context
    ctx = Context.default()
    out = torch.empty(2500, dtype=torch.int32, device="cuda")
    ctx.bind_stream()
    r9 = D.Rng(9)
    ctx.check(ctx.lib.splat_pool_sample(ctx.h, r9.h, 100_000, 2500, out.data_ptr()))
    assert np.array_equal(out.cpu().numpy(), ref.fisher_yates(9, 100_000, 2500))


def test_identify_critical_random_with_library_draws(ref, scene):
    s, cams = scene
    want, want_n = ref.identify_critical_views(s, cams, CRITERIA["random"], 0.6, seed=1234)
    rnd = D.random_scores(D.Rng(1234), s.n)
    got, got_n = D.identify_critical(s, cams, "random", 0.6, random_scores=rnd)
    assert got_n == want_n
    assert_bitwise(got.cpu().numpy(), want, "random-criterion selection")


@pytest.mark.parametrize("case", ["mixed", "all_positive", "all_zero", "deficit", "ties"])
def test_importance_sample_matches_reference(ref, case):
    rng = np.random.default_rng(5)
    n = 30_000
    s = scenes.make_gaussians(n, seed=2)
    imp = rng.gamma(0.5, 2.0, n)
    targets = (1, 999, n)
    if case == "mixed":
        imp[rng.random(n) < 0.3] = 0.0
        targets = (1, 17, 15_000, n)
    elif case == "all_zero":
        imp[:] = 0.0
    elif case == "deficit":
        imp[:] = 0.0
        imp[rng.choice(n, 2000, replace=False)] = rng.random(2000) + 0.1
        imp[5] = -1.0
        targets = (1500, 2000, 2001, 20_000, n)
    elif case == "ties":
        imp = np.where(np.arange(n) % 3 == 0, 1.0, 2.0)
        targets = (10, 10_000)
    ds = DeviceGaussians.from_host(s)
    for t in targets:
        for seed in (0, 2**40 + 1):
            kept_set, kept = D.importance_sample(ds, _cuda(imp), t, seed)
            want = ref.importance_sample(imp, t, seed, s=s)
            assert_bitwise(kept.cpu().numpy(), want, f"{case} target {t} seed {seed}")
            assert kept_set.n == t
    with pytest.raises(Exception):
        D.importance_sample(ds, _cuda(imp), 0, 0)
    with pytest.raises(Exception):
        D.importance_sample(ds, _cuda(imp), n + 1, 0)


@pytest.mark.parametrize("seed", [0, 7])
def test_vanilla_clone_split_matches_reference(ref, seed):
    rng = np.random.default_rng(seed)
    n = 40_000
    s = scenes.make_gaussians(n, seed=seed + 1)
    cnt = rng.integers(0, 5, n).astype(np.int32)
    acc = (rng.random(n) * 4e-4 * np.maximum(cnt, 1)).astype(np.float32)
    ds = DeviceGaussians.from_host(s)
    for thr, sthr, ext in ((2e-4, 0.01, 3.3), (0.0, 0.02, 1.0), (1.0, 0.01, 3.3)):
        out, ms, nc, ns = D.vanilla_clone_split(ds, _cuda(acc), _cuda(cnt), thr, sthr, ext, D.Rng(seed))
        want, wms, wc, ws = ref.vanilla_clone_split(s, acc, cnt, thr, sthr, ext, seed)
        assert (nc, ns) == (wc, ws)
        assert_bitwise(ms.cpu().numpy(), wms, "moment source")
        got = out.to_host()
        for k in ("centers", "log_scales", "rotations", "opacity_logits", "sh"):
            assert_bitwise(getattr(got, k), getattr(want, k), f"{k} thr {thr}")
