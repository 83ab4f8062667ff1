"""The reference's random draws (include/splat_rng.h: std::mt19937 / mt19937_64 and libstdc++'s
uniform_real / uniform_int / normal distributions, restated in C) and the §8f functions that
consume them — importance_sample (simplify.cpp:36-92) and vanilla_clone_split +
apply_densify_plan's Progressive branch (densify.cpp:132-163, 182-191) — pinned bit for bit
against the reference's own code compiled in place (oracle/_ref, mode B)."""
import numpy as np
import pytest

from paper_2411_12788_b200 import scenes


def test_normal_draws_pinned(oracle, ref):
    for seed in (0, 1, 5489, 2**31 + 7):
        a, b = oracle.rng_normal_f32(seed, 5001), ref.rng_normal_f32(seed, 5001)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), seed


def test_uniform_f64_mt32_pinned(oracle, ref):
    for seed in (0, 3, 1234):
        assert np.array_equal(oracle.rng_uniform_f64_32(seed, 3000), ref.rng_uniform_f64_32(seed, 3000))


def test_mixed_64_pinned(oracle, ref):
    rng = np.random.default_rng(0)
    n = 4000
    kinds = (rng.random(n) < 0.5).astype(np.int32)
    lo = rng.integers(0, 1000, n).astype(np.int32)
    hi = lo + rng.integers(0, 2**30, n).astype(np.int32)
    hi[::7] = lo[::7]  # single-value ranges still consume a draw
    for seed in (0, 99, 2**40 + 3):
        assert np.array_equal(oracle.rng_mixed_64(seed, kinds, lo, hi), ref.rng_mixed_64(seed, kinds, lo, hi))


def test_fisher_yates_pinned(oracle, ref):
    for seed, pool, take in ((0, 1, 1), (7, 1000, 1000), (11, 100_000, 2500), (3, 12, 5)):
        assert np.array_equal(oracle.rng_fisher_yates(seed, pool, take), ref.rng_fisher_yates(seed, pool, take))


@pytest.mark.parametrize("case", ["mixed", "all_positive", "all_zero", "deficit", "ties"])
def test_importance_sample_pinned(oracle, ref, case):
    rng = np.random.default_rng(5)
    n = 3000
    s = scenes.make_gaussians(n, seed=2)
    imp = rng.gamma(0.5, 2.0, n)
    if case == "mixed":
        imp[rng.random(n) < 0.3] = 0.0
        targets = (1, 17, 1500, n)
    elif case == "all_positive":
        targets = (1, 999, n)
    elif case == "all_zero":
        imp[:] = 0.0
        targets = (1, 40, n)
    elif case == "deficit":  # fewer positive weights than the target: uniform filler from the zeros
        imp[:] = 0.0
        imp[rng.choice(n, 200, replace=False)] = rng.random(200) + 0.1
        imp[5] = -1.0  # non-positive weights are filler too
        targets = (150, 200, 201, 2000, n)
    else:
        imp = np.where(np.arange(n) % 3 == 0, 1.0, 2.0)
        targets = (10, 1000)
    for t in targets:
        for seed in (0, 42):
            got = oracle.importance_sample(imp, t, seed)
            want = ref.importance_sample(imp, t, seed, s=s)
            assert got.size == t and np.array_equal(got, want), (case, t, seed)
    with pytest.raises(RuntimeError):
        oracle.importance_sample(imp, 0, 0)
    with pytest.raises(RuntimeError):
        oracle.importance_sample(imp, n + 1, 0)


def _assert_set_equal(a, b, what):
    for k in ("centers", "log_scales", "rotations", "opacity_logits", "sh"):
        x, y = getattr(a, k), getattr(b, k)
        assert x.shape == y.shape and np.array_equal(x.view(np.uint32), y.view(np.uint32)), (what, k)


@pytest.mark.parametrize("seed", [0, 7])
def test_vanilla_clone_split_pinned(oracle, ref, seed):
    rng = np.random.default_rng(seed)
    n = 4000
    s = scenes.make_gaussians(n, seed=seed + 1)
    cnt = rng.integers(0, 5, n).astype(np.int32)
    acc = (rng.random(n) * 4e-4 * np.maximum(cnt, 1)).astype(np.float32)
    for thr, sthr, ext in ((2e-4, 0.01, 3.3), (0.0, 0.02, 1.0), (1.0, 0.01, 3.3)):
        got, gms, gc, gs = oracle.vanilla_clone_split(s, acc, cnt, thr, sthr, ext, seed)
        want, wms, wc, ws = ref.vanilla_clone_split(s, acc, cnt, thr, sthr, ext, seed)
        assert (gc, gs) == (wc, ws)
        assert np.array_equal(gms, wms)
        _assert_set_equal(got, want, (thr, sthr))
        if thr < 1.0:
            assert gc > 0 and gs > 0
