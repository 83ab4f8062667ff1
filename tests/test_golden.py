"""The C restatement oracle and the CUDA path against fixtures produced by the REFERENCE's own code
(tests/golden/make_golden.py, oracle/_ref mode B).  CPU part: bitwise oracle == reference."""
import numpy as np
import pytest

from helpers import GOLDEN, assert_bitwise, assert_grads_close, load_golden

GRADS = ("d_centers", "d_log_scales", "d_rotations", "d_opacity_logits", "d_sh", "grad2d_accum", "grad2d_count")


@pytest.mark.parametrize("path", GOLDEN, ids=[p.stem for p in GOLDEN])
def test_oracle_matches_reference_fixture(oracle, path):
    s, cam, cfg, bg, mask, d_color, d = load_golden(path)
    r = oracle.render(s, cam, cfg, mask=mask, bg=bg)
    for k in ("color", "alpha", "depth", "transmittance", "max_contributor", "importance", "max_weight",
              "max_pixel_count"):
        assert_bitwise(r[k], d[f"B_{k}"], k)
    t = oracle.tiles(s, cam, cfg, mask=mask)
    assert_bitwise(t["ranges"], d["B_ranges"], "ranges")
    assert_bitwise(t["gaussian"], d["B_lists"], "lists")
    p = oracle.project(s, cam, cfg, mask=mask)
    assert_bitwise(p["order"], d["B_order"], "order")
    g = oracle.render_backward(s, cam, d_color, cfg, mask=mask, bg=bg)
    for k in GRADS:
        assert_bitwise(g[k], d[f"B_{k}"], k)


@pytest.mark.parametrize("path", GOLDEN, ids=[p.stem for p in GOLDEN])
def test_mode_a_vs_mode_b_images_close(path):
    """glibc expf (the reference as shipped) vs splat_expf: images within the forward tolerance
    except where a gate flips at an exp ulp (counted, must be rare)."""
    _, _, _, _, _, _, d = load_golden(path)
    diff = np.abs(d["A_color"].astype(np.float64) - d["B_color"])
    flips = int((diff > 1e-5).sum())
    assert flips <= max(3, diff.size // 2000), f"{flips} colour values differ by > 1e-5"


@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLDEN, ids=[p.stem for p in GOLDEN])
def test_cuda_matches_reference_fixture(path):
    from paper_2411_12788_b200 import rasterizer as R
    s, cam, cfg, bg, mask, d_color, d = load_golden(path)
    out, rep = R.render(s, cam, cfg, mask=mask, background=bg, report=True)
    for k in ("color", "alpha", "depth", "transmittance", "max_contributor"):
        assert_bitwise(getattr(out, k), d[f"B_{k}"], k)
    assert_bitwise(rep.max_weight, d["B_max_weight"], "max_weight")
    assert_bitwise(rep.max_pixel_count, d["B_max_pixel_count"], "max_pixel_count")
    fw = R.forward_debug()
    assert_bitwise(fw["ranges"], d["B_ranges"], "ranges")
    assert_bitwise(fw["gaussian"], d["B_lists"], "lists")
    g = R.render_backward(s, cam, cfg, d_color, mask=mask, background=bg)
    assert_grads_close(g, {k: d[f"B_{k}"] for k in GRADS}, what=path.stem)
