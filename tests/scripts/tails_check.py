"""Parity with tile lists cut to a short prefix (run by tests/test_gpu_list_tails.py with
SPLAT_LIST_PREFIX set): blocks walk the rest of their lists from the supertile lists (StagePipe
tails), so the forward images, importance report and gradients must equal the oracle's exactly as
with complete lists, and the bit-exact list getter must still see the full lists."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
from helpers import assert_bitwise, assert_grads_close, rel_err  # noqa: E402
from oracle_lib import OracleLib  # noqa: E402
from paper_2411_12788_b200 import scenes  # noqa: E402
from paper_2411_12788_b200 import rasterizer as R  # noqa: E402
from paper_2411_12788_b200.capi import RasterConfig  # noqa: E402

oracle = OracleLib()
cases = [(scenes.make_gaussians(20_000, seed=0), scenes.config0_camera()),
         (scenes.make_gaussians(60_000, seed=3), scenes.ring_camera(5, 64, width=400, height=300))]
for k, (s, cam) in enumerate(cases):
    for rep in (False, True):
        got = R.render(s, cam, report=rep)
        out = got[0] if rep else got
        want = oracle.render(s, cam, report=rep)
        for key in ("color", "alpha", "depth", "transmittance", "max_contributor"):
            assert_bitwise(getattr(out, key), want[key], f"case {k} report={rep} {key}")
        if rep:
            assert_bitwise(got[1].max_weight, want["max_weight"], f"case {k} max_weight")
            assert_bitwise(got[1].max_pixel_count, want["max_pixel_count"], f"case {k} max_pixel_count")
            assert rel_err(got[1].importance, want["importance"], floor_frac=1e-6) <= 1e-4
    target = oracle.render(scenes.perturbed(s), cam, report=False)["color"]
    _, d_color = oracle.l1_loss(want["color"], target)
    assert_grads_close(R.render_backward(s, cam, RasterConfig(), d_color), oracle.render_backward(s, cam, d_color),
                       what=f"case {k} tails")
    # the getter completes the lists; a backward after it uses the complete lists
    R.render(s, cam)
    fw = R.forward_debug()
    to = oracle.tiles(s, cam)
    assert fw["n_pairs"] == to["n_pairs"]
    assert_bitwise(fw["ranges"], to["ranges"], f"case {k} ranges")
    assert_bitwise(fw["gaussian"], to["gaussian"], f"case {k} per-tile lists")
print("tails check ok")
