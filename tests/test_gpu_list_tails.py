"""Tile lists materialised only up to a prefix (binning.cu bin_emit, StagePipe tails): with the
prefix cut to 64 / 256 entries every block walks into the supertile-list tails, in the forward
(training and importance), in the backward's re-culling paths (the one-pixel-per-thread backward
re-culls every tile list) and after the bit-exact getter completed the lists; results must be the
oracle's as with complete lists.  Separate processes: the prefix is fixed at context creation."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("env", [{"SPLAT_LIST_PREFIX": "64"}, {"SPLAT_LIST_PREFIX": "256", "SPLAT_BWD_PX2": "0"},
                                 {"SPLAT_LIST_PREFIX": "100", "SPLAT_BLEND_PERSISTENT": "0"}])
def test_parity_with_list_tails(env):
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "scripts" / "tails_check.py")], capture_output=True,
                       text=True, timeout=550, env=dict(os.environ, **env), cwd=str(ROOT))
    assert r.returncode == 0 and "tails check ok" in r.stdout, (r.stdout + r.stderr)[-4000:]
