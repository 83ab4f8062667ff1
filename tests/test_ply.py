"""PLY checkpoints (paper_2411_12788_b200/ply.py) against the reference's own write_ply / read_ply
(ply_io.cpp, compiled in oracle/_ref and driven through the oracle/_ref/ply_ref helper process):
byte-identical files, identical sets after reading each other's files, the reference's parse
errors."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2411_12788_b200 import ply, scenes

HELPER = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "ply_ref"


def _flat(s):
    return np.concatenate([np.asarray(a, np.float32).reshape(-1) for a in
                           (s.centers, s.log_scales, s.rotations, s.opacity_logits, s.sh)])


@pytest.mark.skipif(not HELPER.exists(), reason="oracle/_ref/ply_ref not built")
def test_ply_byte_identical_and_cross_readable(tmp_path):
    s = scenes.make_gaussians(777, seed=4)
    ours, theirs, raw = tmp_path / "ours.ply", tmp_path / "ref.ply", tmp_path / "a.bin"
    ply.write_ply(ours, s)
    _flat(s).tofile(raw)
    subprocess.run([str(HELPER), "write", str(raw), str(s.n), str(theirs)], check=True)
    assert ours.read_bytes() == theirs.read_bytes()
    back = ply.read_ply(theirs)
    assert np.array_equal(_flat(back).view(np.uint32), _flat(s).view(np.uint32))
    subprocess.run([str(HELPER), "read", str(ours), str(raw)], check=True)
    assert np.array_equal(np.fromfile(raw, np.float32).view(np.uint32), _flat(s).view(np.uint32))


def test_ply_errors(tmp_path):
    p = tmp_path / "bad.ply"
    p.write_bytes(b"plx\n")
    with pytest.raises(RuntimeError, match="missing 'ply' magic"):
        ply.read_ply(p)
    p.write_bytes(b"ply\nformat ascii 1.0\nend_header\n")
    with pytest.raises(RuntimeError, match="unsupported format"):
        ply.read_ply(p)
    s = scenes.make_gaussians(3, seed=1)
    ply.write_ply(p, s)
    p.write_bytes(p.read_bytes()[:-10])
    with pytest.raises(RuntimeError, match="truncated vertex data"):
        ply.read_ply(p)
    with pytest.raises(RuntimeError, match="cannot open"):
        ply.read_ply(tmp_path / "missing.ply")
