"""The C++ drop-in (include/splat_b200_adapter.hpp) in the reference's own types: the check binary
oracle/_ref/adapter_check (built with the reference present, see oracle/Makefile) runs the
reference's CPU functions and the GPU drop-ins side by side."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "oracle" / "_ref" / "adapter_check"


@pytest.mark.gpu
def test_cpp_adapter_matches_reference():
    if not EXE.exists():
        pytest.skip("adapter_check not built (needs /root/reference at build time)")
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED" in r.stdout
