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


@pytest.mark.gpu
def test_cpp_adapter_timing_config1():
    """The drop-in at BASELINE config 1 scale (1 M Gaussians, 1237 x 822) through the adapter, by
    value and with a resident set: the measured cost of switching the reference's call sites."""
    if not EXE.exists():
        pytest.skip("adapter_check not built (needs /root/reference at build time)")
    r = subprocess.run([str(EXE), "--time", "1000000"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("ADAPTER_TIME")]
    print("\n".join(lines))
    assert len(lines) == 2
