"""The shared exponential (include/splat_expf.h): accuracy, and splat_expf_core / splat_expf_gate ==
splat_expf on the ranges the blend kernels use them for."""
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
SRC = r'''
#include "splat_expf.h"
#include <stdio.h>
#include <stdlib.h>
int main(void) {
    long n = 0, over1ulp = 0, core_diff = 0, gate_diff = 0;
    /* every 61st float in [-103.9, 88.7]; exhaustive for core on every 7th float in [-87.3, 0] */
    for (uint32_t u = 0; u < 0xFFFFFFFFu - 61; u += 61) {
        float x; memcpy(&x, &u, 4);
        if (!(x > -103.9f && x < 88.7f)) continue;
        ++n;
        float a = splat_expf(x);
        float r = (float)exp((double)x);
        int32_t ia, ir; memcpy(&ia, &a, 4); memcpy(&ir, &r, 4);
        if (r != 0 && abs(ia - ir) > 1) ++over1ulp;
    }
    for (uint32_t u = 0x80000000u; u <= 0xC2AE9999u; u += 7) {
        float x; memcpy(&x, &u, 4);
        if (!(x >= -87.3f)) continue;
        float a = splat_expf(x), b = splat_expf_core(x);
        if (memcmp(&a, &b, 4)) ++core_diff;
        if (x >= -86.6f) {
            float c = splat_expf_gate(x);
            if (memcmp(&a, &c, 4)) ++gate_diff;
        }
    }
    printf("%ld %ld %ld %ld\n", n, over1ulp, core_diff, gate_diff);
    return 0;
}
'''


def test_splat_expf_accuracy_and_core(tmp_path):
    c = tmp_path / "t.c"
    c.write_text(SRC)
    exe = tmp_path / "t"
    subprocess.run(["gcc", "-O2", "-mfma", "-ffp-contract=off", f"-I{ROOT / 'include'}", str(c), "-o", str(exe), "-lm"],
                   check=True)
    n, over, core, gate = (int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                                          check=True).stdout.split())
    assert n > 10_000_000
    assert over == 0, f"{over} samples off by more than 1 ulp"
    assert core == 0, f"splat_expf_core differs from splat_expf on {core} samples"
    assert gate == 0, f"splat_expf_gate differs from splat_expf on {gate} samples"


def test_oracle_exp_modes():
    import sys
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import OracleLib
    b, a = OracleLib("oracle", "B"), OracleLib("oracle", "A")
    xs = np.linspace(-20, 5, 20001, dtype=np.float32)
    gb = np.array([b.exp(float(x)) for x in xs], np.float32)
    ga = np.array([a.exp(float(x)) for x in xs], np.float32)
    assert np.all(np.abs(gb.view(np.int32) - ga.view(np.int32)) <= 1)


LOG_SRC = r'''
#include "splat_expf.h"
#include <stdio.h>
#include <stdlib.h>
int main(void) {
    long n = 0, over1 = 0; double worst = 0;
    for (uint32_t u = 1; u < 0x7f800000u; u += 97) {   /* every 97th positive finite float */
        float x; memcpy(&x, &u, 4);
        ++n;
        const float a = splat_logf(x);
        const double r = log((double)x);
        const float rf = (float)r;
        const double ulp = fabs((double)nextafterf(rf, INFINITY) - (double)rf);
        const double e = fabs((double)a - r) / ulp;
        if (e > worst) worst = e;
        if (e > 1.0) ++over1;
    }
    printf("%ld %ld %.4f %a %a %a\n", n, over1, worst, splat_logf(1.0f), splat_logf(0.0f), splat_logf(-1.0f));
    return 0;
}
'''


def test_splat_logf_accuracy(tmp_path):
    """splat_logf (the log shared by densify.cu and the mode-B oracle): < 1 ulp everywhere."""
    c = tmp_path / "l.c"
    c.write_text(LOG_SRC)
    exe = tmp_path / "l"
    subprocess.run(["gcc", "-O2", "-mfma", "-ffp-contract=off", f"-I{ROOT / 'include'}", str(c), "-o", str(exe), "-lm"],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    n, over, worst = int(out[0]), int(out[1]), float(out[2])
    assert n > 20_000_000 and over == 0 and worst < 1.0, out
    assert out[3] == "0x0p+0" and out[4] == "-inf" and out[5] in ("nan", "-nan"), out
