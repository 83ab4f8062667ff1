"""The C-ABI boundary: libsplat_b200.so loads without a GPU and exports every entry point declared
in include/splat_b200.h; the ctypes mirror matches the header's struct layouts."""
import ctypes as C
import re
from pathlib import Path

from paper_2411_12788_b200 import capi

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    text = (ROOT / "include" / "splat_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void|const char\*)\s+(splat_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(str(capi.LIB_PATH))
    names = declared_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, f"missing exports: {missing}"
    assert set(names) == set(capi.EXPORTED_SYMBOLS), "ctypes mirror out of sync with the header"


def test_load_library_declares_prototypes():
    lib = capi.load_library()
    assert lib.splat_render.restype is C.c_int


def test_struct_layouts():
    # sizes implied by include/splat_b200.h (x86-64 SysV)
    assert C.sizeof(capi.Camera) == 4 * (2 + 4 + 9 + 3 + 2)
    assert C.sizeof(capi.RasterConfig) == 8 + 5 * 8
    assert C.sizeof(capi.Gaussians) == 5 * 8 + 8
    assert C.sizeof(capi.AdamConfig) == 5 * 8 + 8 + 6 * 8
    assert C.sizeof(capi.ParamGrads) == 7 * 8


def test_ctx_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        return
    lib = capi.load_library()
    h = C.c_void_p()
    assert lib.splat_ctx_create(0, C.byref(h)) != 0
