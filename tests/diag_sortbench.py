import sys, ctypes as C, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2411_12788_b200.rasterizer import Context
ctx = Context.default(); lib = ctx.lib
def bench(n, bits, keys):
    k = torch.from_numpy(keys.view(np.int32)).cuda(); v = torch.arange(n, dtype=torch.int32, device='cuda')
    ka, va = torch.empty_like(k), torch.empty_like(v); alt = C.c_int()
    for _ in range(3): lib.splat_sort_pairs(ctx.h, k.data_ptr(), v.data_ptr(), ka.data_ptr(), va.data_ptr(), n, 0, bits, C.byref(alt))
    torch.cuda.synchronize()
    lib.splat_profile_enable(ctx.h, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): lib.splat_sort_pairs(ctx.h, k.data_ptr(), v.data_ptr(), ka.data_ptr(), va.data_ptr(), n, 0, bits, C.byref(alt))
    e1.record(); torch.cuda.synchronize()
    names = C.create_string_buffer(4096); tot = (C.c_double*64)(); cnt=(C.c_int64*64)(); nk=C.c_int()
    lib.splat_profile_read(ctx.h, names, 4096, tot, cnt, 64, C.byref(nk)); lib.splat_profile_enable(ctx.h, 0)
    nm = names.value.decode().split('\n')[:nk.value]
    print(f"n={n} bits={bits}: {e0.elapsed_time(e1)/20*1000:.1f} us/sort;", {a: round(tot[i]/20*1000,1) for i,a in enumerate(nm)})
rng = np.random.default_rng(0)
bench(1_000_000, 32, rng.uniform(2.3, 3.8, 1_000_000).astype(np.float32).view(np.uint32))
bench(3_400_000, 9, rng.integers(0, 260, 3_400_000).astype(np.uint32))
bench(1_000_000, 24, rng.integers(0, 1<<24, 1_000_000).astype(np.uint32))
