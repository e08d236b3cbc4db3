"""Measurement helper (not product code): what the peer-memory combine (CGX_COMBINE_P2P,
group.cu) costs on ONE GPU.  A group of P ranks that all sit on device 0 runs the c2 / c4 apply
on device-resident row shards; the ranks' kernels share the GPU (they never wait on each other:
streams ordered by events), so the wall time of one call is about the single-context step plus
what the mode adds -- segmented stores from the gather, the slot sums, P host-thread phases --
and NOT a multi-GPU number.  Printed beside: the single-context apply on the whole X."""
import ctypes as C
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1606_05732_b200 as cg  # noqa: E402
from paper_1606_05732_b200 import bench_data  # noqa: E402
from paper_1606_05732_b200._lib import CGX_COMBINE_P2P, CGX_F32, CGX_MEM_DEVICE, CGX_ROW_MAJOR, lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n, d, B, m = {"c2": (1 << 24, 32, 65536, 64), "c4": (1 << 25, 128, 131072, 32)}[cfg]
ctx = cg.context()
seed = 12345
x = bench_data.dense_normal(n, d, seed=7)
t1 = cg.countgauss_new(m, B, n, cg.SeededRng(seed), ctx=ctx)
z1 = torch.empty((d, m), dtype=torch.float64, device="cuda").t()


def wall(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - a) * 1e3)
    return statistics.median(ts)


print(f"{cfg}: single context, wall per apply: {wall(lambda: cg.api.countgauss_apply_into(t1, x, z1)):.3f} ms")
t_seed = cg.SeededRng(seed).next_u64()
for P in (1, 2, 4, 8):
    g = C.c_void_p()
    devs = (C.c_int * P)(*([0] * P))
    assert lib.cgx_group_init(P, devs, C.byref(g)) == 0, lib.cgx_last_error()
    t = C.c_void_p()
    assert lib.cgx_group_countgauss_new(g, t_seed, m, B, n, C.byref(t)) == 0, lib.cgx_last_error()
    shards = []
    for p in range(P):
        r0, rows = C.c_int64(), C.c_int64()
        lib.cgx_gxform_shard(t, p, C.byref(r0), C.byref(rows))
        shards.append(x[r0.value:r0.value + rows.value])
    xs = (C.c_void_p * P)(*[s.data_ptr() for s in shards])
    zd = [torch.empty((d, m), dtype=torch.float64, device="cuda") for _ in range(P)]
    zs = (C.c_void_p * P)(*[z.data_ptr() for z in zd])

    def call():
        rc = lib.cgx_group_countgauss_apply_dense(g, t, xs, CGX_F32, CGX_ROW_MAJOR, d, n, d, CGX_MEM_DEVICE, zs,
                                                  CGX_MEM_DEVICE, CGX_COMBINE_P2P)
        assert rc == 0, lib.cgx_last_error()

    ms = wall(call)
    f, c = C.c_int64(), C.c_int64()
    lib.cgx_group_stats(g, C.byref(f), C.byref(c))
    err = (torch.linalg.norm(zd[0].t() - z1) / torch.linalg.norm(z1)).item()
    print(f"  P={P}: {ms:.3f} ms wall per group apply (all ranks on one GPU), fused/copied sketches {f.value}/{c.value}, "
          f"Z vs single context {err:.1e}")
    lib.cgx_gxform_free(t)
    lib.cgx_group_free(g)
