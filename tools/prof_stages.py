"""Measurement helper (not product code): time the CountGauss stages separately on c2-sized
inputs, for ncu runs and quick A/B checks.

  python tools/prof_stages.py [--fuse 0|1] [--reps N] [--what apply|gauss|sketch]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1606_05732_b200 as cg  # noqa: E402
from paper_1606_05732_b200 import bench_data  # noqa: E402
from paper_1606_05732_b200._lib import CGX_MEM_DEVICE, check, lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fuse", type=int, default=1)
    ap.add_argument("--fuse_mode", type=int, default=2)
    ap.add_argument("--rows_per_task", type=int, default=1024)
    ap.add_argument("--grid_waves", type=int, default=1)
    ap.add_argument("--ws_gw", type=int, default=0)
    ap.add_argument("--explicit_g", type=int, default=0)
    ap.add_argument("--async_stages", type=int, default=0)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--what", default="apply")
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--d", type=int, default=32)
    ap.add_argument("--B", type=int, default=65536)
    ap.add_argument("--m", type=int, default=64)
    a = ap.parse_args()
    ctx = cg.context(0)
    ctx.set_option("fuse", a.fuse)
    ctx.set_option("fuse_mode", a.fuse_mode)
    ctx.set_option("rows_per_task", a.rows_per_task)
    ctx.set_option("grid_waves", a.grid_waves)
    ctx.set_option("ws_gw", a.ws_gw)
    ctx.set_option("async_stages", a.async_stages)
    t = cg.countgauss_new(a.m, a.B, a.n, cg.SeededRng(12345))
    x = bench_data.dense_normal(a.n, a.d, seed=7)
    if a.dtype == "f64":
        x = x.double()
    if a.explicit_g:  # G read from memory instead of generated (isolates the generation cost)
        gmat = torch.empty((a.B, a.m), dtype=torch.float64, device="cuda")
        check(lib.cgx_fill_gaussian(ctx.h, t._xf.h, gmat.data_ptr(), CGX_MEM_DEVICE, C.c_void_p(1)))
        check(lib.cgx_xform_set_gaussian_explicit(ctx.h, t._xf.h, a.m, gmat.data_ptr(), CGX_MEM_DEVICE))
    z = torch.empty((a.d, a.m), dtype=torch.float64, device="cuda").t()
    g = torch.empty((a.B, a.m), dtype=torch.float64, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ctx.profile(True)
    for rep in range(a.reps):
        ev[0].record()
        if a.what == "apply":
            cg.api.countgauss_apply_into(t, x, z)
        elif a.what == "gauss":
            check(lib.cgx_fill_gaussian(ctx.h, t._xf.h, g.data_ptr(), CGX_MEM_DEVICE, C.c_void_p(1)))
        elif a.what == "sketch":
            cg.countsketch_apply(t, x)
        ev[1].record()
        torch.cuda.synchronize()
        print(f"{a.what} fuse={a.fuse} rep {rep}: {ev[0].elapsed_time(ev[1]):.3f} ms")
    for st in (0, 1):
        ms, n = ctx.profile_read(st)
        if n:
            print(f"  stage {st}: {ms / n:.3f} ms/launch over {n} (includes warm-up)")


if __name__ == "__main__":
    main()
