"""Measurement helper (not product code): time stage 2 (Z = G . S.X) alone, with G
generated in chunks (seeded) or read from memory (explicit), at a config's shape.

  python tools/prof_gemm.py [--config c5] [--reps 5] [--explicit 0|1]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1606_05732_b200 as cg  # noqa: E402
from paper_1606_05732_b200._lib import CGX_MEM_DEVICE, CGX_ROW_MAJOR, check, lib  # noqa: E402

SHAPES = {"c3": (262144, 128, 256), "c5": (1 << 20, 256, 512), "c4": (131072, 32, 128), "c2": (65536, 64, 32)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--explicit", type=int, default=0)
    ap.add_argument("--opt", action="append", default=[], metavar="KEY=VALUE")
    ap.add_argument("--shape", default="", help="B,m,d instead of a config")
    ap.add_argument("--check", type=int, default=0, help="1: relative Frobenius error vs cuBLAS fp64")
    a = ap.parse_args()
    B, m, d = [int(v) for v in a.shape.split(",")] if a.shape else SHAPES[a.config]
    ctx = cg.context(0)
    for kv in a.opt:
        k, v = kv.split("=", 1)
        ctx.set_option(k, int(v))
    t = cg.countgauss_new(m, B, 10, cg.SeededRng(12345))
    if a.explicit:
        g = torch.empty((B, m), dtype=torch.float64, device="cuda")
        check(lib.cgx_fill_gaussian(ctx.h, t._xf.h, g.data_ptr(), CGX_MEM_DEVICE, C.c_void_p(1)))
        check(lib.cgx_xform_set_gaussian_explicit(ctx.h, t._xf.h, m, g.data_ptr(), CGX_MEM_DEVICE))
    sx = torch.randn((B, d), dtype=torch.float64, device="cuda")
    z = torch.empty((d, m), dtype=torch.float64, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    flops = 2.0 * m * B * d
    for rep in range(a.reps):
        ev[0].record()
        check(lib.cgx_gauss_gemm(ctx.h, t._xf.h, sx.data_ptr(), CGX_ROW_MAJOR, d, CGX_MEM_DEVICE, z.data_ptr(),
                                 CGX_MEM_DEVICE, C.c_void_p(1)))
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1])
        print(f"{a.config} {B},{m},{d} {a.opt} explicit={a.explicit} rep {rep}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s")
    if a.check:
        g = torch.empty((B, m), dtype=torch.float64, device="cuda")
        check(lib.cgx_fill_gaussian(ctx.h, t._xf.h, g.data_ptr(), CGX_MEM_DEVICE, C.c_void_p(1)))
        torch.cuda.synchronize()
        zr = sx.t() @ g
        err = ((z - zr).norm() / zr.norm()).item()
        print(f"check {B},{m},{d} {a.opt}: rel Frobenius err vs cuBLAS fp64 {err:.3e}  max abs {(z - zr).abs().max().item():.3e}")
        if err > 1e-10:  # per 64-column tile of Z (rows of the (d, m) tensor) and 128-row tile
            for c0 in range(0, d, 64):
                for r0 in range(0, m, 128):
                    zt, rt = z[c0:c0 + 64, r0:r0 + 128], zr[c0:c0 + 64, r0:r0 + 128]
                    print(f"  tile cols {c0}.. rows {r0}..: {((zt - rt).norm() / rt.norm()).item():.3e}")


if __name__ == "__main__":
    main()
