"""Measurement helper (not product code): stage-2 (Z = G.SX) timing with G regenerated
in-kernel vs G read from memory (explicit), on random S.X of a given shape.

  python tools/prof_gemm.py --B 262144 --m 128 --d 256
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1606_05732_b200 as cg  # noqa: E402
from paper_1606_05732_b200._lib import CGX_MEM_DEVICE, CGX_ROW_MAJOR, check, lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=262144)
    ap.add_argument("--m", type=int, default=128)
    ap.add_argument("--d", type=int, default=256)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    ctx = cg.context(0)
    t = cg.countgauss_new(a.m, a.B, 10, cg.SeededRng(1))
    sx = torch.randn(a.B, a.d, dtype=torch.float64, device="cuda")
    z = torch.empty(a.d, a.m, dtype=torch.float64, device="cuda")
    s1 = C.c_void_p(1)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def run(label):
        for rep in range(a.reps):
            ev[0].record()
            check(lib.cgx_gauss_gemm(ctx.h, t._xf.h, sx.data_ptr(), CGX_ROW_MAJOR, a.d, CGX_MEM_DEVICE,
                                     z.data_ptr(), CGX_MEM_DEVICE, s1))
            ev[1].record()
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1])
        flops = 2.0 * a.m * a.B * a.d
        print(f"{label}: {ms:.3f} ms  {flops / ms / 1e9:.2f} TFLOP/s (last rep)")

    run("regenerated G")
    g = torch.empty(a.B, a.m, dtype=torch.float64, device="cuda")  # col-major m x B
    ev[0].record()
    check(lib.cgx_fill_gaussian(ctx.h, t._xf.h, g.data_ptr(), CGX_MEM_DEVICE, s1))
    ev[1].record()
    torch.cuda.synchronize()
    print(f"fill_gaussian alone: {ev[0].elapsed_time(ev[1]):.3f} ms for {a.m * a.B} normals")
    check(lib.cgx_xform_set_gaussian_explicit(ctx.h, t._xf.h, a.m, g.data_ptr(), CGX_MEM_DEVICE))
    run("explicit G")


if __name__ == "__main__":
    main()
