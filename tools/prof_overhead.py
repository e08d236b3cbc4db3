"""Measurement helper (not product code): host-side cost per countgauss_apply call
(enqueue rate with no synchronisation) against the GPU time per call, at small n where
fixed costs dominate.

  python tools/prof_overhead.py [--n 65536] [--calls 2000] [--fuse 1]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1606_05732_b200 as cg  # noqa: E402
from paper_1606_05732_b200 import bench_data  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 16)
    ap.add_argument("--d", type=int, default=32)
    ap.add_argument("--B", type=int, default=65536)
    ap.add_argument("--m", type=int, default=64)
    ap.add_argument("--calls", type=int, default=2000)
    ap.add_argument("--fuse", type=int, default=1)
    a = ap.parse_args()
    ctx = cg.context(0)
    ctx.set_option("fuse", a.fuse)
    t = cg.countgauss_new(a.m, a.B, a.n, cg.SeededRng(12345))
    x = bench_data.dense_normal(a.n, a.d, seed=7)
    z = torch.empty((a.d, a.m), dtype=torch.float64, device="cuda").t()
    for _ in range(20):
        cg.api.countgauss_apply_into(t, x, z)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    t0 = time.perf_counter()
    ev[0].record()
    for _ in range(a.calls):
        cg.api.countgauss_apply_into(t, x, z)
    ev[1].record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"n={a.n} fuse={a.fuse}: host enqueue {1e6 * (t1 - t0) / a.calls:.1f} us/call, "
          f"GPU {1e3 * ev[0].elapsed_time(ev[1]) / a.calls:.1f} us/call, wall {1e6 * (t2 - t0) / a.calls:.1f} us/call, "
          f"launches/call {ctx.launches / (a.calls + 20):.1f}")


if __name__ == "__main__":
    main()
