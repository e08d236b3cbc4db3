"""Measurement helper (not product code): the per-rank GPU work of a strong-scaled c2/c4
step on P ranks, run on ONE GPU rank by rank (no collective is emulated -- ranks never wait
on each other here; the NCCL volumes are printed beside): for each combine mode,
  z : apply on rank p's n/P rows (sketch + full stage 2)       + all-reduce of Z
  g : sketch of n/P rows -> partial S.X, rows [m p/P, ...) of G.(S.X) + all-reduce of S.X
  sx: sketch of n/P rows, split-K stage 2 on B/P buckets       + reduce-scatter of S.X
CUDA events around each rank's work (median of 20), max over ranks = the step's compute."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1606_05732_b200 as cg  # noqa: E402
from paper_1606_05732_b200 import bench_data  # noqa: E402
from paper_1606_05732_b200.distributed import bucket_range, g_row_range, shard_range  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n, d, B, m = {"c2": (1 << 24, 32, 65536, 64), "c4": (1 << 25, 128, 131072, 32)}[cfg]
ctx = cg.context()
t_seed = cg.SeededRng(12345).next_u64()
x = bench_data.dense_normal(n, d, seed=7)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = ev(), ev()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


for P in (1, 2, 4, 8):
    res = {}
    for mode in ("z", "g", "sx"):
        worst = 0.0
        for p in range(P):
            r0, r1 = shard_range(n, P, p)
            t = cg.api.countgauss_new_shard(m, B, n, r0, r1 - r0, t_seed, ctx=ctx)
            xs = x[r0:r1]
            z = torch.empty((d, m), dtype=torch.float64, device="cuda").t()
            sx = torch.empty((B, d), dtype=torch.float64, device="cuda")
            if mode == "z":
                ms = timed(lambda: cg.api.countgauss_apply_into(t, xs, z))
            elif mode == "g":
                g0, g1 = g_row_range(m, P, p)
                ms = timed(lambda: (cg.api.countsketch_apply_into(t, xs, sx), cg.api.gauss_gemm_rows(t, sx, g0, g1)))
            else:
                b0, b1 = bucket_range(B, P, p)
                ms = timed(lambda: (cg.api.countsketch_apply_into(t, xs, sx),
                                    cg.api.gauss_gemm_range(t, sx[b0:b1], b0, b1)))
            worst = max(worst, ms)
        res[mode] = worst
    vol = {"z": m * d * 8, "g": B * d * 8, "sx": (P - 1) / P * B * d * 8}
    print(f"{cfg} P={P}: per-rank compute (max over ranks) z {res['z']:.3f} ms, g {res['g']:.3f} ms, "
          f"sx {res['sx']:.3f} ms; ideal {0.42 * (1 if cfg == 'c2' else 6.5) / P:.3f} ms; collective bytes per rank "
          f"z {vol['z'] / 1e6:.3f} MB, g {vol['g'] / 1e6:.1f} MB (all-reduce), sx {vol['sx'] / 1e6:.1f} MB")
