"""Measurement helper (not product code): where the c2 e2e call's time goes -- a bare pinned
H2D of X, the C-ABI apply on pinned host X, and the apply on device X (wall clock, median
of 5)."""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1606_05732_b200 as cg  # noqa: E402
from paper_1606_05732_b200 import bench_data  # noqa: E402

n, d, B, m = 1 << 24, 32, 65536, 64
x = bench_data.dense_normal(n, d, seed=7)
t = cg.countgauss_new(m, B, n, cg.SeededRng(12345))
pinned = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
pinned.copy_(x)
xd = torch.empty_like(x)


def med(f, reps=5):
    f()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - a)
    return statistics.median(ts) * 1e3


print(f"bare H2D (torch copy_): {med(lambda: xd.copy_(pinned, non_blocking=True)):.2f} ms")
print(f"apply, pinned host X (numpy view): {med(lambda: cg.countgauss_apply(t, pinned.numpy())):.2f} ms")
print(f"apply, pinned host X (torch cpu tensor): {med(lambda: cg.countgauss_apply(t, pinned)):.2f} ms")
print(f"apply, device X: {med(lambda: cg.countgauss_apply(t, xd)):.2f} ms")
