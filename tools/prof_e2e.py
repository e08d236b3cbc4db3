"""Measurement helper (not product code): c2 through the C ABI with host X -- pinned fp32
row-major (bench e2e), pageable fp32, pageable fp64 column-major (drop-in layout) -- wall
clock per call (median of 5), with the staging trace when CGX_TRACE_STAGE is set."""
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1606_05732_b200 as cg  # noqa: E402
from paper_1606_05732_b200 import bench_data  # noqa: E402

n, d, B, m = 1 << 24, 32, 65536, 64
x = bench_data.dense_normal(n, d, seed=7)
t = cg.countgauss_new(m, B, n, cg.SeededRng(12345))
pinned = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
pinned.copy_(x)
pageable = x.cpu().numpy().copy()
col64 = np.asfortranarray(pageable.astype(np.float64))
for label, arr in [("pinned f32", pinned.numpy()), ("pageable f32", pageable), ("pageable f64 col-major", col64)]:
    cg.countgauss_apply(t, arr)
    ts = []
    for _ in range(5):
        a = time.perf_counter()
        cg.countgauss_apply(t, arr)
        ts.append(time.perf_counter() - a)
    print(f"{label}: {statistics.median(ts) * 1e3:.1f} ms ({arr.nbytes / statistics.median(ts) / 1e9:.1f} GB/s of X)")
