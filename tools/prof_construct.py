"""Measurement helper (not product code): countgauss_new wall time (first call pays the
pool and scratch allocations; later calls reuse them) at the CSR/dense config shapes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1606_05732_b200 as cg  # noqa: E402

ctx = cg.context(0)
for m, B, n in [(128, 262144, 1 << 26), (64, 65536, 1 << 24), (256, 1 << 20, 1 << 27)]:
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        t = cg.countgauss_new(m, B, n, cg.SeededRng(12345 + rep))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(f"m={m} B={B} n={n} rep {rep}: construct {1e3 * (t1 - t0):.1f} ms")
        del t
