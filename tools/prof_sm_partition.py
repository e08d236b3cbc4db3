"""Measurement helper (not product code): is the c5 CSR gather bound by SM issue or by DRAM?
Time the sketch alone on all 148 SMs and with K SMs pinned by tools/microbench/occupy.so.
If it barely slows with fewer SMs, stage 2 could run beside it on the freed SMs.

  python tools/prof_sm_partition.py [K ...]
"""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_05732_b200 as cg  # noqa: E402
from paper_1606_05732_b200 import bench_data  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1].startswith("c") else "c5"
ks = [int(a) for a in sys.argv[1:] if not a.startswith("c")] or [0, 16, 32, 48]
occ = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "microbench", "occupy.so"))
ctx = cg.context()
if cfg == "c5":
    n, d, B, m = 1 << 27, 512, 1 << 20, 256
    x = bench_data.csr_zipf(n, d, seed=5, s_len=1.5, cap=512, s_col=1.1)
else:
    n, d, B, m = 1 << 26, 256, 1 << 18, 128
    x = bench_data.csr_bernoulli(n, d, 0.01, seed=3)
t = cg.countgauss_new(m, B, n, cg.SeededRng(1), ctx=ctx)
sx = torch.empty((B, d), dtype=torch.float64, device="cuda")
side = torch.cuda.Stream()
flag = torch.ones(1, dtype=torch.int32, device="cuda")
started = torch.zeros(1, dtype=torch.int32, device="cuda")
for k in ks:
    times = []
    for rep in range(4):
        if k:
            flag.fill_(1)
            started.zero_()
            torch.cuda.synchronize()
            occ.occupy(k, ctypes.c_void_p(flag.data_ptr()), ctypes.c_void_p(started.data_ptr()),
                       ctypes.c_void_p(side.cuda_stream))
            while int(started.item()) < k:  # item() syncs the default stream only
                time.sleep(0.001)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        cg.api.countsketch_apply_into(t, x, sx)
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b))
        if k:
            flag.zero_()
            torch.cuda.synchronize()
    print(f"{cfg} sketch with {k:3d} SMs pinned ({148 - k} free): " + " ".join(f"{v:.2f}" for v in times) + " ms",
          flush=True)
