"""Measurement helper (not product code): the CSR record path (csr_mode=3, csr_atomic.cu)
against the bit-exact gather (csr_mode=1) on a BASELINE CSR config: S.X agreement and
per-launch sketch time (CUDA events around the stage-1 kernels)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1606_05732_b200 as cg  # noqa: E402
from paper_1606_05732_b200 import bench_data  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
modes = [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "3"])]
C = {"c3": dict(n=1 << 26, d=256, B=262144, m=128), "c5": dict(n=1 << 27, d=512, B=1 << 20, m=256)}[cfg]
ctx = cg.context()
for kv in sys.argv[3:]:  # extra KEY=VALUE context options
    k, v = kv.split("=")
    ctx.set_option(k, int(v))
if cfg == "c3":
    x = bench_data.csr_bernoulli(C["n"], C["d"], 0.01, seed=oracle.mix64(12345, 3))
else:
    x = bench_data.csr_zipf(C["n"], C["d"], seed=oracle.mix64(12345, 5))
t = cg.countgauss_new(C["m"], C["B"], C["n"], cg.SeededRng(12345))
res = {}
for mode in modes:
    ctx.set_option("csr_mode", mode)
    sx = cg.countsketch_apply(t, x)
    torch.cuda.synchronize()
    ctx.profile(True)
    for _ in range(5):
        cg.countsketch_apply(t, x)
    ms, k = ctx.profile_read(0)
    ctx.profile(False)
    res[mode] = sx.clone()
    print(f"{cfg} csr_mode={mode}: sketch {ms / k:.3f} ms/launch")
if 1 in res:
    for mode, sx in res.items():
        if mode == 1:
            continue
        a, b = sx, res[1]
        eq = (a == b).double().mean().item()
        rel = ((a - b).norm() / b.norm()).item()
        mx = ((a - b).abs().max() / b.abs().max()).item()
        print(f"  mode {mode} vs gather: equal entries {eq:.4f}, rel Frobenius {rel:.2e}, max rel {mx:.2e}")
