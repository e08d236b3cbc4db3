import sys, torch
sys.path.insert(0, ".")
import paper_1606_05732_b200 as cg
from paper_1606_05732_b200 import bench_data
n, d, B, m = 1 << 24, 32, 65536, 64
P = 8
ctx = cg.context()
t_seed = cg.SeededRng(12345).next_u64()
rows = n // P
x = bench_data.dense_normal(rows, d, seed=7)
t = cg.api.countgauss_new_shard(m, B, n, 0, rows, t_seed, ctx=ctx)
z = torch.empty((d, m), dtype=torch.float64, device="cuda").t()
sx = torch.empty((B, d), dtype=torch.float64, device="cuda")
for _ in range(5):
    cg.api.countgauss_apply_into(t, x, z)
    cg.api.countsketch_apply_into(t, x, sx)
    cg.api.gauss_gemm_rows(t, sx, 0, 8)
torch.cuda.synchronize()
