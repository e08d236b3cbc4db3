import sys, torch
sys.path.insert(0, ".")
import oracle
import paper_1606_05732_b200 as cg
from paper_1606_05732_b200 import bench_data
ctx = cg.context(); ctx.set_option("csr_mode", 3)
x = bench_data.csr_bernoulli(1 << 26, 256, 0.01, seed=oracle.mix64(12345, 3))
t = cg.countgauss_new(128, 262144, 1 << 26, cg.SeededRng(12345))
sx = torch.empty((262144, 256), dtype=torch.float64, device="cuda")
for _ in range(3):
    cg.api.countsketch_apply_into(t, x, sx)
torch.cuda.synchronize()
