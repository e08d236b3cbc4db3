import sys, torch, statistics
sys.path.insert(0, ".")
import paper_1606_05732_b200 as cg
from paper_1606_05732_b200 import bench_data
n, d, B, m = 1 << 24, 32, 65536, 64
ctx = cg.context()
t_seed = cg.SeededRng(12345).next_u64()
for P in (8, 4):
    rows = n // P
    x = bench_data.dense_normal(rows, d, seed=7)
    t = cg.api.countgauss_new_shard(m, B, n, 0, rows, t_seed, ctx=ctx)
    sx = torch.empty((B, d), dtype=torch.float64, device="cuda")
    for rpt in (32, 64, 128, 256, 512, 1024):
        ctx.set_option("rows_per_task", rpt)
        for tt in (0, 1, 2, 4):
            ctx.set_option("tail_tasks", tt)
            ctx.profile(True)
            for _ in range(10):
                cg.api.countsketch_apply_into(t, x, sx)
            ms, k = ctx.profile_read(0)
            ctx.profile(False)
            print(f"P={P} rows_per_task={rpt} tail={tt}: sketch {1000*ms/k:.1f} us")
