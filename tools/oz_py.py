import ctypes as C, sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1606_05732_b200 as cg
from paper_1606_05732_b200._lib import CGX_MEM_DEVICE, CGX_ROW_MAJOR, check, lib
B, m, d = 1000, 100, 70
ctx = cg.context(0)
t = cg.countgauss_new(m, B, 10, cg.SeededRng(12345), ctx=ctx)
g = torch.empty((B, m), dtype=torch.float64, device="cuda")
check(lib.cgx_fill_gaussian(ctx.h, t._xf.h, g.data_ptr(), CGX_MEM_DEVICE, C.c_void_p(1)))
sx = torch.randn((B, d), dtype=torch.float64, device="cuda")
zr = sx.t() @ g
for S in (0, 7):
    ctx.set_option("oz_slices", S)
    z = torch.empty((d, m), dtype=torch.float64, device="cuda")
    check(lib.cgx_gauss_gemm(ctx.h, t._xf.h, sx.data_ptr(), CGX_ROW_MAJOR, d, CGX_MEM_DEVICE, z.data_ptr(), CGX_MEM_DEVICE, C.c_void_p(1)))
    torch.cuda.synchronize()
    print(S, ((z - zr).norm() / zr.norm()).item(), z[0, :4].tolist(), zr[0, :4].tolist(), z[:4, 0].tolist(), zr[:4,0].tolist())
