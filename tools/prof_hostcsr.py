"""Measurement helper (not product code): the drop-in's small-CSR case -- acceptance
criterion 11 (acceptance.cpp:318-382: m=16, B=80, d=16, 8 nnz/row, 0.5M..4M nnz) -- through
the C ABI with host arrays (int64 columns, fp64 values), against the same call on device
arrays, to split the host-staging cost from the kernel."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1606_05732_b200 as cg  # noqa: E402
from paper_1606_05732_b200._lib import (CGX_COL_MAJOR, CGX_F64, CGX_I64, CGX_MEM_DEVICE, CGX_MEM_HOST,  # noqa: E402
                                        check, lib)


def main():
    import torch

    ctx = cg.context()
    for nnz in (500000, 1000000, 2000000, 4000000):
        rows, d, B, m = nnz // 8, 16, 80, 16
        t = cg.countgauss_new(m, B, rows, cg.SeededRng(nnz))
        rng = np.random.default_rng(1)
        rp = np.arange(0, nnz + 1, 8, dtype=np.int64)
        cols = np.sort(rng.integers(0, d, (rows, 8)), axis=1).astype(np.int64).ravel()
        vals = rng.uniform(-1, 1, nnz)
        out = np.empty((d, B))
        res = {}
        for label, mem, arrs in [("host", CGX_MEM_HOST, (rp, cols, vals)), ("device", CGX_MEM_DEVICE, None)]:
            if mem == CGX_MEM_DEVICE:
                dt = [torch.from_numpy(a).cuda() for a in (rp, cols, vals)]
                ptrs = [a.data_ptr() for a in dt]
            else:
                ptrs = [a.ctypes.data for a in arrs]
            best = 1e9
            for _ in range(8):
                a = time.perf_counter()
                check(lib.cgx_countsketch_apply_csr(ctx.h, t._xf.h, ptrs[0], ptrs[1], CGX_I64, ptrs[2], CGX_F64, rows,
                                                    d, nnz, mem, out.ctypes.data, CGX_COL_MAJOR, CGX_MEM_HOST, None))
                best = min(best, time.perf_counter() - a)
            res[label] = best * 1e3
        print(f"nnz {nnz}: host-array apply {res['host']:.3f} ms, device-array apply {res['device']:.3f} ms")


if __name__ == "__main__":
    main()
