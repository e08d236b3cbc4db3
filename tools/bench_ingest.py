"""Measurement helper (not product code): binary CSR ingestion rate -- a c3-shaped CSR
(2^26 x 256, 1%) saved as CGXCSR1, then streamed file -> pinned -> HBM by
SparseMatrix.load(device=0) (cgx_csr_load).  The file is read right after being written,
so it comes from the page cache: the number is the loader's pipeline rate, PCIe-bound.

  python tools/bench_ingest.py [--rows 67108864] [--path /tmp/c3.cgxcsr]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1606_05732_b200 as cg  # noqa: E402
from paper_1606_05732_b200 import bench_data  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1 << 26)
    ap.add_argument("--d", type=int, default=256)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--path", default="/tmp/c3.cgxcsr")
    a = ap.parse_args()
    x = bench_data.csr_bernoulli(a.rows, a.d, a.density, seed=11)
    h = cg.SparseMatrix(x.rows, x.cols, x.row_offsets.cpu().numpy(), x.col_indices.cpu().numpy(), x.values.cpu().numpy())
    t0 = time.perf_counter()
    h.save(a.path)
    t1 = time.perf_counter()
    size = os.path.getsize(a.path)
    for rep in range(3):
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        y = cg.SparseMatrix.load(a.path, device=0)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"load rep {rep}: {size / 1e9:.2f} GB in {1e3 * (t3 - t2):.1f} ms = {size / (t3 - t2) / 1e9:.1f} GB/s")
    assert torch.equal(y.values, x.values)
    print(f"save: {size / (t1 - t0) / 1e9:.1f} GB/s")
    os.remove(a.path)


if __name__ == "__main__":
    main()
