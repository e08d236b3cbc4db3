"""Binary CSR ingestion: the CGXCSR1 container round-trips every dtype /
index type, and malformed files fail with ValueError.  Host-side (no GPU); the streamed
device load is covered in test_gpu_parity.py."""
import os

import numpy as np
import pytest

from paper_1606_05732_b200.api import SparseMatrix


def _rand(rng, n, d, density, idx, val):
    mask = rng.uniform(size=(n, d)) < density
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(mask.sum(1), out=rp[1:])
    _, c = np.nonzero(mask)
    return SparseMatrix(n, d, rp, c.astype(idx), rng.standard_normal(len(c)).astype(val))


@pytest.mark.parametrize("idx,val", [(np.int32, np.float32), (np.int64, np.float64), (np.int32, np.float64)])
@pytest.mark.parametrize("n,d,density", [(1000, 50, 0.1), (7, 3, 0.0), (1, 1, 1.0)])
def test_roundtrip(tmp_path, idx, val, n, d, density):
    x = _rand(np.random.default_rng(n + d), n, d, density, idx, val)
    p = str(tmp_path / "x.cgxcsr")
    x.save(p)
    assert os.path.getsize(p) == 64 + 8 * (n + 1) + x.nnz() * (np.dtype(idx).itemsize + np.dtype(val).itemsize)
    y = SparseMatrix.load(p)
    assert (y.rows, y.cols) == (n, d)
    assert y.col_indices.dtype == idx and y.values.dtype == val
    assert np.array_equal(y.row_offsets, x.row_offsets)
    assert np.array_equal(y.col_indices, x.col_indices)
    assert np.array_equal(y.values, x.values)


def test_bad_files(tmp_path):
    p = tmp_path / "bad"
    p.write_bytes(b"not a csr file at all" * 4)
    with pytest.raises(ValueError, match="not a CGXCSR1 file"):
        SparseMatrix.load(str(p))
    x = _rand(np.random.default_rng(0), 100, 10, 0.3, np.int32, np.float32)
    q = str(tmp_path / "x")
    x.save(q)
    data = open(q, "rb").read()
    open(q, "wb").write(data[:-10])  # truncated values
    with pytest.raises(ValueError, match="truncated"):
        SparseMatrix.load(q)
    with pytest.raises(ValueError, match="cannot open"):
        SparseMatrix.load(str(tmp_path / "missing"))
