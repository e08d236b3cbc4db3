"""Out-of-bounds writes, checked by hand (compute-sanitizer is closed on this pool,
profiles/r02_sanitizer_refused.log): every device output of the path -- S.X (row- and
column-major) and Z -- is carved out of a larger allocation whose bytes before and after it
hold a sentinel pattern, the inputs sit in carved allocations too, and after the call the
guards must be untouched and the output must be fully written (no sentinel left) and equal to
the same call into a plain tensor.  Shapes are ragged on purpose: d and B off every tile and
vector width, rows off the 32-row chunks, the sub-warp kernels (d <= 16), the cp.async gather,
the CSR gather, the record path, the chunked CSR branch, and the DMMA and tcgen05 stage 2."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GUARD = 4096  # doubles on each side
SENT = -1.2345678e300


def _carve(shape_elems, dtype=torch.float64, fill=None):
    g = GUARD if dtype == torch.float64 else GUARD * 2
    buf = torch.full((shape_elems + 2 * g,), SENT if fill is None else fill, dtype=dtype, device="cuda")
    return buf, buf[g:g + shape_elems], g


def _guards_ok(buf, g):
    return bool((buf[:g] == buf[0]).all() and (buf[-g:] == buf[0]).all() and buf[0].item() == buf[-1].item())


DENSE = [  # n, d, B, m, dtype
    (50001, 1, 97, 3, torch.float64),
    (50001, 3, 4099, 5, torch.float32),
    (33333, 7, 1, 4, torch.float64),
    (70001, 12, 513, 9, torch.float32),
    (65537, 24, 2049, 16, torch.float32),     # cp.async gather, 96 B rows
    (65537, 33, 2049, 16, torch.float64),     # odd d
    (40003, 130, 1031, 20, torch.float32),    # 520 B rows: register-batch stream kernel
    (40003, 132, 1031, 70, torch.float32),    # V = 4 gather
    (30001, 260, 777, 129, torch.float64),    # m.d >= 16384: tcgen05 stage 2, ragged tiles
]


@pytest.mark.parametrize("n,d,B,m,dtype", DENSE)
def test_dense_outputs_stay_inside_their_buffers(cg, n, d, B, m, dtype):
    gen = torch.Generator(device="cuda").manual_seed(n + d)
    xbuf, xflat, gx = _carve(n * d, dtype, fill=0.5)
    xflat.copy_(torch.randn(n * d, generator=gen, device="cuda", dtype=dtype))
    x = xflat.view(n, d)
    t = cg.countgauss_new(m, B, n, cg.SeededRng(77))
    # S.X row-major, S.X column-major, Z
    sbuf, sflat, gs = _carve(B * d)
    cg.api.countsketch_apply_into(t, x, sflat.view(B, d))
    cbuf, cflat, gc = _carve(B * d)
    cg.api.countsketch_apply_into(t, x, cflat.view(d, B).t())
    zbuf, zflat, gz = _carve(m * d)
    cg.api.countgauss_apply_into(t, x, zflat.view(d, m).t())
    torch.cuda.synchronize()
    for buf, g in ((sbuf, gs), (cbuf, gc), (zbuf, gz), (xbuf, gx)):
        assert _guards_ok(buf, g)
    sx = sflat.view(B, d)
    assert not (sx == SENT).any() and not (zflat == SENT).any() and not (cflat == SENT).any()
    assert torch.equal(cflat.view(d, B).t(), sx)
    sx_plain = torch.empty((B, d), dtype=torch.float64, device="cuda")
    cg.api.countsketch_apply_into(t, x, sx_plain)
    z_plain = cg.countgauss_apply(t, x)
    torch.cuda.synchronize()
    assert torch.equal(sx_plain, sx)
    assert torch.equal(z_plain, zflat.view(d, m).t())


CSR = [  # n, d, B, m, max row length, csr_mode
    (50001, 1, 97, 3, 2, 0),
    (40001, 37, 1025, 6, 9, 0),       # B.d <= 2^16: the chunked branch
    (60001, 300, 5003, 16, 12, 0),    # lean gather
    (60001, 300, 5003, 16, 12, 3),    # record path forced
    (20001, 515, 300, 130, 40, 0),    # tcgen05 stage 2 after the gather (column maxima folded in)
    (300001, 256, 8192, 128, 4, 3),   # record path + tcgen05 stage 2
]


@pytest.mark.parametrize("n,d,B,m,maxlen,csr_mode", CSR)
def test_csr_outputs_stay_inside_their_buffers(cg, n, d, B, m, maxlen, csr_mode):
    rng = np.random.default_rng(n + d)
    lens = rng.integers(0, maxlen + 1, n)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    nnz = int(rp[-1])
    cols = rng.integers(0, d, nnz).astype(np.int32)
    vals = rng.standard_normal(nnz).astype(np.float32)
    # the inputs in carved allocations as well: a read past their ends would at least not fault
    # silently into a neighbour holding the same data
    cbuf, cflat, _ = _carve(nnz, torch.int32, fill=0x7FFFFFF0)
    cflat.copy_(torch.from_numpy(cols))
    vbuf, vflat, _ = _carve(nnz, torch.float32, fill=float("nan"))
    vflat.copy_(torch.from_numpy(vals))
    x = cg.SparseMatrix(n, d, torch.from_numpy(rp).cuda(), cflat, vflat)
    ctx = cg.context()
    ctx.set_option("csr_mode", csr_mode)
    try:
        t = cg.countgauss_new(m, B, n, cg.SeededRng(91))
        sbuf, sflat, gs = _carve(B * d)
        cg.api.countsketch_apply_into(t, x, sflat.view(B, d))
        zbuf, zflat, gz = _carve(m * d)
        cg.api.countgauss_apply_into(t, x, zflat.view(d, m).t())
        torch.cuda.synchronize()
        assert _guards_ok(sbuf, gs) and _guards_ok(zbuf, gz)
        assert not (sflat == SENT).any() and not (zflat == SENT).any()
        assert not torch.isnan(sflat).any() and not torch.isnan(zflat).any()  # no guard value was read
        sx_plain = torch.empty((B, d), dtype=torch.float64, device="cuda")
        cg.api.countsketch_apply_into(t, x, sx_plain)
        torch.cuda.synchronize()
        if csr_mode == 3:  # the record path's adds run in no fixed order
            assert (torch.linalg.norm(sx_plain - sflat.view(B, d)) / torch.linalg.norm(sx_plain)).item() <= 1e-14
        else:
            assert torch.equal(sx_plain, sflat.view(B, d))
    finally:
        ctx.set_option("csr_mode", 0)
