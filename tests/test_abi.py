"""CPU: the C-ABI library loads, exports every symbol include/cgx.h declares, its pure host
functions agree with the oracle, and the Python mirror's argument checks raise the
reference's exceptions before any GPU work (no compute calls here: no GPU)."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    from paper_1606_05732_b200 import _lib

    declared = _lib.header_symbols()
    assert len(declared) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert set(declared) == set(_lib.SIGNATURES), "ctypes table out of sync with cgx.h"


def test_library_is_sm100a_only():
    from paper_1606_05732_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    archs = {line.split(".")[-2] for line in out.splitlines() if ".cubin" in line}
    assert archs == {"sm_100a"}, archs


def test_host_seed_functions_match_oracle():
    from paper_1606_05732_b200._lib import lib

    rng = np.random.default_rng(1)
    for _ in range(200):
        a, b = (int(v) for v in rng.integers(0, 2 ** 63, size=2))
        assert lib.cgx_mix64(a, b) == oracle.mix64(a, b)
        assert lib.cgx_rng_draw(a, b % 100000) == oracle.draw(a, b % 100000)


def test_seeded_rng_mirror(golden):
    import paper_1606_05732_b200 as cg

    r = cg.SeededRng(12345)
    assert [r.next_u64() for _ in range(64)] == [int(v) for v in golden["rng_u64_12345"]]
    r = cg.SeededRng(7)
    for _ in range(1000):  # test_rng.cpp:55-62
        u = r.next_uniform()
        assert 0.0 < u < 1.0
    a = cg.SeededRng(9)
    b = a.split()
    assert b.seed() == oracle.draw(9, 0)


def test_argument_errors_raise_before_gpu():
    import paper_1606_05732_b200 as cg

    rng = cg.SeededRng(1)
    with pytest.raises(ValueError, match="buckets and input_dim must be >= 1"):
        cg.countsketch_new(0, 5, rng)
    with pytest.raises(ValueError, match="buckets and input_dim must be >= 1"):
        cg.countsketch_new(5, 0, rng)
    with pytest.raises(ValueError, match="m, buckets and input_dim must be >= 1"):
        cg.countgauss_new(0, 5, 10, rng)
    with pytest.raises(ValueError, match="needs buckets >= input_dim"):
        cg.countsketch_injective(3, 10, rng)
    with pytest.raises(ValueError, match="m must be >= 1"):
        cg.cg_nmf(np.zeros((4, 3)), 0, 5, rng)
    with pytest.raises(ValueError, match="at least one column"):
        cg.cg_nmf(np.zeros((4, 0)), 2, 5, rng)


def test_context_fails_loudly_without_gpu():
    """No silent CPU path: with no usable GPU, creating a context raises."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1606_05732_b200 import _lib
    from paper_1606_05732_b200.api import Context

    with pytest.raises(_lib.CgxError):
        Context(0)
    h = C.c_void_p()
    assert _lib.lib.cgx_init(0, C.byref(h)) != _lib.CGX_OK
    assert _lib.lib.cgx_last_error()


def test_null_arguments_rejected():
    from paper_1606_05732_b200._lib import CGX_EINVAL, lib

    assert lib.cgx_countgauss_new(None, 1, 1, 1, 1, None) == CGX_EINVAL
    assert b"null context" in lib.cgx_last_error()
    assert lib.cgx_xform_info(None, None, None, None, None, None, None) == CGX_EINVAL


def test_library_carries_tcgen05_int8_and_tma():
    """The stage-2 tensor-core kernel is compiled in: tcgen05 int8 MMAs (UTCIMMA), TMEM loads
    and TMA/bulk copies appear in the sm_100a SASS of libcgx.so."""
    import shutil
    import subprocess

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    lib = os.path.join(os.path.dirname(__file__), "..", "paper_1606_05732_b200", "libcgx.so")
    sass = subprocess.run([cuobjdump, "-sass", lib], capture_output=True, text=True).stdout
    for mnemonic in ("UTCIMMA", "UTMALDG", "UBLKCP"):
        assert mnemonic in sass, mnemonic


def test_bench_stage2_roofline_line():
    """bench.py's stage-2 roofline object: the tcgen05 path for large Z (int8 digit products
    against the nominal int8 rate), the DMMA path otherwise."""
    import argparse
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    big = bench.stage2_line(argparse.Namespace(opt=[]), 256, 1 << 20, 512, 4.0)
    assert big["unit"] == "int8 TOPS" and abs(big["achieved"] - 28 * 2.0 * 256 * (1 << 20) * 512 / 4e-3 / 1e12) < 1e-6
    assert abs(big["fp64_equiv_tflops"] - 2.0 * 256 * (1 << 20) * 512 / 4e-3 / 1e12) < 1e-9
    small = bench.stage2_line(argparse.Namespace(opt=[]), 64, 65536, 32, 0.03)
    assert small["unit"] == "TFLOP/s" and "DMMA" in small["kernel"]
    off = bench.stage2_line(argparse.Namespace(opt=["oz_slices=0"]), 256, 1 << 20, 512, 8.0)
    assert off["unit"] == "TFLOP/s"
    assert bench.stage2_line(argparse.Namespace(opt=[]), 256, 1 << 20, 512, 0.0) is None


@pytest.mark.parametrize("seed,r,cols,alpha", [(oracle.mix64(12345, 4), 16, 112, 0.5), (7, 3, 40, 2.5),
                                               (99, 1, 5, 0.5), (5, 8, 0, 1.0)])
def test_separable_mixing_matches_oracle(seed, r, cols, alpha):
    """Config 4's Dirichlet mixing weights (host code in libcgx) == the C twin, bit for bit;
    columns are on the simplex."""
    from paper_1606_05732_b200 import bench_data

    h = bench_data.separable_mixing(seed, r, cols, alpha)
    assert np.array_equal(h, oracle.Restatement().separable_mixing(seed, r, cols, alpha))
    if cols:
        assert np.allclose(h.sum(0), 1.0, atol=1e-12) and (h >= 0).all()
    with pytest.raises(ValueError):
        bench_data.separable_mixing(seed, 0, cols, alpha)
    with pytest.raises(ValueError):
        bench_data.separable_mixing(seed, r, cols, 0.0)
