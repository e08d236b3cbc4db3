"""ctypes binding of ``libcgx.so`` -- the C-ABI declared in ``include/cgx.h``.

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).  There
is no fallback: if the library is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcgx.so")

CGX_OK, CGX_EINVAL, CGX_ENOMEM, CGX_ECUDA, CGX_ENCCL, CGX_ERANGE = range(6)
CGX_F64, CGX_F32 = 0, 1
CGX_I64, CGX_I32 = 0, 1
CGX_COL_MAJOR, CGX_ROW_MAJOR = 0, 1
CGX_MEM_HOST, CGX_MEM_DEVICE = 0, 1
CGX_COMBINE_Z, CGX_COMBINE_G, CGX_COMBINE_SX, CGX_COMBINE_P2P = 0, 1, 2, 3

_P, _I64, _U64, _I, _D, _SZ = C.c_void_p, C.c_int64, C.c_uint64, C.c_int, C.c_double, C.c_size_t

# name -> (restype, argtypes); mirrors include/cgx.h one-to-one.
SIGNATURES = {
    "cgx_last_error": (C.c_char_p, []),
    "cgx_version": (C.c_char_p, []),
    "cgx_init": (_I, [_I, _P]),
    "cgx_free": (_I, [_P]),
    "cgx_synchronize": (_I, [_P, _P]),
    "cgx_trim": (_I, [_P]),
    "cgx_device_alloc": (_I, [_P, _SZ, _P]),
    "cgx_device_free": (_I, [_P, _P]),
    "cgx_host_alloc": (_I, [_P, _SZ, _P]),
    "cgx_host_free": (_I, [_P, _P]),
    "cgx_memcpy": (_I, [_P, _P, _P, _SZ, _P]),
    "cgx_mix64": (_U64, [_U64, _U64]),
    "cgx_rng_draw": (_U64, [_U64, _U64]),
    "cgx_countsketch_new": (_I, [_P, _U64, _I64, _I64, _P]),
    "cgx_countsketch_injective": (_I, [_P, _U64, _I64, _I64, _P]),
    "cgx_countsketch_explicit": (_I, [_P, _I64, _I64, _P, _P, _I, _P]),
    "cgx_countgauss_new": (_I, [_P, _U64, _I64, _I64, _I64, _P]),
    "cgx_countgauss_new_shard": (_I, [_P, _U64, _I64, _I64, _I64, _I64, _I64, _P]),
    "cgx_gauss_gemm_range": (_I, [_P, _P, _P, _I64, _I64, _I64, _I, _P, _I, _P]),
    "cgx_gauss_gemm_rows": (_I, [_P, _P, _P, _I64, _I64, _I64, _I, _P, _I, _P]),
    "cgx_countgauss_bucket_shard": (_I, [_P, _U64, _I64, _I64, _I64, _I64, _I64, _P]),
    "cgx_xform_rows": (_I, [_P, _P, _P, _I, _P]),
    "cgx_gen_dense_normal_rows": (_I, [_P, _U64, _P, _I64, _I64, _I, _I, _P, _P]),
    "cgx_xform_set_gaussian_seeded": (_I, [_P, _P, _I64, _U64]),
    "cgx_xform_set_gaussian_explicit": (_I, [_P, _P, _I64, _P, _I]),
    "cgx_xform_info": (_I, [_P, _P, _P, _P, _P, _P, _P]),
    "cgx_xform_free": (_I, [_P]),
    "cgx_fill_hash_sign": (_I, [_P, _P, _P, _P, _I, _P]),
    "cgx_fill_gaussian": (_I, [_P, _P, _P, _I, _P]),
    "cgx_inverse_normal_cdf": (_I, [_P, _P, _P, _I64, _I, _P]),
    "cgx_countsketch_apply_dense": (_I, [_P, _P, _P, _I, _I, _I64, _I64, _I64, _I, _P, _I, _I, _P]),
    "cgx_countsketch_apply_csr": (_I, [_P, _P, _P, _P, _I, _P, _I, _I64, _I64, _I64, _I, _P, _I, _I, _P]),
    "cgx_countgauss_apply_dense": (_I, [_P, _P, _P, _I, _I, _I64, _I64, _I64, _I, _P, _I, _P]),
    "cgx_countgauss_apply_csr": (_I, [_P, _P, _P, _P, _I, _P, _I, _I64, _I64, _I64, _I, _P, _I, _P]),
    "cgx_gauss_gemm": (_I, [_P, _P, _P, _I, _I64, _I, _P, _I, _P]),
    "cgx_select_extremes": (_I, [_P, _P, _I64, _I64, _I, _P, _P, _P, _P]),
    "cgx_gaussian_project_dense": (_I, [_P, _U64, _I64, _P, _I, _I, _I64, _I64, _I64, _I, _P, _I, _P]),
    "cgx_csr_save": (_I, [C.c_char_p, _P, _P, _I, _P, _I, _I64, _I64, _I64]),
    "cgx_csr_info": (_I, [C.c_char_p, _P, _P, _P, _P, _P]),
    "cgx_csr_load": (_I, [_P, C.c_char_p, _P, _P, _P, _I, _P]),
    "cgx_countgauss_materialize": (_I, [_P, _P, _P, _I, _P]),
    "cgx_gaussian_project_csr": (_I, [_P, _U64, _I64, _P, _P, _I, _P, _I, _I64, _I64, _I64, _I, _P, _I, _P]),
    "cgx_countsketch_batch_gram": (_I, [_P, _U64, _I64, _I64, _I64, _P, _I64, _I64, _I64, _I, _P, _P, _I, _P]),
    "cgx_gen_dense_normal": (_I, [_P, _U64, _I64, _I64, _I64, _I, _I, _P, _P]),
    "cgx_gen_csr_bernoulli": (_I, [_P, _U64, _I64, _I64, _D, _P, _P, _P, _P, _P]),
    "cgx_gen_csr_zipf": (_I, [_P, _U64, _I64, _I64, _D, _I64, _D, _P, _P, _P, _P, _P]),
    "cgx_gen_separable": (_I, [_P, _U64, _I64, _I64, _I64, _I64, _D, _D, _I, _I, _P, _P]),
    "cgx_separable_mixing": (_I, [_U64, _I64, _I64, _D, _P]),
    "cgx_host_checksum": (_I, [_P, _P, _SZ, _P]),
    "cgx_group_init": (_I, [_I, _P, _P]),
    "cgx_group_stats": (_I, [_P, _P, _P]),
    "cgx_group_supports": (_I, [_P, _I]),
    "cgx_ipc_export": (_I, [_P, _P, _P]),
    "cgx_ipc_open": (_I, [_P, _P, _P]),
    "cgx_ipc_close": (_I, [_P, _P]),
    "cgx_countsketch_apply_dense_to": (_I, [_P, _P, _P, _I, _I, _I64, _I64, _I64, _I, _P, _I, _I64, _P]),
    "cgx_countsketch_apply_csr_to": (_I, [_P, _P, _P, _P, _I, _P, _I, _I64, _I64, _I64, _I, _P, _I, _I64, _P]),
    "cgx_sum_slots": (_I, [_P, _P, _I, _I64, _I64, _P, _P]),
    "cgx_group_free": (_I, [_P]),
    "cgx_group_size": (_I, [_P]),
    "cgx_group_context": (_I, [_P, _I, _P]),
    "cgx_group_countgauss_new": (_I, [_P, _U64, _I64, _I64, _I64, _P]),
    "cgx_gxform_free": (_I, [_P]),
    "cgx_gxform_shard": (_I, [_P, _I, _P, _P]),
    "cgx_group_countgauss_apply_dense": (_I, [_P, _P, _P, _I, _I, _I64, _I64, _I64, _I, _P, _I, _I]),
    "cgx_group_countgauss_apply_csr": (_I, [_P, _P, _P, _P, _I, _P, _I, _I64, _I64, _I64, _P, _I, _I]),
    "cgx_launch_count": (_U64, [_P]),
    "cgx_set_option": (_I, [_P, C.c_char_p, _I64]),
    "cgx_profile_enable": (_I, [_P, _I]),
    "cgx_profile_read": (_I, [_P, _I, _P, _P]),
}


def header_symbols() -> list[str]:
    """Every function name declared in include/cgx.h (parsed, for the export test)."""
    import re

    hdr = os.path.join(os.path.dirname(HERE), "include", "cgx.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"\b(cgx_[a-z0-9_]+)\s*\(", text)))


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the CountGauss path)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class CgxError(RuntimeError):
    pass


def check(rc: int) -> None:
    if rc == CGX_OK:
        return
    msg = lib.cgx_last_error().decode(errors="replace")
    if rc == CGX_EINVAL:
        raise ValueError(msg)          # std::invalid_argument in the reference
    if rc == CGX_ERANGE:
        raise OverflowError(msg)       # std::length_error
    if rc == CGX_ENOMEM:
        raise MemoryError(msg)
    raise CgxError(f"cgx error {rc}: {msg}")
