"""oracle -- TEST INFRASTRUCTURE ONLY: ctypes bindings for the two parity checkers.

* ``Restatement`` wraps ``oracle/liboracle.so`` (``oracle/cgoracle.c``), the plain-C
  restatement of the reference CountGauss path, each function citing the reference
  file:line it follows.
* ``Reference`` wraps ``oracle/_ref/libcgref.so``: the unmodified reference library
  (``/root/reference/proj/src``) compiled by ``oracle/Makefile`` behind a small
  ``extern "C"`` shim (``oracle/ref_shim.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg
and ``--impl reference`` arm) may import this package -- as the checker or the CPU
baseline, never as the thing measured or shipped.  The product package
(``paper_1606_05732_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GAMMA = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1

_P = C.c_void_p
_I64 = C.c_int64
_U64 = C.c_uint64
_D = C.c_double


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def build() -> None:
    """Compile liboracle.so and (when /root/reference exists) _ref/libcgref.so."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


# ---------------------------------------------------------------- pure-python pins
def fin(z: int) -> int:
    """SplitMix64 finalizer (rng.hpp:31-37)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def mix64(a: int, b: int) -> int:
    """mix64 (rng.hpp:12-17)."""
    return fin(a + GAMMA + b * 0xBF58476D1CE4E5B9)


def draw(seed: int, k: int) -> int:
    """Draw k of SeededRng(seed) (rng.hpp:31-37)."""
    return fin(seed + (k + 1) * GAMMA)


class Restatement:
    """oracle/cgoracle.c via ctypes."""

    def __init__(self):
        L = self.lib = _load(os.path.join(HERE, "liboracle.so"))
        L.cgo_mix64.restype = _U64
        L.cgo_mix64.argtypes = [_U64, _U64]
        L.cgo_draw.restype = _U64
        L.cgo_draw.argtypes = [_U64, _U64]
        L.cgo_inverse_normal_cdf.restype = _D
        L.cgo_inverse_normal_cdf.argtypes = [_D]
        L.cgo_countgauss_seeds.argtypes = [_U64, _P, _P, _P]
        L.cgo_hash_sign.argtypes = [_U64, _I64, _I64, _I64, _P, _P]
        L.cgo_gaussian.argtypes = [_U64, _I64, _I64, _I64, _P]
        L.cgo_sketch_dense.argtypes = [_P, _P, _I64, _P, C.c_int, _I64, _I64, _I64, _I64, _P]
        L.cgo_sketch_csr.argtypes = [_P, _P, _I64, _P, _P, C.c_int, _P, C.c_int, _I64, _I64, _P]
        L.cgo_gemm.argtypes = [_P, _I64, _I64, _P, _I64, _P]
        L.cgo_select_extremes.restype = _I64
        L.cgo_select_extremes.argtypes = [_P, _I64, _I64, _P, _P]
        L.cgo_normal_f32.restype = C.c_float
        L.cgo_normal_f32.argtypes = [_U64, _U64]
        L.cgo_gen_dense_f32.argtypes = [_U64, _I64, _I64, _P]
        L.cgo_gen_dense_f64_colmajor.argtypes = [_U64, _I64, _I64, _P]
        L.cgo_sketch_csr_buckets.argtypes = [_P, _P, _I64, _I64, _P, _P, C.c_int, _P, C.c_int, _I64, _I64, _P]
        L.cgo_gen_separable_f64_colmajor.argtypes = [_U64, _I64, _I64, _I64, _D, _D, _P]
        L.cgo_separable_mixing.argtypes = [_U64, _I64, _I64, _D, _P]
        L.cgo_gen_separable_f32.argtypes = [_U64, _I64, _I64, _I64, _I64, _D, _D, _P]

    def mix64(self, a, b):
        return int(self.lib.cgo_mix64(a, b))

    def inverse_normal_cdf(self, p):
        return float(self.lib.cgo_inverse_normal_cdf(p))

    def countgauss_seeds(self, caller_seed):
        t, c, g = _U64(), _U64(), _U64()
        self.lib.cgo_countgauss_seeds(caller_seed, C.byref(t), C.byref(c), C.byref(g))
        return t.value, c.value, g.value

    def hash_sign(self, cs_seed, B, n, i0=0):
        h = np.empty(n, np.int64)
        s = np.empty(n, np.float64)
        self.lib.cgo_hash_sign(cs_seed, B, i0, n, _ptr(h), _ptr(s))
        return h, s

    def gaussian(self, g_seed, m, B, c0=0):
        g = np.empty((B, m), np.float64)  # column-major m x B == row-major B x m
        self.lib.cgo_gaussian(g_seed, m, c0, B, _ptr(g))
        return g.T  # (m, B) view, Fortran-ordered

    def sketch_dense(self, hash_, sign, B, x):
        """x: (n, d) numpy array, any of C/F order, float32/float64. Returns (B, d) F-order."""
        n, d = x.shape
        if x.dtype not in (np.float32, np.float64):
            x = x.astype(np.float64)
        if x.flags.c_contiguous:
            rs, cs = d, 1
        else:
            x = np.asfortranarray(x)
            rs, cs = 1, n
        out = np.empty((d, B), np.float64)
        self.lib.cgo_sketch_dense(_ptr(np.ascontiguousarray(hash_, np.int64)),
                                  _ptr(np.ascontiguousarray(sign, np.float64)), B, _ptr(x),
                                  int(x.dtype == np.float32), n, d, rs, cs, _ptr(out))
        return out.T

    def sketch_csr(self, hash_, sign, B, rowptr, cols, vals, n, d):
        rowptr = np.ascontiguousarray(rowptr, np.int64)
        cols = np.ascontiguousarray(cols)
        vals = np.ascontiguousarray(vals)
        assert cols.dtype in (np.int32, np.int64) and vals.dtype in (np.float32, np.float64)
        out = np.empty((d, B), np.float64)
        self.lib.cgo_sketch_csr(_ptr(np.ascontiguousarray(hash_, np.int64)),
                                _ptr(np.ascontiguousarray(sign, np.float64)), B, _ptr(rowptr),
                                _ptr(cols), int(cols.dtype == np.int64), _ptr(vals),
                                int(vals.dtype == np.float32), n, d, _ptr(out))
        return out.T

    def sketch_csr_buckets(self, hash_, sign, b0, b1, rowptr, cols, vals, n, d):
        """Rows [b0, b1) of the serial CSR S.X (bit-identical to the full result's rows)."""
        rowptr = np.ascontiguousarray(rowptr, np.int64)
        cols = np.ascontiguousarray(cols)
        vals = np.ascontiguousarray(vals)
        out = np.empty((d, b1 - b0), np.float64)
        self.lib.cgo_sketch_csr_buckets(_ptr(np.ascontiguousarray(hash_, np.int64)),
                                        _ptr(np.ascontiguousarray(sign, np.float64)), b0, b1, _ptr(rowptr),
                                        _ptr(cols), int(cols.dtype == np.int64), _ptr(vals),
                                        int(vals.dtype == np.float32), n, d, _ptr(out))
        return out.T

    def gemm(self, a, b):
        a = np.asfortranarray(a, np.float64)
        b = np.asfortranarray(b, np.float64)
        out = np.empty((b.shape[1], a.shape[0]), np.float64)
        self.lib.cgo_gemm(_ptr(a), a.shape[0], a.shape[1], _ptr(b), b.shape[1], _ptr(out))
        return out.T

    def select_extremes(self, z):
        """Per-row (amax, amin, tie_rows) and the nmf.cpp:119-131 sorted-unique sets."""
        z = np.asfortranarray(z, np.float64)
        m, d = z.shape
        amax = np.empty(m, np.int64)
        amin = np.empty(m, np.int64)
        ties = int(self.lib.cgo_select_extremes(_ptr(z), m, d, _ptr(amax), _ptr(amin)))
        i_max = np.unique(amax)
        i_min = np.unique(amin)
        return dict(amax=amax, amin=amin, tie_rows=ties, i_max=i_max, i_min=i_min,
                    unioned=np.union1d(i_max, i_min))

    def countgauss(self, caller_seed, m, B, x=None, csr=None):
        """Full CountGauss T.X as the reference computes it (sketch.cpp:115-138)."""
        t_seed, cs_seed, g_seed = self.countgauss_seeds(caller_seed)
        if x is not None:
            n = x.shape[0]
        else:
            n = len(csr[0]) - 1
        h, s = self.hash_sign(cs_seed, B, n)
        g = self.gaussian(g_seed, m, B)
        if x is not None:
            sx = self.sketch_dense(h, s, B, x)
        else:
            rowptr, cols, vals, d = csr
            sx = self.sketch_csr(h, s, B, rowptr, cols, vals, n, d)
        return self.gemm(g, sx), sx

    def gen_dense_f32(self, seed, n, d):
        x = np.empty((n, d), np.float32)
        self.lib.cgo_gen_dense_f32(seed, n, d, _ptr(x))
        return x

    def separable_mixing(self, seed, r, cols, alpha=0.5):
        """H (r x cols) of the config-4 generator: Dirichlet(alpha) columns."""
        h = np.empty((cols, r), np.float64)
        self.lib.cgo_separable_mixing(seed, r, cols, alpha, _ptr(h))
        return h.T

    def gen_separable_f32(self, seed, n, d, r=16, alpha=0.5, sigma=0.01, row0=0):
        """Rows [row0, row0+n) of the config-4 near-separable X, row-major fp32."""
        x = np.empty((n, d), np.float32)
        self.lib.cgo_gen_separable_f32(seed, row0, n, d, r, alpha, sigma, _ptr(x))
        return x


class Reference:
    """The reference library itself (oracle/_ref/libcgref.so) via ctypes."""

    def __init__(self):
        L = self.lib = _load(os.path.join(HERE, "_ref", "libcgref.so"))
        L.cgref_last_error.restype = C.c_char_p
        L.cgref_mix64.restype = _U64
        L.cgref_mix64.argtypes = [_U64, _U64]
        L.cgref_max_threads.restype = C.c_int
        L.cgref_set_threads.argtypes = [C.c_int]
        L.cgref_rng_u64.argtypes = [_U64, _I64, _P]
        L.cgref_rng_normal.argtypes = [_U64, _I64, _P]
        L.cgref_inverse_normal_cdf.argtypes = [_D, _P]
        L.cgref_countgauss_new.argtypes = [_I64, _I64, _I64, _U64, _P]
        L.cgref_countsketch_new.argtypes = [_I64, _I64, _U64, _P]
        L.cgref_countsketch_injective.argtypes = [_I64, _I64, _U64, _P]
        L.cgref_xform_explicit.argtypes = [_I64, _I64, _P, _P, _I64, _P, _P]
        L.cgref_xform_free.argtypes = [_P]
        L.cgref_xform_info.argtypes = [_P, _P, _P, _P, _P, _P]
        L.cgref_xform_hash_sign.argtypes = [_P, _P, _P]
        L.cgref_xform_g.argtypes = [_P, _P]
        L.cgref_dense_new.argtypes = [_P, _I64, _I64, _P]
        L.cgref_dense_free.argtypes = [_P]
        L.cgref_dense_alloc.argtypes = [_I64, _I64, _P, _P]
        L.cgref_csr_new.argtypes = [_P, _P, _P, _I64, _I64, _P]
        L.cgref_csr_free.argtypes = [_P]
        L.cgref_apply.argtypes = [_P, _P, C.c_int, C.c_int, _P]
        L.cgref_time_apply.argtypes = [_P, _P, C.c_int, C.c_int, C.c_int, _P, _P]
        L.cgref_gemm.argtypes = [_P, _I64, _I64, _P, _I64, _I64, _P]
        L.cgref_materialized_sketch.argtypes = [_P, _P, _I64, _I64, _P]
        L.cgref_cg_nmf.argtypes = [_P, C.c_int, _I64, _I64, _U64] + [_P] * 7
        L.cgref_random_sparse.argtypes = [_I64, _I64, _I64, _U64, _P, _P, _P]
        L.cgref_gp_nmf.argtypes = [_P, _I64, _U64] + [_P] * 7
        L.cgref_generate_separable.argtypes = [_I64, _I64, _I64, _U64, _P]
        L.cgref_sketch_gram_trials.argtypes = [_U64, _I64, _I64, _I64, _P, _I64, _I64, _P, _P]

    def _check(self, rc):
        if rc == 1:
            raise ValueError(self.lib.cgref_last_error().decode())
        if rc != 0:
            raise RuntimeError(self.lib.cgref_last_error().decode())

    def rng_u64(self, seed, count):
        out = np.empty(count, np.uint64)
        self.lib.cgref_rng_u64(seed, count, _ptr(out))
        return out

    def rng_normal(self, seed, count):
        out = np.empty(count, np.float64)
        self.lib.cgref_rng_normal(seed, count, _ptr(out))
        return out

    def inverse_normal_cdf(self, p):
        out = _D()
        self._check(self.lib.cgref_inverse_normal_cdf(p, C.byref(out)))
        return out.value

    def set_threads(self, t):
        self.lib.cgref_set_threads(int(t))

    def max_threads(self):
        return int(self.lib.cgref_max_threads())

    # -- transforms
    def countgauss_new(self, m, B, n, caller_seed):
        h = C.c_void_p()
        self._check(self.lib.cgref_countgauss_new(m, B, n, caller_seed, C.byref(h)))
        return RefXform(self, h)

    def countsketch_new(self, B, n, caller_seed):
        h = C.c_void_p()
        self._check(self.lib.cgref_countsketch_new(B, n, caller_seed, C.byref(h)))
        return RefXform(self, h)

    def countsketch_injective(self, B, n, caller_seed):
        h = C.c_void_p()
        self._check(self.lib.cgref_countsketch_injective(B, n, caller_seed, C.byref(h)))
        return RefXform(self, h)

    def xform_explicit(self, B, hash_, sign, g=None):
        hash_ = np.ascontiguousarray(hash_, np.int64)
        sign = np.ascontiguousarray(sign, np.float64)
        m = 0
        if g is not None:
            g = np.asfortranarray(g, np.float64)
            m = g.shape[0]
        h = C.c_void_p()
        self._check(self.lib.cgref_xform_explicit(B, len(hash_), _ptr(hash_), _ptr(sign), m,
                                                  _ptr(g), C.byref(h)))
        return RefXform(self, h)

    # -- matrices
    def dense(self, x):
        x = np.asfortranarray(x, np.float64)
        h = C.c_void_p()
        self._check(self.lib.cgref_dense_new(_ptr(x), x.shape[0], x.shape[1], C.byref(h)))
        return RefMatrix(self, h, False, x.shape[0], x.shape[1])

    def dense_generated(self, n, d, seed, restatement):
        """n x d DenseMatrix filled in place with the synthetic N(0,1) entries
        (cgo_gen_dense_f64_colmajor) -- the bench's CPU input, never copied twice."""
        h = C.c_void_p()
        data = C.c_void_p()
        self._check(self.lib.cgref_dense_alloc(n, d, C.byref(h), C.byref(data)))
        restatement.lib.cgo_gen_dense_f64_colmajor(seed, n, d, data)
        return RefMatrix(self, h, False, n, d)

    def dense_alloc(self, n, d):
        """A zero n x d DenseMatrix held by the reference and a writable numpy view of its
        column-major storage (d x n, row j = column j), filled in place by the caller so a
        multi-GB input is never held twice."""
        h = C.c_void_p()
        data = C.c_void_p()
        self._check(self.lib.cgref_dense_alloc(n, d, C.byref(h), C.byref(data)))
        view = np.ctypeslib.as_array((C.c_double * (n * d)).from_address(data.value)).reshape(d, n)
        return RefMatrix(self, h, False, n, d), view

    def dense_separable_generated(self, n, d, seed, restatement, r=16, alpha=0.5, sigma=0.01):
        """n x d DenseMatrix filled in place with config 4's near-separable X
        (cgo_gen_separable_f64_colmajor, the twin of the GPU generator)."""
        h = C.c_void_p()
        data = C.c_void_p()
        self._check(self.lib.cgref_dense_alloc(n, d, C.byref(h), C.byref(data)))
        restatement.lib.cgo_gen_separable_f64_colmajor(seed, n, d, r, alpha, sigma, data)
        return RefMatrix(self, h, False, n, d)

    def csr(self, rowptr, cols, vals, n, d):
        rowptr = np.ascontiguousarray(rowptr, np.int64)
        cols = np.ascontiguousarray(cols, np.int64)
        vals = np.ascontiguousarray(vals, np.float64)
        h = C.c_void_p()
        self._check(self.lib.cgref_csr_new(_ptr(rowptr), _ptr(cols), _ptr(vals), n, d, C.byref(h)))
        return RefMatrix(self, h, True, n, d)

    def gemm(self, a, b):
        a = np.asfortranarray(a, np.float64)
        b = np.asfortranarray(b, np.float64)
        out = np.empty((b.shape[1], a.shape[0]), np.float64)
        self._check(self.lib.cgref_gemm(_ptr(a), a.shape[0], a.shape[1], _ptr(b), b.shape[0],
                                        b.shape[1], _ptr(out)))
        return out.T

    def cg_nmf(self, xm, m, B, caller_seed):
        cap = max(2 * m, 1)
        bufs = [np.empty(cap, np.int64) for _ in range(3)]
        cnt = [_I64() for _ in range(4)]
        self._check(self.lib.cgref_cg_nmf(xm.h, int(xm.sparse), m, B, caller_seed,
                                          _ptr(bufs[0]), C.byref(cnt[0]), _ptr(bufs[1]),
                                          C.byref(cnt[1]), _ptr(bufs[2]), C.byref(cnt[2]),
                                          C.byref(cnt[3])))
        return dict(i_max=bufs[0][:cnt[0].value].copy(), i_min=bufs[1][:cnt[1].value].copy(),
                    unioned=bufs[2][:cnt[2].value].copy(), tie_rows=cnt[3].value)

    def sketch_gram_trials(self, master, t0, trials, B, u):
        """distcheck.cpp:107-113 for trials [t0, t0+trials): (su, gram), trial-major."""
        u = np.asfortranarray(u, dtype=np.float64)
        n, d = u.shape
        su = np.empty((trials, d, B), np.float64)
        gm = np.empty((trials, d, d), np.float64)
        self._check(self.lib.cgref_sketch_gram_trials(master, t0, trials, B, _ptr(u), n, d, _ptr(su),
                                                      _ptr(gm)))
        return su.transpose(0, 2, 1), gm.transpose(0, 2, 1)

    def gp_nmf(self, xm, m, caller_seed):
        cap = max(2 * m, 1)
        bufs = [np.empty(cap, np.int64) for _ in range(3)]
        cnt = [_I64() for _ in range(4)]
        self._check(self.lib.cgref_gp_nmf(xm.h, m, caller_seed, _ptr(bufs[0]), C.byref(cnt[0]), _ptr(bufs[1]),
                                          C.byref(cnt[1]), _ptr(bufs[2]), C.byref(cnt[2]), C.byref(cnt[3])))
        return dict(i_max=bufs[0][:cnt[0].value].copy(), i_min=bufs[1][:cnt[1].value].copy(),
                    unioned=bufs[2][:cnt[2].value].copy(), tie_rows=cnt[3].value)

    def random_sparse(self, rows, cols, per_row, seed):
        rowptr = np.empty(rows + 1, np.int64)
        ci = np.empty(rows * per_row, np.int64)
        v = np.empty(rows * per_row, np.float64)
        self._check(self.lib.cgref_random_sparse(rows, cols, per_row, seed, _ptr(rowptr), _ptr(ci),
                                                 _ptr(v)))
        return rowptr, ci, v

    def generate_separable(self, d, n, k, seed):
        x = np.empty((n, d), np.float64)
        self._check(self.lib.cgref_generate_separable(d, n, k, seed, _ptr(x)))
        return x.T


class RefXform:
    def __init__(self, ref, h):
        self.ref, self.h = ref, h
        t, c, m, B, n = _U64(), _U64(), _I64(), _I64(), _I64()
        ref.lib.cgref_xform_info(h, C.byref(t), C.byref(c), C.byref(m), C.byref(B), C.byref(n))
        self.seed, self.cs_seed, self.m, self.B, self.n = t.value, c.value, m.value, B.value, n.value

    def __del__(self):
        try:
            self.ref.lib.cgref_xform_free(self.h)
        except Exception:
            pass

    def hash_sign(self):
        h = np.empty(self.n, np.int64)
        s = np.empty(self.n, np.float64)
        self.ref.lib.cgref_xform_hash_sign(self.h, _ptr(h), _ptr(s))
        return h, s

    def g(self):
        g = np.empty((self.B, self.m), np.float64)
        self.ref.lib.cgref_xform_g(self.h, _ptr(g))
        return g.T

    def apply(self, xm, kind):
        """kind 0: countsketch_apply -> (B,d); 1: countgauss_apply -> (m,d); 2: serial sketch."""
        rows = self.m if kind == 1 else self.B
        out = np.empty((xm.d, rows), np.float64)
        self.ref._check(self.ref.lib.cgref_apply(self.h, xm.h, int(xm.sparse), kind, _ptr(out)))
        return out.T

    def time_apply(self, xm, kind, reps):
        rows = self.m if kind == 1 else self.B
        out = np.empty((xm.d, rows), np.float64)
        ms = np.empty(reps, np.float64)
        self.ref._check(self.ref.lib.cgref_time_apply(self.h, xm.h, int(xm.sparse), kind, reps,
                                                      _ptr(ms), _ptr(out)))
        return ms, out.T

    def materialized_sketch(self, x):
        x = np.asfortranarray(x, np.float64)
        out = np.empty((x.shape[1], self.B), np.float64)
        self.ref._check(self.ref.lib.cgref_materialized_sketch(self.h, _ptr(x), x.shape[0],
                                                               x.shape[1], _ptr(out)))
        return out.T


class RefMatrix:
    def __init__(self, ref, h, sparse, n, d):
        self.ref, self.h, self.sparse, self.n, self.d = ref, h, sparse, n, d

    def __del__(self):
        try:
            (self.ref.lib.cgref_csr_free if self.sparse else self.ref.lib.cgref_dense_free)(self.h)
        except Exception:
            pass
