"""Measurement helper (not product code): what one tiny trial of distcheck's Monte-Carlo loop
costs through the C ABI the way the drop-in shim calls it (acceptance criterion 3: n = 3,
B = 2, 100000 trials): cgx_countsketch_new + cgx_fill_hash_sign to host + cgx_countsketch_apply_dense
host -> host, microseconds per call."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1606_05732_b200 as cg  # noqa: E402
from paper_1606_05732_b200._lib import CGX_COL_MAJOR, CGX_F64, CGX_MEM_HOST, lib  # noqa: E402

n, B, d = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (3, 2, 1)
trials = 3000
ctx = cg.context(0)
u = np.full((n, d), 1.0 / np.sqrt(n), order="F")
out = np.zeros((B, d), order="F")
hh = np.zeros(n, np.int64)
ss = np.zeros(n, np.float64)
acc = {"new": 0.0, "fill": 0.0, "apply": 0.0, "free": 0.0}
for k in range(trials + 100):
    if k == 100:
        acc = dict.fromkeys(acc, 0.0)
    h = C.c_void_p()
    t0 = time.perf_counter()
    assert lib.cgx_countsketch_new(ctx.h, 1000 + k, B, n, C.byref(h)) == 0
    t1 = time.perf_counter()
    assert lib.cgx_fill_hash_sign(ctx.h, h, hh.ctypes.data, ss.ctypes.data, CGX_MEM_HOST, None) == 0
    t2 = time.perf_counter()
    assert lib.cgx_countsketch_apply_dense(ctx.h, h, u.ctypes.data, CGX_F64, CGX_COL_MAJOR, n, n, d, CGX_MEM_HOST,
                                           out.ctypes.data, CGX_COL_MAJOR, CGX_MEM_HOST, None) == 0
    t3 = time.perf_counter()
    lib.cgx_xform_free(h)
    t4 = time.perf_counter()
    for key, dt in zip(acc, (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
        acc[key] += dt
print(f"n={n} B={B} d={d}: " + ", ".join(f"{k} {1e6 * v / trials:.1f} us" for k, v in acc.items())
      + f"; launches/trial {ctx.launches / (trials + 100):.1f}")
