"""The drop-in boundary exercised as a reference caller uses it (GPU).

* The reference's own acceptance suite (proj/tests/acceptance.cpp), compiled from the
  reference sources with integration/countgauss_gpu.cpp + libcgx.so supplying every
  CountSketch / CountGauss symbol (oracle/Makefile `acceptance`), must pass criteria 1-11
  and print the same statistics as the CPU build for the deterministic criteria.
  (Criterion 12 needs the reference CLI, which cannot be built here: CLI11 is absent; it
  fails for the CPU build too.)
* integration/dropin_bench.cpp drives cg::countgauss_apply(t, DenseMatrix / SparseMatrix)
  -- the seeded fast path and the pipelined host staging -- and must agree with the same
  program linked against the reference library.
The binaries are prebuilt in this container (they need /root/reference) and travel with
the repo snapshot; the test skips when they are absent.
"""
import json
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


def _bin(name):
    p = os.path.join(REF, name)
    if not os.path.exists(p):
        pytest.skip(f"{p} not built (needs /root/reference at build time)")
    return p


def _criteria(out):
    res = {}
    for line in out.splitlines():
        m = re.match(r"\[(PASS|FAIL)\] criterion\s+(\d+): (.*?)\(\s*[\d.]+s\)\s*(.*)$", line)
        if m:
            res[int(m.group(2))] = (m.group(1), m.group(4).strip())
    return res


def test_reference_acceptance_suite_on_gpu_backend():
    cli = os.path.join(REF, "countgauss")  # absent: criterion 12 fails on both builds
    gpu = subprocess.run([_bin("acceptance_gpu"), cli], capture_output=True, text=True, timeout=600, cwd=REF)
    cpu = subprocess.run([_bin("acceptance_cpu"), cli], capture_output=True, text=True, timeout=600, cwd=REF)
    g, c = _criteria(gpu.stdout), _criteria(cpu.stdout)
    print(gpu.stdout, gpu.stderr[-2000:], "rc", gpu.returncode)
    for k in range(1, 12):
        assert g[k][0] == "PASS", (k, g[k])
    for k in (1, 2, 3, 4, 6, 7, 8, 9, 10):  # deterministic statistics: identical text
        assert g[k][1] == c[k][1], (k, g[k][1], c[k][1])


@pytest.mark.parametrize("values", ["fp32", "fp64"])
def test_dropin_countgauss_apply_matches_reference_library(values):
    args = ["c1", "3"] + (["fp64"] if values == "fp64" else [])
    g = json.loads(subprocess.run([_bin("dropin_bench_gpu")] + args, capture_output=True, text=True, timeout=300,
                                  check=True).stdout.strip().splitlines()[-1])
    c = json.loads(subprocess.run([_bin("dropin_bench_cpu")] + args, capture_output=True, text=True, timeout=300,
                                  check=True).stdout.strip().splitlines()[-1])
    assert abs(g["z_abs_sum"] - c["z_abs_sum"]) <= 1e-12 * abs(c["z_abs_sum"])


@pytest.mark.parametrize("devices", ["0,0", "0,0,0"])
@pytest.mark.parametrize("cfg", ["c1", "c3s"])
def test_dropin_spans_a_device_group(cfg, devices):
    """CGX_DEVICES: cg::countgauss_apply on a seeded transform runs row-sharded over a device
    group (here ranks sharing device 0, so the combine is the peer-memory one), and must agree
    with the reference library like the single-GPU drop-in does."""
    args = [cfg, "2"]
    env = dict(os.environ, CGX_DEVICES=devices, CGX_SHIM_TRACE="1")
    run = subprocess.run([_bin("dropin_bench_gpu")] + args, capture_output=True, text=True, timeout=300, check=True,
                         env=env)
    assert f"over {len(devices.split(','))} ranks" in run.stderr
    g = json.loads(run.stdout.strip().splitlines()[-1])
    c = json.loads(subprocess.run([_bin("dropin_bench_cpu")] + args, capture_output=True, text=True, timeout=300,
                                  check=True).stdout.strip().splitlines()[-1])
    assert abs(g["z_abs_sum"] - c["z_abs_sum"]) <= 1e-12 * abs(c["z_abs_sum"])
    one = json.loads(subprocess.run([_bin("dropin_bench_gpu")] + args, capture_output=True, text=True, timeout=300,
                                    check=True).stdout.strip().splitlines()[-1])
    assert g["z_abs_sum"] != 0 and abs(g["z_abs_sum"] - one["z_abs_sum"]) <= 1e-12 * abs(one["z_abs_sum"])
