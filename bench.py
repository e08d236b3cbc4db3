#!/usr/bin/env python
"""CountGauss T.X = G.(S.X) throughput on B200 (BASELINE.json metric), one JSON line.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

Workload (N=1 default): BASELINE config 2 -- dense X, n = 2^24 rows x d = 32 fp32,
B = 65536 buckets, m = 64 -- the configuration the metric is quoted on (configs[1]).  A
step is one countgauss_apply over the whole X; X (2.15 GB) is generated in HBM before the
timed region and is larger than L2 (126 MB), so no L2 flush is needed.  For N > 1
(torchrun, one process per GPU over NCCL) the config's rows are sharded contiguously
("strong", the north star's split): each rank sketches its shard with the shared seed into
a partial S.X, and the partials are combined the north star's way -- all-reduce of S.X and
G's m rows split across ranks for dense configs (--combine g), reduce-scatter of S.X by
bucket range with split-K stage 2 for CSR configs (--combine sx); --combine z / --scaling
weak are the labelled alternatives.  Time is the max over ranks.

Reported beside `value` (device-resident X):
  roofline      -- the sketch kernel (stage 1), CUDA events on its launch stream,
                   algorithmic bytes n*d*4 + B*d*8 per launch vs MEASURED_PEAKS hbm_gbs;
                   roofline.ceiling: the measured hardware rate that bounds it where that
                   is not HBM bandwidth (random-row gather, random DRAM accesses, the CSR
                   record path's RED + copy floor);
  stage2        -- the G.(S.X) kernel against its own peak (int8 tensor or FP64 DMMA);
  e2e           -- the same metric through the C-ABI with X in pinned HOST memory
                   (H2D of X and D2H of Z inside the timed region);
  e2e_dropin    -- cg::countgauss_apply through the reference's own C++ API (pageable fp64
                   DenseMatrix / SparseMatrix), drop-in vs the reference library, same host;
  cpu_baseline  -- the reference's own countgauss_apply (oracle/_ref, compiled from the
                   reference sources) on the box's host cores, full c2 in fp64;
  clocks        -- NVML SM clock and clock-event reasons sampled during the timed region.
--impl reference times that CPU implementation alone (rank 0), as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CountGauss T·X throughput: nnz(X)/s and HBM GB/s at 1/2/4/8 B200 vs CPU ref"
SEED = 12345  # CLI default seed (countgauss_main.cpp:46)

CONFIGS = {
    "c1": dict(kind="dense", n=65536, d=8, B=2048, m=16, dtype="f64"),
    "c2": dict(kind="dense", n=1 << 24, d=32, B=65536, m=64, dtype="f32"),
    "c3": dict(kind="csr", n=1 << 26, d=256, B=262144, m=128, density=0.01),
    "c4": dict(kind="dense", n=1 << 25, d=128, B=131072, m=32, dtype="f32", gen="separable", r=16, alpha=0.5,
               sigma=0.01),
    "c5": dict(kind="csr", n=1 << 27, d=512, B=1 << 20, m=256, zipf=(1.5, 512, 1.1)),
}


def mix64(a, b):
    M = (1 << 64) - 1
    z = (a + 0x9E3779B97F4A7C15 + b * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def workload_name(cfg_name, c):
    if c.get("gen") == "separable":
        return (f"{cfg_name}: near-separable dense X {c['n']}x{c['d']} f32 row-major = max(A.[I_{c['r']}|H] + "
                f"N(0,{c['sigma']}^2), 0), H Dirichlet({c['alpha']}); cg_nmf: CountGauss B={c['B']}, m={c['m']} "
                f"+ anchor selection")
    if c["kind"] == "dense":
        return (f"{cfg_name}: dense X {c['n']}x{c['d']} {c['dtype']} row-major, CountGauss B={c['B']}, "
                f"m={c['m']}")
    if "zipf" in c:
        s_len, cap, s_col = c["zipf"]
        return (f"{cfg_name}: CSR X {c['n']}x{c['d']} row lengths Zipf({s_len}) cap {cap}, columns Zipf({s_col}), "
                f"fp32/int32, B={c['B']}, m={c['m']}")
    return f"{cfg_name}: CSR X {c['n']}x{c['d']} Bernoulli({c['density']}) fp32/int32, B={c['B']}, m={c['m']}"


def data_seed(cfg_name):
    """Seed of a config's synthetic X: mix64(s0, config id)."""
    return mix64(SEED, int(cfg_name[1:]))


def units_of(c, nnz=None):
    return c["n"] * c["d"] if c["kind"] == "dense" else nnz


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every ~0.5 ms
    on a side thread while the timed region runs (a c2 step is 0.42 ms, so a 50 ms
    nvidia-smi poll would see nothing).  Raises if NVML cannot be read at all."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake_slowdown": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, index):
        import pynvml as nv

        self.nv = nv
        nv.nvmlInit()
        self.h = None
        try:  # the CUDA ordinal's physical GPU, by PCI bus id (CUDA_VISIBLE_DEVICES-safe)
            import torch

            p = torch.cuda.get_device_properties(index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            self.h = nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            self.h = nv.nvmlDeviceGetHandleByIndex(index)
        self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
        self.samples = []
        self.reasons = 0
        self.stop = threading.Event()

    def _sample(self):
        nv = self.nv
        self.samples.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
        self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))

    def _run(self):
        while not self.stop.is_set():
            self._sample()
            time.sleep(0.0005)

    def __enter__(self):
        self._sample()  # fails loudly here if NVML is unusable
        self.samples.clear()
        self.reasons = 0
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join()
        if not self.samples:
            self._sample()

    def summary(self):
        nv = self.nv
        names = sorted(k for k, attr in self.REASONS.items() if self.reasons & int(getattr(nv, attr, 0)))
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples), "how": "NVML every ~0.5 ms during the timed region"}


# ---------------------------------------------------------------- CPU baseline (reference)
def cpu_reference_run(cfg_name, c, steps, warmup):
    """The reference's production countgauss_apply (OpenMP) on the host cores."""
    import oracle

    R = oracle.Reference()
    O = oracle.Restatement()
    threads = os.cpu_count() or 1
    R.set_threads(threads)
    cores = R.max_threads()
    t_seed_rng = SEED
    if c["kind"] != "dense":
        return _cpu_reference_csr(cfg_name, c, R, steps, cores)
    t0 = time.time()
    xf = R.countgauss_new(c["m"], c["B"], c["n"], t_seed_rng)
    construct_s = time.time() - t0
    if c.get("gen") == "separable":
        xm = R.dense_separable_generated(c["n"], c["d"], data_seed(cfg_name), O, r=c["r"], alpha=c["alpha"],
                                         sigma=c["sigma"])
    else:
        xm = R.dense_generated(c["n"], c["d"], data_seed(cfg_name), O)
    # cgref_time_apply runs one untimed call, then the timed ones; the first (warmup - 1)
    # timed samples are discarded too, so `warmup` untimed calls precede the kept samples
    ms, _ = xf.time_apply(xm, 1, max(1, steps + warmup - 1))
    ms = list(ms)[warmup - 1:] if warmup > 1 else list(ms)
    med = statistics.median(ms)
    units = c["n"] * c["d"]
    what = "countgauss_apply (cg_nmf's product; its countgauss_new is outside the step on both arms)" \
        if c.get("gen") == "separable" else "countgauss_apply"
    return dict(value=units / (med / 1e3), ms=ms, median_ms=med, cores=cores, construct_s=construct_s,
                warmup=max(warmup, 1),
                sample=(f"full {cfg_name}: {what} on fp64 column-major X (the reference layout), "
                        f"{len(ms)} timed calls after {max(warmup, 1)} warm-up calls, median; reference code as-is"))


def _cpu_reference_csr(cfg_name, c, R, steps, cores, sample_nnz=20_000_000, full_nnz_max=400_000_000):
    """CSR configs: the reference's countgauss_apply (serial CSR branch + OpenMP gemm) on the
    config's X.  c3 (172 M nnz, ~5 s per call) runs at FULL size, median of 3 after a
    warm-up.  c5 (2.33e9 nnz, ~2 min per call on this host) runs a bounded row sample (its
    first rows, same generator), timed as the whole apply and as the sketch alone, and the
    full-size time is extrapolated as sketch_ms * nnz/nnz_sample + (apply_ms - sketch_ms):
    the serial CSR sketch is linear in nnz, and the GEMM stage (m x B by B x d) does not
    depend on n."""
    import numpy as np
    import torch

    from paper_1606_05732_b200 import bench_data

    mean = c.get("mean_row_nnz") or (c["d"] * c.get("density", 0.0) or 17.36)
    full = c["n"] * mean <= full_nnz_max
    rows = c["n"] if full else int(min(c["n"], max(1024, sample_nnz / mean)))
    if "zipf" in c:
        s_len, cap, s_col = c["zipf"]
        x = bench_data.csr_zipf(rows, c["d"], seed=data_seed(cfg_name), s_len=s_len, cap=cap, s_col=s_col)
    else:
        x = bench_data.csr_bernoulli(rows, c["d"], c["density"], seed=data_seed(cfg_name))
    rp = x.row_offsets.cpu().numpy()
    ci = x.col_indices.cpu().numpy().astype(np.int64)
    vv = x.values.cpu().numpy().astype(np.float64)
    nnz_s = int(rp[-1])
    del x
    torch.cuda.empty_cache()
    xm = R.csr(rp, ci, vv, rows, c["d"])
    del rp, ci, vv
    t0 = time.time()
    xf = R.countgauss_new(c["m"], c["B"], rows, SEED)
    construct_s = time.time() - t0
    if full:
        reps = 3
        ms_all, _ = xf.time_apply(xm, 1, reps)  # one untimed call first (cgref_time_apply)
        med = statistics.median(ms_all)
        return dict(value=nnz_s / (med / 1e3), ms=list(ms_all), median_ms=med, cores=cores, construct_s=construct_s,
                    warmup=1, sample=(f"full {cfg_name} ({nnz_s} nnz, int64 columns / fp64 values, the reference "
                                      f"SparseMatrix): countgauss_apply (serial CSR branch + OpenMP gemm), median of "
                                      f"{reps} after 1 warm-up call"))
    reps = max(1, min(steps, 5))
    ms_all, _ = xf.time_apply(xm, 1, reps)
    ms_sk, _ = xf.time_apply(xm, 0, reps)
    t_all, t_sk = statistics.median(ms_all), statistics.median(ms_sk)
    nnz_full = c.get("nnz_full") or nnz_s * (c["n"] / rows)
    est_ms = t_sk * nnz_full / nnz_s + max(0.0, t_all - t_sk)
    return dict(value=nnz_full / (est_ms / 1e3), ms=[est_ms] * reps, median_ms=est_ms, cores=cores,
                construct_s=construct_s, warmup=1,
                sample=(f"{cfg_name} rows 0..{rows} ({nnz_s} nnz) through the reference's countgauss_apply "
                        f"(serial CSR branch + OpenMP gemm): apply {t_all:.0f} ms, sketch {t_sk:.0f} ms, median of "
                        f"{reps}; full size extrapolated as sketch x nnz ratio + gemm"))


def run_dropin(cfg_name, c, reps=3):
    """Times cg::countgauss_apply through the drop-in and through the reference library, in
    one program (integration/dropin_bench.cpp), on the config's shape with fp32-valued fp64
    entries (BASELINE's configs hold fp32 data) and, for dense configs, full-fp64 entries."""
    ref = os.path.join(ROOT, "oracle", "_ref")
    gpu_bin, cpu_bin = os.path.join(ref, "dropin_bench_gpu"), os.path.join(ref, "dropin_bench_cpu")
    if not (os.path.exists(gpu_bin) and os.path.exists(cpu_bin)):
        return {"unavailable": "oracle/_ref/dropin_bench_{gpu,cpu} not built (needs /root/reference at build time)"}
    import subprocess

    def run(b, extra):
        out = subprocess.run([b, cfg_name, str(reps)] + extra, capture_output=True, text=True, timeout=900,
                             check=True).stdout
        return json.loads(out.strip().splitlines()[-1])

    res = {}
    for label, extra in [("fp32_valued", [])] + ([("fp64", ["fp64"])] if cfg_name != "c3" else []):
        gj, cj = run(gpu_bin, extra), run(cpu_bin, extra)
        res[label] = {"value": gj["nnz_per_s"], "unit": "nnz/s", "ms_per_step": gj["ms"],
                      "h2d_bytes_per_step": int(gj["input_bytes"]), "d2h_bytes_per_step": c["m"] * c["d"] * 8,
                      "reference_ms": cj["ms"], "speedup_vs_reference": cj["ms"] / gj["ms"],
                      "z_match": abs(gj["z_abs_sum"] - cj["z_abs_sum"]) <= 1e-12 * abs(cj["z_abs_sum"]),
                      "values": gj["values"]}
    res["how"] = ("cg::countgauss_apply(t, X) with X a reference DenseMatrix/SparseMatrix in pageable host memory "
                  f"(fp64; CSR int64+fp64), median of {reps} after a warm-up, wall clock, through the drop-in shim "
                  "(seeded fast path + pipelined pinned staging) vs the same program linked with the reference library "
                  "on this host's cores; h2d_bytes = the bytes the API hands over")
    return res


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    c = CONFIGS[args.config]
    # each CPU step is a full c2 countgauss_apply (~0.1-0.3 s on a multi-core host): bound
    # the sample so the whole arm ends within a few minutes
    r = cpu_reference_run(args.config, c, min(args.steps, 20), min(max(args.warmup, 1), 3))
    line = {
        "metric": METRIC, "impl": "reference", "value": r["value"], "unit": "nnz/s", "n_gpus": args.gpus,
        "steps": len(r["ms"]), "warmup": r["warmup"], "ms_per_step": r["median_ms"], "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, c), "layout": "fp64 column-major (reference DenseMatrix)"},
        "cpu_baseline": {"value": r["value"], "unit": "nnz/s", "cores": r["cores"], "kind": "reference",
                         "sample": r["sample"]},
        "e2e": {"value": r["value"], "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "construct_s": r["construct_s"],
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- our arm
def stage2_line(args, m, B, d, gemm_ms):
    """Stage 2 (Z = G.(S.X)) against its own roofline: the int8 tcgen05 kernel (ozgemm.cu)
    for large Z -- S(S+1)/2 digit products of 2*m*B*d int8 ops each, against the nominal
    dense int8 rate (4.5 POPS; MEASURED_PEAKS.json holds no int8 figure) -- else the FP64
    DMMA kernels against the measured 37.2 TFLOP/s DMMA peak."""
    if gemm_ms <= 0:
        return None
    opts = dict(o.split("=", 1) for o in args.opt)
    S = int(opts.get("oz_slices", 7))
    min_z = int(opts.get("oz_min_z", 16384))
    g_mem = m * B * 8 <= (4 << 30) and opts.get("g_resident", "1") != "0"
    fp64_flop = 2.0 * m * B * d
    if S > 0 and g_mem and m * d >= min_z and m <= 4096 and d <= 4096:
        ops = S * (S + 1) / 2 * fp64_flop
        tops = ops / (gemm_ms / 1e3) / 1e12
        return {"kernel": f"oz_gemm<{S}> (tcgen05.mma kind::i8, FP64 emulated by {S} digit planes)",
                "bound": "tensor", "achieved": tops, "peak": 4500.0, "unit": "int8 TOPS", "frac": tops / 4500.0,
                "peak_source": "nominal dense int8 (B200)", "fp64_equiv_tflops": fp64_flop / (gemm_ms / 1e3) / 1e12,
                "ms": gemm_ms}
    tf = fp64_flop / (gemm_ms / 1e3) / 1e12
    return {"kernel": "gemm_dmma (FP64 DMMA, mma.sync m8n8k4)", "bound": "tensor", "achieved": tf, "peak": 37.2,
            "unit": "TFLOP/s", "frac": tf / 37.2, "peak_source": "measured DMMA (tools/microbench/fp64_peak.cu)",
            "ms": gemm_ms}


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    # CGX_BENCH_BACKEND=gloo: functional check of the N>1 plumbing with every rank on the
    # visible GPU(s) (host-side collectives, no device-side waits between ranks); its
    # timings mean nothing.  The measured path is NCCL with one GPU per rank.
    backend = os.environ.get("CGX_BENCH_BACKEND", "nccl")
    if backend == "gloo":
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    import paper_1606_05732_b200 as cg
    from paper_1606_05732_b200 import bench_data
    from paper_1606_05732_b200.distributed import shard_range

    c = CONFIGS[args.config]
    ctx = cg.context(local)
    for kv in args.opt:
        k, v = kv.split("=", 1)
        ctx.set_option(k, int(v))
    n, d, B, m = c["n"], c["d"], c["B"], c["m"]
    if args.scaling == "weak":
        # X grows with N: N shards of the config's n rows each (rows are independent units;
        # the only exchange is the all-reduce of the m x d partial Z)
        n = n * world
    r0, r1 = shard_range(n, world, rank)
    rows = r1 - r0
    t_seed = cg.SeededRng(SEED).next_u64()
    hash_place = args.placement == "hash"
    if hash_place and (c["kind"] != "dense" or args.combine != "z"):
        raise SystemExit("--placement hash: dense configs and --combine z only")

    # inputs in HBM
    t_hash = None
    if hash_place:
        from paper_1606_05732_b200.distributed import bucket_range

        b0, b1 = bucket_range(B, world, rank)
        t0 = time.perf_counter()
        t_hash = cg.api.countgauss_bucket_shard(m, B, n, b0, b1, t_seed, ctx=ctx)
        torch.cuda.synchronize()
        construct_hash_ms = (time.perf_counter() - t0) * 1e3
        grows = cg.api.xform_rows(t_hash, device=dev)
        rows = grows.numel()
    if c["kind"] == "dense" and hash_place:
        dt = torch.float32 if c["dtype"] == "f32" else torch.float64
        if c.get("gen") == "separable":
            raise SystemExit("--placement hash: not for the separable generator")
        x = bench_data.dense_normal_rows(grows, d, seed=data_seed(args.config), dtype=dt, device=local)
        nnz_local = rows * d
        x_bytes = rows * d * x.element_size()
        del grows
    elif c["kind"] == "dense":
        dt = torch.float32 if c["dtype"] == "f32" else torch.float64
        if c.get("gen") == "separable":
            x = bench_data.dense_separable(rows, d, seed=data_seed(args.config), r=c["r"], alpha=c["alpha"],
                                           sigma=c["sigma"], dtype=dt, row0=r0, device=local)
        else:
            x = bench_data.dense_normal(rows, d, seed=data_seed(args.config), dtype=dt, row0=r0, device=local)
        nnz_local = rows * d
        x_bytes = rows * d * x.element_size()
    else:
        if "zipf" in c:
            s_len, cap, s_col = c["zipf"]
            x = bench_data.csr_zipf(rows, d, seed=data_seed(args.config) + r0, s_len=s_len, cap=cap, s_col=s_col,
                                    device=local)
        else:
            x = bench_data.csr_bernoulli(rows, d, c["density"], seed=data_seed(args.config) + r0, device=local)
        nnz_local = x.nnz()
        x_bytes = nnz_local * 8 + (rows + 1) * 8
    torch.cuda.synchronize()

    # transform construction (per-transform work, timed separately: the reference's
    # countgauss_new is likewise outside countgauss_apply)
    if hash_place:
        t, construct_ms = t_hash, construct_hash_ms
    else:
        t0 = time.perf_counter()
        t = cg.api.countgauss_new_shard(m, B, n, r0, rows, t_seed, ctx=ctx)
        torch.cuda.synchronize()
        construct_ms = (time.perf_counter() - t0) * 1e3

    stream = torch.cuda.current_stream(dev)
    zbuf = torch.empty((d, m), dtype=torch.float64, device=dev)  # contiguous storage of Z^T
    z = zbuf.t()  # column-major m x d view (the reference layout)

    from paper_1606_05732_b200.distributed import PeerLanding, combine, combine_p2p

    landing = PeerLanding(ctx, world, rank, B, d) if world > 1 and args.combine == "p2p" else None

    sxbuf = torch.empty((B, d), dtype=torch.float64, device=dev) if world > 1 and args.combine in ("sx", "sxo", "g") else None
    sxT = torch.empty((d, B), dtype=torch.float64, device=dev) if world > 1 and args.combine == "cols" else None

    comb_ev = []  # (start, end) CUDA events around the combine phase of each timed step

    def mark():
        if timing_combine:
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            return e
        return None

    def step():
        if world == 1 or args.combine == "z":
            cg.api.countgauss_apply_into(t, x, z)
            if world > 1:
                e0 = mark()
                dist.all_reduce(zbuf)  # partial Z of every row shard -> full Z on every rank
                if e0 is not None:
                    comb_ev.append((e0, mark()))
            return z
        if args.combine == "p2p":  # the sketch stores its rows into the owners' landing slots (peer memory)
            e0 = mark()
            out = combine_p2p(landing, lambda bases, per: cg.api.countsketch_apply_to(t, x, bases, per),
                              lambda sl, b0, b1: cg.api.gauss_gemm_range(t, sl, b0, b1), m=m)
            if e0 is not None:
                comb_ev.append((e0, mark()))
            return out
        if args.combine == "cols":
            cg.api.countsketch_apply_into(t, x, sxT.t())  # partial S.X, column-major
            e0 = mark()
            out = combine("cols", world=world, rank=rank, B=B, d=d, m=m, partial_sx=sxT,
                          stage2=lambda blk, c0, c1: cg.api.gauss_gemm(t, blk.t()).t())
        else:
            cg.api.countsketch_apply_into(t, x, sxbuf)  # partial S.X (row-major B x d)
            e0 = mark()
            if args.combine in ("sx", "sxo"):
                out = combine(args.combine, world=world, rank=rank, B=B, d=d, m=m, partial_sx=sxbuf,
                              stage2=lambda sl, b0, b1: cg.api.gauss_gemm_range(t, sl, b0, b1))
            else:
                out = combine("g", world=world, rank=rank, B=B, d=d, m=m, partial_sx=sxbuf,
                              stage2=lambda sx, r0, r1: cg.api.gauss_gemm_rows(t, sx, r0, r1))
        if e0 is not None:
            comb_ev.append((e0, mark()))
        return out

    timing_combine = False
    nmf = c.get("gen") == "separable"
    anchors = []

    def full_step():
        zz = step()
        if nmf:  # cg_nmf (nmf.cpp:141-153): the anchors of Z, read back to the host
            anchors.append(cg.select_extremes(zz, ctx=ctx))
        return zz

    for _ in range(args.warmup):
        full_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ctx.profile(True)
    launches0 = ctx.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        timing_combine = world > 1
        ev0.record(stream)
        for _ in range(args.steps):
            full_step()
        ev1.record(stream)
        torch.cuda.synchronize()
        timing_combine = False
        if world > 1:
            dist.barrier()
    launches = ctx.launches - launches0
    elapsed_ms = ev0.elapsed_time(ev1)
    sk_ms, sk_n = ctx.profile_read(0)
    gm_ms, gm_n = ctx.profile_read(1)
    ctx.profile(False)

    tot_units = nnz_local
    if world > 1:
        tt = torch.tensor([elapsed_ms, float(nnz_local)], dtype=torch.float64, device=dev)
        mx = tt.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = tt.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        elapsed_ms = float(mx[0])
        tot_units = float(sm[1])
    ms_per_step = elapsed_ms / args.steps
    value = tot_units / (ms_per_step / 1e3)

    # Roofline of the dominant kernel, per launch.  Stage 0 is the one-pass kernel
    # (sketch + G generation + contraction: S.X and G never touch HBM) when gm_n == 0,
    # else the stage-1 sketch kernel, which also writes S.X (B*d*8 bytes).
    peak, peak_kind = peaks()
    fused = gm_n == 0
    bytes_alg = x_bytes + (0 if fused else B * d * 8)
    if c["kind"] == "dense":
        kernel_name = ("countgauss_dense_ws (one pass: sketch + G + G.(S.X))" if fused
                       else "sketch_dense_async (stage 1: cp.async row gather -> S.X)")
    else:
        opts = dict(o.split("=", 1) for o in args.opt)
        mode = int(opts.get("csr_mode", 0))
        record = mode == 3 or (mode == 0 and nnz_local / rows < 8.0 and B * d >= (1 << 22) and nnz_local >= (1 << 22))
        kernel_name = ("sketch phase, CSR record path (csr_atomic.cu: count + scatter + L2-atomic accumulate -> S.X)"
                       if record else "sketch_csr_lean (stage 1: bucket-ordered row gather -> S.X)")
    sk_avg_ms = sk_ms / max(sk_n, 1)
    achieved = bytes_alg / (sk_avg_ms / 1e3) / 1e9
    traffic = None  # DRAM bytes per launch of this kernel, from the committed ncu capture
    try:
        tr = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")))
        ent = tr.get(args.config)
        if ent and world == 1 and ent["kernel"] in kernel_name and ent.get("bytes"):
            traffic = ent["bytes"]
    except (OSError, ValueError, KeyError):
        traffic = None

    # The hardware rate that bounds the kernel when it is not HBM bandwidth,
    # each measured on this GPU by a committed microbenchmark: random 128 B rows for the dense
    # gather (d*4 <= 128 B rows), random 64 B DRAM accesses for the CSR gather, and for the
    # record path the sum of its three kernels' floors (count and scatter at the measured copy
    # rate on their DRAM bytes, the accumulate at the L2 atomic-unit rate on its nnz REDs).
    ceiling = None
    if world == 1 and not fused:
        if c["kind"] == "dense" and d * x.element_size() <= 128:
            ceiling = {"what": "random 128 B-row gather rate (tools/microbench/gather_bw.cu)", "rate": 5950.0,
                       "unit": "GB/s", "achieved": achieved, "frac": achieved / 5950.0}
        elif c["kind"] == "csr" and "record" in kernel_name:
            # count: row offsets + a 4 B row record; scatter: row offsets + row records +
            # the nonzeros (8 B) read and their 8 B records written (ncu on c3: 0.78, 3.52 GB)
            count_b = (rows + 1) * 8 + rows * 4
            scatter_b = (rows + 1) * 8 + rows * 4 + nnz_local * 16
            floor_ms = (count_b + scatter_b) / (peak * 1e9) * 1e3 + nnz_local / 187e9 * 1e3
            ceiling = {"what": "count + scatter DRAM bytes at the measured copy rate, plus one L2 RED per "
                               "nonzero at 187 G/s (tools/microbench/red_types.cu)",
                       "floor_ms": floor_ms, "achieved_ms": sk_avg_ms, "frac": floor_ms / sk_avg_ms}
        elif c["kind"] == "csr" and traffic:
            acc = traffic / 64.0 / (sk_avg_ms / 1e3)
            ceiling = {"what": "random 64 B DRAM accesses per second (ncu DRAM bytes / 64) against the best "
                               "rate of independent random loads on this GPU (tools/microbench/random_access.cu "
                               "sweep: 36.5-49.7e9/s)",
                       "rate": 49.7e9, "unit": "accesses/s", "achieved": acc, "frac": acc / 49.7e9}

    # e2e: same call with X in pinned host memory (H2D + D2H inside the timed region)
    e2e = None
    if c["kind"] == "csr" and not args.no_e2e:
        hx = cg.SparseMatrix(x.rows, x.cols, *(torch.empty(a.shape, dtype=a.dtype, pin_memory=True).copy_(a).numpy()
                                               for a in (x.row_offsets, x.col_indices, x.values)))
        cg.countgauss_apply(t, hx)
        if world > 1:
            dist.barrier()
        ts = []
        k_e2e = max(1, min(args.steps, 5))
        for _ in range(k_e2e):
            a = time.perf_counter()
            zh = cg.countgauss_apply(t, hx)  # synchronous: returns with Z on the host
            if world > 1:
                zt = torch.from_numpy(zh.copy()).to(dev)
                dist.all_reduce(zt)
                zh = zt.cpu().numpy()
            ts.append(time.perf_counter() - a)
        e_s = statistics.median(ts)
        if world > 1:
            tt = torch.tensor([e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_s = float(tt[0])
        e2e = {"value": tot_units / e_s, "unit": "nnz/s", "h2d_bytes_per_step": int(x_bytes),
               "d2h_bytes_per_step": int(m * d * 8), "ms_per_step": e_s * 1e3, "steps": k_e2e,
               "how": "cgx_countgauss_apply_csr with host (pinned) int64 row offsets, int32 columns, fp32 values; "
                      "wall clock, median"}
        del hx
    if c["kind"] == "dense" and not args.no_e2e:
        xh = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        xh.copy_(x)
        zh = None
        for _ in range(1):
            zh = cg.countgauss_apply(t, xh.numpy())
        if world > 1:
            dist.barrier()
        ts = []
        k_e2e = max(1, min(args.steps, 5))
        for _ in range(k_e2e):
            a = time.perf_counter()
            zh = cg.countgauss_apply(t, xh.numpy())  # synchronous: returns with Z on the host
            if world > 1:
                zt = torch.from_numpy(zh.copy()).to(dev)
                dist.all_reduce(zt)
                zh = zt.cpu().numpy()
            ts.append(time.perf_counter() - a)
        e_s = statistics.median(ts)
        if world > 1:
            tt = torch.tensor([e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_s = float(tt[0])
        e2e = {"value": tot_units / e_s, "unit": "nnz/s", "h2d_bytes_per_step": int(x_bytes),
               "d2h_bytes_per_step": int(m * d * 8), "ms_per_step": e_s * 1e3, "steps": k_e2e,
               "how": "cgx_countgauss_apply_dense with x_mem=HOST (pinned), wall clock, median"}
        del xh

    # e2e through the reference's own C++ API (cg::countgauss_apply(t, DenseMatrix /
    # SparseMatrix): fp64 column-major / int64+fp64 CSR in pageable std::vector storage),
    # the drop-in (integration/countgauss_gpu.cpp + libcgx) against the same program linked
    # with the reference library (integration/dropin_bench.cpp, built by oracle/Makefile).
    e2e_dropin = None
    if rank == 0 and world == 1 and not args.no_e2e and args.config in ("c1", "c2", "c3", "c4"):
        e2e_dropin = run_dropin(args.config, c)

    # Ablation (the reference's bench reports it too, countgauss_main.cpp:535-547): the
    # dense-Gaussian projection G~.X (m x n Gaussian, generated on the GPU, never stored) on
    # the same X -- dense or CSR -- untimed by the main metric.
    ablation = None
    if world == 1 and not args.no_ablation:
        rng = cg.SeededRng(SEED)
        cg.gaussian_project(x, m, rng)  # warm-up
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3 if c["kind"] == "dense" else 1
        e0.record(stream)
        for _ in range(reps):
            cg.gaussian_project(x, m, rng)
        e1.record(stream)
        torch.cuda.synchronize()
        dense_ms = e0.elapsed_time(e1) / reps
        ablation = {"dense_gaussian_ms": dense_ms, "countgauss_ms": ms_per_step,
                    "speedup_vs_dense": dense_ms / ms_per_step,
                    "what": (f"G~.X with G~ = gaussian_matrix({m}, {n}, rng) generated in-GPU (gp_nmf, nmf.cpp:155-159)"
                             if c["kind"] == "dense" else
                             f"G~.X for CSR X, G~ = gaussian_matrix({m}, {n}, rng) generated in-GPU: the reference "
                             "bench's O(nnz*m) loop (countgauss_main.cpp:535-547), the config-5 ablation")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            r = cpu_reference_run(args.config, c, 1, 1)
            cpu = {"value": r["value"], "unit": "nnz/s", "cores": r["cores"], "kind": "reference",
                   "sample": r["sample"]}
        except Exception as exc:  # reported, not fatal
            cpu = {"value": None, "unit": "nnz/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {
                "workload": workload_name(args.config, c), "n": n, "d": d, "B": B, "m": m,
                "rows_per_rank": rows, "nnz_per_rank": int(nnz_local), "mean_row_nnz": nnz_local / rows,
                "placement": ("hash: each rank holds the rows hashing into its bucket range, in (bucket, row) order "
                              "(SURVEY 8e ablation C): the sketch reads X sequentially, S.X slices are final, stage 2 "
                              "is split-K over G[:, b0:b1)") if hash_place else "rows: contiguous row shards",
                "parallelism": f"rows sharded x{world} ({args.scaling} scaling: "
                + ("the config's n rows per rank" if args.scaling == "weak" else "the config's n rows split across ranks")
                + ")" + ({"z": ", NCCL all-reduce of Z", "sx": ", NCCL reduce-scatter of S.X + split-K stage 2 + all-reduce of Z",
                       "p2p": ", sketch kernels store S.X rows into the owners' landing buffers over peer memory (CUDA IPC), host barrier, slot sums in rank order + split-K stage 2 + all-gather of Z summed in rank order",
                       "sxo": ", NCCL all-to-all of S.X bucket ranges summed in rank order + split-K stage 2 + all-gather of Z summed in rank order",
                       "g": ", NCCL all-reduce of S.X + G's m rows split over ranks + all-gather of Z",
                       "cols": ", NCCL column reduce-scatter of S.X + split-N stage 2 + all-gather of Z"}[args.combine]
                      if world > 1 else ""),
                "input_dtype": c.get("dtype", "f32"), "accumulate": "f64 (S.X and G.(S.X))",
                "l2": f"inputs larger than L2 ({x_bytes / 1e9:.2f} GB X per rank), no flush",
                "construct_ms": construct_ms,
                "G": ("materialized once per transform (countgauss_new, like the reference's t.g), read by apply"
                      if c["m"] * c["B"] * 8 <= (4 << 30) and not any(o.startswith("g_resident=0") for o in args.opt)
                      else "generated inside the apply kernels"),
                "options": args.opt,
                **({"anchors": anchors[-1].unioned, "anchors_stable": all(a == anchors[-1] for a in anchors),
                    "step": "countgauss_apply + select_extremes (cg_nmf without its countgauss_new)"}
                   if nmf else {}),
                "stage_ms": {"sketch": sk_avg_ms, "gemm": gm_ms / max(gm_n, 1),
                             **({"combine": sum(a.elapsed_time(b) for a, b in comb_ev) / len(comb_ev),
                                 "combine_what": "rank 0: the NCCL collectives"
                                 + (" and the stage 2 inside the combine" if args.combine != "z" else "")}
                                if comb_ev else {})},
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "kernel": kernel_name,
                         "bytes_per_launch": bytes_alg, "peak_source": peak_kind, "ceiling": ceiling},
            "stage2": stage2_line(args, m, B, d, gm_ms / max(gm_n, 1)),
            "e2e": e2e,
            "e2e_dropin": e2e_dropin,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "ablation": ablation,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        if landing is not None:
            landing.close()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=600)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ablation", action="store_true", help="skip the dense-Gaussian G~.X ablation")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default, the north star's split): the config's n rows split N ways; weak: each "
                         "rank sketches the config's n rows (X has N*n rows)")
    ap.add_argument("--opt", action="append", default=[], metavar="KEY=VALUE",
                    help="cgx_set_option before timing (A/B of kernel variants)")
    ap.add_argument("--placement", default="rows", choices=["rows", "hash"],
                    help="rows: contiguous row shards; hash: each rank holds the rows hashing into its bucket "
                         "range, in bucket order (SURVEY 8e ablation C; dense configs; combine = all-reduce of Z)")
    ap.add_argument("--combine", default="auto", choices=["auto", "z", "sx", "sxo", "p2p", "g", "cols"],
                    help="N>1 combine (auto: g for dense configs, sx for CSR -- the north star's schemes): z = all-reduce of Z; sx = reduce-scatter of S.X + split-K stage 2 + "
                         "all-reduce; sxo = sx with all-to-all / all-gather and sums in rank order (same bits on every rank); p2p = sxo with the S.X exchange fused into the sketch kernels' stores over peer memory (CUDA IPC landing buffers; host barrier per step); g = all-reduce of S.X + G's m rows split over ranks + all-gather; "
                         "cols = column reduce-scatter of S.X + split-N stage 2 + all-gather")
    args = ap.parse_args()
    if args.combine == "auto":
        args.combine = "g" if CONFIGS[args.config]["kind"] == "dense" else "sx"
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3", file=sys.stderr)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
