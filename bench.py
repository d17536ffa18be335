#!/usr/bin/env python
"""ACE hot-path benchmark (BASELINE.json metric: ACE points/sec, hash + insert
+ score, on 1 B200; roofline fraction reported beside it).

Prints one JSON line per BASELINE configuration, configs 1-4 first and the
headline last: config 5, the largest single-GPU workload (100M points,
streamed in 65,536-point batches: score against the counts at batch start,
flag score <= mean - alpha, insert; ace_cli.cpp:173-186 / detect.cpp:76-84).
A batch-config step is reset + build_sketch + detect_batch over the config's
rows (ace_sketch_build_detect); the stream step is the whole 100M-row stream
from an empty sketch (ace_sketch_stream_run).  Inputs are resident in HBM
(all larger than the 126 MB L2, so no flush is needed) for `value`; `e2e`
is the same call with the rows in pinned host memory and the flags returned to
the host.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C ...]
  python bench.py --impl reference ...   # the reference's CPU implementation
  python bench.py --api point [--impl reference]   # the per-point API

--api point times the reference's only API, one query at a time, as
ace_cli stream --adapt drives it (ace_cli.cpp:173-183): detect_stream then
insert per query through the C++ drop-in headers (include/ace/*.hpp,
tests/cpp/point_bench.cpp) after a sketch built from one 65,536-row batch;
a step is 1,000 queries.

Multi-GPU (torchrun): replicas only -- each rank runs the full workload on its
own GPU (the north star is single-GPU, no inter-GPU exchange); value = total
points of all ranks / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ACE points/sec (hash+insert+score) on 1 B200; % of binding FP32/HBM/L2-atomic roofline"
UNIT = "points/s"
ORDER = [1, 2, 3, 4, 5]  # the headline (config 5) last
STREAM_PIPE = 90  # config 5: projection SMs while pipelined beside the stream kernel (0 = not pipelined)
STREAM_GROUP = 8  # config 5: batches per hashing launch (lookahead of the stream driver)

# bounded CPU samples (rows): cpu_baseline leg (~10 s of reference CPU work
# per config) and the --impl reference arm (~1 s per step)
CPU_SAMPLE = {1: 100_000, 2: 150_000, 3: 40_000, 4: 1_500, 5: 3 * 65_536}
REF_SAMPLE = {1: 20_000, 2: 10_000, 3: 4_000, 4: 160, 5: 16_384}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d, src = json.loads(p.read_text()), "measured (MEASURED_PEAKS.json)"
    else:
        d, src = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"
    # dense TF32: the tcgen05 peak of the fp32 input dtype,
    # measured on this pool's B200 by scripts/tf32_peak.py; else half of bf16
    t = ROOT / "profiles" / "r2_tf32_peak.json"
    if t.exists():
        d["tf32_tflops"] = json.loads(t.read_text())["tf32_tflops"]
        d["tf32_source"] = "measured (profiles/r2_tf32_peak.json, torch.matmul fp32+TF32 8192^3)"
    else:
        d["tf32_tflops"] = 0.5 * d["bf16_tflops"]
        d["tf32_source"] = "half the bf16 dense peak (fallback)"
    return d, src


def step_roofline(w, value, pk):
    """The metric's binding roofline for the whole step:
    points/s = min(projection peak / (2 d K L), HBM / (4 d), L2 RED rate / L),
    with the tcgen05 dense peak of the fp32 input dtype (TF32, measured), the
    measured HBM copy bandwidth and the
    measured random-address L2 RED rate (profiles/r1_peaks_probe.json) for
    this counter array.  This design counts in shared-memory histograms, so
    the L2-atomic term is the metric's definition rather than a limit of the
    implementation; the binding term without it is reported beside it."""
    probe = ROOT / "profiles" / "r1_peaks_probe.json"
    red = None
    if probe.exists():
        d = json.loads(probe.read_text())
        rates = {int(k): v for k, v in d.get("l2_red_u32_gops", {}).items()}
        if rates:
            size = w.num_tables * (4 << w.k_bits)
            red = rates[min(rates, key=lambda k: abs(k - size))] * 1e9
    f = 2.0 * w.dim * w.k_bits * w.num_tables
    proj = pk["tf32_tflops"] * 1e12 / f
    hbm = pk["hbm_gbs"] * 1e9 / (4.0 * w.dim)
    terms = {"projection_pts_s": proj, "hbm_x_read_pts_s": hbm}
    if red:
        terms["l2_atomic_pts_s"] = red / w.num_tables
    bind = min(terms, key=terms.get)
    no_atomic = min(proj, hbm)
    return {"binding": bind.replace("_pts_s", ""), "binding_pts_s": terms[bind], "frac": value / terms[bind],
            "terms": terms, "frac_without_atomic_term": value / no_atomic,
            "source": "SURVEY.md 8(d); HBM from MEASURED_PEAKS.json, TF32 from profiles/r2_tf32_peak.json, "
                      "L2 RED rate from profiles/r1_peaks_probe.json"}


class Clocks:
    """nvidia-smi sampling during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [v.strip() for v in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def _profiled_traffic(kernel: str, cfg: int):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    summaries (profiles/traffic.json), or None."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return d.get(f"cfg{cfg}", {}).get(kernel)


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(value: float, ws: int) -> float:
    """Replicas: the job's time is the slowest rank's (all-reduce MAX; CUDA
    tensor under NCCL, CPU tensor under gloo)."""
    if ws <= 1:
        return value
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([value], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(points_per_rank: int, ws: int, ms_max: float) -> float:
    """Whole-job points/s of N independent replicas (weak scaling)."""
    return points_per_rank * ws / (ms_max * 1e-3)


def sample_rows(cfg: int, rows: int):
    """Host rows of a bounded CPU sample, generated in this process only for
    the compiled reference (the reference arm does not load the repo's
    generator library: see ref_rows)."""
    from paper_1706_06664_b200 import workloads as W
    return W.host_rows(cfg, 0, rows)[0]


def cpu_baseline(cfg: int, x) -> dict:
    """The compiled reference (oracle/_ref) on a bounded sample of the
    workload on the host cores: batch configs insert on one core (single
    writer, sketch.hpp:23-24) then detect_batch on all cores; config 5 in
    stream order (per 65,536-row batch: detect_stream on all cores, then the
    inserts on one core).  The C restatement (oracle/) if the reference was
    not built."""
    from oracle import REF_SO, Oracle, Reference
    from paper_1706_06664_b200 import workloads as W
    w = W.CONFIGS[cfg]
    n = x.shape[0]
    cores = os.cpu_count() or 1
    if REF_SO.exists():
        ref = Reference()
        if w.mode == "stream":
            ts, ti, _ = ref.time_stream(w.w_seed, x, w.k_bits, w.num_tables, w.batch, w.alpha)
            what = (f"first {n} rows of config {cfg} in {w.batch}-row batches: detect_stream on {cores} threads "
                    f"({ts:.2f} s), inserts on 1 core ({ti:.2f} s)")
            secs = ts + ti
        else:
            ti, td, _ = ref.time_build_detect(w.w_seed, x, w.k_bits, w.num_tables, 0)
            what = f"first {n} rows of config {cfg}: insert on 1 core ({ti:.2f} s), detect_batch on {cores} threads ({td:.2f} s)"
            secs = ti + td
        kind = "reference"
    else:
        o = Oracle()
        t0 = time.perf_counter()
        wm = o.directions(w.w_seed, w.dim, w.k_bits, w.num_tables)
        ids, _ = o.buckets(wm, x, w.k_bits, w.num_tables, threads=1, fast=False)
        sk = o.sketch(w.k_bits, w.num_tables, 32)
        sk.insert_ids(ids)
        sk.score_ids(ids)
        secs = time.perf_counter() - t0
        kind, cores = "port", 1
        what = f"first {n} rows of config {cfg}, the C restatement on one core"
    return {"value": n / secs, "unit": UNIT, "cores": cores, "kind": kind, "sample": what}


def ref_rows(cfg: int, rows: int):
    """Reference-arm input rows, generated by a separate process into a .npy
    file so this process loads only the compiled reference (oracle/_ref)."""
    out = Path("/tmp") / f"ace_ref_rows_cfg{cfg}_{rows}.npy"
    if not out.exists():
        code = ("import sys, numpy as np; sys.path.insert(0, %r); "
                "from paper_1706_06664_b200 import workloads as W; "
                "np.save(%r, W.host_rows(%d, 0, %d)[0])") % (str(ROOT), str(out), cfg, rows)
        subprocess.run([sys.executable, "-c", code], check=True)
    return np.load(out)


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref, compiled from the unmodified sources) on the box's host
    cores, each step a bounded sample of the config's workload."""
    ws, rank, _ = dist_setup()
    if rank != 0:
        return
    from paper_1706_06664_b200 import workloads as W
    if args.api == "point":
        for cfg in args.config:
            cb = run_point_ref(args, cfg, args.steps, args.warmup)
            line = point_line(cfg, "reference", cb["value"], cb["ms_per_step"], args, ws)
            line["impl"] = "reference"
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            line["e2e"] = {"value": cb["value"], "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
            line["reported"] = cb["reported"]
            print(json.dumps(line), flush=True)
        return
    for cfg in args.config:
        w = W.CONFIGS[cfg]
        x = ref_rows(cfg, REF_SAMPLE[cfg])
        times = []
        cb = None
        for i in range(args.warmup + args.steps):
            cb = cpu_baseline(cfg, x)
            if i >= args.warmup:
                times.append(x.shape[0] / cb["value"])
        t = statistics.mean(times)
        value = x.shape[0] / t
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (datagen cfg {cfg}, seed {w.data_seed})",
            "config": {"workload": f"cfg{cfg} {w.name}: {'stream' if w.mode == 'stream' else 'build_sketch + detect_batch'}"
                                   f" (reference CPU, sample of {x.shape[0]} rows per step)",
                       "N": x.shape[0], "d": w.dim, "K": w.k_bits, "L": w.num_tables},
            "cpu_baseline": {**cb, "value": value},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)


POINT_BUILD, POINT_STEP = 65_536, 1_000  # per-point API: sketch built from one batch; queries per step


def point_rows(cfg: int, queries: int):
    """Rows of the per-point workload (build batch + queries), float32, in a
    file (the C++ program reads it)."""
    n = POINT_BUILD + queries
    f = Path("/tmp") / f"ace_point_rows_cfg{cfg}_{n}.f32"
    if not f.exists():
        ref_rows(cfg, n).astype(np.float32).tofile(f)
    return f, n


def run_point_ref(args, cfg: int, steps: int, warmup: int) -> dict:
    """The reference's per-point loop (oracle/_ref ref_time_point: the
    unmodified reference's detect_stream + insert per query, one core)."""
    from oracle import REF_SO, Oracle, Reference
    from paper_1706_06664_b200 import workloads as W
    w = W.CONFIGS[cfg]
    q = (steps + warmup) * POINT_STEP
    x = ref_rows(cfg, POINT_BUILD + q)
    if REF_SO.exists():
        # warm-up queries are the first `warmup` steps of the same loop: time
        # the whole loop and each part by its query count (per-query cost is flat)
        sec, rep = Reference().time_point(w.w_seed, x, POINT_BUILD, w.k_bits, w.num_tables, w.alpha)
        kind = "reference"
    else:
        o = Oracle()
        wm = o.directions(w.w_seed, w.dim, w.k_bits, w.num_tables)
        t0 = time.perf_counter()
        ids, _ = o.buckets(wm, x, w.k_bits, w.num_tables, threads=1, fast=False)
        sk = o.sketch(w.k_bits, w.num_tables, 32)
        sk.insert_ids(np.ascontiguousarray(ids[:, :POINT_BUILD]))
        t1 = time.perf_counter()
        rep = 0
        for i in range(POINT_BUILD, x.shape[0]):
            f, _ = sk.stream_ids(np.ascontiguousarray(ids[:, i:i + 1]), w.alpha)
            rep += int(f[0])
        sec = time.perf_counter() - t1 + (t1 - t0) * q / x.shape[0]
        kind = "port"
    per_q = sec / q
    return {"value": 1.0 / per_q, "unit": "queries/s", "cores": 1, "kind": kind,
            "sample": f"cfg {cfg}: sketch from {POINT_BUILD} rows, then {q} queries of detect_stream + insert "
                      f"one at a time on one core ({sec:.2f} s)", "ms_per_step": per_q * POINT_STEP * 1e3,
            "reported": rep}


def point_line(cfg: int, impl: str, value: float, ms: float, args, ws: int) -> dict:
    from paper_1706_06664_b200 import workloads as W
    w = W.CONFIGS[cfg]
    return {
        "metric": "per-point API queries/s (detect_stream + insert per query, ace_cli stream --adapt)",
        "value": value, "unit": "queries/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (datagen cfg {cfg}, seed {w.data_seed})",
        "config": {"workload": f"cfg{cfg} {w.name}: per-point detect_stream + insert through the C++ drop-in "
                               f"(include/ace/*.hpp), sketch built from {POINT_BUILD} rows, {POINT_STEP} queries "
                               f"per step", "d": w.dim, "K": w.k_bits, "L": w.num_tables, "alpha": w.alpha,
                   "api": "point"},
    }


def run_point(args, cfg, ws, rank, local, N):
    """--api point, this implementation: tests/cpp/point_bench.cpp (the C++
    drop-in, libace.so over libace_dev.so) runs the loop; wall clock around
    the timed queries (a host API: every query's row goes in and its score
    and flag come back)."""
    from paper_1706_06664_b200 import workloads as W
    w = W.CONFIGS[cfg]
    q, wq = args.steps * POINT_STEP, max(3, args.warmup) * POINT_STEP
    f, _ = point_rows(cfg, wq + q)
    clocks = Clocks(local)
    clocks.start()
    r = subprocess.run([str(N.LIB_DIR / "ace_point_bench"), str(w.dim), str(w.k_bits), str(w.num_tables),
                        str(w.w_seed), repr(w.alpha), str(POINT_BUILD), str(wq), str(q), str(f)],
                       capture_output=True, text=True, check=True)
    clk = clocks.stop()
    sec, rep, p50, p99, tdet, launches = r.stdout.split()
    sec = max_over_ranks(float(sec), ws)
    value = q * ws / sec
    ms = sec / args.steps * 1e3
    line = point_line(cfg, "ace", value, ms, args, ws)
    pk, pk_src = peaks()
    per_q_s = sec / q
    bytes_q = w.num_tables * w.k_bits * w.dim * 8.0  # W (binary64) read per query's folds
    line.update({
        "latency_us": {"p50": float(p50), "p99": float(p99), "detect_stream_mean": float(tdet),
                       "definition": "wall clock of one detect_stream + insert pair"},
        "roofline": {"bound": "hbm", "achieved": bytes_q / per_q_s / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": bytes_q / per_q_s / 1e9 / pk["hbm_gbs"], "traffic": None,
                     "peak_source": pk_src,
                     "note": "latency-bound: one point_kernel launch (a cluster of 8 CTAs) per query; algorithmic "
                             "bytes = the query's binary64 W read (K L d x 8 B, L2-resident) per query time"},
        "gpu_launches": int(launches) // args.steps, "clocks": clk,
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": POINT_STEP * w.dim * 8,
                "d2h_bytes_per_step": POINT_STEP * 32,
                "note": "the per-point API is the host call itself: the row (binary64) travels in the launch "
                        "parameters, score, sum and state snapshot come back through mapped host memory"},
        "reported": int(rep),
    })
    return line


def roofline_of(kernel_ms, flops, pk, pk_src, w, cfg, ms_step, kname, desc):
    """Dominant-kernel roofline: algorithmic flops (2 d K L per point) per
    launch / live launch time, against the dense tcgen05 peak of the fp32
    input dtype (TF32: "the dense tcgen05 peak of the input
    dtype for tensor kernels"); the bf16 dense fraction and the fraction of
    the 3-pass fp16 split's own ceiling (bf16 peak / 3) are reported beside."""
    peak = pk["tf32_tflops"]
    bf16 = pk["bf16_tflops"]
    ach = flops / (kernel_ms * 1e-3) / 1e12 if kernel_ms > 0 else None
    return {
        "bound": "tensor", "kernel": f"{kname} ({desc})", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
        "frac": ach / peak if ach else None, "traffic": _profiled_traffic(kname, cfg),
        "peak_source": f"dense TF32, {pk['tf32_source']}; algorithmic flops = 2*d*K*L per point, "
                       "the 3 split passes count against achieved",
        "peak_bf16_dense": bf16, "peak_bf16_source": f"{pk_src} (burst)",
        "frac_vs_bf16_dense": ach / bf16 if ach else None,
        "algorithmic_flops_per_launch": flops, "kernel_ms": kernel_ms,
        "kernel_share_of_step": kernel_ms / ms_step if ms_step else None,
        # the exact-sign split runs 3 fp16 MMA passes per projection: bf16
        # peak / 3 is the kernel's ceiling in algorithmic flops
        "split_passes": 3, "frac_of_split_ceiling": 3.0 * ach / bf16 if ach else None,
    }


def run_batch(args, cfg, ws, rank, local, torch, N, ace, W):
    w = W.CONFIGS[cfg]
    n = w.n
    x = torch.empty((n, w.dim), dtype=torch.float32, device="cuda")
    W.device_rows(cfg, 0, n, x.data_ptr())
    torch.cuda.synchronize()
    fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    stream = torch.cuda.current_stream()
    sk.set_stream(stream.cuda_stream)
    flags = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")

    def step():
        sk.reset()
        return sk.build_detect(x, flags_out=flags)

    for _ in range(max(3, args.warmup)):
        rep = step()
    torch.cuda.synchronize()
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    launches0 = N.dev().ace_kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        rep = step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = (N.dev().ace_kernel_launches() - launches0) / args.steps
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, ws)
    # per-phase breakdown: a separate pass with per-phase CUDA events on the
    # sketch's stream (outside the timed region)
    N.dev().ace_sketch_set_timing(sk.handle, 1)
    phase = np.zeros(5)
    ms5 = (C.c_double * 5)()
    phase_steps = max(3, min(args.steps, 10))
    for _ in range(phase_steps):
        step()
        N.dev().ace_sketch_timings(sk.handle, ms5)
        phase += np.array(ms5[:])
    N.dev().ace_sketch_set_timing(sk.handle, 0)
    phase /= phase_steps
    value = replica_value(n, ws, ms)

    e2e = None
    if not args.no_e2e:
        xh = torch.empty((n, w.dim), dtype=torch.float32, pin_memory=True)
        xh.copy_(x)
        xnp = xh.numpy()
        sk_e = ace.AceSketch(fam, ace.CounterWidth.k32)
        sk_e.set_stream(stream.cuda_stream)
        bits = np.zeros((n + 31) // 32, dtype=np.uint32)
        rep_e, st_e = N.AceBatchReport(), N.AceHashStats()
        fn = N.dev().ace_sketch_build_detect

        def e2e_call():
            sk_e.reset()
            rc = fn(sk_e._h, xnp.ctypes.data, N.ACE_F32, n, w.dim, N.ACE_HOST, bits.ctypes.data, None, N.ACE_HOST,
                    C.byref(rep_e), C.byref(st_e))
            if rc != 0:
                raise RuntimeError(N.dev().ace_last_error().decode())

        for _ in range(2):
            e2e_call()
        torch.cuda.synchronize()
        reps = max(3, args.steps // 2)
        t0 = time.perf_counter()
        for _ in range(reps):
            e2e_call()
        torch.cuda.synchronize()
        te = max_over_ranks((time.perf_counter() - t0) / reps, ws)
        e2e = {"value": replica_value(n, ws, te * 1e3), "unit": UNIT, "h2d_bytes_per_step": n * w.dim * 4,
               "d2h_bytes_per_step": ((n + 31) // 32) * 4 + 200,
               "note": "wall clock around the C-ABI call ace_sketch_build_detect (+ sketch reset) with pinned host "
                       "rows in (copied in chunks, each hashed as it lands) and the flag bitmap out to host memory"}
        del xh, xnp, sk_e

    pk, pk_src = peaks()
    flops = 2.0 * w.dim * w.k_bits * w.num_tables * n
    kstream = w.dim > 256
    kname = "hash_tck_kernel" if kstream else "hash_tc_kernel"
    desc = ("tcgen05 fp16x3-split projection, TMEM accumulators, A and W streamed in K chunks" if kstream else
            "tcgen05 fp16x3-split projection of raw fp32 rows loaded by tensor-map TMA, split in-kernel into a "
            "TMEM A operand; sign / near-tie epilogue; bucket packing")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": f"synthetic (datagen cfg {cfg}, seed {w.data_seed})",
        "config": {"workload": f"cfg{cfg} {w.name}: build_sketch + detect_batch",
                   "N": n, "d": w.dim, "K": w.k_bits, "L": w.num_tables, "counter_width": 32,
                   "l2": f"inputs {n * w.dim * 4 / 1e6:.0f} MB > 126 MB L2 (no flush needed)",
                   "parallelism": f"replicas x{ws}"},
        "roofline": roofline_of(phase[4], flops, pk, pk_src, w, cfg, ms, kname, desc),
        "step_roofline": step_roofline(w, value, pk),
        "phases_ms": {"hash_insert": phase[0], "score": phase[1], "threshold_flags": phase[2],
                      "convert_x": phase[3], "projection_kernel": phase[4]},
        "gpu_launches": int(round(launches)),
        "clocks": clk,
        "e2e": e2e,
        "exactness": {"near_ties_1e-6": int(rep.stats.near_ties), "rechecked": int(rep.stats.rechecked),
                      "flipped": int(rep.stats.flipped), "ambiguous": int(rep.ambiguous),
                      "replayed": bool(rep.replayed), "reported": int(rep.reported)},
    }
    del x, flags, sk
    torch.cuda.empty_cache()
    return line


def run_stream(args, cfg, ws, rank, local, torch, N, ace, W):
    """Config 5: the streaming driver over the 100M rows in 65,536-row
    batches; one step = the whole stream from an empty sketch.  Reports
    points/s and p50/p99 of the per-batch latency (start of the batch's work
    to the end of the launch that writes its flags)."""
    w = W.CONFIGS[cfg]
    n = w.n if args.rows is None else min(w.n, args.rows)
    x = torch.empty((n, w.dim), dtype=torch.float32, device="cuda")
    chunk = 8 * 1024 * 1024
    for r0 in range(0, n, chunk):
        m = min(chunk, n - r0)
        W.device_rows(w.cfg, r0, m, x[r0:r0 + m].data_ptr())
    torch.cuda.synchronize()
    fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
    G = args.stream_group
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    sk.set_option(N.ACE_OPT_STREAM_GROUP, G)
    sk.set_option(N.ACE_OPT_STREAM_PIPE, args.stream_pipe)
    stream = torch.cuda.current_stream()
    sk.set_stream(stream.cuda_stream)
    flags = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")

    def step(lat=False):
        sk.reset()
        return sk.stream_run(x, w.batch, w.alpha, flags_out=flags, latencies=lat)

    # per-batch latency from one run with CUDA events around every batch (the
    # timed steps replay the driver's CUDA graph, which records no events)
    _, lat_all, _ = step(lat=True)
    for _ in range(max(3, args.warmup)):
        _, _, rep = step()
    torch.cuda.synchronize()
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    launches0 = N.dev().ace_kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        _, _, rep = step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = (N.dev().ace_kernel_launches() - launches0) / args.steps
    clk = clocks.stop()
    st = sk.last_stats
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, ws)
    value = replica_value(n, ws, ms)
    # phase totals of one more run (events around every launch group)
    N.dev().ace_sketch_set_timing(sk.handle, 1)
    step(lat=False)
    ms5 = (C.c_double * 5)()
    N.dev().ace_sketch_timings(sk.handle, ms5)
    N.dev().ace_sketch_set_timing(sk.handle, 0)
    hash_ms, apply_ms = ms5[4], ms5[2]

    # the throughput / latency trade-off of the driver's options: smaller
    # hashing groups without the pipeline flag each batch sooner
    modes = []
    for g_m, p_m in ((1, 0), (2, 0), (4, 0)):
        if args.rows is not None:
            break
        sk_m = ace.AceSketch(fam, ace.CounterWidth.k32)
        sk_m.set_option(N.ACE_OPT_STREAM_GROUP, g_m)
        sk_m.set_option(N.ACE_OPT_STREAM_PIPE, p_m)
        sk_m.set_stream(stream.cuda_stream)

        def step_m(lat=False):
            sk_m.reset()
            return sk_m.stream_run(x, w.batch, w.alpha, flags_out=flags, latencies=lat)

        _, lat_m, _ = step_m(lat=True)
        for _ in range(3):
            step_m()
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record(stream)
        for _ in range(3):
            step_m()
        m1.record(stream)
        torch.cuda.synchronize()
        modes.append({"hash_group_batches": g_m, "pipeline_sms": p_m,
                      "points_per_s": replica_value(n, ws, max_over_ranks(m0.elapsed_time(m1) / 3, ws)),
                      "p50_ms": float(np.percentile(lat_m, 50)), "p99_ms": float(np.percentile(lat_m, 99))})
        del sk_m

    e2e = None
    if not args.no_e2e:
        # the same call with the rows in pinned host memory (the next hashing
        # group's H2D copy overlaps this group's work) and the flag bitmap
        # returned to host memory
        xh = torch.empty((n, w.dim), dtype=torch.float32, pin_memory=True)
        xh.copy_(x)
        bits = np.zeros((n + 31) // 32, dtype=np.uint32)
        rep_e = N.AceStreamReport()
        st_e = N.AceHashStats()
        fn = N.dev().ace_sketch_stream_run
        sk_e = ace.AceSketch(fam, ace.CounterWidth.k32)
        sk_e.set_option(N.ACE_OPT_STREAM_GROUP, G)
        sk_e.set_option(N.ACE_OPT_STREAM_PIPE, args.stream_pipe)
        sk_e.set_stream(stream.cuda_stream)

        def e2e_call():
            sk_e.reset()
            rc = fn(sk_e._h, xh.data_ptr(), N.ACE_F32, n, w.dim, N.ACE_HOST, w.batch, float(w.alpha),
                    bits.ctypes.data, N.ACE_HOST, None, C.byref(rep_e), C.byref(st_e))
            if rc != 0:
                raise RuntimeError(N.dev().ace_last_error().decode())

        e2e_call()
        torch.cuda.synchronize()
        reps = 3
        t0 = time.perf_counter()
        for _ in range(reps):
            e2e_call()
        torch.cuda.synchronize()
        te = max_over_ranks((time.perf_counter() - t0) / reps, ws)
        e2e = {"value": replica_value(n, ws, te * 1e3), "unit": UNIT, "h2d_bytes_per_step": n * w.dim * 4,
               "d2h_bytes_per_step": ((n + 31) // 32) * 4 + 200,
               "note": "wall clock around the C-ABI call ace_sketch_stream_run (+ sketch reset) with pinned host "
                       "rows in and the flag bitmap out to host memory"}
        del xh, sk_e

    pk, pk_src = peaks()
    nb = -(-n // w.batch)
    groups = -(-nb // G)  # hashing launches of G batches each
    flops_per_launch = 2.0 * w.dim * w.k_bits * w.num_tables * (n / groups)
    roof = roofline_of(hash_ms / groups, flops_per_launch, pk, pk_src, w, cfg, ms / groups, "hash_tc_kernel",
                       "tcgen05 fp16x3-split projection of raw fp32 rows loaded by tensor-map TMA, split in-kernel; "
                       f"per launch: one {G}-batch hashing group ({G * w.batch:,} rows) with its near-tie pass")
    roof["kernel_share_of_step"] = hash_ms / ms if ms else None
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    P = args.stream_pipe
    pipe_on = (P > 0 and w.k_bits <= 15 and w.batch <= 65536 and w.batch % 32 == 0 and nb > G
               and w.num_tables + 4 + P <= sms and P >= 8)
    if pipe_on and roof["achieved"]:
        # pipelined: the projection launch has P of the GPU's SMs (the stream
        # kernel of the previous group runs on the others at the same time), so
        # its roofline is the peak of those P SMs; the whole-GPU fraction beside
        share = P / sms
        ach = roof["achieved"]
        roof.update({
            "sm_share": share, "peak_whole_gpu": roof["peak"], "peak": roof["peak"] * share,
            "frac": ach / (roof["peak"] * share), "frac_of_whole_gpu_peak": ach / roof["peak"],
            "frac_vs_bf16_dense": ach / (roof["peak_bf16_dense"] * share),
            "frac_of_split_ceiling": 3.0 * ach / (roof["peak_bf16_dense"] * share),
            "note": f"the projection launch runs on {P} of {sms} SMs beside the previous group's stream kernel "
                    f"(ACE_OPT_STREAM_PIPE): peak = measured whole-GPU peak x {P}/{sms}; kernel_ms is measured "
                    "in that concurrent run, so the kernels' shares of the step add up to more than 1",
        })
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": f"synthetic (datagen cfg {cfg}, seed {w.data_seed})",
        "config": {"workload": f"cfg{cfg} {w.name}: streaming score -> flag (mean - alpha) -> insert",
                   "N": n, "d": w.dim, "K": w.k_bits, "L": w.num_tables, "batch": w.batch,
                   "hash_group_batches": G,
                   "pipeline": (f"projection of group g+1 on {P} SMs beside the stream kernel of group g on "
                                f"{sms - P} (ACE_OPT_STREAM_PIPE)") if pipe_on else "off",
                   "graph": "the stream driver's device work replayed as one CUDA graph",
                   "alpha": w.alpha, "counter_width": 32,
                   "l2": f"inputs {n * w.dim * 4 / 1e9:.1f} GB > 126 MB L2",
                   "parallelism": f"replicas x{ws}"},
        "roofline": roof,
        "step_roofline": step_roofline(w, value, pk),
        "phases_ms": {"hashing": hash_ms, "stream_kernels": apply_ms},
        "batch_latency_ms": {"p50": float(np.percentile(lat_all, 50)),
                             "p99": float(np.percentile(lat_all, 99)),
                             "max": float(lat_all.max()), "batches_per_step": int(len(lat_all)),
                             "definition": "start of the batch's work (its group's hashing for a group's first "
                                           "batch) to the end of the launch that writes its flags; CUDA events "
                                           "around every batch in one extra run (no graph)"},
        "latency_modes": modes,
        "gpu_launches": int(round(launches)), "clocks": clk, "e2e": e2e,
        "exactness": {"near_ties_1e-6": int(st.near_ties), "rechecked": int(st.rechecked),
                      "flipped": int(st.flipped), "ambiguous": int(rep.ambiguous), "reported": int(rep.reported)},
    }
    del x, flags, sk
    torch.cuda.empty_cache()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, nargs="+", default=ORDER,
                    help="configurations to run, in order (default: 1 2 3 4 5, the headline last)")
    ap.add_argument("--impl", default="ace", choices=["ace", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--rows", type=int, default=None, help="stream mode: limit N (smoke runs)")
    ap.add_argument("--stream-group", type=int, default=STREAM_GROUP,
                    help="stream mode: batches per hashing launch and per stream-kernel launch")
    ap.add_argument("--stream-pipe", type=int, default=STREAM_PIPE,
                    help="stream mode: SMs of the next group's projection beside the stream kernel (0 = off)")
    ap.add_argument("--api", default="batch", choices=["batch", "point"],
                    help="batch: the hot path over each config (default); point: the per-point API")
    args = ap.parse_args()
    if args.api == "point" and args.config == ORDER:
        args.config = [5, 2]
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_1706_06664_b200 import _native as N
    from paper_1706_06664_b200 import ace
    from paper_1706_06664_b200 import workloads as W

    ws, rank, local = dist_setup()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    for cfg in args.config:
        if args.api == "point":
            line = run_point(args, cfg, ws, rank, local, N)
            if rank == 0 and ws == 1 and not args.no_cpu_baseline:
                cb = run_point_ref(args, cfg, 2, 0)
                line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            if rank == 0:
                print(json.dumps(line), flush=True)
            continue
        w = W.CONFIGS[cfg]
        run = run_stream if w.mode == "stream" else run_batch
        line = run(args, cfg, ws, rank, local, torch, N, ace, W)
        if rank == 0 and ws == 1 and not args.no_cpu_baseline:
            n_cpu = min(CPU_SAMPLE[cfg], line["config"]["N"])
            line["cpu_baseline"] = cpu_baseline(cfg, sample_rows(cfg, n_cpu))
        if rank == 0:
            print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
