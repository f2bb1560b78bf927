#!/usr/bin/env python
"""Benchmark of the adaptive solve of A X = B (arXiv 2007.11208) on B200.

One "step" = one call of the public C-ABI entry point ``as_solve_ex`` on the
BASELINE.json workload: structure detection -> dispatch -> factor -> rcond
estimate -> gate -> solve (or SVD fallback), one graph launch and one stream
sync, inputs resident in HBM.  The default workload is configs[1] (C2: banded
fp64 n=8192, kl=ku=8, 4 RHS); ``--config`` selects another BASELINE config.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

Under torchrun (N > 1) every rank solves its own independent system (the solve
does not shard): weak scaling, no
collective on the data path; timing is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 GFLOP/s and solves/s per structure class; fraction of fp64/HBM roofline"


# ------------------------------------------------------------------ workload accounting
def workload(tag: str):
    import workloads as W
    kw = dict(W.CONFIGS[tag][1])
    n, nrhs = kw["n"], kw["nrhs"]
    es = 4 if tag == "C5f" else 8
    info = {"tag": tag, "n": n, "nrhs": nrhs, "es": es, "desc": W.CONFIGS[tag][0]}
    if tag == "C2":
        kl, ku = kw["kl"], kw["ku"]
        info["flops"] = n * (2 * kl * (kl + ku) + kl) + nrhs * 2 * n * (2 * kl + ku)   # gbtrf + gbtrs
        info["detect_bytes"] = n * n * es                       # a banded matrix must be read entirely
        info["factor_bytes"] = (kl + ku + 1) * n * es + 2 * (2 * kl + ku + 1) * n * es   # pack read + ab write/rw
        info["solve_bytes"] = 2 * n * nrhs * es + (2 * kl + ku + 1) * n * es
    elif tag in ("C3a",):
        info["flops"] = n ** 3 / 3 + 2 * n * n * nrhs            # potrf + potrs
        info["detect_bytes"] = n * n * es
        info["factor_flops"] = n ** 3 / 3
    elif tag == "C3b":
        info["flops"] = n * n * nrhs                             # trtrs
        info["detect_bytes"] = n * (n + 1) // 2 * es             # strict lower + diagonal
        info["solve_bytes"] = n * (n + 1) // 2 * es + 2 * n * nrhs * es
    elif tag in ("C1", "C5", "C5f"):
        info["flops"] = 2 * n ** 3 / 3 + 2 * n * n * nrhs        # getrf + getrs
        info["factor_flops"] = 2 * n ** 3 / 3
        info["detect_bytes"] = None                              # exits after the first tile pair
    elif tag == "C4":
        info["flops"] = 2 * n ** 3 / 3 + 4 * n ** 3 / 3          # getrf + QR (Jacobi sweeps added at run time)
        info["detect_bytes"] = None
    return info


def make_inputs(tag: str):
    import workloads as W
    if tag == "C5f":
        return W.make("C5f")
    return W.make(tag)


def load_traffic():
    """{config: {kernel, dram_bytes, source}} written from ncu --set full captures (profiles/)."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def clocks_peak_ghz() -> float:
    """Max SM clock (GHz) from MEASURED_PEAKS.json (1.965 on this pool's B200s)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f).get("sm_max_mhz", 1965.0)) / 1e3
    except (OSError, ValueError):
        return 1.965


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "MEASURED_PEAKS.json (measured copy)"
    return 6650.0, "B200_PROFILING.md fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sms)) if sms else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args, tag: str, rank: int, world: int):
    if rank != 0:
        return
    import oracle
    A, B = make_inputs(tag)
    info = workload(tag)
    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    # bounded sample: the full system for C1/C2 (fast on CPU); otherwise a scaled-down system of the same recipe
    sample = f"full {tag} system"
    if tag in ("C3a", "C3b", "C4", "C5", "C5f"):
        import workloads as W
        small = {"C3a": dict(n=1024, nrhs=16), "C3b": dict(n=2048, nrhs=16), "C4": dict(n=256),
                 "C5": dict(n=1024, nrhs=4), "C5f": dict(n=1024, nrhs=4)}[tag]
        A, B = W.make(tag, **small)
        sample = f"{tag} recipe at n={small['n']} (full size exceeds a minutes-long CPU budget)"
    for _ in range(args.warmup if tag in ("C1",) else min(args.warmup, 1)):
        oracle.solve(A, B)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.solve(A, B)
    dt = time.perf_counter() - t0
    v = args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "solves/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64" if tag != "C5f" else "f32",
            "data": "synthetic (seeded BASELINE.json recipe)",
            "config": {"workload": f"{tag}: {info['desc']}", "sample": sample},
            "cpu_baseline": {"value": v, "unit": "solves/s", "cores": oracle.get_threads(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(tag: str, A, B, budget_s: float = 12.0):
    import oracle
    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    sample = f"full {tag} system"
    if tag not in ("C1", "C2"):
        import workloads as W
        small = {"C3a": dict(n=1024, nrhs=16), "C3b": dict(n=2048, nrhs=16), "C4": dict(n=256),
                 "C5": dict(n=1024, nrhs=4), "C5f": dict(n=1024, nrhs=4)}[tag]
        A, B = W.make(tag, **small)
        sample = f"{tag} recipe at n={small['n']}"
    reps = 0
    t0 = time.perf_counter()
    while True:
        oracle.solve(A, B)
        reps += 1
        if time.perf_counter() - t0 >= budget_s or reps >= 200:
            break
    dt = time.perf_counter() - t0
    return {"value": reps / dt, "unit": "solves/s", "cores": oracle.get_threads(), "kind": "oracle",
            "sample": f"{sample}, {reps} solve(s) in {dt:.1f} s"}


# ------------------------------------------------------------------ multi-rank aggregation
def aggregate_time(t_ms: float, dist=None, device=None) -> float:
    """Max over ranks of this rank's timed-region duration (replicas: the job ends with the slowest)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return t_ms
    import torch
    t = torch.tensor([t_ms], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(world: int, steps: int, t_max_ms: float) -> float:
    """Whole-job solves/s: every rank solves `steps` independent systems in t_max."""
    return world * steps / (t_max_ms * 1e-3)


# ------------------------------------------------------------------ main (CUDA arm)
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3a", "C3b", "C4", "C5", "C5f"])
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true",
                    help="launch the plan's kernels directly instead of through its CUDA graph (for ncu launch "
                         "lists: ncu cannot profile kernel nodes of graphs with conditional nodes)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    tag = args.config

    if args.impl == "reference":
        run_reference(args, tag, rank, world)
        return

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2007_11208_b200 as AS
    AS.set_instrumentation(True)
    if args.eager:
        AS.set_exec_mode(True)
    info = workload(tag)
    A, B = make_inputs(tag)
    dA, dB = AS.to_device(A), AS.to_device(B)
    X = AS.empty_colmajor(B.shape[0], B.shape[1], dB.dtype)
    stream = torch.cuda.current_stream()
    # C5f: the fp32 rcond sits at the 0.5*eps gate: run with NO_FALLBACK and
    # report the LU data point (the gate bit is still set in the flags)
    opts = AS.make_options(no_fallback=True) if tag == "C5f" else None

    # warm-up (builds + instantiates the plan's graph)
    for _ in range(args.warmup):
        ret, _, rep = AS.as_solve_ex(dA, dB, X=X, options=opts)
        assert ret == 0, AS.strerror(ret)
    torch.cuda.synchronize()
    fp64_peak = AS.measure_fp64_peak(40000)

    # ---- timed region: K public-API calls, inputs resident (A is larger than L2 for C2/C3/C5;
    # for C1/C4 the 126 MB L2 is flushed by a 256 MB write between steps, outside the per-call timing)
    flush = None
    if A.nbytes < 256 * 2 ** 20:
        flush = torch.empty(64 * 2 ** 20, dtype=torch.float32, device="cuda")
    clock = ClockSampler(local)
    clock.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    stage = np.zeros(4)
    launches = 0
    step_ms = []
    reports = []
    for _ in range(args.steps):
        if flush is not None:
            flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ret, _, rep = AS.as_solve_ex(dA, dB, X=X, options=opts)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        st = AS.last_stage_ms()
        if st:
            stage += np.array(st)
        launches += AS.last_kernel_nodes()
        reports.append(rep)
    torch.cuda.synchronize()
    blocking_ms = float(np.sum(step_ms)) / args.steps
    # Device throughput (inputs larger than L2): the same K public-API solves issued back to back
    # with as_solve_async (one graph launch each, no host sync between them), bracketed by a
    # barrier + synchronize; the host-side enqueue of call k+1 overlaps the GPU work of call k.
    # With L2 flushes between steps (small inputs) the blocking per-call loop above is the number.
    if flush is None and not args.eager:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        for _ in range(args.steps):
            r = AS.as_solve_async(dA, dB, X, options=opts, stream=stream)
            assert r == 0, AS.strerror(r)
        eb.record(stream)
        eb.synchronize()
        torch.cuda.synchronize()
        step_ms = [ea.elapsed_time(eb) / args.steps] * args.steps
    if dist:
        dist.barrier()
    clocks = clock.stop()
    t_ms = aggregate_time(float(np.sum(step_ms)), dist, device="cuda")
    ms_per_step = t_ms / args.steps
    value = job_throughput(world, args.steps, t_ms)
    stage /= args.steps
    rep = reports[-1]

    # ---- end to end: host buffers through as_solve_host (H2D + solve + D2H inside the timing)
    pin_A = torch.from_numpy(np.ascontiguousarray(A.T)).pin_memory()
    pin_B = torch.from_numpy(np.ascontiguousarray(B.T)).pin_memory()
    pin_X = torch.empty_like(pin_B).pin_memory()
    import ctypes as C
    e2e_ms = []
    rep_h = AS.Report()
    dtc = AS.AS_F32 if A.dtype == np.float32 else AS.AS_F64
    n, nrhs = B.shape
    for i in range(max(3, min(args.steps, 10)) + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = AS.lib().as_solve_host(dtc, pin_A.data_ptr(), n, n, pin_B.data_ptr(), n, nrhs, pin_X.data_ptr(),
                                   C.byref(opts) if opts is not None else None, C.byref(rep_h), stream.cuda_stream)
        e1.record(stream)
        e1.synchronize()
        if i > 0:   # first call allocates the staging buffers / plan
            e2e_ms.append(e0.elapsed_time(e1))
    e2e = {"value": world * len(e2e_ms) / (np.sum(e2e_ms) * 1e-3), "unit": "solves/s",
           "h2d_bytes_per_step": int(A.nbytes + B.nbytes), "d2h_bytes_per_step": int(B.nbytes)}

    # ---- roofline of the dominant stage
    hbm_peak, hbm_src = load_peaks()
    names = ["detect", "factor+rcond", "solve/fallback"]
    dom = int(np.argmax(stage[:3]))
    roof = {"stage": names[dom], "stage_ms": [round(x, 4) for x in stage.tolist()]}
    if dom == 0 and info.get("detect_bytes"):
        ach = info["detect_bytes"] / (stage[0] * 1e-3) / 1e9
        roof.update({"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                     "traffic": None, "algorithmic_bytes": info["detect_bytes"], "peak_source": hbm_src})
    elif info.get("factor_flops") and dom == 1 and tag == "C5f":
        # fp32 runs on the SIMT FFMA pipe (tf32 tensor cores would miss the fp32 accuracy bar):
        # plain ALU arithmetic against the unit-count peak
        ffma_peak = 148 * 128 * 2 * clocks_peak_ghz() / 1e3
        ach = info["factor_flops"] / (stage[1] * 1e-3) / 1e12
        roof.update({"bound": "alu", "achieved": ach, "peak": ffma_peak, "unit": "TFLOP/s",
                     "frac": ach / ffma_peak, "traffic": None, "algorithmic_flops": info["factor_flops"],
                     "peak_source": "FP32 FFMA unit count: 148 SMs x 128 lanes x 2 flop x max SM clock"})
    elif info.get("factor_flops") and dom == 1:
        ach = info["factor_flops"] / (stage[1] * 1e-3) / 1e12
        roof.update({"bound": "tensor", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
                     "frac": ach / fp64_peak, "traffic": None, "algorithmic_flops": info["factor_flops"],
                     "peak_source": "fp64 DMMA register loop measured in this run"})
    elif tag == "C2":
        byts = info["factor_bytes"] if dom == 1 else info["solve_bytes"]
        ach = byts / (stage[dom] * 1e-3) / 1e9
        roof.update({"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                     "traffic": None, "algorithmic_bytes": byts, "peak_source": hbm_src,
                     "note": "banded factor/solve is a latency-bound chain of n pivot steps (SURVEY 8(a) a4)"})
    else:
        flops = info["flops"]
        ach = flops / (stage[dom] * 1e-3) / 1e12
        roof.update({"bound": "tensor", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s", "frac": ach / fp64_peak,
                     "traffic": None, "peak_source": "fp64 DMMA register loop measured in this run"})
    # DRAM traffic of the dominant kernel per launch, from the committed ncu --set full capture
    tr = load_traffic().get(tag)
    if tr:
        roof["traffic"] = tr["dram_bytes"]
        roof["traffic_kernel"] = tr["kernel"]
        roof["traffic_source"] = tr["source"]
    # detection stage fraction is always reported when it is HBM-graded
    extra = {}
    if info.get("detect_bytes"):
        ach = info["detect_bytes"] / (stage[0] * 1e-3) / 1e9
        extra["detect_hbm"] = {"achieved_gbs": ach, "frac": ach / hbm_peak, "bytes": info["detect_bytes"]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(tag, A, B)

    gflops = info["flops"] / (ms_per_step * 1e-3) / 1e9
    line = {"metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if tag == "C5f" else "f64", "data": "synthetic (seeded BASELINE.json recipe)",
            "config": {"workload": f"{tag}: {info['desc']}", "n": info["n"], "nrhs": info["nrhs"],
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                       "l2": "inputs larger than L2" if flush is None else "L2 flushed between steps (256 MB write)",
                       "timing": ("K back-to-back as_solve_async calls between two synchronizes (device throughput)"
                                  if flush is None and not args.eager else
                                  "per-call CUDA events around blocking as_solve_ex (host launch + sync included)"),
                       "ms_per_call_blocking": blocking_ms,
                       "method": rep["method"], "flags": hex(rep["flags"]), "rcond": rep["rcond"]},
            "gflops": gflops, "roofline": roof, **extra, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clocks, "fp64_dmma_peak_tflops": fp64_peak}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
