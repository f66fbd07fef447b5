#!/usr/bin/env python
"""Benchmark: batched VQE energy + adjoint-gradient evaluations per second.

One step = one batched evaluation (energy + full gradient) of every parameter
set of the workload.  Default workload = BASELINE.json configs[1] (C2): 20-qubit
hardware-efficient ansatz, depth 8 (P = 320), open-chain TFIM g = 1 (39 terms),
global batch 1024 parameter sets, complex64, adjoint gradients.  N GPUs split
the batch (strong scaling: total work fixed), one NCCL all-reduce per step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

`value` is measured on device-resident parameter sets (CUDA events on the
engine stream, max over ranks); `e2e` goes through the public host-buffer C-ABI
call (qf_energy_grad_batch: pinned H2D of theta, kernels, collective, D2H of
energies + gradients) timed on the host clock.  `--impl reference` times the
reference algorithm (energy + parameter-shift gradient = 1 + 2P energies per
eval, reference src/variational.cpp:38-81) through the CPU oracle on all host
cores: the reference itself cannot be built here (no Eigen).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "VQE energy+gradient evals/sec"
UNIT = "evals/s"

# SURVEY.md section 8 config restatement (depths/anisotropy fixed there where BASELINE.json is silent)
CONFIGS = {
    "C1": dict(n=10, layers=4, ham="tfim", batch=16, prec="c64"),
    "C2": dict(n=20, layers=8, ham="tfim", batch=1024, prec="c64"),
    "C3": dict(n=26, layers=10, ham="xxz", batch=64, prec="c64"),
    "C4": dict(n=30, layers=8, ham="random2000", batch=1, prec="c64", shard="terms"),
    "C5": dict(n=16, layers=8, ham="random1000", batch=4096, prec="c128"),
}
CFG_INDEX = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5}
PREWARM_S = 1.0  # untimed evaluation before the warm-up steps (clock ramp; reported in config)


def hea_template(n, layers):
    """SURVEY.md 8 HEA: per layer ry(q), rz(q) on every site, then cx(q, q+1)."""
    ops, k = [], 0
    for _ in range(layers):
        for q in range(n):
            ops.append(("ry", q, -1, k, 1.0, 0.0, -1)); k += 1
        for q in range(n):
            ops.append(("rz", q, -1, k, 1.0, 0.0, -1)); k += 1
        for q in range(n - 1):
            ops.append(("cx", q, q + 1, -1, 1.0, 0.0, -1))
    return ops, k


def hamiltonian(cfg_name, cfg):
    from paper_2602_14167_b200 import qforge as qf
    from paper_2602_14167_b200.rng import RngStream

    n = cfg["n"]
    if cfg["ham"] == "tfim":
        h = qf.tfim_terms(qf.build_lattice("chain", [n], [False]), 1.0)
    elif cfg["ham"] == "xxz":
        h = qf.heisenberg_terms(qf.build_lattice("chain", [n], [False]), 1.0, 1.0, 0.5)
    else:
        T = int(cfg["ham"].replace("random", ""))
        h = qf.random_pauli_sum(n, T, RngStream(2000 + CFG_INDEX[cfg_name]), True)
    return h


def thetas_for(cfg_name, batch, P):
    """theta row b = RngStream(1000 + cfg).split(B)[b].normal() x P."""
    from paper_2602_14167_b200.rng import RngStream

    streams = RngStream(1000 + CFG_INDEX[cfg_name]).split(batch)
    return np.array([[s.normal() for _ in range(P)] for s in streams], dtype=np.float64)


class ClockSampler:
    """SM clocks / clock-event (throttle) reasons sampled during the timed region
    (NVML in process; nvidia-smi as the fallback)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        # in-process NVML (microsecond queries); spawning nvidia-smi would stall
        # short timed regions on its driver initialisation
        if self._nv is not None:
            nv, hdl = self._nv
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            mx = nv.nvmlDeviceGetMaxClockInfo(hdl, nv.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(hdl, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(hdl)
                flags = ["Active" if r & b else "Not Active" for b in bits]
                self.samples.append([str(sm), str(mx), "", *flags])
                self._stop.wait(0.05)
            return
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def start(self):
        self._nv = None
        try:  # NVML initialised before the timed region starts
            import pynvml as nv
            nv.nvmlInit()
            self._nv = (nv, nv.nvmlDeviceGetHandleByIndex(self.gpu))
        except Exception:
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if self._nv is not None and not self.samples:  # regions shorter than one sampling period
            try:
                nv, hdl = self._nv
                bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                        nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(hdl)
                self.samples.append([str(nv.nvmlDeviceGetClockInfo(hdl, nv.NVML_CLOCK_SM)),
                                     str(nv.nvmlDeviceGetMaxClockInfo(hdl, nv.NVML_CLOCK_SM)), "",
                                     *["Active" if r & b else "Not Active" for b in bits]])
            except Exception:
                pass
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def measured_fp_peaks():
    """FP32 / FP64 CUDA-core peaks measured on this pool's B200 (tools/micro/peaks.cu,
    committed as profiles/r2_fp_peaks.json): (fp32 TFLOP/s, fp64 TFLOP/s, source)."""
    p = os.path.join(ROOT, "profiles", "r2_fp_peaks.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["fp32_ffma_3reg_tflops"]), float(d["fp64_dfma_tflops"]), "measured (profiles/r2_fp_peaks.json)"
    except Exception:
        return 74.45, 37.2, "nominal (148 SMs x 128 FP32 lanes x 1965 MHz; FP64 half rate)"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def ncu_compute(cfg_name, cls_name, batch):
    """FP32-pipe view of the same committed capture (the sweeps are FMA-pipe bound,
    not HBM bound), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            e = json.load(f).get(cfg_name, {}).get(cls_name)
    except Exception:
        return None
    if not e or e.get("batch") != batch or "sm__pipe_fma_cycles_active_pct" not in e:
        return None
    return {"fma_pipe_active_pct": e["sm__pipe_fma_cycles_active_pct"], "issue_active_pct": e.get("smsp__issue_active_pct"),
            "top_stall": e.get("top_stall"), "source": e.get("source")}


def ncu_traffic(cfg_name, cls_name, batch):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the kernel class,
    from the committed `ncu --set full` capture (profiles/ncu_traffic.json) of the
    same workload and batch; None when no capture matches."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            e = json.load(f).get(cfg_name, {}).get(cls_name)
    except Exception:
        return None
    if not e or e.get("batch") != batch:
        return None
    return e.get("bytes_per_launch")


# --------------------------------------------------------------------------- CPU (oracle)
def cpu_sample(cfg_name, cfg, ops, P, h, thetas, seconds=12.0):
    """Times the reference algorithm (energy + parameter-shift gradient = 1 + 2P
    energy evaluations per eval, src/variational.cpp:38-81) via the CPU oracle
    on all host cores: a bounded sample of energy() calls, extrapolated."""
    from oracle import pyoracle as po

    cores = os.cpu_count() or 1
    a = po.Ansatz(cfg["n"], ops_to_ids(ops), P)
    hh = po.Hamil(cfg["n"], *h.arrays())
    # calibrate with one energy on one core
    t0 = time.perf_counter()
    po.energy(a, thetas[0], hh)
    t1 = time.perf_counter() - t0
    per_round = max(t1, 1e-6)
    rounds = max(1, int(seconds / per_round))
    count = min(cores * rounds, 4096)
    rows = np.resize(thetas, (count, P)) if P else np.zeros((count, 0))
    t0 = time.perf_counter()
    po.energy_grad_batch(a, rows, hh, workers=cores, grads=False)
    dt = time.perf_counter() - t0
    energies_per_s = count / dt
    evals_per_s = energies_per_s / (1 + 2 * P)
    return {"value": evals_per_s, "unit": UNIT, "cores": cores, "kind": "port", "cpu_model": cpu_model(),
            "compiler": "gcc -O2 (no -ffast-math / -march, like proj/src/CMakeLists.txt:8; oracle/Makefile)",
            "precision": "c128 (the reference's complex<double>)",
            "sample": f"{count} energy() calls of {cfg_name} (n={cfg['n']}, P={P}) on {cores} threads in "
                      f"{dt:.1f} s; eval = 1 + 2P = {1 + 2 * P} energies (parameter shift, "
                      f"variational.cpp:54-81), extrapolated"}


def ops_to_ids(ops):
    from oracle.pyoracle import GID
    return [(GID[o[0]] if isinstance(o[0], str) else o[0],) + tuple(o[1:]) for o in ops]


def run_reference(args, cfg_name, cfg, rank, world):
    if rank != 0:
        return 0
    ops, P = hea_template(cfg["n"], cfg["layers"])
    h = hamiltonian(cfg_name, cfg)
    thetas = thetas_for(cfg_name, min(cfg["batch"], 64), P)
    vals = []
    sample = None
    for s in range(args.warmup + args.steps):
        cb = cpu_sample(cfg_name, cfg, ops, P, h, thetas, seconds=args.ref_seconds)
        if s >= args.warmup:
            vals.append(cb["value"])
            sample = cb
    value = statistics.mean(vals)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * cfg["batch"] / value, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "impl": "reference",
            "config": config_block(cfg_name, cfg, P, h, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": sample["cores"], "kind": "port",
                             "sample": sample["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def l2_note(cfg):
    state = cfg["batch"] * (2 ** cfg["n"]) * (8 if cfg["prec"] == "c64" else 16)
    if state > 126 * 2 ** 20:
        return "inputs larger than L2 (batch of states = {:.1f} GiB per step)".format(state / 2 ** 30)
    return ("inputs fit in L2 ({:.1f} MiB of states per step) and are not flushed between timed steps "
            "(latency-bound configuration)".format(state / 2 ** 20))


def config_block(cfg_name, cfg, P, h, world):
    return {"workload": f"{cfg_name}: {cfg['n']}-qubit HEA depth {cfg['layers']} (P={P}), "
                        f"{cfg['ham']} ({len(h.terms)} terms), batch {cfg['batch']}, {cfg['prec']}, adjoint gradient",
            "n_qubits": cfg["n"], "layers": cfg["layers"], "n_params": P, "hamiltonian": cfg["ham"],
            "n_terms": len(h.terms), "global_batch": cfg["batch"], "precision": cfg["prec"],
            "parallelism": f"{cfg.get('shard', 'batch')}-sharded x{world}",
            "prewarm_s": PREWARM_S,
            "l2": l2_note(cfg)}


# --------------------------------------------------------------------------- GPU
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=0, help="override global batch")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-c128", action="store_true", help="skip the same-precision (complex128) leg")
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    cfg_name = args.config
    cfg = dict(CONFIGS[cfg_name])
    if args.batch:
        cfg["batch"] = args.batch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, cfg_name, cfg, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2602_14167_b200 import _lib, engine

    torch.cuda.set_device(local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    ctx = engine.Context(local_rank)
    if world > 1:
        obj = [engine.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx.set_comm(rank, world, obj[0])

    n, B = cfg["n"], cfg["batch"]
    ops, P = hea_template(n, cfg["layers"])
    h = hamiltonian(cfg_name, cfg)
    codes, w = h.arrays()
    prog = engine.Program(ctx, n, ops, P, cfg["prec"])
    obs = engine.Observable(ctx, n, codes, w)
    term_shard = cfg.get("shard") == "terms" and world > 1
    if term_shard:
        obs.set_sharding(_lib.QF_SHARD_TERMS)
    thetas = thetas_for(cfg_name, B, P)
    dev = torch.device("cuda", local_rank)
    ext = torch.cuda.ExternalStream(ctx.stream, device=dev)
    th_d = torch.tensor(thetas, dtype=torch.float64, device=dev)
    out_d = torch.zeros(B * (1 + P), dtype=torch.float64, device=dev)
    E_d = out_d[:B]
    G_d = out_d[B:].view(B, P)
    # The engine shards itself (qf_energy_grad_batch_device with a communicator:
    # the rank's batch rows or term block, one NCCL all-reduce on its stream):
    # every rank passes the full batch and receives the full result.
    def step_device():
        with torch.cuda.stream(ext):
            engine.energy_grad_batch_device(ctx, prog, obs, th_d, E_d, G_d)

    def agreed_count(seconds, one_call):
        """iterations covering `seconds`, identical on every rank (the calls run collectives)"""
        t0 = time.perf_counter()
        one_call()
        torch.cuda.synchronize(dev)
        dt = max(time.perf_counter() - t0, 1e-6)
        c = torch.tensor([min(100000, int(seconds / dt) + 1)], dtype=torch.int64, device=dev)
        if world > 1:
            dist.all_reduce(c, op=dist.ReduceOp.MAX)
        return int(c.item())

    # ---- device-resident value ----
    # pre-warm: ~PREWARM_S of untimed evaluation before the W warm-up steps, so
    # small configurations (microsecond calls) run at ramped-up clocks
    for _ in range(agreed_count(PREWARM_S, step_device)):
        step_device()
    torch.cuda.synchronize(dev)
    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    # The timed region runs exactly as a user's call does (per-class event
    # timing off, so single-chunk calls replay their CUDA graph); the per-class
    # split for the roofline comes from a second, instrumented pass below.
    sampler = ClockSampler(local_rank)
    sampler.start()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(ext)
    for _ in range(args.steps):
        step_device()
    ev1.record(ext)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms_local = ev0.elapsed_time(ev1)
    # instrumented pass: the same K steps with per-class CUDA events on the
    # engine stream (kernel launches counted, graphs off)
    ctx.reset_stats()
    ctx.set_timing(2)  # per class and per launch
    for _ in range(args.steps):
        step_device()
    torch.cuda.synchronize(dev)
    launches, cls_launches, cls_ms, cls_bytes = ctx.stats()
    cls_flops = ctx.flops()
    per_launch = ctx.launch_times()
    ctx.set_timing(False)
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    value = B * args.steps / (ms_total / 1000.0)

    # ---- end to end through the public host-buffer call ----
    E_h = np.empty(B)
    G_h = np.empty((B, P))
    def e2e_call():
        engine.energy_grad_batch(ctx, prog, obs, thetas)

    for _ in range(max(2, agreed_count(PREWARM_S / 2, e2e_call))):  # clock ramp, graph capture
        e2e_call()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        E_h, G_h = engine.energy_grad_batch(ctx, prog, obs, thetas)
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = B * args.steps / float(te.item())
    # consistency of the two legs (same numbers through both APIs)
    torch.cuda.synchronize(dev)
    E_dev = E_d.cpu().numpy()
    G_dev = G_d.cpu().numpy()
    agree = float(max(np.abs(E_dev - E_h).max(), np.abs(G_dev - G_h).max()))
    if agree != 0.0:  # both legs run the same kernels on the same inputs: bitwise equal
        raise SystemExit(f"device-resident and end-to-end results differ: max |d| = {agree}")

    # ---- roofline of the dominant kernel class ----
    names = ["forward_sweep", "hpsi_energy", "adjoint_sweep", "reduction"]
    dom = max(range(3), key=lambda i: cls_ms[i])
    peak, peak_src = measured_hbm_peak()
    fp32_peak, fp64_peak, fp_src = measured_fp_peaks()
    fpeak = fp64_peak if cfg["prec"] == "c128" else fp32_peak
    achieved = (cls_bytes[dom] / 1e9) / (cls_ms[dom] / 1e3) if cls_ms[dom] > 0 else 0.0
    bytes_per_launch = cls_bytes[dom] / max(1, cls_launches[dom])
    ftf = (cls_flops[dom] / 1e12) / (cls_ms[dom] / 1e3) if cls_ms[dom] > 0 else 0.0
    # Both rooflines of the dominant class are measured: HBM (algorithmic bytes
    # over the copy peak) and the FP32/FP64 pipe (minimal algorithmic flops over the
    # measured FMA peak).  The top-level entry is the BINDING one (the larger
    # fraction): since the round-2 schedule (6 + 6 sweeps for C2) the adjoint sweeps
    # move a quarter of the round-1 bytes in less time and are FP32-pipe bound, so
    # their HBM fraction is small by construction; both are kept in the line.
    hbm_part = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_source": peak_src, "algorithmic_bytes_per_launch": bytes_per_launch}
    fp_part = {"bound": "fp64" if cfg["prec"] == "c128" else "fp32", "achieved": ftf, "peak": fpeak,
               "unit": "TFLOP/s", "frac": ftf / fpeak, "peak_source": fp_src,
               "flops_per_launch": cls_flops[dom] / max(1, cls_launches[dom]),
               "counting": "minimal algorithmic flops per amplitude (FMA = 2; SURVEY.md 8(d)): 6 per "
                           "real rotation (ry/rx/h), 14 per dense complex 1q gate, 6 per diagonal "
                           "phase, 0 for x/cx, 4 per gradient tap or Pauli term; adjoint gates count "
                           "twice (psi and lambda)"}
    binding = fp_part if fp_part["frac"] > hbm_part["frac"] else hbm_part
    roofline = {"bound": binding["bound"], "kernel": names[dom], "achieved": binding["achieved"],
                "peak": binding["peak"], "unit": binding["unit"], "frac": binding["frac"],
                "traffic": ncu_traffic(cfg_name, names[dom], B),
                "hbm": hbm_part, "flops": dict(fp_part, binding=binding is fp_part),
                "compute": ncu_compute(cfg_name, names[dom], B),
                "avg_launch_ms": cls_ms[dom] / max(1, cls_launches[dom]),
                "classes": {names[i]: {"ms": cls_ms[i], "launches": cls_launches[i], "bytes": cls_bytes[i],
                                       "GBps": (cls_bytes[i] / 1e9) / (cls_ms[i] / 1e3) if cls_ms[i] else None,
                                       "TFLOPs": (cls_flops[i] / 1e12) / (cls_ms[i] / 1e3) if cls_ms[i] else None}
                            for i in range(4)},
                "per_launch_ms": {("fwd%d" % k if k < 1000 else "hpsi" if k == 1000 else "bwd%d" % (k - 2000)):
                                  round(v[0] / max(1, v[1]), 4) for k, v in sorted(per_launch.items())}}

    # ---- same-precision leg: the reference computes in complex<double>
    # (common.hpp:12); the headline workload is c64 (BASELINE configs[1]), so the
    # c128 program of the same workload is timed too (device-resident and e2e) ----
    c128_leg = None
    if cfg["prec"] == "c64" and not args.no_c128:
        prog2 = engine.Program(ctx, n, ops, P, "c128")
        E2_d = torch.zeros(B, dtype=torch.float64, device=dev)
        G2_d = torch.zeros(B, P, dtype=torch.float64, device=dev)

        def step2():
            with torch.cuda.stream(ext):
                engine.energy_grad_batch_device(ctx, prog2, obs, th_d, E2_d, G2_d)

        k2 = max(2, args.steps // 2)
        for _ in range(args.warmup):
            step2()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        for _ in range(k2):
            step2()
        e1.record(ext)
        torch.cuda.synchronize(dev)
        t2 = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        engine.energy_grad_batch(ctx, prog2, obs, thetas)  # e2e warm-up (graph capture)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(k2):
            E2_h, G2_h = engine.energy_grad_batch(ctx, prog2, obs, thetas)
        te2 = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te2, op=dist.ReduceOp.MAX)
        # the two precisions agree to float32 accuracy on the same inputs
        d64 = float(max(np.abs(E2_h - E_h).max() / max(1.0, np.abs(E2_h).max()),
                        np.abs(G2_h - G_h).max() / max(1.0, np.abs(G2_h).max())))
        c128_leg = {"dtype": "c128", "value": B * k2 / (float(t2.item()) / 1e3), "unit": UNIT, "steps": k2,
                    "ms_per_step": float(t2.item()) / k2,
                    "e2e": {"value": B * k2 / float(te2.item()), "unit": UNIT, "h2d_bytes_per_step": B * P * 8,
                            "d2h_bytes_per_step": B * (1 + P) * 8},
                    "c64_vs_c128_max_rel_diff": d64,
                    "note": "same workload in the reference's precision (complex<double>, common.hpp:12): the "
                            "like-for-like comparison with the reference arm"}
        prog2.close()
        del E2_d, G2_d

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        if cfg["n"] <= 26:
            cpu = cpu_sample(cfg_name, cfg, ops, P, h, thetas[:64])
        else:  # one complex128 energy() at n = 30 needs 16 GiB and hours of CPU time
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                   "sample": f"not sampled: n = {cfg['n']} exceeds what the CPU reference evaluates in minutes"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": cfg["prec"], "data": "synthetic",
                "config": config_block(cfg_name, cfg, P, h, world),
                "roofline": roofline, "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": B * P * 8,
                        "d2h_bytes_per_step": B * (1 + P) * 8},
                "gpu_launches": launches, "clocks": clocks,
                "program": dict(prog.info(), jit=prog.jit_status()), "e2e_vs_device_max_abs_diff": agree,
                "c128": c128_leg}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
