"""`qforge`-compatible command line for the GPU-backed experiments on the hot
path: vqe-tfim, mipt-haar and shadow-gen (8f row 4).

    python -m paper_2602_14167_b200.cli {vqe-tfim,mipt-haar,shadow-gen} [--config F] [--seed S] [--workers W]
                                                  [--out DIR] [--set key=value ...]
    python -m paper_2602_14167_b200.cli emit-summary DIR

Mirrors tools/qforge_main.cpp (flags :45-56, --set JSON-or-string overrides
:14-30, exit codes 0 / 2 config error / 3 numerical contract violation :92-100)
and the vqe-tfim experiment of src/experiments.cpp:83-141 (ramp start, seed
perturbations from RngStream(seed).split(seeds), CSV `step,seed,energy`,
`.params.json`, `.meta.json`, FNV-1a config digest :37-46).  vqe_run runs on the
GPU; `grad_mode` additionally accepts "adjoint" and the config key `precision`
("c128" default, "c64") selects the device precision.  Outputs are identical
for every `--workers` value.
"""
from __future__ import annotations

import json
import os
import sys
import time

EXPERIMENTS = ["vqe-tfim", "mipt-haar", "shadow-gen"]


class ConfigError(Exception):
    pass


def _fmt(x: float) -> str:
    """std::ostream with setprecision(17) (experiments.cpp:55)."""
    return format(float(x), ".17g")


def config_digest(name: str, cfg: dict, seed: int) -> str:  # experiments.cpp:37-46
    s = name + "|" + json.dumps(cfg, separators=(",", ":"), sort_keys=True) + "|" + str(seed)
    h = 0xCBF29CE484222325
    for c in s.encode():
        h ^= c
        h = (h * 0x100000001B3) & ((1 << 64) - 1)
    return f"{h:016x}"


def merge_overrides(cfg: dict, sets: list) -> dict:  # qforge_main.cpp:14-30
    for kv in sets:
        eq = kv.find("=")
        if eq <= 0:
            raise ConfigError(f"--set expects key=value, got '{kv}'")
        key, value = kv[:eq], kv[eq + 1:]
        try:
            cfg[key] = json.loads(value)
        except json.JSONDecodeError:
            cfg[key] = value
    return cfg


def _get(cfg, key, fallback, typ):
    if key not in cfg:
        return fallback
    v = cfg[key]
    ok = (isinstance(v, bool) is False and isinstance(v, (int, float))) if typ is float else \
        (isinstance(v, int) and not isinstance(v, bool)) if typ is int else isinstance(v, typ)
    if not ok:
        raise ConfigError(f"config field '{key}' has the wrong type")
    return typ(v)


def exp_vqe_tfim(cfg, out, base, seed, workers):  # experiments.cpp:83-141
    from . import qforge as qf
    from .rng import RngStream

    n = _get(cfg, "n", 2, int)
    g = _get(cfg, "g", 1.0, float)
    layers = _get(cfg, "layers", 2, int)
    steps = _get(cfg, "steps", 300, int)
    lr = _get(cfg, "lr", 2e-2, float)
    seeds = _get(cfg, "seeds", 8, int)
    mode_name = _get(cfg, "grad_mode", "parameter_shift", str)
    precision = _get(cfg, "precision", "c128", str)
    if n < 2:
        raise ConfigError("vqe-tfim: n must be >= 2")
    if seeds < 1:
        raise ConfigError("vqe-tfim: seeds must be >= 1")
    modes = {"parameter_shift": qf.GradMode.parameter_shift, "finite_diff": qf.GradMode.finite_diff,
             "adjoint": qf.GradMode.adjoint}
    if mode_name not in modes:
        raise ConfigError("vqe-tfim: grad_mode must be parameter_shift, finite_diff or adjoint")
    if precision not in ("c64", "c128"):
        raise ConfigError("vqe-tfim: precision must be c64 or c128")
    qf.set_precision(precision)
    h = qf.tfim_terms(qf.build_lattice("chain", [n], [False]), g)
    ansatz = qf.tfim_chain_ansatz(n, layers)
    # annealing-ramp start (experiments.cpp:101-113)
    ramp = []
    dt = 1.0
    for l in range(layers):
        s = (l + 0.5) / layers
        ramp += [-2.0 * dt * (1.0 - s) * g] * n
        ramp += [-2.0 * dt * s] * (n - 1)
    streams = RngStream(seed).split(seeds)
    theta0 = []
    for sd in range(seeds):
        t = list(ramp)
        if sd > 0:
            t = [t[j] + 0.1 * streams[sd].normal() for j in range(ansatz.n_params)]
        theta0.append(t)
    res = qf.vqe_run(ansatz, theta0, h, steps, lr, modes[mode_name], workers)
    with open(os.path.join(out, base + ".csv"), "w") as f:
        f.write("step,seed,energy\n")
        for sd in range(seeds):
            for step, e in enumerate(res.traces[sd]):
                f.write(f"{step},{sd},{_fmt(e)}\n")
    params = [float(x) for x in res.final_thetas[res.best_index]]
    with open(os.path.join(out, base + ".params.json"), "w") as f:
        f.write(json.dumps({"theta": params}, indent=2) + "\n")
    return {"best_energy": res.best_energy, "best_index": res.best_index, "n": n, "g": g, "layers": layers}


def exp_mipt_haar(cfg, out, base, seed, workers):  # experiments.cpp:210-250
    from . import engine

    n = _get(cfg, "N", 12, int)
    depth = _get(cfg, "D", 24, int)
    p = _get(cfg, "p", 0.1, float)
    trajectories = _get(cfg, "trajectories", 100, int)
    precision = _get(cfg, "precision", "c128", str)
    if n < 2 or n > 20:
        raise ConfigError("mipt-haar: N must lie in [2, 20]")
    if p < 0.0 or p > 1.0:
        raise ConfigError("mipt-haar: p must lie in [0, 1]")
    if trajectories < 1:
        raise ConfigError("mipt-haar: trajectories must be >= 1")
    if precision not in ("c64", "c128"):
        raise ConfigError("mipt-haar: precision must be c64 or c128")
    ent, _ = engine.mipt_haar(engine.default_context(), n, depth, p, trajectories, seed, precision)
    mean = 0.0
    with open(os.path.join(out, base + ".csv"), "w") as f:
        f.write("L,p,trajectory,entropy_bits\n")
        for tr in range(trajectories):
            f.write(f"{n},{_fmt(p)},{tr},{_fmt(ent[tr])}\n")
            mean += float(ent[tr])
    return {"mean_entropy": {str(n): mean / trajectories}, "p": p, "trajectories": trajectories, "N": n, "D": depth}


def exp_shadow_gen(cfg, out, base, seed, workers):  # experiments.cpp:252-274
    from . import engine
    from .rng import RngStream

    n = _get(cfg, "n", 20, int)
    m = _get(cfg, "M", 256, int)
    depth = _get(cfg, "depth", 0, int)
    precision = _get(cfg, "precision", "c128", str)
    if n < 1 or n > 24:
        raise ConfigError("shadow-gen: n must lie in [1, 24]")
    if m < 1:
        raise ConfigError("shadow-gen: M must be >= 1")
    if precision not in ("c64", "c128"):
        raise ConfigError("shadow-gen: precision must be c64 or c128")
    streams = RngStream(seed).split(3)
    ops = []
    for _ in range(depth):
        for q in range(n):
            ops.append(("ry", q, -1, -1, 1.0, 2.0 * 3.14159265358979323846 * streams[0].uniform(), -1))
        for q in range(n - 1):
            ops.append(("cx", q, q + 1, -1, 1.0, 0.0, -1))
    bases = [[1 + streams[1].uniform_below(3) for _ in range(n)] for _ in range(m)]  # random_bases, shadows.cpp:24-29
    us = [s.uniform() for s in streams[2].split(m)]
    ctx = engine.default_context()
    prep = engine.Program(ctx, n, ops, 0, precision)
    outcomes = engine.shadow_snapshots(ctx, prep, None, bases, us)
    name = base + ".dataset.csv"
    with open(os.path.join(out, name), "w") as f:  # save_dataset, shadows.cpp:124-136
        f.write(f"{n},{m}\n")
        for r in range(m):
            f.write("".join(str(c) for c in bases[r]) + ";" + "".join(str(int(b)) for b in outcomes[r]) + "\n")
    return {"n": n, "M": m, "depth": depth, "dataset": name}


def run_experiment(name, cfg, out_dir, seed, workers):  # experiments.cpp:434-467
    if not isinstance(cfg, dict):
        raise ConfigError("config must be a JSON object")
    if name not in EXPERIMENTS:
        raise ConfigError(f"unknown experiment '{name}'")
    os.makedirs(out_dir, exist_ok=True)
    base = name + "_" + config_digest(name, cfg, seed)
    t0 = time.monotonic()
    extra = {"vqe-tfim": exp_vqe_tfim, "mipt-haar": exp_mipt_haar, "shadow-gen": exp_shadow_gen}[name](
        cfg, out_dir, base, seed, workers)
    wall = time.monotonic() - t0
    meta = {"experiment": name, "seed": seed, "config": cfg, "workers": workers, "wall_time_s": wall,
            "data": base + ".csv"}
    meta.update(extra)
    with open(os.path.join(out_dir, base + ".meta.json"), "w") as f:
        f.write(json.dumps(meta, indent=2, sort_keys=True) + "\n")
    return meta


def emit_summary(d):  # experiments.cpp:469-509 (vqe subset)
    if not os.path.isdir(d):
        raise ConfigError(f"summary: not a directory: {d}")
    metas = sorted(fn for fn in os.listdir(d) if fn.endswith(".meta.json") and len(fn) > 10)
    if not metas:
        raise ConfigError(f"summary: no run metadata in {d}")
    runs, best = [], float("inf")
    for fn in metas:
        with open(os.path.join(d, fn)) as f:
            m = json.load(f)
        runs.append(m)
        if "best_energy" in m:
            best = min(best, m["best_energy"])
    summary = {"runs": runs}
    if best < float("inf"):
        summary["best_energy"] = best
    with open(os.path.join(d, "summary.json"), "w") as f:
        f.write(json.dumps(summary, indent=2, sort_keys=True) + "\n")
    return summary


def main(argv=None) -> int:
    import argparse

    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser(prog="qforge", description="seeded, configuration-driven VQE on B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("emit-summary")
    s.add_argument("dir")
    for name in EXPERIMENTS:
        e = sub.add_parser(name)
        e.add_argument("--config", default="")
        e.add_argument("--seed", type=int, default=0)
        e.add_argument("--workers", type=int, default=1)
        e.add_argument("--out", default=".")
        e.add_argument("--set", action="append", default=[], dest="sets")
    try:
        args = ap.parse_args(argv)
    except SystemExit as ex:
        return 2 if ex.code else 0
    try:
        if args.cmd == "emit-summary":
            print(json.dumps(emit_summary(args.dir), indent=2, sort_keys=True))
            return 0
        cfg = {}
        if args.config:
            try:
                with open(args.config) as f:
                    cfg = json.load(f)
            except OSError:
                raise ConfigError(f"cannot open config file {args.config}")
            except json.JSONDecodeError as ex:
                raise ConfigError(f"config parse error: {ex}")
        cfg = merge_overrides(cfg, args.sets)
        if args.workers < 1:
            raise ConfigError("--workers must be >= 1")
        meta = run_experiment(args.cmd, cfg, args.out, args.seed, args.workers)
        print(json.dumps(meta, indent=2, sort_keys=True))
        return 0
    except (ConfigError, ValueError) as ex:
        print(f"config error: {ex}", file=sys.stderr)
        return 2
    except Exception as ex:  # noqa: BLE001
        print(f"numerical contract violation: {ex}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
