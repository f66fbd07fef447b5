"""CLI parity with tools/qforge_main.cpp + experiments.cpp vqe-tfim
(test_experiments.cpp:77-158): exit codes, config/--set precedence, digest-named
outputs, byte-identical CSV for the same seed, worker-count invariance."""
import json
import os

import pytest

from paper_2602_14167_b200 import cli


def test_exit_codes_and_config_errors(tmp_path, capsys):
    assert cli.main(["vqe-tfim", "--out", str(tmp_path), "--set", "n=1"]) == 2
    assert cli.main(["vqe-tfim", "--out", str(tmp_path), "--set", "grad_mode=bogus"]) == 2
    assert cli.main(["vqe-tfim", "--out", str(tmp_path), "--set", "nokey"]) == 2
    assert cli.main(["vqe-tfim", "--config", str(tmp_path / "missing.json")]) == 2
    assert cli.main(["vqe-tfim", "--workers", "0"]) == 2
    assert cli.main(["no-such-experiment"]) == 2
    assert cli.main(["emit-summary", str(tmp_path / "nothing")]) == 2
    assert cli.main(["mipt-haar", "--out", str(tmp_path), "--set", "N=21"]) == 2
    assert cli.main(["mipt-haar", "--out", str(tmp_path), "--set", "p=1.5"]) == 2
    assert cli.main(["mipt-haar", "--out", str(tmp_path), "--set", "trajectories=0"]) == 2


def test_overrides_and_digest():
    cfg = cli.merge_overrides({"n": 3, "g": 1.0}, ["n=4", "grad_mode=adjoint", "lr=0.05", "tag=[1,2]"])
    assert cfg == {"n": 4, "g": 1.0, "grad_mode": "adjoint", "lr": 0.05, "tag": [1, 2]}
    d1 = cli.config_digest("vqe-tfim", {"n": 2, "g": 1.0}, 7)
    assert d1 == cli.config_digest("vqe-tfim", {"g": 1.0, "n": 2}, 7)  # key order independent
    assert d1 != cli.config_digest("vqe-tfim", {"n": 2, "g": 1.0}, 8)
    assert len(d1) == 16 and int(d1, 16) >= 0


@pytest.mark.gpu
def test_vqe_tfim_outputs_deterministic_and_worker_invariant(ctx, tmp_path):
    args = ["vqe-tfim", "--seed", "7", "--set", "n=2", "--set", "layers=2", "--set", "steps=300",
            "--set", "seeds=8"]
    a, b = tmp_path / "a", tmp_path / "b"
    assert cli.main(args + ["--out", str(a), "--workers", "1"]) == 0
    assert cli.main(args + ["--out", str(b), "--workers", "3"]) == 0
    csv_a = [f for f in os.listdir(a) if f.endswith(".csv")]
    assert len(csv_a) == 1
    assert open(a / csv_a[0]).read() == open(b / csv_a[0]).read()
    meta = json.load(open(a / csv_a[0].replace(".csv", ".meta.json")))
    assert meta["best_energy"] == pytest.approx(-5 ** 0.5, rel=1e-3)
    lines = open(a / csv_a[0]).read().splitlines()
    assert lines[0] == "step,seed,energy" and len(lines) == 1 + 8 * 301
    s = cli.emit_summary(str(a))
    assert s["best_energy"] == meta["best_energy"]
    assert cli.main(args + ["--out", str(a), "--set", "grad_mode=adjoint", "--set", "precision=c64"]) == 0


@pytest.mark.gpu
def test_mipt_haar_outputs_match_oracle(ctx, tmp_path):
    """mipt-haar (experiments.cpp:210-250): CSV L,p,trajectory,entropy_bits with the
    per-trajectory entropies of the oracle restatement, worker invariant."""
    from oracle import pyoracle as po
    args = ["mipt-haar", "--seed", "11", "--set", "N=6", "--set", "D=8", "--set", "p=0.25",
            "--set", "trajectories=5"]
    a, b = tmp_path / "a", tmp_path / "b"
    assert cli.main(args + ["--out", str(a)]) == 0
    assert cli.main(args + ["--out", str(b), "--workers", "4"]) == 0
    csv = [f for f in os.listdir(a) if f.endswith(".csv")][0]
    assert open(a / csv).read() == open(b / csv).read()
    lines = open(a / csv).read().splitlines()
    assert lines[0] == "L,p,trajectory,entropy_bits" and len(lines) == 6
    ent = [float(x.split(",")[3]) for x in lines[1:]]
    ref = po.mipt_haar(6, 8, 0.25, 5, 11)
    assert max(abs(x - y) for x, y in zip(ent, ref)) < 1e-9
    meta = json.load(open(a / csv.replace(".csv", ".meta.json")))
    assert meta["N"] == 6 and meta["D"] == 8 and meta["mean_entropy"]["6"] == pytest.approx(sum(ent) / 5)
