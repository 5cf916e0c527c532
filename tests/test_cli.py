"""CLI (reference cli.py surface): run-config files and --set overrides, the
header, exit codes, gen-fields on CPU; bench-dirac and solve records on the GPU."""

import csv
import hashlib
import json

import numpy as np
import pytest

from paper_2601_05816_b200 import config as C
from paper_2601_05816_b200.__main__ import main


def _lines(capsys):
    return capsys.readouterr().out.strip().splitlines()


def test_gen_fields_config_file_and_header(tmp_path, capsys):
    cfgfile = tmp_path / "run.cfg"
    cfgfile.write_text("lattice.dims = 2 2 2 4   # T X Y Z\nclover.mode = random\nblock.b = 4\nblock.layout = 2\n"
                       f"output.path = {tmp_path}/\n")
    rc = main(["gen-fields", "--config", str(cfgfile), "--set", "seed=3"])
    assert rc == 0
    out = _lines(capsys)
    head = json.loads(out[0])
    assert set(head) == {"version", "config_hash", "seed", "rng"} and head["rng"] == "pcg64" and head["seed"] == 3
    cfg = C.load_config(str(cfgfile))
    C.set_key(cfg, "seed", "3")
    assert head["config_hash"] == hashlib.sha256(C.canonical(cfg).encode()).hexdigest()[:12] == C.config_hash(cfg)
    import paper_2601_05816_b200 as P
    psi = P.read_spinor(tmp_path / "psi.snap")
    assert psi.n_sites == 32 and psi.b == 4
    assert np.array_equal(P.read_gauge(tmp_path / "gauge.snap").data,
                          P.gen_gauge(P.LatticeGeometry((2, 2, 2, 4)), "random", seed=3).data)


def test_config_canonical_form_and_extensions():
    cfg = C.parse_config("block.b = 12\nsolver.odd_even = yes\n")
    text = C.canonical(cfg)
    assert text.splitlines()[0] == "lattice.dims = 4 4 4 4" and "solver.odd_even = true" in text
    assert "device.dtype" not in text  # extensions appear only when set
    C.set_key(cfg, "device.dtype", "c64")
    assert C.canonical(cfg).endswith("device.dtype = c64\n")
    assert C.parse_config(C.canonical(cfg)) == cfg  # round trip
    assert "solver.orthogonalization" not in C.canonical(cfg)
    C.set_key(cfg, "solver.orthogonalization", "cgs")
    assert C.canonical(cfg).endswith("solver.orthogonalization = cgs\n")
    assert C.parse_config(C.canonical(cfg)) == cfg
    C.set_key(cfg, "solver.orthogonalization", "qr")
    with pytest.raises(C.ConfigError, match="orthogonalization"):
        C.validate(cfg)


def test_usage_errors_exit_1(capsys):
    assert main(["gen-fields", "--set", "lattice.dims=2 3 2 4"]) == 1  # odd extent
    assert main(["gen-fields", "--set", "block.b"]) == 1  # no value
    assert main(["gen-fields", "--set", "no.such.key=1"]) == 1
    assert main(["no-such-command"]) == 1
    assert main(["stream", "--kind", "triad"]) == 1  # reference CPU-model tool, not provided


@pytest.mark.gpu
def test_bench_dirac_records(capsys):
    rc = main(["bench-dirac", "--set", "lattice.dims=8 8 8 8", "--set", "lattice.antiperiodic_time=true",
               "--set", "dirac.m0=0.1", "--b-list", "1 4", "--layout-list", "1 2", "--reps", "2"])
    assert rc == 0
    text = "\n".join(_lines(capsys)[1:])
    recs = json.loads(text)["records"]
    assert [(r["b"], r["layout"]) for r in recs] == [(1, 1), (1, 2), (4, 1), (4, 2)]
    for r in recs:
        assert r["seconds"] > 0 and r["device_seconds"] > 0 and 0 < r["roofline_frac"] < 2
        assert r["bytes"] == (168 * r["b"] + 114) * 16 * 4096


@pytest.mark.gpu
@pytest.mark.parametrize("grid", ["1 1 1 1", "2 1 1 1"])
def test_solve_writes_history_and_snapshot(tmp_path, capsys, grid):
    rc = main(["solve", "--set", "lattice.dims=8 4 4 4", "--set", "gauge.mode=near-unit",
               "--set", "lattice.antiperiodic_time=true", "--set", "block.b=3", "--set", "block.layout=2",
               "--set", "dirac.m0=0.1", "--set", "clover.mode=zero", "--set", "solver.odd_even=true",
               "--set", "solver.tol=1e-10", "--set", "solver.restart_len=30", "--set", "solver.restarts=20",
               "--set", f"ranks.grid={grid}", "--set", f"output.path={tmp_path}/"])
    assert rc == 0
    res = json.loads(_lines(capsys)[-1])
    assert res["odd_even"] and res["converged"] and res["iterations"] > 0
    rows = list(csv.reader(open(tmp_path / "history.csv")))
    assert rows[0] == ["iter", "rhs", "relnorm"] and len(rows) == 1 + 3 * res["iterations"]
    rc = main(["solve", "--set", "lattice.dims=8 4 4 4", "--set", "block.b=2", "--set", "dirac.m0=0.1",
               "--set", "clover.mode=zero", "--set", f"ranks.grid={grid}", "--set", "solver.restart_len=2",
               "--set", "solver.restarts=1", "--set", "solver.tol=1e-12", "--set", f"output.path={tmp_path}/x"])
    assert rc == 2  # did not converge -> numerical failure


@pytest.mark.gpu
def test_oracle_check_suites(capsys):
    base = ["oracle-check", "--set", "lattice.dims=4 4 4 8", "--set", "clover.mode=random", "--set", "block.b=3"]
    assert main(base) == 0
    out = _lines(capsys)
    assert sum(line.endswith(")") and ": PASS (" in line for line in out) == 5
    assert main(base + ["--set", "lattice.antiperiodic_time=true", "--set", "device.dtype=c64"]) == 0
    capsys.readouterr()
    assert main(base + ["--corrupt-gauge"]) == 2  # unitarity fails, detected
    assert "gauge-unitarity: FAIL" in capsys.readouterr().out
