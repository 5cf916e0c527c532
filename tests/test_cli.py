"""CLI (reference cli.py surface): header, exit codes, gen-fields on CPU;
bench-dirac and solve records on the GPU."""

import csv
import json

import numpy as np
import pytest

from paper_2601_05816_b200.__main__ import main


def _lines(capsys):
    return capsys.readouterr().out.strip().splitlines()


def test_gen_fields_and_header(tmp_path, capsys):
    rc = main(["gen-fields", "--dims", "2 2 2 4", "--clover", "random", "--out", str(tmp_path) + "/"])
    assert rc == 0
    out = _lines(capsys)
    head = json.loads(out[0])
    assert set(head) == {"version", "config_hash", "seed", "rng"} and head["rng"] == "pcg64"
    import paper_2601_05816_b200 as P
    psi = P.read_spinor(tmp_path / "psi.snap")
    assert psi.n_sites == 32 and psi.b == 4
    assert np.array_equal(P.read_gauge(tmp_path / "gauge.snap").data,
                          P.gen_gauge(P.LatticeGeometry((2, 2, 2, 4)), "random", seed=0).data)


def test_usage_errors_exit_1(capsys):
    assert main(["gen-fields", "--dims", "2 3 2 4"]) == 1  # odd extent
    assert main(["no-such-command"]) == 1


@pytest.mark.gpu
def test_bench_dirac_records(capsys):
    rc = main(["bench-dirac", "--dims", "8 8 8 8", "--b-list", "1 4", "--layouts", "1 2", "--reps", "2",
               "--antiperiodic"])
    assert rc == 0
    text = "\n".join(_lines(capsys)[1:])
    recs = json.loads(text)["records"]
    assert [(r["b"], r["layout"]) for r in recs] == [(1, 1), (1, 2), (4, 1), (4, 2)]
    for r in recs:
        assert r["seconds"] > 0 and r["device_seconds"] > 0 and 0 < r["roofline_frac"] < 2
        assert r["bytes"] == (168 * r["b"] + 114) * 16 * 4096


@pytest.mark.gpu
def test_solve_writes_history_and_snapshot(tmp_path, capsys):
    rc = main(["solve", "--dims", "8 4 4 4", "--gauge", "near-unit", "--antiperiodic", "--b", "3",
               "--odd-even", "--tol", "1e-10", "--out", str(tmp_path) + "/"])
    assert rc == 0
    res = json.loads(_lines(capsys)[-1])
    assert res["odd_even"] and res["converged"] and res["iterations"] > 0
    rows = list(csv.reader(open(tmp_path / "history.csv")))
    assert rows[0] == ["iter", "rhs", "relnorm"] and len(rows) == 1 + 3 * res["iterations"]
    rc = main(["solve", "--dims", "8 4 4 4", "--b", "2", "--restart-len", "2", "--restarts", "1",
               "--tol", "1e-12", "--out", str(tmp_path) + "/x"])
    assert rc == 2  # did not converge -> numerical failure
