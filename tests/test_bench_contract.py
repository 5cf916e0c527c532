"""bench.py --impl reference (the CPU reference arm) keeps the driver's JSON-line
contract on CPU: one line, the own arm's metric / unit / config, W >= 3, and
under torchrun only rank 0 prints while the other ranks exit 0 without work."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _lines(out: str) -> list[dict]:
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_reference_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    (line,) = _lines(r.stdout)
    assert KEYS <= set(line)
    assert line["impl"] == "reference" and line["warmup"] >= 3 and line["n_gpus"] == 1
    assert line["config"]["lattice"] == [32, 16, 16, 16] and line["config"]["nrhs"] == 16
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    # the reference itself when baseline/_ref holds lqcdlab, else the oracle port
    want = "reference" if (ROOT / "baseline" / "_ref" / "lqcdlab").exists() else "port"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == want


def test_reference_arm_under_torchrun_rank0_only():
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
                        "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _lines(r.stdout)
    assert line["n_gpus"] == 2 and line["config"]["lattice"] == [64, 16, 16, 16]


@pytest.mark.gpu
def test_own_arm_line_on_gpu():
    """bench.py's own arm (GMRES records skipped for time): the driver's keys, the
    roofline and e2e objects, the clocks line and a launch count."""
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-gmres"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _lines(r.stdout)
    assert (KEYS - {"impl"}) | {"roofline", "gpu_launches", "clocks"} <= set(line)
    assert line["config"]["lattice"] == [32, 16, 16, 16] and line["dtype"] == "c128"
    roof = line["roofline"]
    assert roof["bound"] == "hbm" and 0 < roof["frac"] < 1 and abs(roof["achieved"] / roof["peak"] - roof["frac"]) < 1e-9
    field, links = 32 * 16 ** 3 * 12 * 16 * 16, 32 * 16 ** 3 * 4 * 9 * 16
    assert line["e2e"]["d2h_bytes_per_step"] == line["e2e"]["h2d_bytes_per_step"] == field
    assert line["e2e"]["links_cached"] is True
    v = line["e2e_variants"]
    assert v["pageable_links_every_call"]["host_buffers"] == "pageable"
    assert v["pinned_links_every_call"]["h2d_bytes_per_step"] == field + links
    assert 0 < line["e2e"]["value"] < line["value"] and line["gpu_launches"] >= 3
    assert line["cpu_baseline"]["cores"] >= 1 and line["cpu_baseline"]["value"] > 0


@pytest.mark.gpu
def test_multi_gpu_arm_logic_with_thread_ranks():
    """The N-GPU arm (weak-scaled headline, e2e through the comm= seam, halo
    stats, configs[4]-style strong-scaling block and its odd-even GMRES(8))
    run by 2 thread ranks sharing one GPU (tsplit.ThreadGroup instead of
    NCCL) on a reduced strong lattice: the code path the driver's N-GPU run
    takes, minus NCCL.  Timings here are not bench numbers."""
    import threading

    import torch

    sys.path.insert(0, str(ROOT))
    import bench
    import paper_2601_05816_b200 as P
    from paper_2601_05816_b200.tsplit import ThreadGroup
    grp = ThreadGroup(2)
    args = bench.argparse.Namespace(steps=3, warmup=3, no_gmres=False, no_cpu=True, strong_dims=[8, 8, 8, 16],
                                    sample_clocks=False)
    out, errs = [None, None], []

    def body(r):
        try:
            torch.cuda.set_device(0)
            out[r] = bench.multi_gpu(args, torch, P, bench.ThreadBenchGroup(grp, r, torch.device("cuda", 0)))
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            grp.barrier.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    if errs:
        raise errs[0]
    line = out[0]
    assert line["n_gpus"] == 2 and line["config"]["lattice"] == [64, 16, 16, 16]
    assert line["gpu_launches"] == 3 * 3  # pack, interior, both boundary slices in one launch, per apply
    assert len(line["epoch_stats"]) == 2 and all(e["interior_ms"] > 0 for e in line["epoch_stats"])
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
    recs = line["strong"]["records"]
    assert [r["dtype"] for r in recs] == ["c128", "c64"] and all(r["base_n1_ms"] > 0 for r in recs)
    gm = line["strong"]["gmres"]
    assert gm["converged"] and gm["iterations"] > 0 and gm["max_final_relnorm"] <= 1e-8
