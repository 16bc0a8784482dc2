"""bench.py's contract pieces that run without a GPU: the reference arm (the reference library on
the host cores, one JSON line with impl / cpu_baseline / e2e) and the cost-model report."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    from oracle import REF_SO

    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "1", "--ref-threads", "2"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "iters/s"
    assert line["cpu_baseline"]["cores"] == 2 and line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["higher_is_better"] is True and line["config"]["workload"].startswith("c1")
    # the same config dict as our arm (same_config), the extrapolation to the oracle's full-run
    # mix (tests/golden/c1_poisson7_32.json), and no product library in the process
    sys.path.insert(0, ROOT)
    import bench
    from paper_2203_08498_b200.configs import CONFIGS

    assert line["config"] == bench.config_dict(CONFIGS["c1"], line["config"]["n"], line["config"]["nnz"])
    m = line["sequence_model"]
    assert m["mix"]["iccg"] == 34 and m["iterations"] == 34 + 29 + 29 + 30 and m["t_rr_s"] > 0
    assert line["time_to_solution_ms_per_rhs"] > 0 and "model" in line["cpu_baseline"]["host"]
    assert line["repo_libraries_mapped"] and all(p.startswith("oracle/") for p in line["repo_libraries_mapped"])


def test_cost_model_report_fields():
    sys.path.insert(0, ROOT)
    import bench

    rep = bench.cost_model_report(2097152, 14581760, 16, {"solve1_iterations": 168, "solve1_ms": 190.4,
                                                          "accelerated_iterations": [68, 157], "accelerated_ms": 80.0})
    assert rep["gamma_predicted"] > 1.0 and 0 < rep["iccg_model_fraction"] < 1.0
    assert rep["gamma_measured"] == pytest.approx((80.0 / 225) / (190.4 / 168), rel=1e-3)


@pytest.mark.gpu
def test_bench_line_contract_on_gpu():
    """The default workload through bench.py (short run): one JSON line with every key the
    driver and the judge read."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "cpu_baseline", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 1 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1 and r["peak"] > 0 and r["achieved"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] == 1
    assert d["config"]["workload"] == "c3_q1_27pt_256" and "time_to_solution_ms_per_rhs" in d


@pytest.mark.gpu
def test_bench_row_slabs_two_ranks():
    """bench.py --gpus 2 (the N > 1 headline: the sequence over two row slabs, run_slabs) under
    torch.distributed.run, both ranks on the one GPU over the host-staged transport (gloo; NCCL
    refuses two ranks per GPU): one JSON line, strong scaling, and block-Jacobi iteration counts
    within +-2 of the oracle's ic0_factorize(a, 0, 2) sequence on C1."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--config", "c1", "--slab-transport", "host", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")][-1])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["parallelism"].startswith("row slabs x2")
    from oracle import Oracle
    from oracle.sequence import run_sequence
    from paper_2203_08498_b200 import problems

    ref = run_sequence(Oracle(), problems.CONFIGS["c1"], problems.generate(problems.CONFIGS["c1"]), blocks=2)
    assert len(d["iterations_block_jacobi"]) == len(ref["iterations"])
    assert all(abs(a - b) <= 2 for a, b in zip(d["iterations_block_jacobi"], ref["iterations"])), (
        d["iterations_block_jacobi"], ref["iterations"])
    assert d["iterations_single_gpu"] and len(d["iterations_single_gpu"]) == len(ref["iterations"])
