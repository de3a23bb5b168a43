"""GPU: bench.py keeps its contract (one JSON line with the driver's keys) --
run end to end, so a broken report leg cannot first show up at round end."""

import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _run(*args):
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [line for line in res.stdout.splitlines() if line.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run("--steps", "3", "--warmup", "3")
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline"):
        assert key in d, key
    assert d["steps"] == 3 and d["warmup"] >= 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["unit"] == "GDOF/s" and d["dtype"] == "f64"
    assert "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] <= 1.2 and r["achieved"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["gpu_launches"] >= 3
    if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "hexbench")):
        # the installed reference travels with the snapshot (tools/install_reference.sh)
        assert d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"]["api"]["value"] > 0
    # per_bp is the line's LAST key (the driver keeps the tail) and slim
    assert list(d)[-1] == "per_bp"
    assert set(d["per_bp"]) == {"BP3.5 E=32768", "BP1.0 E=4096", "BP3.0 E=32768",
                                "BP1.0 E=32768"}
    for rep in d["per_bp"].values():
        assert rep["gdof_per_s"] > 0 and 0 < rep["frac_of_measured_peak"] < 1.3
        assert 0 < rep["smem_roofline_frac"] < 1.0
    assert len(json.dumps(d["per_bp"])) < 1200
    with open(os.path.join(ROOT, d["details"]["file"])) as fh:
        details = json.load(fh)
    for leg in ("per_bp", "cg", "cg_assembled", "unfused_baseline", "calibration", "e2e_api"):
        assert details.get(leg), leg


def test_bench_gpus_2_relaunches_itself():
    """Plain `python bench.py --gpus 2` (how the driver calls it) runs two
    ranks: it re-launches itself under torch.distributed.run (here over gloo,
    sharing the one GPU; NCCL with one GPU per rank on a multi-GPU node)."""
    env = dict(os.environ, HX_BENCH_BACKEND="gloo")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--quick", "--steps", "3", "--warmup", "3"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [line for line in res.stdout.splitlines() if line.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and "x2" in d["config"]["parallelism"] and d["value"] > 0


def test_bench_refuses_more_nccl_ranks_than_gpus():
    if torch.cuda.device_count() > 1:
        pytest.skip("multi-GPU node")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--quick", "--steps", "3"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode != 0
    assert "need 2 GPUs" in res.stderr


def test_bench_two_ranks_weak_scaling_line():
    """The N>1 path of bench.py (torchrun, barrier, max-over-ranks time,
    summed DOFs, rank-0 line) with two ranks sharing the one GPU over gloo
    (NCCL needs one GPU per rank; the driver's multi-GPU runs use it)."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, HX_BENCH_BACKEND="gloo")
    res = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
         "--gpus", "2", "--quick", "--steps", "3", "--warmup", "3"],
        capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [line for line in res.stdout.splitlines() if line.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert "x2" in d["config"]["parallelism"]


def test_scaling_tool_two_ranks(tmp_path):
    """tools/scaling.py (config 5) through its multi-rank path: strong and
    weak modes on two ranks sharing the GPU over gloo, small meshes."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "scaling.jsonl"
    env = dict(os.environ, HX_BENCH_BACKEND="gloo")
    res = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", str(port),
         os.path.join(ROOT, "tools", "scaling.py"), "--strong-side", "8", "--weak-side", "6",
         "--steps", "3", "--warmup", "3", "--out", str(out)],
        capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    recs = [json.loads(line) for line in out.read_text().splitlines()]
    assert len(recs) == 6 and all(r["gpus"] == 2 and r["gdof_per_s"] > 0 for r in recs)
    strong = [r for r in recs if r["mode"] == "strong"]
    assert all(r["n_el_total"] == 512 and r["n_el_per_gpu_max"] == 256 for r in strong)
