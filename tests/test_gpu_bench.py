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
    for leg in ("per_bp", "cg", "cg_assembled", "unfused_baseline", "calibration"):
        assert d.get(leg), leg


def test_reference_arm_contract():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["value"] == d["value"]


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
