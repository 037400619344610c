"""bench.py's JSON line keeps the driver's contract (keys, units, the reference arm's
shape). CPU: the reference arm on a small sample. GPU: the device arm on a small graph."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def _metric():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        return json.load(f)["metric"]


def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "2", "--warmup", "1", "--nrows", "20000")
    assert d["impl"] == "reference" and d["metric"] == _metric()
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["steps"] == 2 and d["warmup"] == 1 and d["n_gpus"] == 1
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_device_arm_line():
    d = _run("--steps", "2", "--warmup", "3", "--nrows", "200000", "--no-cpu-baseline", "--no-solver", "--no-completion",
             "--no-solve")
    assert d["metric"] == _metric() and d["unit"] == "GB/s" and d["value"] > 0
    assert d["steps"] == 2 and d["warmup"] == 3 and d["dtype"] == "f64" and d["vs_baseline"] is None
    assert d["config"]["workload"] and "model" not in d["config"]
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] <= 1.5
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == "GB/s" and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


@pytest.mark.gpu
def test_device_arm_two_ranks_gloo():
    """The N>1 launch (torchrun, one process per rank, row-sharded factors with halo
    exchange): rank 0 prints one line for the whole job. gloo lets both ranks share the
    one visible GPU; the NCCL launch differs only in the collective backend."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--nrows", "200000", "--no-cpu-baseline",
           "--no-solver", "--no-e2e", "--dist-backend", "gloo"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["config"]["halo_bytes_per_spmm_per_rank"] > 0


@pytest.mark.gpu
def test_device_arm_two_ranks_strong_scaling_gloo():
    """--scaling strong: the two ranks split one graph of --nrows vertices."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--nrows", "300000", "--scaling", "strong",
           "--no-cpu-baseline", "--no-e2e", "--dist-backend", "gloo"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["n"] == 300000 and d["config"]["n_per_gpu"] == 150000


@pytest.mark.gpu
def test_device_arm_two_ranks_peer_memory_gloo():
    """The N>1 bench with the peer-memory ghost rows forced (CULORADS_HALO=nvlink): the two
    ranks map each other's factor allocations by CUDA IPC and the SpMM reads remote rows in
    place (on an NVLink box with NCCL this plan is the default)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--nrows", "300000", "--scaling", "strong",
           "--no-cpu-baseline", "--no-e2e", "--dist-backend", "gloo"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                         env=dict(os.environ, CULORADS_HALO="nvlink"))
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["halo"]["plan"] == "NvlinkHaloPlan" and d["halo"]["bytes_per_spmm_per_rank"] > 0
