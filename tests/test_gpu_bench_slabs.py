"""bench.py's torchrun path (run_slabs) end to end on ONE GPU: the ranks share
the GPU and the interface planes are staged through the host
(ST_DIST_BACKEND=gloo) -- a functional check of the rendezvous, the balanced
partition, the per-rank slab operators, the split steps with the exchange on
the communication stream, the cross-rank stability reduction and the JSON
line; never a measurement.  The slab fields themselves are compared bitwise
with the single-GPU field in test_gpu_slabs*.py."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _torchrun(n, *args):
    port = _free_port()
    env = dict(os.environ, ST_DIST_BACKEND="gloo", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "4", "--warmup", "3", *args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]   # rank 0 alone prints, one line
    return json.loads(lines[0])


def test_strong_scaling_line_two_and_three_slabs():
    """Config 4 at 1/8 volume cut into 2 and 3 slabs balanced by DoFs: the
    line carries the contract's keys and both partitions reach the same
    maximum temperature to the last bit."""
    d2 = _torchrun(2, "--workload", "config4_s2")
    d3 = _torchrun(3, "--workload", "config4_s2")
    for d, n in ((d2, 2), (d3, 3)):
        assert d["n_gpus"] == n and d["scaling"] == "strong" and d["steps"] == 4
        assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
        assert d["roofline"]["bytes_per_dof"] == 24.0
        parts = d["config"]["partition"]
        assert len(parts) == n and parts[0][0] == 0 and parts[-1][1] == 1500
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    assert d2["config"]["dofs"] == d3["config"]["dofs"] == 120334881
    assert d2["t_max"] == d3["t_max"]


def test_weak_scaling_line():
    d = _torchrun(2, "--workload", "config1", "--scaling", "weak")
    assert d["scaling"] == "weak" and d["n_gpus"] == 2
    assert d["config"]["workload"].endswith("_x2") and d["value"] > 0


def test_reference_arm_under_torchrun_prints_one_line():
    env = dict(os.environ)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "2",
           "--warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "port"
