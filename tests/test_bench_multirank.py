"""bench.py's N>1 plumbing on CPU (gloo, world_size 2): barrier, max over ranks, whole-job
aggregation (value = tokens of all ranks / slowest rank), rank 0 alone prints one JSON line.
The step itself is replaced by the --simulate-step-ms test hook (no GPU here)."""
import json
import os
import pathlib
import socket
import subprocess
import sys

REPO = pathlib.Path(__file__).resolve().parents[1]


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_aggregation_gloo():
    env = dict(os.environ, PYTHONPATH=str(REPO))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(free_port()), str(REPO / "bench.py"), "--gpus", "2", "--steps", "4",
           "--warmup", "3", "--simulate-step-ms", "20"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=REPO)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["simulated"]
    # rank 1 sleeps 1.5x longer: the reported time must be the slowest rank's
    assert d["rank_seconds_max"] >= 4 * 0.020 * 1.5 * 0.95
    tokens = (512 + 64) * 4 * 2
    assert abs(d["value"] - tokens / d["rank_seconds_max"]) < 1e-6 * d["value"]
