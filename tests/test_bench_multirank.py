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


_FAKE_WORKER = r'''
import json, os, sys
sys.path.insert(0, os.environ["REPO"])
import torch.distributed as dist
import paper_2508_01989_b200 as pkg
import bench

PUSHED = []


class FakeRemote:
    def __init__(self, exported, device):
        assert exported["handle"] == b"h" * 64 and device == 0
        self.dst_rank = exported["rank"]

    def close(self):
        pass


class FakeEvent:
    def __init__(self, n):
        self.n = n

    def wait(self):
        return 0.5, self.n * 2097152

    def close(self):
        pass


class FakeInstance:
    def __init__(self, rank):
        self.rank, self.held = rank, {}

    def kv_reserve(self, rid, n):
        self.held[rid] = list(range(100 * self.rank, 100 * self.rank + (n + 15) // 16))

    def kv_release(self, rid):
        del self.held[rid]

    def kv_pages(self, rid):
        return self.held[rid]

    def export_pool(self):
        return {"handle": b"h" * 64, "page_bytes": 2097152, "n_pages": 1000, "device": 0, "rank": self.rank}

    def push_pages(self, remote, sp, dp):
        assert len(sp) == len(dp) == 256 and dp[0] == 100 * remote.dst_rank
        PUSHED.append((self.rank, remote.dst_rank))
        return FakeEvent(len(sp))


pkg.RemotePool = FakeRemote
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
inst = FakeInstance(rank)
out = bench.migration_nvlink(inst, rank, world, 0, n_tokens=4096, reps=3)
assert not inst.held, "every reservation released"
if rank == 0:
    print(json.dumps(out))
dist.destroy_process_group()
'''


def test_cross_gpu_migration_leg_pairs_ranks_gloo(tmp_path):
    """bench.migration_nvlink's rank pairing and aggregation (4 ranks, gloo, fake instances):
    rank 2k pushes into rank 2k+1's exported pool with that rank's page list; every rank releases
    its reservation; rank 0 reports one entry per pair with the GB/s of its copies."""
    w = tmp_path / "worker.py"
    w.write_text(_FAKE_WORKER)
    env = dict(os.environ, PYTHONPATH=str(REPO), REPO=str(REPO))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "4", "--master-addr",
           "127.0.0.1", "--master-port", str(free_port()), str(w)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=REPO)
    assert p.returncode == 0, p.stderr[-3000:]
    d = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][0])
    assert [(x["src"], x["dst"]) for x in d["pairs"]] == [(0, 1), (2, 3)]
    gb = 256 * 2097152 / 0.5 / 1e6
    assert all(abs(x["gb_s"] - gb) < 1e-6 * gb for x in d["pairs"])
    assert abs(d["min_nvlink_frac"] - gb / 900.0) < 1e-9
