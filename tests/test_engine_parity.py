"""Bit-exact scheduler parity of the product host engine (include/pdsim) against the oracle.

Schedule logs carry every plan (instance, start time, chunk slices, decode set),
every request's lifecycle (assignment, first token, completion, migrations as
(time, from, to, reason)) and instance stats, with doubles as hexfloats.
"""
import hashlib
import json
import pathlib
import subprocess

import pytest

REPO = pathlib.Path(__file__).resolve().parents[1]
GOLDEN = json.loads((REPO / "tests" / "golden" / "schedules.json").read_text())
ORACLE = REPO / "oracle" / "_ref" / "pdsim_oracle"


def sim_log(built, cfg: pathlib.Path, seed: int, tmp_path):
    log = tmp_path / f"ours.{cfg.stem}.{seed}.log"
    p = subprocess.run([str(built / "taichi_sim"), "run", "--config", str(cfg), "--seed", str(seed), "--log", str(log)],
                       capture_output=True, text=True, timeout=600)
    return p.returncode, (log.read_bytes() if log.exists() else b""), p.stdout, p.stderr


@pytest.mark.parametrize("key", sorted(GOLDEN))
def test_schedule_log_matches_golden(built, key, tmp_path):
    cfg_name, seed = key.split("/seed")
    code, data, out, err = sim_log(built, REPO / "configs" / f"{cfg_name}.json", int(seed), tmp_path)
    g = GOLDEN[key]
    assert code == g["exit"], err
    assert hashlib.sha256(data).hexdigest() == g["sha256"]
    if code == 0:
        assert json.loads(out) == g["summary"]
    else:
        assert err.strip() == g["stderr"]


@pytest.mark.skipif(not ORACLE.exists(), reason="oracle not built")
@pytest.mark.parametrize("qps", [1.0, 4.0, 16.0])
@pytest.mark.parametrize("mode,n_p,n_d,s_p,s_d,cap,prof", [
    ("hybrid", 2, 2, 1024, 256, 12000, "short_chat"),
    ("hybrid", 3, 1, 2048, 128, 30000, "long_doc"),
    ("aggregation", 4, 0, 512, 512, 20000, "short_chat"),
    ("disaggregation", 2, 2, 4096, 0, 40000, "long_doc"),
    ("hybrid", 1, 3, 512, 64, 9000, "short_chat"),
])
def test_live_random_grid_vs_oracle(built, tmp_path, qps, mode, n_p, n_d, s_p, s_d, cap, prof):
    """Fresh grid (not in the golden set): tight capacities force degrade/backflow and re-entrancy."""
    cfg = {"mode": mode,
           "cluster": {"n_p_heavy": n_p, "n_d_heavy": n_d, "s_p_tokens": s_p, "s_d_tokens": s_d,
                       "kv_capacity_tokens": cap},
           "slo": {"ttft_ms": 3000.0, "tpot_ms": 60.0},
           "policy": {"approach_factor": 0.9},
           "workload": {"synthetic": {"profile": prof, "n_records": 300}, "qps": qps, "seed": 7, "n_requests": 200}}
    path = tmp_path / "cfg.json"
    path.write_text(json.dumps(cfg))
    for seed in (3, 4):
        code, data, out, _ = sim_log(built, path, seed, tmp_path)
        olog = tmp_path / "oracle.log"
        p = subprocess.run([str(ORACLE), "run", "--config", str(path), "--seed", str(seed), "--log", str(olog)],
                           capture_output=True, text=True, timeout=600)
        assert code == p.returncode
        assert data == (olog.read_bytes() if olog.exists() else b"")
        if code == 0:
            assert out == p.stdout


REF_TESTS = ["cost_model_test", "cluster_test", "proxy_test", "decode_flow_test", "metrics_test",
             "workload_test", "engine_test"]


def test_reference_unit_tests_against_our_headers(built):
    """Drop-in acceptance: the reference's 7 test files compile against
    include/pdsim and give 93/94; the single failure is the reference test's own
    102-ULP defect (cost_model_test.cpp:33-36), which also fails under real gtest."""
    binaries = [built / "reftests" / t for t in REF_TESTS]
    if not all(b.exists() for b in binaries):
        pytest.skip("reference test sources unavailable on this host")
    passed, failed = 0, []
    for b in binaries:
        p = subprocess.run([str(b)], capture_output=True, text=True, timeout=600)
        passed += sum(1 for l in p.stdout.splitlines() if l.startswith("[       OK ]"))
        failed += [l.split()[-1] for l in p.stdout.splitlines() if l.startswith("[  FAILED  ]")]
    assert passed == 93
    assert failed == ["IterationTime.SlopeIsPerPrefillToken"]
