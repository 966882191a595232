#!/usr/bin/env python3
"""Regenerate tests/golden/schedules.json from the ORACLE (reference scheduler compiled
from /root/reference by oracle/Makefile, guarded + hooked engine).

For every config in configs/*.json and seeds 0-2: sha256 of the canonical schedule
log (oracle/harness.cpp format) plus the run's JSON summary (or its error text).
The c1_* logs are also stored gzipped for human diffs.

    python tests/golden/make_golden.py
"""
import gzip
import hashlib
import json
import pathlib
import subprocess
import tempfile

REPO = pathlib.Path(__file__).resolve().parents[2]
ORACLE = REPO / "oracle" / "_ref" / "pdsim_oracle"
SEEDS = [0, 1, 2]


def run_oracle(cfg: pathlib.Path, seed: int):
    with tempfile.TemporaryDirectory() as td:
        log = pathlib.Path(td) / "log.txt"
        p = subprocess.run([str(ORACLE), "run", "--config", str(cfg), "--seed", str(seed), "--log", str(log)],
                           capture_output=True, text=True)
        data = log.read_bytes() if log.exists() else b""
        return p.returncode, p.stdout.strip(), p.stderr.strip(), data


def main():
    out = {}
    for cfg in sorted((REPO / "configs").glob("*.json")):
        for seed in SEEDS:
            code, so, se, data = run_oracle(cfg, seed)
            key = f"{cfg.stem}/seed{seed}"
            out[key] = {"exit": code, "sha256": hashlib.sha256(data).hexdigest(),
                        "summary": json.loads(so) if code == 0 else None, "stderr": se}
            if cfg.stem.startswith("c1_") and code == 0:
                (REPO / "tests" / "golden" / f"{cfg.stem}.seed{seed}.log.gz").write_bytes(gzip.compress(data, mtime=0))
            print(key, code, out[key]["sha256"][:16])
    (REPO / "tests" / "golden" / "schedules.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
