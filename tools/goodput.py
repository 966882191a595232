#!/usr/bin/env python3
"""SLO goodput on B200 in wall-clock mode (BASELINE.json metric).

For each mode (aggregation / disaggregation / hybrid) and QPS grid point, runs lib/taichi_serve
--clock wall: the host engine makes the reference's decisions while every hybrid step runs on the
GPU and its measured device time advances the clock (same-device KV copies priced at the measured
NVLink bandwidth when instances are emulated on one GPU). Goodput = highest grid QPS whose
seed-mean attainment >= target (metrics.hpp:200-225 semantics).

  python tools/goodput.py --base configs/c3_llama8b_4p4d.json --modes hybrid,aggregation,disaggregation \
      --qps 100,150,200 --seeds 0 --model llama3_8b --out gpurun_out/goodput.json
"""
import argparse
import json
import pathlib
import subprocess
import tempfile
import time

REPO = pathlib.Path(__file__).resolve().parents[1]


def mode_config(base, mode):
    c = json.loads(json.dumps(base))
    c["mode"] = mode
    cl = c["cluster"]
    if mode == "aggregation":
        cl["s_d_tokens"] = cl["s_p_tokens"]
    elif mode == "disaggregation":
        cl["s_d_tokens"] = 0
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--base", required=True)
    ap.add_argument("--modes", default="hybrid")
    ap.add_argument("--qps", required=True)
    ap.add_argument("--seeds", default="0")
    ap.add_argument("--model", default="llama3_8b")
    ap.add_argument("--devices", default="0")
    ap.add_argument("--pool-tokens", type=int, default=0)
    ap.add_argument("--kv-cap", default="auto",
                    help="taichi_serve --kv-cap: logical KV capacity consistent with the physical pool (auto), "
                         "the config's (config) or N tokens")
    ap.add_argument("--n-requests", type=int, default=0)
    ap.add_argument("--profile", default="", help="calibration JSON whose 'profile' replaces the config's")
    ap.add_argument("--slo", default="", help="TTFT_ms,TPOT_ms override of the config's SLO (config-4 SLO sets)")
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    base = json.loads(pathlib.Path(args.base).read_text())
    if args.profile:
        base["profile"] = json.loads(pathlib.Path(args.profile).read_text())["profile"]
    if args.n_requests:
        base["workload"]["n_requests"] = args.n_requests
    if args.slo:
        ttft, tpot = (float(x) for x in args.slo.split(","))
        base["slo"]["ttft_ms"], base["slo"]["tpot_ms"] = ttft, tpot
    target = base["slo"].get("attainment_target", 0.9)
    grid = [float(q) for q in args.qps.split(",")]
    seeds = [int(s) for s in args.seeds.split(",")]
    results = {"base": args.base, "model": args.model, "slo": base["slo"], "modes": {}}
    for mode in args.modes.split(","):
        pts = []
        for q in grid:
            atts = []
            runs = []
            for sd in seeds:
                c = mode_config(base, mode)
                c["workload"]["qps"] = q
                with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
                    json.dump(c, f)
                cmd = [str(REPO / "paper_2508_01989_b200" / "lib" / "taichi_serve"), "--config", f.name, "--seed",
                       str(sd), "--model", args.model, "--devices", args.devices, "--clock", "wall"]
                if args.pool_tokens:
                    cmd += ["--pool-tokens", str(args.pool_tokens)]
                cmd += ["--kv-cap", args.kv_cap]
                t0 = time.time()
                p = subprocess.run(cmd, capture_output=True, text=True)
                if p.returncode == 3:  # physical KV pool exhausted: an invalid point, not an SLO miss
                    runs.append({"seed": sd, "invalid": "pool exhausted", "error": p.stderr.strip()[-300:]})
                    continue
                if p.returncode != 0:
                    runs.append({"seed": sd, "error": p.stderr.strip()[-300:]})
                    atts.append(0.0)
                    continue
                s = json.loads(p.stdout)
                s["seed"], s["host_s"] = sd, time.time() - t0
                runs.append(s)
                atts.append(s["attainment"])
            if not atts:  # every seed invalid
                pts.append({"qps": q, "mean_attainment": None, "passed": False, "invalid": True, "runs": runs})
                print(mode, q, "INVALID (pool exhausted)", flush=True)
                continue
            mean = sum(atts) / len(atts)
            pts.append({"qps": q, "mean_attainment": mean, "passed": mean >= target, "runs": runs,
                        "seeds_valid": len(atts), "seeds": len(seeds)})
            print(mode, q, round(mean, 4), [r.get("p90_ttft_ms") for r in runs], [r.get("p90_tpot_ms") for r in runs],
                  flush=True)
        # goodput: the highest passing grid QPS (metrics.hpp:198-209); invalid points never pass
        good = max([p["qps"] for p in pts if p["passed"]], default=0.0)
        results["modes"][mode] = {"goodput_qps": good, "points": pts}
        print("GOODPUT", mode, good, flush=True)
    pathlib.Path(args.out).write_text(json.dumps(results, indent=1))


if __name__ == "__main__":
    main()
