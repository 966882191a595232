#!/usr/bin/env python3
"""bench.py -- hybrid-step throughput of the B200 TaiChi instance (BASELINE.json config 2).

Workload (N=1): one aggregated Llama-3-8B-shaped instance (random-init bf16 weights,
synthetic token ids), chunk size 512. One "step" = one hybrid iteration: a 512-token
prefill chunk of a 1024-token prompt (positions 512..1023, so it attends to a 512-token
paged prefix) piggybacked with 64 decode requests at context 1024 -- T = 576 rows through
32 layers + LM head on the 65 sampled rows + greedy argmax. Weights (15 GB) and the KV
cache (8.6 GB of decode context) are far larger than L2 (126 MB), so no flush is needed.

  value     tokens/s from device time (CUDA events on the instance stream, inputs resident)
  e2e       tokens/s through the C ABI (tc_step_launch / tc_step_wait) with host token ids in
            and sampled ids out, wall clock around the step loop
  roofline  the dominant kernel (gate_up GEMM, fused SwiGLU) vs measured bf16 tensor peak
  cpu_baseline  the oracle port of the same step (all 32 layers, bf16 torch) on the host cores

N>1 (torchrun): every rank drives its own instance on its own GPU (independent TaiChi
instances; the step has no collective) -> "scaling": "weak", value = sum over ranks.
--impl reference: the CPU implementation (oracle port) on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import tempfile
import time

REPO = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))


# GPU-vs-oracle parity tests that run the exact step a bench line measures (layer-reduced model,
# same shapes, same concurrent prefill/decode attention split)
PARITY = {
    ("llama3_8b", 512, 512, 64, 1024): "tests/test_gpu_bench_shapes.py::test_config2_bench_step_llama_shape",
    ("qwen2_5_14b", 1024, 4096, 32, 8192): "tests/test_gpu_bench_shapes.py::test_config5_bench_step_qwen_shape",
    ("llama3_8b", 0, 0, 64, 1024): "tests/test_gpu_bench_shapes.py::test_config2_bench_step_llama_shape (its decode rows)",
}


def step_cost(d, P, prefix, D, ctx, n_logit):
    """Algorithmic flops / bytes per kernel class for one step."""
    H, Hk, dh, dm, F, V, L = d["n_heads"], d["n_kv_heads"], d["head_dim"], d["d_model"], d["ffn_dim"], d["vocab"], d["n_layers"]
    T = P + D
    qkv_n = (H + 2 * Hk) * dh
    kv_tok = 2 * Hk * dh * 2  # bytes of K+V per token per layer
    k = {}
    def gemm(name, m, n, kk):
        k[name] = {"flops": 2.0 * m * n * kk * L, "bytes": (n * kk * 2 + m * kk * 2 + m * n * 2) * L}
    gemm("gemm_qkv", T, qkv_n, dm)
    gemm("gemm_o", T, dm, H * dh)
    gemm("gemm_gate_up", T, 2 * F, dm)
    gemm("gemm_down", T, dm, F)
    pairs_p = P * prefix + P * (P + 1) // 2
    pairs_d = D * (ctx + 1)
    k["attn"] = {"flops": 4.0 * H * dh * (pairs_p + pairs_d) * L,
                 "bytes": ((prefix + P) + D * (ctx + 1)) * kv_tok * L + T * (qkv_n + H * dh) * 2 * L}
    k["lm_head"] = {"flops": 2.0 * n_logit * V * dm, "bytes": V * dm * 2 + n_logit * V * 4}
    k["elementwise"] = {"flops": 0.0, "bytes": T * dm * (4 + 2) * 2 * L * 2}
    return k


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        rows = [r.split(", ") for r in pathlib.Path(self.f.name).read_text().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for i, n in enumerate(names):
                if len(r) >= 9 and r[5 + i].strip() == "Active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def measured_peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return j["hbm_gbs"], j["bf16_tflops"], j["bf16_tflops_sustained"], "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


def cpu_baseline(dims, P, prefix, D, ctx, n_logit, repeats=3):
    from oracle import cpu_step, model_ref as mr
    import torch
    d = mr.Dims(**dims)
    threads = os.cpu_count() or 1
    sec, det = cpu_step.time_step(d, P, prefix, D, ctx, n_logit, repeats=repeats, threads=threads)
    return {"value": (P + D) / sec, "unit": "tokens/s", "cores": torch.get_num_threads(), "kind": "port",
            "sample": f"the full step (P={P} prefix={prefix} D={D} ctx={ctx}), all {d.n_layers} layers + LM head on "
                      f"{n_logit} rows, bf16 torch on the host cores, median of {repeats} after 1 warm-up",
            "seconds_per_step": sec, **det}


def scheduler_baseline(config="configs/c3_llama8b_4p4d.json", repeat=5):
    """the reference scheduler/engine on the host cores, single-threaded, on the
    config-3 trace (4P1024 + 4D256, short_chat, 2000 requests) -- oracle/_ref/pdsim_oracle is the
    reference's own pdsim headers compiled here (oracle/Makefile) -- next to this repo's drop-in
    host engine (lib/taichi_sim), which makes the identical decisions (tests/test_engine_parity.py)."""
    import platform
    out = {"config": config, "threads": 1, "repeat": repeat, "cpu": platform.processor() or None,
           "nproc": os.cpu_count()}
    try:
        out["cpu"] = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    for name, exe in (("reference", REPO / "oracle" / "_ref" / "pdsim_oracle"),
                      ("ours", REPO / "paper_2508_01989_b200" / "lib" / "taichi_sim")):
        if not exe.exists():
            out[name] = {"unavailable": f"{exe.relative_to(REPO)} not built"}
            continue
        r = subprocess.run([str(exe), "bench", "--config", str(REPO / config), "--repeat", str(repeat)],
                           capture_output=True, text=True, timeout=300)
        out[name] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {"error": r.stderr[-300:]}
    return out


def memcpy_baseline(nbytes=512 << 20, reps=5):
    """BASELINE.md 3.3 (context for the migration leg): a host memcpy of one 4096-token Llama-3-8B
    request's KV (512 MiB), single thread, median of reps."""
    import numpy as np
    a = np.ones(nbytes, dtype=np.uint8)
    b = np.empty_like(a)
    ts = []
    for _ in range(reps + 1):
        t0 = time.perf_counter()
        np.copyto(b, a)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts[1:])
    return {"bytes": nbytes, "ms": t * 1e3, "gb_s": nbytes / t / 1e9, "threads": 1}


def migration_bench(src, model, dev, hbm_gbs, n_tokens=(1024, 4096), reps=8):
    """KV migration: tc_kv_migrate of a request's first n_tokens rows
    between two instances, timed by the library with CUDA events around the page-copy kernel.
    This box exposes one GPU, so both instances sit on it (weights shared) and the copy is an
    HBM read + write of whole 2 MiB pages; across GPUs the same kernel pushes over NVLink."""
    from paper_2508_01989_b200 import Instance
    dst = Instance(model, device=dev, weight_seed=1, kv_pool_tokens=max(n_tokens) + 1024, max_step_tokens=512,
                   max_seqs=8, max_context=max(n_tokens) + 64, share_weights=src)
    out = []
    rid = 1 << 40
    for n in n_tokens:
        src.kv_reserve(rid, n)
        a, b = src, dst
        ms, nbytes = [], 0
        for i in range(reps + 2):
            a.migrate_to(b, rid, n)
            t, nbytes = a.migrate_wait()
            if i >= 2:
                ms.append(t)
            a, b = b, a
        a.kv_release(rid)
        t = statistics.median(ms)
        out.append({"tokens": n, "bytes": nbytes, "ms": t, "copy_gb_s": nbytes / t / 1e6,
                    "hbm_gb_s": 2 * nbytes / t / 1e6, "hbm_frac": 2 * nbytes / t / 1e6 / hbm_gbs})
    dst.close()
    return {"kernel": "kv_copy_pages (whole 2 MiB pages, 16 B vectors)", "path": "same-GPU pool-to-pool copy "
            "(1-GPU box): bound = HBM read+write; cross-GPU it is an NVLink P2P push (target 900 GB/s, not "
            "measurable on one GPU)", "median_of": reps, "sizes": out}


def migration_nvlink(inst, rank, world, dev, n_tokens=4096, reps=8):
    """KV migration across GPUs (K11 over NVLink), one process per GPU: rank 2k
    (a prefill-heavy instance) pushes a 4096-token request's pages into rank 2k+1's pool (its
    decode-heavy partner) through a CUDA IPC mapping (tc_kv_push_pages), all pairs at once after a
    barrier. Device time per copy from CUDA events on the source's copy stream; GB/s vs 900."""
    import torch.distributed as dist
    from paper_2508_01989_b200 import RemotePool
    rid = (1 << 41) + rank
    info, res = None, None
    try:
        if rank % 2 == 1:
            inst.kv_reserve(rid, n_tokens)
            info = (inst.export_pool(), [int(x) for x in inst.kv_pages(rid)])
    except Exception as e:  # noqa: BLE001 -- reported in the line, the step numbers stand
        info = ("error", repr(e))
    infos = [None] * world
    dist.all_gather_object(infos, info)
    remote = None
    if rank % 2 == 0 and rank + 1 < world:
        try:
            peer = infos[rank + 1]
            if peer[0] == "error":
                raise RuntimeError(peer[1])
            exported, dpages = peer
            inst.kv_reserve(rid, n_tokens)
            spages = [int(x) for x in inst.kv_pages(rid)]
            remote = RemotePool(exported, device=dev)
            ms, nbytes = [], 0
            for i in range(reps + 2):
                ev = inst.push_pages(remote, spages, dpages[:len(spages)])
                t, nbytes = ev.wait()
                ev.close()
                if i >= 2:
                    ms.append(t)
            t = statistics.median(ms)
            res = {"src": rank, "dst": rank + 1, "bytes": nbytes, "ms": t, "gb_s": nbytes / t / 1e6,
                   "nvlink_frac": nbytes / t / 1e6 / 900.0}
        except Exception as e:  # noqa: BLE001
            res = {"src": rank, "dst": rank + 1, "error": repr(e)}
    dist.barrier()
    if remote is not None:
        remote.close()
    for r in (rid,):
        try:
            inst.kv_release(r)
        except Exception:  # noqa: BLE001 -- not reserved on this rank
            pass
    out = [None] * world
    dist.all_gather_object(out, res)
    pairs = [r for r in out if r]
    ok = [r for r in pairs if "gb_s" in r]
    return {"kernel": "kv_migrate_pages via tc_kv_push_pages (CUDA IPC mapping of the peer's pool, NVLink P2P stores)",
            "tokens": n_tokens, "median_of": reps, "pairs": pairs,
            "min_pair_gb_s": min((r["gb_s"] for r in ok), default=None),
            "min_nvlink_frac": min((r["nvlink_frac"] for r in ok), default=None),
            "peak": "900 GB/s per direction per GPU (NVLink 5, nominal)"}


def reduce_max(vals, device=None):
    """Max over ranks of a list of floats (timing rule: multi-GPU numbers are the max over ranks)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(vals)
    t = torch.tensor(list(vals), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def simulated(args, rank, world, metric, config, P, D):
    """CPU stand-in for the multi-rank path (gloo): same barrier / max-over-ranks / whole-job
    aggregation as the GPU path, with a sleep in place of the step."""
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    for _ in range(args.warmup):
        time.sleep(args.simulate_step_ms / 1e3)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        time.sleep(args.simulate_step_ms / 1e3 * (1 + 0.5 * rank))  # ranks deliberately unequal
    local = time.perf_counter() - t0
    (slowest,) = reduce_max([local])
    if world > 1:
        dist.barrier()
    tokens = (P + D) * args.steps * world
    if rank == 0:
        print(json.dumps({"metric": metric, "value": tokens / slowest, "unit": "tokens/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": slowest / args.steps * 1e3,
                          "higher_is_better": True, "scaling": "weak", "simulated": True,
                          "data": "SIMULATED (test hook, no GPU)", "config": config, "rank_seconds_max": slowest}))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama3_8b")
    ap.add_argument("--prefill", type=int, default=512)
    ap.add_argument("--prefix", type=int, default=512)
    ap.add_argument("--decode", type=int, default=64)
    ap.add_argument("--ctx", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--simulate-step-ms", type=float, default=0.0,
                    help="TEST HOOK (CPU, gloo): replace the GPU step by a sleep to exercise the multi-rank "
                         "timing / aggregation path; the output is marked simulated and is not a measurement")
    ap.add_argument("--profile-window", action="store_true",
                    help="cudaProfilerStart/Stop around the timed steps only (ncu --profile-from-start off)")
    args = ap.parse_args()
    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    P, prefix, D, ctx = args.prefill, args.prefix, args.decode, args.ctx
    n_logit = D + 1
    workload = (f"{args.model} hybrid step: {P}-token prefill chunk (prefix {prefix}) + {D} decodes @ ctx {ctx}; "
                f"chunk size 512, single aggregated instance per GPU")
    config = {"workload": workload, "model_shape": args.model, "step_rows": P + D, "prefill_tokens": P,
              "prefill_prefix": prefix, "decode_reqs": D, "decode_ctx": ctx, "instances": world,
              "l2": None}
    metric = "hybrid-step tokens/s"

    if args.impl == "reference":
        if rank != 0:
            return
        from oracle import cpu_step, model_ref as mr
        import torch
        d = mr.preset(args.model)
        cs = cpu_step.CpuStep(d, P, prefix, D, ctx, n_logit, threads=os.cpu_count())
        vals = []
        for i in range(args.warmup + args.steps):
            sec_i, det = cs.run()
            if i >= args.warmup:
                vals.append(sec_i)
        sec = statistics.median(vals)
        v = (P + D) / sec
        cb = {"value": v, "unit": "tokens/s", "cores": torch.get_num_threads(), "kind": "port",
              "sample": f"per step: the full step, all {d.n_layers} layers + LM head on {n_logit} rows, bf16 torch on "
                        f"the host cores; median of {args.steps} steps after {args.warmup} warm-up",
              "seconds_per_step": sec}
        print(json.dumps({"metric": metric, "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
                          "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                          "config": config, "impl": "reference", "cpu_baseline": cb,
                          "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    import torch
    import torch.distributed as dist

    if args.simulate_step_ms > 0:
        return simulated(args, rank, world, metric, config, P, D)
    from paper_2508_01989_b200 import Instance

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local
    inst = Instance(args.model, device=dev, weight_seed=1, kv_pool_tokens=(D + 2) * (ctx + 64) + prefix + P + 8192,
                    max_step_tokens=max(P + D, 512), max_seqs=D + 8, max_context=max(ctx, prefix + P, 4096) + 64)
    dims = inst.dims.as_dict()
    H_, Hk_, dh_, dm_, F_ = dims["n_heads"], dims["n_kv_heads"], dims["head_dim"], dims["d_model"], dims["ffn_dim"]
    w_gb = 2 * (dims["n_layers"] * ((H_ + 2 * Hk_) * dh_ * dm_ + dm_ * H_ * dh_ + 3 * F_ * dm_) + 2 * dims["vocab"] * dm_) / 1e9
    kv_gb = (D * (ctx + 1) + prefix + P) * 2 * dims["n_kv_heads"] * dims["head_dim"] * 2 * dims["n_layers"] / 1e9
    config["l2"] = (f"inputs larger than L2 ({w_gb:.1f} GB weights + {kv_gb:.1f} GB KV read per step vs 126 MB L2), "
                    f"no flush needed")
    V = dims["vocab"]
    import numpy as np
    rng = np.random.default_rng(1000 + rank)
    # setup (untimed): prefill the chunk's prefix and every decode context
    prompt = rng.integers(0, V, prefix + P).tolist()
    if prefix:
        for s in range(0, prefix, 512):
            inst.step(prefill=[(0, s, prompt[s:min(prefix, s + 512)], False)])
    for rid in range(1, D + 1):
        toks = rng.integers(0, V, ctx).tolist()
        for s in range(0, ctx, 512):
            inst.step(prefill=[(rid, s, toks[s:s + 512], False)])
    dec_tok = rng.integers(0, V, D).tolist()
    step_prefill = [(0, prefix, prompt[prefix:prefix + P], True)] if P else []
    step_decode = [(rid, ctx, dec_tok[rid - 1]) for rid in range(1, D + 1)]

    def one_step():
        return inst.step(prefill=step_prefill, decode=step_decode)

    for _ in range(args.warmup):
        one_step()
    # timed region
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    gpu_ms, launches, h2d, d2h = [], 0, 0, 0
    if args.profile_window:
        torch.cuda.profiler.start()
    with ClockSampler(dev) as clocks:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            o = one_step()
            gpu_ms.append(o.gpu_ms)
            launches += o.launches
            h2d, d2h = o.h2d_bytes, o.d2h_bytes
        t1 = time.perf_counter()
    torch.cuda.synchronize(dev)
    if args.profile_window:
        torch.cuda.profiler.stop()
    dev_s, wall_s = sum(gpu_ms) / 1e3, t1 - t0
    dev_s, wall_s = reduce_max([dev_s, wall_s], device=f"cuda:{dev}")
    if world > 1:
        dist.barrier()
    tokens = (P + D) * args.steps * world
    value = tokens / dev_s
    e2e = tokens / wall_s

    # per-phase device times (separate pass with per-kernel events) -> dominant-kernel roofline
    inst.set_profiling(True)
    phases = {}
    prof_steps = max(3, min(args.steps, 5))
    prof_step_ms = []
    for _ in range(prof_steps):
        o = one_step()
        prof_step_ms.append(o.gpu_ms)
        for ph in ["gemm_qkv", "gemm_o", "gemm_gate_up", "gemm_down", "attn", "norm", "lm_head", "embed"]:
            phases.setdefault(ph, []).append(inst.phase_ms(ph))
    inst.set_profiling(False)
    phases = {k: statistics.median(v) for k, v in phases.items()}
    # context: a decode-only step of the same decodes (half of all serving steps are decode-only,
    # SURVEY.md App. B); weight-streaming bound = weight bytes / HBM bandwidth
    dec_ms = statistics.median([inst.step(decode=step_decode).gpu_ms for _ in range(5)]) if D else float("nan")
    hbm, peak, peak_sus, peak_kind = measured_peaks()
    cost = step_cost(dims, P, prefix, D, ctx, n_logit)
    L = dims["n_layers"]
    gu = cost["gemm_gate_up"]
    gu_launch_s = phases["gemm_gate_up"] / 1e3 / L
    achieved = gu["flops"] / L / gu_launch_s / 1e12
    traffic = None
    tf = REPO / "profiles" / "gemm_gate_up_traffic.json"
    if tf.exists():
        # per model shape: only an ncu capture of THIS model's gate_up launch counts as its traffic
        traffic = json.loads(tf.read_text()).get(args.model, {}).get("dram_bytes_per_launch")
    roofline = {"bound": "tensor", "kernel": "gemm_gate_up (tcgen05, fused SwiGLU)", "achieved": achieved,
                "peak": peak_sus, "unit": "TFLOP/s", "frac": achieved / peak_sus, "traffic": traffic,
                "peak_kind": f"{peak_kind} sustained bf16 (kernel timed inside a long step)",
                "flops_per_launch": gu["flops"] / L, "avg_launch_ms": gu_launch_s * 1e3,
                "share_of_step": phases["gemm_gate_up"] / statistics.median(prof_step_ms)}
    # whole-step roofline: sum over kernel classes of max(F/peak, B/BW) vs the step time
    bound_s = sum(max(c["flops"] / (peak_sus * 1e12), c["bytes"] / (hbm * 1e9)) for c in cost.values())
    step_ms = dev_s / args.steps * 1e3 if world == 1 else statistics.median(gpu_ms)
    step_roofline = {"bound_ms": bound_s * 1e3, "measured_ms": step_ms, "frac": bound_s * 1e3 / step_ms,
                     "phase_ms": phases, "profiled_step_ms": statistics.median(prof_step_ms),
                     "kernels": {k: {"flops": v["flops"], "bytes": v["bytes"],
                                     "bound_ms": 1e3 * max(v["flops"] / (peak_sus * 1e12), v["bytes"] / (hbm * 1e9)),
                                     "measured_ms": phases.get(k)} for k, v in cost.items()}}

    migration = migration_bench(inst, args.model, dev, hbm)
    if world > 1:
        migration["cross_gpu"] = migration_nvlink(inst, rank, world, dev)

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(dims, P, prefix, D, ctx, n_logit, repeats=3)
    if rank == 0:
        line = {"metric": metric, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, random token ids)",
                "config": config, "clocks": clocks.summary(),
                "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
                "gpu_launches": launches * world, "roofline": roofline, "step_roofline": step_roofline,
                "decode_only_step": None if not D else {"decode_reqs": D, "ctx": ctx, "ms": dec_ms, "tokens_per_s": D / dec_ms * 1e3,
                                     "weight_stream_bound_ms": 1e3 * sum(c["bytes"] for k, c in
                                                                         step_cost(dims, 0, 0, D, ctx, D).items()) /
                                                               (measured_peaks()[0] * 1e9)},
                "migration": migration, "cpu_baseline": cb,
                "parity": PARITY.get((args.model, P, prefix, D, ctx), "tests/test_gpu_step.py (shape-generic step parity)")}
        if cb is not None:
            line["cpu_baselines_extra"] = {"scheduler": scheduler_baseline(), "migration_memcpy": memcpy_baseline()}
        print(json.dumps(line))
    inst.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
