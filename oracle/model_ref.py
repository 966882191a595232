"""CPU oracle of the hybrid-step arithmetic (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module, and only as the checker -- never as the thing measured or shipped.

Parity status: UNPINNED. The reference (/root/reference/proj) is a simulator
whose hybrid step is the affine formula iteration_time_ms
(proj/include/pdsim/cost_model.hpp:43-53); it contains no model arithmetic, and
the paper's numerics live in vLLM, which is not vendored and has no pinned
version under /root/reference. This module therefore restates
our own written spec of a standard Llama-3 /
Qwen2 decoder:

  x = E[token]                                  (fp32 residual stream)
  per layer:  h = bf16(RMSNorm(x) * w_attn)
              qkv = h @ Wqkv^T [+ b]            q|k|v rows, fp32 accumulate (no rounding yet)
              q, k = bf16(RoPE(q, k)), v = bf16(v)   half-split rotation, theta, fp64 table;
                                                ONE bf16 rounding after RoPE, as the fused
                                                QKV epilogue stores it (gemm_ws.cuh)
              o = bf16(softmax(q k^T / sqrt(dh), causal, GQA h -> h // G) v)
              x += o @ Wo^T
              h = bf16(RMSNorm(x) * w_mlp)
              x += bf16(silu(h Wg^T) * (h Wu^T)) @ Wd^T
  logits = bf16(RMSNorm(x_last) * w_final) @ Wlm^T ; token = argmax (lowest index on ties)

Weights are the library's deterministic init, re-derived here bit-for-bit from
the same splitmix64 hash (include/taichi_b200.h tc_weight_value).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)

# tensor ids / scales (must match csrc/taichi_b200.cu)
TID_EMBED, TID_LM_HEAD, TID_FINAL_NORM = 1, 2, 3
LIN_SCALE = np.float32(0.034641016)
BIAS_SCALE = np.float32(0.1)
NORM_SCALE = np.float32(0.1)


def tid_layer(l: int, j: int) -> int:
    return 16 + 16 * l + j


def _sm64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def bf16_bits_from_f32(v: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 (finite inputs)."""
    b = v.astype(np.float32).view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    return ((b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)


def gen_bits(seed: int, tid: int, rows: int, cols: int, scale, offset, chunk: int = 1 << 22) -> np.ndarray:
    """bf16 bits of logical tensor `tid` [rows, cols] (csrc/elementwise.cuh init_weights)."""
    key = _sm64(np.array([seed], dtype=np.uint64) ^ _sm64(np.array([tid], dtype=np.uint64)))[0]
    n = rows * cols
    out = np.empty(n, dtype=np.uint16)
    for s in range(0, n, chunk):
        idx = np.arange(s, min(n, s + chunk), dtype=np.uint64)
        with np.errstate(over="ignore"):
            h = _sm64(idx + key)
        u = (h >> np.uint64(40)).astype(np.float32) * np.float32(5.9604644775390625e-08)
        c = u * np.float32(2.0) - np.float32(1.0)
        v = (c * np.float32(scale)).astype(np.float32) + np.float32(offset)
        out[s:s + len(idx)] = bf16_bits_from_f32(v.astype(np.float32))
    return out.reshape(rows, cols)


@dataclass
class Dims:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn_dim: int
    vocab: int
    qkv_bias: int
    rope_theta: float
    rms_eps: float

    @staticmethod
    def from_any(d) -> "Dims":
        if isinstance(d, Dims):
            return d
        if isinstance(d, dict):
            return Dims(**d)
        return Dims(**{k: getattr(d, k) for k in Dims.__dataclass_fields__})


PRESETS = {
    "tiny": Dims(2, 256, 4, 2, 64, 512, 1024, 0, 1.0e4, 1e-5),
    "llama3_8b": Dims(32, 4096, 32, 8, 128, 14336, 128256, 0, 5.0e5, 1e-5),
    "qwen2_5_14b": Dims(48, 5120, 40, 8, 128, 13824, 152064, 1, 1.0e6, 1e-6),
}


def preset(name: str) -> Dims:
    base, _, lay = name.partition(":L")
    d = Dims(**PRESETS[base].__dict__)
    if lay:
        d.n_layers = int(lay)
    # the GPU stores rope_theta / eps as fp32
    d.rope_theta = float(np.float32(d.rope_theta))
    d.rms_eps = float(np.float32(d.rms_eps))
    return d


def _t(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(bf16_bits_to_f32(bits).copy())


def generate_weights(dims: Dims, seed: int) -> dict:
    """All weights as fp32 torch tensors holding bf16-exact values (logical layout)."""
    m = dims
    H, Hk, dh, dm, F = m.n_heads, m.n_kv_heads, m.head_dim, m.d_model, m.ffn_dim
    qkv_n = (H + 2 * Hk) * dh
    w = {
        "embed": _t(gen_bits(seed, TID_EMBED, m.vocab, dm, np.float32(1.0), 0.0)),
        "lm_head": _t(gen_bits(seed, TID_LM_HEAD, m.vocab, dm, LIN_SCALE, 0.0)),
        "final_norm": _t(gen_bits(seed, TID_FINAL_NORM, 1, dm, NORM_SCALE, np.float32(1.0)))[0],
        "layers": [],
    }
    for l in range(m.n_layers):
        w["layers"].append({
            "qkv": _t(gen_bits(seed, tid_layer(l, 0), qkv_n, dm, LIN_SCALE, 0.0)),
            "o": _t(gen_bits(seed, tid_layer(l, 1), dm, H * dh, LIN_SCALE, 0.0)),
            "gate": _t(gen_bits(seed, tid_layer(l, 2), F, dm, LIN_SCALE, 0.0)),
            "up": _t(gen_bits(seed, tid_layer(l, 3), F, dm, LIN_SCALE, 0.0)),
            "down": _t(gen_bits(seed, tid_layer(l, 4), dm, F, LIN_SCALE, 0.0)),
            "attn_norm": _t(gen_bits(seed, tid_layer(l, 5), 1, dm, NORM_SCALE, np.float32(1.0)))[0],
            "mlp_norm": _t(gen_bits(seed, tid_layer(l, 6), 1, dm, NORM_SCALE, np.float32(1.0)))[0],
            "qkv_bias": _t(gen_bits(seed, tid_layer(l, 7), 1, qkv_n,
                                    BIAS_SCALE if m.qkv_bias else np.float32(0.0), 0.0))[0],
        })
    return w


def weights_from_device(inst, dims: Dims) -> dict:
    """Logical weights read back from a GPU instance (big shapes, where hashing in numpy is slow)."""
    m = dims
    F = m.ffn_dim

    def get(name):
        return _t(inst.weight(name))

    w = {"embed": get("embed"), "lm_head": get("lm_head"), "final_norm": get("final_norm")[0], "layers": []}
    for l in range(m.n_layers):
        gu = get(f"L{l}.gate_up")  # [2F, dm], 64-row interleaved gate|up
        blocks = gu.view(F // 64, 2, 64, -1)
        w["layers"].append({
            "qkv": get(f"L{l}.qkv"), "o": get(f"L{l}.o"),
            "gate": blocks[:, 0].reshape(F, -1).contiguous(), "up": blocks[:, 1].reshape(F, -1).contiguous(),
            "down": get(f"L{l}.down"), "attn_norm": get(f"L{l}.attn_norm")[0],
            "mlp_norm": get(f"L{l}.mlp_norm")[0], "qkv_bias": get(f"L{l}.qkv_bias")[0],
        })
    return w


def bf16(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32)


def rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    inv = torch.rsqrt((x * x).mean(dim=-1, keepdim=True) + eps)
    return x * inv * w


def rope_table(dims: Dims, max_pos: int) -> tuple[torch.Tensor, torch.Tensor]:
    half = dims.head_dim // 2
    inv = np.array([math.pow(dims.rope_theta, -2.0 * j / dims.head_dim) for j in range(half)], dtype=np.float64)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return torch.from_numpy(np.cos(ang).astype(np.float32)), torch.from_numpy(np.sin(ang).astype(np.float32))


def apply_rope(x: torch.Tensor, pos: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    # x [T, nh, dh]
    half = x.shape[-1] // 2
    c = cos[pos][:, None, :]
    s = sin[pos][:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)


class RefModel:
    """Per-request incremental decoder with a dense KV cache (the token oracle)."""

    def __init__(self, dims: Dims, weights: dict, max_pos: int = 4096, round_bf16: bool = True):
        """round_bf16=False drops every bf16 storage point (pure fp32 math): the mode in which the
        restatement is pinned against an independent Llama / Qwen2 implementation
        (tests/test_oracle_model_pinning.py: HF transformers, tests/golden/hf_*.npz)."""
        self.m = dims
        self.w = weights
        self.cos, self.sin = rope_table(dims, max_pos)
        self.rnd = bf16 if round_bf16 else (lambda t: t)

    def new_cache(self):
        return [{"k": None, "v": None} for _ in range(self.m.n_layers)]

    @torch.no_grad()
    def forward(self, tokens, pos0: int, cache) -> torch.Tensor:
        """Feed tokens at positions pos0.. ; returns final hidden (fp32) [T, d]."""
        m, w, bf16 = self.m, self.w, self.rnd
        H, Hk, dh = m.n_heads, m.n_kv_heads, m.head_dim
        G = H // Hk
        toks = torch.as_tensor(np.asarray(tokens, dtype=np.int64))
        T = toks.shape[0]
        pos = torch.arange(pos0, pos0 + T)
        x = w["embed"][toks].clone()
        for l, L in enumerate(w["layers"]):
            h = bf16(rmsnorm(x, L["attn_norm"], m.rms_eps))
            qkv = h @ L["qkv"].T + L["qkv_bias"]
            q = qkv[:, : H * dh].view(T, H, dh)
            k = qkv[:, H * dh:(H + Hk) * dh].view(T, Hk, dh)
            v = bf16(qkv[:, (H + Hk) * dh:].view(T, Hk, dh))
            q = bf16(apply_rope(q, pos, self.cos, self.sin))
            k = bf16(apply_rope(k, pos, self.cos, self.sin))
            c = cache[l]
            c["k"] = k if c["k"] is None else torch.cat([c["k"], k], 0)
            c["v"] = v if c["v"] is None else torch.cat([c["v"], v], 0)
            K = c["k"].repeat_interleave(G, dim=1)  # [S, H, dh]
            V = c["v"].repeat_interleave(G, dim=1)
            S = K.shape[0]
            scores = torch.einsum("thd,shd->hts", q, K) / math.sqrt(dh)
            qpos = pos[:, None]
            kpos = torch.arange(S)[None, :]
            scores = scores.masked_fill((kpos > qpos)[None], float("-inf"))
            p = torch.softmax(scores, dim=-1)
            o = bf16(torch.einsum("hts,shd->thd", p, V).reshape(T, H * dh))
            x = x + o @ L["o"].T
            h = bf16(rmsnorm(x, L["mlp_norm"], m.rms_eps))
            a = bf16(torch.nn.functional.silu(h @ L["gate"].T) * (h @ L["up"].T))
            x = x + a @ L["down"].T
        return x

    @torch.no_grad()
    def logits(self, x_rows: torch.Tensor) -> torch.Tensor:
        h = self.rnd(rmsnorm(x_rows, self.w["final_norm"], self.m.rms_eps))
        return h @ self.w["lm_head"].T

    @torch.no_grad()
    def generate(self, prompt, n_new: int, chunk: int = 0):
        """Greedy continuation of `prompt`; returns (tokens [n_new], logits [n_new, V])."""
        cache = self.new_cache()
        prompt = list(prompt)
        pos = 0
        step = chunk or len(prompt)
        x = None
        while pos < len(prompt):
            x = self.forward(prompt[pos:pos + step], pos, cache)
            pos += len(prompt[pos:pos + step])
        out_t, out_l = [], []
        lg = self.logits(x[-1:])[0]
        for i in range(n_new):
            t = int(torch.argmax(lg).item())
            out_t.append(t)
            out_l.append(lg)
            if i + 1 == n_new:
                break
            x = self.forward([t], pos, cache)
            pos += 1
            lg = self.logits(x[-1:])[0]
        return out_t, torch.stack(out_l)


def prompt_tokens(seed: int, req_id: int, n: int, vocab: int) -> list[int]:
    """Deterministic synthetic prompt ids: splitmix64(seed ^ req_id << 20 ^ pos) % vocab.
    (Traces carry lengths only -- types.hpp:28-31 -- so ids are synthesised.)"""
    idx = (np.uint64(seed) ^ (np.uint64(req_id) << np.uint64(20))) ^ np.arange(n, dtype=np.uint64)
    return (_sm64(idx) % np.uint64(vocab)).astype(np.int64).tolist()
