"""CPU baseline of the hybrid step (TEST / BENCH INFRASTRUCTURE ONLY).

The reference has no arithmetic for the step (its "step" is the affine cost formula,
cost_model.hpp:43-53), so the CPU baseline is the oracle port (kind = "port"): the same mixed step
-- P prefill rows of one prompt chunk over a paged prefix + D decode rows at context ctx -- through
ALL n_layers layers on the host cores (SURVEY.md 8(d) "CPU baselines"):

  embed -> L x [RMSNorm -> QKV -> RoPE -> paged KV append (block-table scatter) -> causal prefill
  attention over the gathered prefix pages + decode attention over each request's gathered pages
  (GQA) -> O + residual -> RMSNorm -> SwiGLU MLP + residual] -> RMSNorm -> LM head on the
  sampled rows -> argmax.

Arithmetic in bf16 (oneDNN / AMX on this host) with fp32 softmax and residual, i.e. the GPU path's
storage type; fp32 on request. To bound host memory, the n_layers layers share one layer's weights
and one page pool (every layer still does all of its reads and math).
"""
from __future__ import annotations

import math
import time

import torch


def _rms(x, w, eps=1e-5):
    xf = x.float()
    return (xf * torch.rsqrt((xf * xf).mean(-1, keepdim=True) + eps) * w).to(x.dtype)


def _rope(x, cos, sin):
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half].float(), x[..., half:].float()
    c, s = cos[:, None, :], sin[:, None, :]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], -1).to(x.dtype)


class CpuStep:
    """Builds the step's weights, page pool and block tables once; run() times one full step."""

    def __init__(self, d, P: int, prefix: int, D: int, ctx: int, n_logit: int, threads: int | None = None,
                 dtype=torch.bfloat16, page: int = 16):
        if threads:
            torch.set_num_threads(threads)
        self.d, self.P, self.prefix, self.D, self.ctx, self.n_logit, self.dt, self.page = d, P, prefix, D, ctx, n_logit, dtype, page
        H, Hk, dh, dm, F = d.n_heads, d.n_kv_heads, d.head_dim, d.d_model, d.ffn_dim
        g = torch.Generator().manual_seed(0)
        r = lambda *s: (torch.randn(*s, generator=g) * 0.02).to(dtype)  # noqa: E731
        self.W = {"qkv": r((H + 2 * Hk) * dh, dm), "o": r(dm, H * dh), "gate_up": r(2 * F, dm), "down": r(dm, F),
                  "bias": r((H + 2 * Hk) * dh) if d.qkv_bias else None,
                  "n1": torch.ones(dm), "n2": torch.ones(dm), "nf": torch.ones(dm)}
        self.embed = r(d.vocab, dm) * 50
        self.lm = r(d.vocab, dm)
        # page pool [pages, page, 2 (k|v), Hk, dh]: the prefill request's pages, then each decode's
        n_pf_pages = (prefix + P + page - 1) // page
        n_dec_pages = (ctx + 1 + page - 1) // page
        self.n_pages = n_pf_pages + D * n_dec_pages
        self.pool = torch.zeros(self.n_pages, page, 2, Hk, dh, dtype=dtype)
        self.pool.normal_(generator=g)
        self.bt_pf = torch.arange(n_pf_pages)
        self.bt_dec = n_pf_pages + torch.arange(D * n_dec_pages).view(D, n_dec_pages)
        self.tokens = torch.randint(0, d.vocab, (P + D,), generator=g)
        self.pos = torch.cat([prefix + torch.arange(P), torch.full((D,), ctx)]).long()
        half = dh // 2
        inv = torch.tensor([math.pow(d.rope_theta, -2.0 * j / dh) for j in range(half)], dtype=torch.float64)
        ang = self.pos.double()[:, None] * inv[None, :]
        self.cos, self.sin = torch.cos(ang).float(), torch.sin(ang).float()
        # KV slot of every new row: (page, slot)
        pf_rows = prefix + torch.arange(P)
        self.new_page = torch.cat([self.bt_pf[pf_rows // page], self.bt_dec[:, ctx // page]])
        self.new_slot = torch.cat([pf_rows % page, torch.full((D,), ctx % page)])

    @torch.no_grad()
    def _layer(self, x):
        d, W, P, D = self.d, self.W, self.P, self.D
        H, Hk, dh = d.n_heads, d.n_kv_heads, d.head_dim
        G, T = H // Hk, P + D
        h = _rms(x, W["n1"], d.rms_eps).to(self.dt)
        qkv = h @ W["qkv"].T
        if W["bias"] is not None:
            qkv = qkv + W["bias"]
        q = _rope(qkv[:, :H * dh].view(T, H, dh), self.cos, self.sin)
        k = _rope(qkv[:, H * dh:(H + Hk) * dh].view(T, Hk, dh), self.cos, self.sin)
        v = qkv[:, (H + Hk) * dh:].view(T, Hk, dh)
        self.pool[self.new_page, self.new_slot, 0] = k
        self.pool[self.new_page, self.new_slot, 1] = v
        out = torch.empty(T, H, dh, dtype=self.dt)
        sdpa = torch.nn.functional.scaled_dot_product_attention
        if P:
            n_keys = self.prefix + P
            kv = self.pool[self.bt_pf].view(-1, 2, Hk, dh)[:n_keys]
            mask = torch.arange(n_keys)[None, :] <= self.pos[:P, None]  # causal over prefix + chunk
            o = sdpa(q[:P].transpose(0, 1)[None], kv[:, 0].transpose(0, 1)[None], kv[:, 1].transpose(0, 1)[None],
                     attn_mask=mask[None, None], enable_gqa=True)
            out[:P] = o[0].transpose(0, 1)
        if D:
            kv = self.pool[self.bt_dec].view(D, -1, 2, Hk, dh)[:, :self.ctx + 1]
            o = sdpa(q[P:].view(D, H, 1, dh), kv[:, :, 0].transpose(1, 2), kv[:, :, 1].transpose(1, 2), enable_gqa=True)
            out[P:] = o[:, :, 0]
        x = x + (out.reshape(T, H * dh) @ W["o"].T).float()
        h = _rms(x, W["n2"], d.rms_eps).to(self.dt)
        gu = h @ W["gate_up"].T
        F = d.ffn_dim
        a = torch.nn.functional.silu(gu[:, :F]) * gu[:, F:]
        return x + (a @ W["down"].T).float()

    @torch.no_grad()
    def run(self):
        t0 = time.perf_counter()
        x = self.embed[self.tokens].float()
        for _ in range(self.d.n_layers):
            x = self._layer(x)
        rows = torch.cat([torch.tensor([self.P - 1]) if self.P else torch.zeros(0, dtype=torch.long),
                          self.P + torch.arange(self.D)])[-self.n_logit:]
        ids = (_rms(x[rows], self.W["nf"], self.d.rms_eps).to(self.dt) @ self.lm.T).float().argmax(-1)
        t1 = time.perf_counter()
        return t1 - t0, {"layers_timed": self.d.n_layers, "sampled": int(ids.numel())}


def time_step(d, P, prefix, D, ctx, n_logit, repeats: int = 3, threads: int | None = None, dtype=torch.bfloat16):
    """Median seconds per full-depth step over `repeats` runs (after one warm-up run)."""
    cs = CpuStep(d, P, prefix, D, ctx, n_logit, threads, dtype)
    cs.run()
    secs = sorted(cs.run()[0] for _ in range(repeats))
    return secs[len(secs) // 2], {"layers_timed": d.n_layers, "threads": torch.get_num_threads(), "repeats": repeats,
                                  "dtype": str(dtype).replace("torch.", "")}
