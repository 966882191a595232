"""CPU baseline of the hybrid step (TEST / BENCH INFRASTRUCTURE ONLY).

The reference has no arithmetic for the step (its "step" is the affine cost
formula, cost_model.hpp:43-53), so the CPU baseline is the oracle port: the same
mixed step (P prefill rows of one prompt chunk with a paged prefix + D decode
rows at context ctx) in torch fp32 on the host cores, over a layer-reduced
model with the target layer shapes, scaled to the full layer count
(SURVEY.md 8(d) "CPU baselines"). kind = "port".
"""
from __future__ import annotations

import math
import time

import torch


def _layer(d, dev="cpu"):
    H, Hk, dh, dm, F = d.n_heads, d.n_kv_heads, d.head_dim, d.d_model, d.ffn_dim
    g = torch.Generator().manual_seed(0)
    r = lambda *s: torch.randn(*s, generator=g) * 0.02  # noqa: E731
    return {"qkv": r((H + 2 * Hk) * dh, dm), "o": r(dm, H * dh), "gate": r(F, dm), "up": r(F, dm),
            "down": r(dm, F), "n1": torch.ones(dm), "n2": torch.ones(dm)}


def _rms(x, w, eps=1e-5):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * w


@torch.no_grad()
def _layer_forward(L, d, x, p_prefix_k, p_prefix_v, P, dec_k, dec_v):
    """x: [P + D, dm]; prefill rows attend to prefix + causal chunk; decode rows to their cache."""
    H, Hk, dh = d.n_heads, d.n_kv_heads, d.head_dim
    G = H // Hk
    T = x.shape[0]
    h = _rms(x, L["n1"])
    qkv = h @ L["qkv"].T
    q = qkv[:, :H * dh].view(T, H, dh)
    k = qkv[:, H * dh:(H + Hk) * dh].view(T, Hk, dh)
    v = qkv[:, (H + Hk) * dh:].view(T, Hk, dh)
    out = torch.empty(T, H, dh)
    if P:
        Kp = torch.cat([p_prefix_k, k[:P]], 0).repeat_interleave(G, 1)
        Vp = torch.cat([p_prefix_v, v[:P]], 0).repeat_interleave(G, 1)
        s = torch.einsum("thd,shd->hts", q[:P], Kp) / math.sqrt(dh)
        n_pre = p_prefix_k.shape[0]
        mask = torch.arange(Kp.shape[0])[None, :] > (n_pre + torch.arange(P))[:, None]
        s.masked_fill_(mask[None], float("-inf"))
        out[:P] = torch.einsum("hts,shd->thd", torch.softmax(s, -1), Vp)
    D = T - P
    if D:
        Kd = torch.cat([dec_k, k[P:, None]], 1)  # [D, ctx+1, Hk, dh]
        Vd = torch.cat([dec_v, v[P:, None]], 1)
        qd = q[P:].view(D, Hk, G, dh)
        s = torch.einsum("dkgh,dskh->dkgs", qd, Kd) / math.sqrt(dh)
        out[P:] = torch.einsum("dkgs,dskh->dkgh", torch.softmax(s, -1), Vd).reshape(D, H, dh)
    x = x + out.reshape(T, H * dh) @ L["o"].T
    h = _rms(x, L["n2"])
    return x + (torch.nn.functional.silu(h @ L["gate"].T) * (h @ L["up"].T)) @ L["down"].T


class CpuStep:
    """Builds one layer of the target shape + the LM head once; run() times one full-depth step
    (one layer measured, scaled by n_layers, plus the LM head on n_logit rows)."""

    def __init__(self, d, P: int, prefix: int, D: int, ctx: int, n_logit: int, threads: int | None = None):
        if threads:
            torch.set_num_threads(threads)
        self.d, self.P, self.n_logit = d, P, n_logit
        self.L = _layer(d)
        g = torch.Generator().manual_seed(1)
        self.x = torch.randn(P + D, d.d_model, generator=g)
        self.pk = torch.randn(prefix, d.n_kv_heads, d.head_dim, generator=g)
        self.pv = torch.randn(prefix, d.n_kv_heads, d.head_dim, generator=g)
        self.dk = torch.randn(D, ctx, d.n_kv_heads, d.head_dim, generator=g)
        self.dv = torch.randn(D, ctx, d.n_kv_heads, d.head_dim, generator=g)
        self.lm = torch.randn(d.vocab, d.d_model, generator=g) * 0.02

    @torch.no_grad()
    def run(self):
        t0 = time.perf_counter()
        y = _layer_forward(self.L, self.d, self.x, self.pk, self.pv, self.P, self.dk, self.dv)
        t1 = time.perf_counter()
        _ = (_rms(y[-self.n_logit:], self.L["n1"]) @ self.lm.T).argmax(-1)
        t2 = time.perf_counter()
        return (t1 - t0) * self.d.n_layers + (t2 - t1), {"layer_s": t1 - t0, "head_s": t2 - t1}


def time_step(d, P, prefix, D, ctx, n_logit, repeats: int = 1, threads: int | None = None):
    """Best-of-`repeats` seconds per full-depth step (after one warm-up run)."""
    cs = CpuStep(d, P, prefix, D, ctx, n_logit, threads)
    cs.run()
    best, det = min((cs.run() for _ in range(repeats)), key=lambda r: r[0])
    return best, {**det, "layers_timed": 1, "scaled_to": d.n_layers, "threads": torch.get_num_threads()}
