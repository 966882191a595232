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


@torch.no_grad()
def time_step(d, P: int, prefix: int, D: int, ctx: int, n_logit: int, repeats: int = 1, threads: int | None = None):
    """Seconds for one full-depth step, measured on ONE layer (+ LM head on n_logit rows) and
    scaled by n_layers. Returns (seconds_per_step, detail dict)."""
    if threads:
        torch.set_num_threads(threads)
    L = _layer(d)
    g = torch.Generator().manual_seed(1)
    x = torch.randn(P + D, d.d_model, generator=g)
    pk = torch.randn(prefix, d.n_kv_heads, d.head_dim, generator=g)
    pv = torch.randn(prefix, d.n_kv_heads, d.head_dim, generator=g)
    dk = torch.randn(D, ctx, d.n_kv_heads, d.head_dim, generator=g)
    dv = torch.randn(D, ctx, d.n_kv_heads, d.head_dim, generator=g)
    lm = torch.randn(d.vocab, d.d_model, generator=g) * 0.02
    _layer_forward(L, d, x, pk, pv, P, dk, dv)  # warm-up
    best_layer, best_head = float("inf"), float("inf")
    for _ in range(repeats):
        t0 = time.perf_counter()
        y = _layer_forward(L, d, x, pk, pv, P, dk, dv)
        t1 = time.perf_counter()
        lg = _rms(y[-n_logit:], L["n1"]) @ lm.T
        _ = lg.argmax(-1)
        t2 = time.perf_counter()
        best_layer, best_head = min(best_layer, t1 - t0), min(best_head, t2 - t1)
    total = best_layer * d.n_layers + best_head
    return total, {"layer_s": best_layer, "head_s": best_head, "layers_timed": 1, "scaled_to": d.n_layers,
                   "threads": torch.get_num_threads()}
