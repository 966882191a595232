// Weight-stationary pair GEMM for the mixed hybrid step, C = X * W^T
// computed transposed: the MMA's M dimension runs over WEIGHT rows and its N dimension over
// the step's TOKENS.
//
// Why: a step packs T = prefill chunk + decodes rows (576 at the bench config). With tokens
// on M the 128-row tile pads 576 to 640 (11% dead MMA work) and the 256-row pair tile pads it
// to 768. UMMA N, in contrast, is any multiple of 16 up to 256, so the token tile is sized to
// the step: n_tt = ceil(T / 256) tiles of TN = round_up(T / n_tt, 32) tokens (576 -> 3 x 192,
// 512 -> 2 x 256, 1100 -> 5 x 224), padding at most 31 rows per tile.
//
// CTA pair (cluster 2x1, tcgen05.mma.cta_group::2, M = 256, N = TN, K = 16): each CTA stages
// its own 128 weight rows (16 KB per 64-deep k-block) and HALF of the token tile (TN/2 rows),
// so a 256 x 192 pair tile costs each SM 28 KB of L2->SMEM traffic per k-block for 384 MMA
// cycles (73 B/clk) against 96 B/clk for the 128 x 256 single-SM tile. The leader issues the
// MMAs; both CTAs' TMA credit the leader's full barrier; commits multicast to both CTAs.
//
// Unit order: token tile fastest, so the n_tt pairs that share a weight tile run together and
// the 15 GB weight stream leaves DRAM once (the activations, <= 17 MB, stay in L2).
//
// Epilogue (warps 4-7): TMEM holds [128 weight rows (lanes)] x [TN tokens (columns)]. Each
// 32-token chunk is read with tcgen05.ld 32x32b (thread = weight row), transposed through a
// double-buffered, XOR-swizzled fp32 staging tile (bank-conflict-free both ways), and then
// processed token-row-wise: thread (token t, segment s) owns 32 consecutive features of one
// token, which is what every fused op needs (bias, SwiGLU on 64-row interleaved gate/up
// blocks, RoPE pairs (j, j + head_dim/2) inside one head, paged KV append, fp32 residual add;
// split-K partials of the residual GEMMs are reduced with red.global.add.v4.f32).
#pragma once

#include "gemm.cuh"

#ifndef TC_WS_MAX_STAGES
#define TC_WS_MAX_STAGES 12
#endif

namespace tc {

constexpr int kWsMaxStages = TC_WS_MAX_STAGES;  // ring depth cap (barrier area fits 12)
static_assert(kWsMaxStages <= 12, "ws GEMM barrier area holds at most 12 stages");
constexpr int kWsWBytes = 128 * kGemmBK * 2;           // this CTA's 128 weight rows per k-block
constexpr int kWsStagingFloats = 32 * 128;             // one 32-token x 128-feature fp32 chunk
constexpr int kWsSmemBytes = 232448;                   // max dynamic shared memory per CTA (sm_100)
constexpr int kWsBarBytes = 256;
constexpr int kWsMetaBytes = 2 * 2 * 256 * 4;          // per-unit-parity token metadata (pos, kv row)
constexpr int kWsRingBudget = kWsSmemBytes - 1024 - 2 * kWsStagingFloats * 4 - kWsMetaBytes - kWsBarBytes;
// warps 0 + 3 TMA, 1 MMA, 2 TMEM alloc, 4-7 epilogue group 0 (even 32-token chunks),
// 8-11 epilogue group 1 (odd chunks): two groups hide each other's TMEM / smem / store latency
constexpr int kWsThreads = 384;

__host__ __device__ constexpr int ws_stage_bytes(int tn) { return kWsWBytes + (tn / 2) * kGemmBK * 2; }
// ring depth for token tile tn: as deep as the budget allows, even (two producer warps alternate)
__host__ __device__ constexpr int ws_stages(int tn) {
  return (ws_stage_bytes(tn) * kWsMaxStages <= kWsRingBudget ? kWsMaxStages : kWsRingBudget / ws_stage_bytes(tn)) & ~1;
}

// Features [4ch, 4ch + 4) of staged token row t (XOR swizzle: conflict-free transposed writes
// by 32 weight rows and row-wise float4 reads by (2 tokens x 4 segments) quarter-warps).
__device__ __forceinline__ int ws_stg_idx(int t, int ch) { return t * 128 + ((ch ^ ((ch >> 3) & 3) ^ ((t & 1) << 2)) << 2); }
__device__ __forceinline__ float4 ws_ld4(const float* sb, int t, int ch) {
  return *reinterpret_cast<const float4*>(sb + ws_stg_idx(t, ch));
}

// Token-row epilogue: token tok (valid), 32 features of segment s of the CTA's 128 weight rows
// starting at global weight row fbase.
template <int EPI>
__device__ __forceinline__ void ws_row_epilogue(const GemmArgs& args, const float* sb, int t, int s, int tok, int fbase,
                                                int pos, int kv_row, const float4 (&cs_reg)[8]) {
  if constexpr (EPI == EPI_BF16 || EPI == EPI_BF16_BIAS) {
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(args.out) + (size_t)tok * args.ldo + fbase + s * 32;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float4 a = ws_ld4(sb, t, s * 8 + 2 * q), b = ws_ld4(sb, t, s * 8 + 2 * q + 1);
      if constexpr (EPI == EPI_BF16_BIAS) {
        const __nv_bfloat16* bb = args.bias + fbase + s * 32 + q * 8;
        a.x += __bfloat162float(bb[0]); a.y += __bfloat162float(bb[1]);
        a.z += __bfloat162float(bb[2]); a.w += __bfloat162float(bb[3]);
        b.x += __bfloat162float(bb[4]); b.y += __bfloat162float(bb[5]);
        b.z += __bfloat162float(bb[6]); b.w += __bfloat162float(bb[7]);
      }
      st_global_v4(out + q * 8, make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y), pack_bf16(b.z, b.w)));
    }
  } else if constexpr (EPI == EPI_F32) {
    float* out = reinterpret_cast<float*>(args.out) + (size_t)tok * args.ldo + fbase + s * 32;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 a = ws_ld4(sb, t, s * 8 + q);
      st_global_v4(out + q * 4, make_uint4(__float_as_uint(a.x), __float_as_uint(a.y), __float_as_uint(a.z), __float_as_uint(a.w)));
    }
  } else if constexpr (EPI == EPI_RESID_F32) {
    float* out = reinterpret_cast<float*>(args.out) + (size_t)tok * args.ldo + fbase + s * 32;
    if (args.splits > 1) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 a = ws_ld4(sb, t, s * 8 + q);
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(out + q * 4), "f"(a.x), "f"(a.y), "f"(a.z),
                     "f"(a.w)
                     : "memory");
      }
    } else {
      float4 x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = *reinterpret_cast<const float4*>(out + q * 4);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 a = ws_ld4(sb, t, s * 8 + q);
        x[q].x += a.x; x[q].y += a.y; x[q].z += a.z; x[q].w += a.w;
        *reinterpret_cast<float4*>(out + q * 4) = x[q];
      }
    }
  } else if constexpr (EPI == EPI_SWIGLU) {
    // weight rows [fbase, fbase + 64) = gate, [fbase + 64, fbase + 128) = up of outputs fbase / 2 + [0, 64)
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(args.out) + (size_t)tok * args.ldo + fbase / 2 + s * 16;
    uint32_t w[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 g = ws_ld4(sb, t, s * 4 + q), u = ws_ld4(sb, t, 16 + s * 4 + q);
      w[q * 2] = pack_bf16(silu(g.x) * u.x, silu(g.y) * u.y);
      w[q * 2 + 1] = pack_bf16(silu(g.z) * u.z, silu(g.w) * u.w);
    }
    st_global_v4(out, make_uint4(w[0], w[1], w[2], w[3]));
    st_global_v4(out + 8, make_uint4(w[4], w[5], w[6], w[7]));
  } else if constexpr (EPI == EPI_QKV_ROPE) {
    // this thread: rotation pairs (j, j + DH/2), j in [j0, j0 + 16), of head fbase / DH + hh
    const QkvRopeArgs& r = args.rope;
    const int DH = r.head_dim, half = DH >> 1;
    const int hh = (s * 16) / half, j0 = (s * 16) % half;
    const int head = fbase / DH + hh;
    const int lo_f = hh * DH + j0;  // tile-local feature of the first lo element
    const bool is_q = head < r.n_heads, is_k = !is_q && head < r.n_heads + r.n_kv_heads;
    __nv_bfloat16* dst;
    if (is_q) {
      dst = reinterpret_cast<__nv_bfloat16*>(args.out) + (size_t)tok * args.ldo + head * DH;
    } else {
      const int page = kv_row / r.page_size, slot = kv_row - page * r.page_size;
      const int kvh = head - r.n_heads - (is_k ? 0 : r.n_kv_heads);
      dst = r.kv + (size_t)page * r.page_stride +
            ((((size_t)r.layer * r.n_kv_heads + kvh) * 2 + (is_k ? 0 : 1)) * r.page_size + slot) * DH;
    }
    float lo[16], hi[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 a = ws_ld4(sb, t, (lo_f >> 2) + q), b = ws_ld4(sb, t, ((lo_f + half) >> 2) + q);
      lo[q * 4] = a.x; lo[q * 4 + 1] = a.y; lo[q * 4 + 2] = a.z; lo[q * 4 + 3] = a.w;
      hi[q * 4] = b.x; hi[q * 4 + 1] = b.y; hi[q * 4 + 2] = b.z; hi[q * 4 + 3] = b.w;
    }
    if (args.bias) {
      const __nv_bfloat16* bl = args.bias + fbase + lo_f;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        lo[i] += __bfloat162float(bl[i]);
        hi[i] += __bfloat162float(bl[half + i]);
      }
    }
    if (is_q || is_k) {
      // (cos, sin) of this row's pairs j0.., loaded into registers before the accumulator chunk
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const float4 c = cs_reg[i >> 1];  // (cos, sin) x 2
        const float a0 = lo[i], b0 = hi[i], a1 = lo[i + 1], b1 = hi[i + 1];
        lo[i] = a0 * c.x - b0 * c.y;
        hi[i] = b0 * c.x + a0 * c.y;
        lo[i + 1] = a1 * c.z - b1 * c.w;
        hi[i + 1] = b1 * c.z + a1 * c.w;
      }
    }
    uint32_t wl[8], wh[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      wl[i] = pack_bf16(lo[2 * i], lo[2 * i + 1]);
      wh[i] = pack_bf16(hi[2 * i], hi[2 * i + 1]);
    }
    st_global_v4(dst + j0, make_uint4(wl[0], wl[1], wl[2], wl[3]));
    st_global_v4(dst + j0 + 8, make_uint4(wl[4], wl[5], wl[6], wl[7]));
    st_global_v4(dst + half + j0, make_uint4(wh[0], wh[1], wh[2], wh[3]));
    st_global_v4(dst + half + j0 + 8, make_uint4(wh[4], wh[5], wh[6], wh[7]));
  }
}

// Work iterator shared by the producer, MMA and epilogue roles of one pair (identical sequences).
// Default: units u = pair, pair + n_pairs, ... (tile, k-split). Grouped stream-K (residual
// epilogue, where every partial is a TMA bulk add): pair p is token tile p % m_tiles of group
// p / m_tiles; group g takes the contiguous range [W g / G, W (g+1) / G) of the weight-tile-major
// k-block stream (W = n_tiles * kb), cut at weight-tile boundaries. The m_tiles siblings of a
// group issue the same weight k-blocks at the same time (one DRAM read, the rest hit L2), and
// every pair gets the same number of k-blocks whatever the tile count.
struct WsIter {
  long long pos, end;  // stream-K
  int u, mt;           // units / stream-K token tile
};
__device__ __forceinline__ WsIter ws_iter_begin(const GemmArgs& a, int pair, int n_pairs) {
  WsIter it;
  it.u = pair;
  it.mt = pair % a.m_tiles;
  const int grp = pair / a.m_tiles;
  const long long total = (long long)a.n_tiles * a.kb;
  it.pos = total * grp / a.groups;
  it.end = total * (grp + 1) / a.groups;
  return it;
}
__device__ __forceinline__ bool ws_next(const GemmArgs& a, WsIter& it, int n_pairs, Unit& w) {
  if (!a.streamk) {
    if (it.u >= a.units) return false;
    w = unit_of(a, it.u);
    it.u += n_pairs;
    return true;
  }
  if (it.pos >= it.end) return false;
  const int tile = (int)(it.pos / a.kb);
  w.k0 = (int)(it.pos - (long long)tile * a.kb);
  w.k1 = (int)min((long long)a.kb, w.k0 + (it.end - it.pos));
  w.mt = it.mt;
  w.nt = tile;
  w.ks = 0;
  it.pos += w.k1 - w.k0;
  return true;
}

// map_w: weights [N, K], box 64 x 128 rows; map_x: activations [rows, K], box 64 x TN/2 rows;
// map_o (EPI_RESID_F32 only): the fp32 residual [rows, N], box 128 features x 32 tokens, no
// swizzle -- each 32-token chunk is staged densely and added by one TMA bulk reduction
// (cp.reduce.async.bulk.tensor .add), which also reduces the split-K partials.
// args.m_tiles = token tiles, args.n_tiles = 256-row weight pair tiles, args.tn, args.stages.
template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kWsThreads, 1)
    gemm_ws_2sm(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
                const __grid_constant__ CUtensorMap map_o, GemmArgs args) {
  const int TN = args.tn, S = args.stages;
  const int stage_bytes = ws_stage_bytes(TN);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* stg = reinterpret_cast<float*>(smem + S * stage_bytes);  // [group][32][128]
  int* meta = reinterpret_cast<int*>(stg + 2 * kWsStagingFloats);  // [unit parity][pos | kv row][256]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(meta + 2 * 2 * 256);
  uint64_t* empty_bar = full_bar + kWsMaxStages;
  uint64_t* tfull_bar = empty_bar + kWsMaxStages;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;            // [2] (leader's copy is used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  // tools-only timeline: 0 entry, 1 prologue done, 2 first stage landed (MMA), 3 last MMA issued,
  // 4 epilogue of the first unit done, 5 epilogue of the last unit done
  auto stamp = [&](int i) {
    if (args.trace) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      args.trace[blockIdx.x * 16 + i] = t;
    }
  };
  if (threadIdx.x == 0) stamp(0);
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_x);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 16);  // 8 epilogue warps x 2 CTAs
    }
    mbar_fence_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) stamp(1);
  // predecessor kernel's outputs (activations, residual) are visible after pdl_wait; the TMA
  // producer waits later, after it has issued the weight loads of its first stages
  if (!(warp == 0 && lane == 0)) pdl_wait();
  pdl_trigger();

  if (warp == 0 || warp == 3) {
    // Two producer warps (0 and 3) issue the k-block stream together: warp 0 the even issue
    // indices, warp 3 the odd ones (S is even, so every ring stage belongs to one of them). One
    // issuing thread sustains only a limited TMA rate (tools/stream_bench.cu: 16 KiB boxes reach
    // 4.2 / 6.6 TB/s chip-wide with 1 / 2 issuing warps per SM), which capped the decode-only
    // weight stream.
    const int pj = warp == 0 ? 0 : 1;
    if (lane == 0) {
      const int half_tn = TN / 2;
      const int wrow = (int)rank * 128;
      // Weights do not depend on the predecessor kernel: fill the first ring stages with this
      // CTA's weight k-blocks while the predecessor drains (PDL), then wait for the activations.
      int pre = 0;
      WsIter it = ws_iter_begin(args, pair, n_pairs);
      Unit w0;
      if (ws_next(args, it, n_pairs, w0)) {
        pre = min(S, w0.k1 - w0.k0);
        for (int i = pj; i < pre; i += 2) {
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[i], 2 * stage_bytes);
          tma_load_2d_2sm(smem + i * stage_bytes, &map_w, &full_bar[i], (w0.k0 + i) * kGemmBK, w0.nt * 256 + wrow,
                          kEvictNormal);
        }
      }
      pdl_wait();
      int issued = 0;
      it = ws_iter_begin(args, pair, n_pairs);
      Unit w;  // w.mt = token tile, w.nt = weight pair tile
      while (ws_next(args, it, n_pairs, w)) {
        for (int kb = w.k0; kb < w.k1; ++kb, ++issued) {
          if ((issued & 1) != pj) continue;
          const int stage = issued % S;
          const uint32_t phase = (uint32_t)(issued / S) & 1u;
          uint8_t* st = smem + stage * stage_bytes;
          if (issued >= pre) {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * stage_bytes);
            tma_load_2d_2sm(st, &map_w, &full_bar[stage], kb * kGemmBK, w.nt * 256 + wrow, kEvictNormal);
          }
          tma_load_2d_2sm(st + kWsWBytes, &map_x, &full_bar[stage], kb * kGemmBK, w.mt * TN + (int)rank * half_tn,
                          kEvictLast);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      const uint32_t idesc = umma_idesc_bf16(256, TN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      WsIter it = ws_iter_begin(args, pair, n_pairs);
      Unit w;
      while (ws_next(args, it, n_pairs, w)) {
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        ++local;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = w.k0; kb < w.k1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (local == 1 && kb == w.k0 && lane == 0) stamp(2);
          if (elect_one()) {
            const uint32_t w_addr = smem_u32(smem + stage * stage_bytes);
            const uint32_t x_addr = w_addr + kWsWBytes;
#pragma unroll
            for (int k = 0; k < kGemmBK / 16; ++k)
              umma_bf16_2sm(d_tmem, umma_smem_desc<kGemmBK * 2>(w_addr + k * 32),
                            umma_smem_desc<kGemmBK * 2>(x_addr + k * 32), idesc, (kb > w.k0 || k > 0) ? 1u : 0u);
            umma_commit_2sm_multicast(&empty_bar[stage]);
            if (kb == w.k1 - 1) {
              umma_commit_2sm_multicast(&tfull_bar[acc]);
              stamp(3);
            }
          }
          __syncwarp();
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {
    const int grp = (warp - 4) >> 2;            // epilogue group: chunks ci with ci % 2 == grp
    const int ew = warp & 3;                    // TMEM lane quarter (warp % 4)
    const int f = ew * 32 + lane;               // weight row within this CTA's 128 (transposed write)
    const int et = (threadIdx.x - 128) & 127;   // thread within the group
    const int t = et >> 2, s = et & 3;          // token row / 32-feature segment (row phase)
    const int fch = f >> 2, fe = f & 3;
    const uint32_t gbar = 1 + grp;              // named barrier of this group (128 threads)
    float* sb = stg + grp * kWsStagingFloats;
    const int n_chunks = TN / 32;
    int local = 0;
    WsIter it = ws_iter_begin(args, pair, n_pairs);
    Unit w;
    while (ws_next(args, it, n_pairs, w)) {
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      ++local;
      int* mpos = meta + acc * 512;
      int* mkv = mpos + 256;
      if constexpr (EPI == EPI_QKV_ROPE) {
        // this unit's per-token RoPE / KV-append metadata -> smem (both groups), fetched while
        // the MMAs run; the rows' (cos, sin) lines are pulled into L2 (the weight stream evicts
        // the table between layers)
        const int e2 = threadIdx.x - 128;  // 0..255
        const int tok = w.mt * TN + e2;
        if (e2 < TN) {
          const bool ok = tok < args.M;
          const int pos = ok ? __ldg(args.rope.positions + tok) : 0;
          mpos[e2] = pos;
          mkv[e2] = ok ? __ldg(args.rope.row_kv + tok) : 0;
          if (ok) {
            const int half = args.rope.head_dim >> 1;
            for (int c = 0; c < half; c += 32)
              asm volatile("prefetch.global.L2 [%0];" ::"l"(args.rope.rope_cs + (size_t)pos * half + c));
          }
        }
        asm volatile("bar.sync 3, 256;" ::: "memory");
      }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      if (et == 0 && grp == 0) stamp(7);
      const int fbase = w.nt * 256 + (int)rank * 128;
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * 256;
      const int my_last = (n_chunks - 1 - grp) >= 0 ? ((n_chunks - 1 - grp) & ~1) + grp : -1;
      if (my_last < 0) {  // a single-chunk tile leaves group 1 idle: release its share at once
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&tempty_bar[acc]);
      }
#pragma unroll 1
      for (int ci = grp; ci < n_chunks; ci += 2) {
        const int c0 = ci * 32;
        // QKV: this thread's RoPE (cos, sin) pairs for its row phase, fetched before the TMEM read
        // and the staging barriers so the L2 round trip overlaps them (round 1: on the critical path)
        float4 cs_reg[8];
        if constexpr (EPI == EPI_QKV_ROPE) {
          const int half = args.rope.head_dim >> 1;
          const int j0 = (s * 16) % half, head = (w.nt * 256 + (int)rank * 128) / args.rope.head_dim + (s * 16) / half;
          if (head < args.rope.n_heads + args.rope.n_kv_heads && w.mt * TN + c0 + t < args.M) {
            const float4* cs = reinterpret_cast<const float4*>(args.rope.rope_cs + (size_t)mpos[c0 + t] * half + j0);
#pragma unroll
            for (int i = 0; i < 8; ++i) cs_reg[i] = __ldg(cs + i);
          }
        }
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_row + c0, r);
        tmem_ld_wait();
        if (et == 0 && grp == 0 && ci < 6) stamp(8 + ci);      // 8, 10, 12: chunk's accumulator in registers
        if (ci == my_last) {  // this warp's last read of the accumulator: release it early
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_leader(&tempty_bar[acc]);
        }
        if constexpr (EPI == EPI_RESID_F32) {
          // dense [32 tokens][128 features] chunk -> one TMA bulk add into the residual; the
          // group's issuing thread first makes sure its previous reduction finished reading sb
          if (et == 0) bulk_wait_group_read<0>();
          asm volatile("bar.sync %0, 128;" ::"r"(gbar) : "memory");
          const int tok0 = w.mt * TN + c0;
#pragma unroll
          for (int i = 0; i < 32; ++i) sb[i * 128 + f] = tok0 + i < args.M ? __uint_as_float(r[i]) : 0.f;
          fence_async_smem();
          asm volatile("bar.sync %0, 128;" ::"r"(gbar) : "memory");
          if (et == 0) {
            tma_reduce_add_2d(&map_o, smem_u32(sb), fbase, tok0);
            bulk_commit_group();
          }
        } else {
          asm volatile("bar.sync %0, 128;" ::"r"(gbar) : "memory");  // previous row phase done with sb
#pragma unroll
          for (int i = 0; i < 32; ++i) sb[ws_stg_idx(i, fch) + fe] = __uint_as_float(r[i]);
          asm volatile("bar.sync %0, 128;" ::"r"(gbar) : "memory");
          const int tok = w.mt * TN + c0 + t;
          if (tok < args.M) ws_row_epilogue<EPI>(args, sb, t, s, tok, fbase, mpos[c0 + t], mkv[c0 + t], cs_reg);
        }
        if (et == 0 && grp == 0 && ci < 6) stamp(9 + ci);      // 9, 11, 13: chunk done
      }
      if (et == 0 && grp == 0) {
        if (local == 1) stamp(4);
        stamp(5);
      }
    }
  }

  // the staged residual chunks must have been read by the TMA unit before the CTA's smem goes away
  if (EPI == EPI_RESID_F32 && warp >= 4 && ((threadIdx.x - 128) & 127) == 0) bulk_wait_group_read<0>();
  tc_fence_before();
  cluster_sync();  // every MMA retired and both epilogues drained before TMEM is released
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, 512);
    if (lane == 0) stamp(6);
  }
}

}  // namespace tc
