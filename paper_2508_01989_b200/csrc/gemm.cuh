// tcgen05 / TMEM / TMA GEMM for the dense projections of the hybrid step
// (SURVEY.md 2, K3-K7): C[M,N] = A[M,K] * B[N,K]^T, bf16 in, fp32 accumulate.
//
//   A: activations, row-major [M, K]  (M = packed prefill + decode rows of one step)
//   B: weights, row-major [N, K]      (K-major, nn.Linear layout)
//
// Persistent schedule with optional split-K. Work units are (tile, k-split) with
// the M-tile index fastest, so the CTAs that run concurrently share the same
// weight N-tile and k-range and stream it from DRAM once (weights are 15 GB, far
// beyond L2; an order that lets CTAs drift apart in k re-reads them). CTA c runs
// units c, c+G, c+2G, ... (G = min(#SMs, units)). The split count is chosen on the
// host by a wave-quantisation cost model: M = 576 gives 4.5 M-tiles and 80..120
// N-tiles, a partial wave that split-K fills; decode-only steps (M <= 128) use it
// to spread the weight stream over all SMs.
// Residual-add GEMMs (O-proj, down-proj: N = d_model gives only 80 tiles at M = 576)
// reduce their k-splits with red.global.add.v4.f32 straight into the fp32 residual
// stream (summation order across splits is not fixed: ~1 ulp run-to-run jitter).
// Other split GEMMs finish a tile in whichever CTA arrives LAST on the tile's atomic
// counter: every split writes its fp32 partial to its own slot and the last
// arriver sums the slots in split order (deterministic) and applies the epilogue.
// No CTA ever waits for another, so concurrent streams on one GPU cannot deadlock.
//
// Warp roles (256 threads, 1 CTA/SM):
//   warp 0      TMA producer: A/B K-slabs (BK = 32 -> 64 B rows, SWIZZLE_64B) into a
//               deep smem ring (8 stages at BN = 256: 7 x 24 KB in flight covers the
//               ~1 us TMA latency at the MMA consumption rate) guarded by full/empty
//               mbarriers.
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma (M=128, N=BN,
//               K=16) into a double-buffered TMEM accumulator; tcgen05.commit
//               releases smem slots and signals the epilogue.
//   warp 2      TMEM allocator.
//   warps 4-7   epilogue: tcgen05.ld (32 lanes x 32 columns per warp) -> fused op
//               -> 16 B global stores; overlaps the next segment's main loop.
// Fused epilogues: bf16 store, +bias (Qwen2 QKV), fp32 residual add (O / down),
// SwiGLU on 64-row interleaved gate/up weights, fp32 store (LM-head logits).
#pragma once

#include "common.cuh"

namespace tc {

enum EpilogueOp : int {
  EPI_BF16 = 0,       // out_bf16[m, n] = acc
  EPI_BF16_BIAS = 1,  // out_bf16[m, n] = acc + bias[n]
  EPI_RESID_F32 = 2,  // resid_f32[m, n] += acc
  EPI_SWIGLU = 3,     // out_bf16[m, n/2 ...] = silu(gate) * up, 64-interleaved
  EPI_F32 = 4,        // out_f32[m, n] = acc
  EPI_QKV_ROPE = 5    // (+bias) -> RoPE(q, k) -> q to out_bf16, k / v to the paged KV pool
};

// Per-row metadata of the fused QKV epilogue (QKV GEMM + RoPE + KV append).
struct QkvRopeArgs {
  __nv_bfloat16* kv;       // KV pool base
  const float2* rope_cs;   // [position][head_dim / 2] (cos, sin)
  const int* positions;    // [rows]
  const int* row_seq;      // [rows] sequence of the row
  const int* row_kv;       // [rows] KV pool row of the token: page * page_size + slot
  const int* seq_bt_off;   // [seqs] offset into block_tables
  const int* block_tables;
  long long page_stride;   // elements per page
  int layer, n_heads, n_kv_heads, head_dim, page_size;
};

constexpr int kGemmBM = 128;
#ifndef TC_GEMM_BK
#define TC_GEMM_BK 64
#endif
constexpr int kGemmBK = TC_GEMM_BK;  // K per pipeline stage (32 or 64 bf16 = 64 / 128 B rows)
constexpr int kGemmThreads = 256;

struct GemmArgs {
  int M, N, K;
  int m_tiles, n_tiles, kb;  // kb = k-blocks per tile
  int splits;                // k-splits per tile
  int units;                 // m_tiles * n_tiles * splits
  void* out;
  const __nv_bfloat16* bias;
  int ldo;
  float* ws;                 // partial slots [units][BN/32][128][32] (splits > 1)
  int* tile_cnt;             // per-tile arrival counters (zero; last arriver resets)
  QkvRopeArgs rope;          // EPI_QKV_ROPE only
  int tn;                    // gemm_ws_2sm: token tile (multiple of 32, <= 256)
  int stages;                // gemm_ws_2sm: smem ring depth for this token tile
  unsigned long long* trace; // gemm_ws_2sm (tools only): per-CTA %globaltimer stamps [grid][16]
  int streamk;               // gemm_ws_2sm, residual epilogue: grouped stream-K (gemm_ws.cuh WsIter)
  int groups;                // gemm_ws_2sm stream-K: pair groups (m_tiles sibling pairs each)
};

template <int BN>
struct GemmCfg {
  static constexpr int kStages = (BN >= 256 ? 4 : 6) * (64 / kGemmBK);
  static constexpr int kABytes = kGemmBM * kGemmBK * 2;
  static constexpr int kBBytes = BN * kGemmBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
  static constexpr int kSlotFloats = kGemmBM * BN;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 512 /*barriers*/;
};

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

// unit u -> (tile = mt + m_tiles * nt, k-range [k0, k1), split index ks)
struct Unit {
  int mt, nt, ks, k0, k1;
};
__device__ __forceinline__ Unit unit_of(const GemmArgs& a, int u) {
  Unit x;
  x.mt = u % a.m_tiles;
  const int r = u / a.m_tiles;
  x.ks = r % a.splits;
  x.nt = r / a.splits;
  x.k0 = (int)(((long long)a.kb * x.ks) / a.splits);
  x.k1 = (int)(((long long)a.kb * (x.ks + 1)) / a.splits);
  return x;
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Applies the epilogue op to one 32-column chunk of row m held in v[32] (fp32).
template <int BN, int EPI>
__device__ __forceinline__ void epi_store_chunk(const GemmArgs& args, int m, int n0, const float (&v)[32]) {
  if constexpr (EPI == EPI_BF16 || EPI == EPI_BF16_BIAS) {
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(args.out) + (size_t)m * args.ldo + n0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 w;
      uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int c = q * 8 + e * 2;
        float a0 = v[c], a1 = v[c + 1];
        if constexpr (EPI == EPI_BF16_BIAS) {
          a0 += __bfloat162float(args.bias[n0 + c]);
          a1 += __bfloat162float(args.bias[n0 + c + 1]);
        }
        wp[e] = pack_bf16(a0, a1);
      }
      st_global_v4(out + q * 8, w);
    }
  } else if constexpr (EPI == EPI_RESID_F32) {
    float* out = reinterpret_cast<float*>(args.out) + (size_t)m * args.ldo + n0;
    if (args.splits > 1) {  // split-K: every k-split adds its partial straight into the residual
#pragma unroll
      for (int q = 0; q < 8; ++q)
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(out + q * 4), "f"(v[q * 4]),
                     "f"(v[q * 4 + 1]), "f"(v[q * 4 + 2]), "f"(v[q * 4 + 3])
                     : "memory");
      return;
    }
    float4 x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = *reinterpret_cast<float4*>(out + q * 4);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      x[q].x += v[q * 4 + 0];
      x[q].y += v[q * 4 + 1];
      x[q].z += v[q * 4 + 2];
      x[q].w += v[q * 4 + 3];
      *reinterpret_cast<float4*>(out + q * 4) = x[q];
    }
  } else if constexpr (EPI == EPI_F32) {
    float* out = reinterpret_cast<float*>(args.out) + (size_t)m * args.ldo + n0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      st_global_v4(out + q * 4, make_uint4(__float_as_uint(v[q * 4]), __float_as_uint(v[q * 4 + 1]),
                                           __float_as_uint(v[q * 4 + 2]), __float_as_uint(v[q * 4 + 3])));
  }
}

// SwiGLU on a (gate, up) pair of 32-column chunks -> 32 bf16 outputs.
__device__ __forceinline__ void epi_swiglu_chunk(const GemmArgs& args, int m, int out_col, const float (&g)[32],
                                                 const float (&u)[32]) {
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(args.out) + (size_t)m * args.ldo + out_col;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 w;
    uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int c = q * 8 + e * 2;
      wp[e] = pack_bf16(silu(g[c]) * u[c], silu(g[c + 1]) * u[c + 1]);
    }
    st_global_v4(out + q * 8, w);
  }
}

// Fused QKV epilogue for one row m of an N-tile: fetch(chunk, v) yields 32 accumulator
// columns. Each head's columns (j, j + DH/2) are rotated together (rotate_half RoPE).
// fetch may be warp-collective (tcgen05.ld): every lane runs the whole routine and
// only the stores are predicated on row_ok.
template <int BN, typename Fetch>
__device__ __forceinline__ void epi_qkv_rope_row(const GemmArgs& args, int m_in, bool row_ok, int nt, Fetch&& fetch) {
  const QkvRopeArgs& r = args.rope;
  const int m = row_ok ? m_in : 0;
  const int DH = r.head_dim, half = DH / 2, hc = half / 32;  // chunks per half head
  const int pos = r.positions[m];
  const int seq = r.row_seq[m];
  const int page = r.block_tables[r.seq_bt_off[seq] + pos / r.page_size];
  const int slot = pos % r.page_size;
  const float2* cs = r.rope_cs + (size_t)pos * half;
#pragma unroll 1
  for (int hh = 0; hh < BN / DH; ++hh) {
    const int head = (nt * BN) / DH + hh;
    const bool is_q = head < r.n_heads, is_k = !is_q && head < r.n_heads + r.n_kv_heads;
    __nv_bfloat16* dst;
    if (is_q) {
      dst = reinterpret_cast<__nv_bfloat16*>(args.out) + (size_t)m * args.ldo + head * DH;
    } else {
      const int kvh = head - r.n_heads - (is_k ? 0 : r.n_kv_heads);
      dst = r.kv + (size_t)page * r.page_stride +
            ((((size_t)r.layer * r.n_kv_heads + kvh) * 2 + (is_k ? 0 : 1)) * r.page_size + slot) * DH;
    }
#pragma unroll 1
    for (int c = 0; c < hc; ++c) {
      float lo[32], hi[32];
      fetch(hh * (DH / 32) + c, lo);
      fetch(hh * (DH / 32) + hc + c, hi);
      const int n_lo = nt * BN + hh * DH + c * 32;
      if (args.bias) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          lo[i] += __bfloat162float(args.bias[n_lo + i]);
          hi[i] += __bfloat162float(args.bias[n_lo + half + i]);
        }
      }
      if (is_q || is_k) {
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float4 t = *reinterpret_cast<const float4*>(cs + c * 32 + i);  // (cos, sin) x 2
          const float a0 = lo[i], b0 = hi[i], a1 = lo[i + 1], b1 = hi[i + 1];
          lo[i] = a0 * t.x - b0 * t.y;
          hi[i] = b0 * t.x + a0 * t.y;
          lo[i + 1] = a1 * t.z - b1 * t.w;
          hi[i + 1] = b1 * t.z + a1 * t.w;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 wl, wh;
        uint32_t* pl = reinterpret_cast<uint32_t*>(&wl);
        uint32_t* ph = reinterpret_cast<uint32_t*>(&wh);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          pl[e] = pack_bf16(lo[q * 8 + 2 * e], lo[q * 8 + 2 * e + 1]);
          ph[e] = pack_bf16(hi[q * 8 + 2 * e], hi[q * 8 + 2 * e + 1]);
        }
        if (row_ok) {
          st_global_v4(dst + c * 32 + q * 8, wl);
          st_global_v4(dst + half + c * 32 + q * 8, wh);
        }
      }
    }
  }
}

template <int BN>
__device__ __forceinline__ float* slot_ptr(const GemmArgs& a, int slot, int chunk, int row) {  // slot = unit
  return a.ws + (size_t)slot * GemmCfg<BN>::kSlotFloats + ((size_t)chunk * kGemmBM + row) * 32;
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                      GemmArgs args) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + S * Cfg::kABytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;   // [2]
  uint64_t* tempty_bar = tfull_bar + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 128);
    }
    mbar_fence_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // predecessor kernel's outputs (activations, residual) are visible from here on
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < args.units; u += gridDim.x) {
        const Unit w = unit_of(args, u);
        for (int kb = w.k0; kb < w.k1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
          tma_load_2d(smem_a + stage * Cfg::kABytes, &map_a, &full_bar[stage], kb * kGemmBK, w.mt * kGemmBM, kEvictLast);
          tma_load_2d(smem_b + stage * Cfg::kBBytes, &map_b, &full_bar[stage], kb * kGemmBK, w.nt * BN, kEvictNormal);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (single elected lane)
    constexpr uint32_t idesc = umma_idesc_bf16(kGemmBM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    for (int u = blockIdx.x; u < args.units; u += gridDim.x) {
      const Unit w = unit_of(args, u);
      const int k0 = w.k0, k1 = w.k1;
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      ++local;
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = k0; kb < k1; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_addr = smem_u32(smem_a + stage * Cfg::kABytes);
          const uint32_t b_addr = smem_u32(smem_b + stage * Cfg::kBBytes);
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k) {
            const uint64_t ad = umma_smem_desc<kGemmBK * 2>(a_addr + k * 32);
            const uint64_t bd = umma_smem_desc<kGemmBK * 2>(b_addr + k * 32);
            umma_bf16(d_tmem, ad, bd, idesc, (kb > k0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty_bar[stage]);
          if (kb == k1 - 1) umma_commit(&tfull_bar[acc]);
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue warpgroup: thread t owns accumulator row t
    const int ew = warp - 4;  // == warp % 4 -> TMEM lane quarter
    const int row = ew * 32 + lane;
    int local = 0;
    for (int u = blockIdx.x; u < args.units; u += gridDim.x) {
      const Unit w = unit_of(args, u);
      const int mt = w.mt, nt = w.nt;
      const int tile = mt + args.m_tiles * nt;
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      ++local;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int m = mt * kGemmBM + row;
      const bool row_ok = m < args.M;
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
      // residual-add GEMMs reduce split-K partials with red.global.add (no workspace)
      const bool whole = args.splits == 1 || EPI == EPI_RESID_F32;

      if (whole) {
        if constexpr (EPI == EPI_QKV_ROPE) {
          auto fetch = [&](int chunk, float (&v)[32]) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(t_row + chunk * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          };
          epi_qkv_rope_row<BN>(args, m, row_ok, nt, fetch);
        } else if constexpr (EPI == EPI_SWIGLU) {
#pragma unroll 1
          for (int grp = 0; grp < BN / 128; ++grp) {
#pragma unroll 1
            for (int half = 0; half < 2; ++half) {
              uint32_t gr[32], ur[32];
              tmem_ld_32x32b_x32(t_row + grp * 128 + half * 32, gr);
              tmem_ld_32x32b_x32(t_row + grp * 128 + 64 + half * 32, ur);
              tmem_ld_wait();
              float g[32], u[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                g[i] = __uint_as_float(gr[i]);
                u[i] = __uint_as_float(ur[i]);
              }
              if (row_ok) epi_swiglu_chunk(args, m, (nt * BN) / 2 + grp * 64 + half * 32, g, u);
            }
          }
        } else {
#pragma unroll 1
          for (int chunk = 0; chunk < BN / 32; ++chunk) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(t_row + chunk * 32, r);
            tmem_ld_wait();
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
            if (row_ok) epi_store_chunk<BN, EPI>(args, m, nt * BN + chunk * 32, v);
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty_bar[acc]);
        continue;
      }

      // ---- split tile: publish this unit's partial, the last arriver reduces
      const int my_slot = u;
#pragma unroll 1
      for (int chunk = 0; chunk < BN / 32; ++chunk) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_row + chunk * 32, r);
        tmem_ld_wait();
        if (row_ok) {
          float* dst = slot_ptr<BN>(args, my_slot, chunk, row);
#pragma unroll
          for (int q = 0; q < 8; ++q) st_global_v4(dst + q * 4, make_uint4(r[q * 4], r[q * 4 + 1], r[q * 4 + 2], r[q * 4 + 3]));
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);  // accumulator no longer needed
      __threadfence();
      epi_bar();
      if (threadIdx.x == 128) {
        const int old = atomicAdd(&args.tile_cnt[tile], 1);
        const bool last = old == args.splits - 1;
        if (last) args.tile_cnt[tile] = 0;  // ready for the next launch
        *last_flag = last ? 1 : 0;
      }
      epi_bar();
      const bool last = *last_flag != 0;
      epi_bar();  // last_flag is reused by the next segment
      if (!last) continue;
      __threadfence();
      if (!row_ok) continue;
      auto load_sum = [&](int chunk, float (&v)[32]) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
        for (int ks = 0; ks < args.splits; ++ks) {
          const int slot = mt + args.m_tiles * (ks + args.splits * nt);
          const float4* src = reinterpret_cast<const float4*>(slot_ptr<BN>(args, slot, chunk, row));
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 p = __ldcg(src + q);
            v[q * 4] += p.x;
            v[q * 4 + 1] += p.y;
            v[q * 4 + 2] += p.z;
            v[q * 4 + 3] += p.w;
          }
        }
      };
      if constexpr (EPI == EPI_QKV_ROPE) {
        epi_qkv_rope_row<BN>(args, m, true, nt, load_sum);
      } else if constexpr (EPI == EPI_SWIGLU) {
#pragma unroll 1
        for (int grp = 0; grp < BN / 128; ++grp) {
#pragma unroll 1
          for (int half = 0; half < 2; ++half) {
            float g[32], u[32];
            load_sum(grp * 4 + half, g);
            load_sum(grp * 4 + 2 + half, u);
            epi_swiglu_chunk(args, m, (nt * BN) / 2 + grp * 64 + half * 32, g, u);
          }
        }
      } else {
#pragma unroll 1
        for (int chunk = 0; chunk < BN / 32; ++chunk) {
          float v[32];
          load_sum(chunk, v);
          epi_store_chunk<BN, EPI>(args, m, nt * BN + chunk * 32, v);
        }
      }
    }
  }

  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
}

}  // namespace tc
