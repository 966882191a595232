// tcgen05 / TMEM / TMA GEMM for the dense projections of the hybrid step
// (SURVEY.md 2, K3-K7): C[M,N] = A[M,K] * B[N,K]^T, bf16 in, fp32 accumulate.
//
//   A: activations, row-major [M, K]  (M = packed prefill + decode tokens)
//   B: weights, row-major [N, K]      (K-major, PyTorch nn.Linear layout)
//
// Structure (one CTA per SM, persistent, static tile schedule):
//   warp 0      TMA producer: A/B K-slabs (BK = 64 -> 128 B rows, SWIZZLE_128B)
//               into a kStages-deep smem ring guarded by full/empty mbarriers.
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma (M=128, N=BN,
//               K=16) into a double-buffered TMEM accumulator; tcgen05.commit
//               releases smem slots and signals the epilogue.
//   warps 4-7   epilogue: tcgen05.ld (32 lanes x 32 columns per warp) -> fused
//               op -> 16 B global stores. Overlaps the next tile's main loop.
// Fused epilogues: plain bf16 store, +bias (Qwen2 QKV), fp32 residual add
// (O-proj / down-proj), SwiGLU on 64-row interleaved gate/up weights, fp32
// store (LM-head logits), fp32 split-K partials (small-M weight streaming).
#pragma once

#include "common.cuh"

namespace tc {

enum EpilogueOp : int {
  EPI_BF16 = 0,        // out_bf16[m, n] = acc
  EPI_BF16_BIAS = 1,   // out_bf16[m, n] = acc + bias[n]
  EPI_RESID_F32 = 2,   // resid_f32[m, n] += acc
  EPI_SWIGLU = 3,      // out_bf16[m, n/2 ...] = silu(gate) * up, 64-interleaved
  EPI_F32 = 4,         // out_f32[m, n] = acc
  EPI_PARTIAL_F32 = 5  // ws[split][m, n] = acc  (split-K; reduced by a second kernel)
};

struct GemmArgs {
  int M, N, K;
  int m_tiles, n_tiles, k_splits, k_blocks_per_split;
  void* out;           // bf16 / f32 output, or f32 residual (EPI_RESID_F32), or workspace
  const __nv_bfloat16* bias;
  int ldo;             // leading dimension of out (elements)
};

constexpr int kGemmBM = 128;
constexpr int kGemmBK = 64;
constexpr int kGemmThreads = 256;

template <int BN>
struct GemmCfg {
  static constexpr int kStages = BN >= 256 ? 4 : (BN >= 128 ? 6 : 8);
  static constexpr int kABytes = kGemmBM * kGemmBK * 2;
  static constexpr int kBBytes = BN * kGemmBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;  // double-buffered accumulator
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

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

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n_units = args.m_tiles * args.n_tiles * args.k_splits;

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

  // unit -> (m_tile fastest so CTAs sharing a weight tile run together, then n, then split)
  auto decode_unit = [&](int u, int& mt, int& nt, int& ks) {
    mt = u % args.m_tiles;
    const int r = u / args.m_tiles;
    nt = r % args.n_tiles;
    ks = r / args.n_tiles;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        int mt, nt, ks;
        decode_unit(u, mt, nt, ks);
        const int kb0 = ks * args.k_blocks_per_split;
        for (int kb = 0; kb < args.k_blocks_per_split; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
          const int kc = (kb0 + kb) * kGemmBK;
          tma_load_2d(smem_a + stage * Cfg::kABytes, &map_a, &full_bar[stage], kc, mt * kGemmBM, kEvictLast);
          tma_load_2d(smem_b + stage * Cfg::kBBytes, &map_b, &full_bar[stage], kc, nt * BN, kEvictFirst);
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
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < args.k_blocks_per_split; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_addr = smem_u32(smem_a + stage * Cfg::kABytes);
          const uint32_t b_addr = smem_u32(smem_b + stage * Cfg::kBBytes);
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k) {
            const uint64_t ad = umma_smem_desc_sw128(a_addr + k * 32);
            const uint64_t bd = umma_smem_desc_sw128(b_addr + k * 32);
            umma_bf16(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(&empty_bar[stage]);
          if (kb == args.k_blocks_per_split - 1) umma_commit(&tfull_bar[acc]);
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
    const int row_in_tile = ew * 32 + lane;
    int local = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++local) {
      int mt, nt, ks;
      decode_unit(u, mt, nt, ks);
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int m = mt * kGemmBM + row_in_tile;
      const bool row_ok = m < args.M;
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
      if constexpr (EPI == EPI_SWIGLU) {
        // columns [128j, 128j+64) = gate block j, [128j+64, 128j+128) = up block j
#pragma unroll 1
        for (int grp = 0; grp < BN / 128; ++grp) {
#pragma unroll 1
          for (int half = 0; half < 2; ++half) {
            uint32_t g[32], v[32];
            tmem_ld_32x32b_x32(t_row + grp * 128 + half * 32, g);
            tmem_ld_32x32b_x32(t_row + grp * 128 + 64 + half * 32, v);
            tmem_ld_wait();
            if (row_ok) {
              __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(args.out) + (size_t)m * args.ldo +
                                   (nt * BN) / 2 + grp * 64 + half * 32;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                uint4 w;
                uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int c = q * 8 + e * 2;
                  const float a0 = silu(__uint_as_float(g[c])) * __uint_as_float(v[c]);
                  const float a1 = silu(__uint_as_float(g[c + 1])) * __uint_as_float(v[c + 1]);
                  wp[e] = pack_bf16(a0, a1);
                }
                st_global_v4(out + q * 8, w);
              }
            }
          }
        }
      } else {
#pragma unroll 1
        for (int chunk = 0; chunk < BN / 32; ++chunk) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_row + chunk * 32, r);
          tmem_ld_wait();
          if (!row_ok) continue;
          const int n0 = nt * BN + chunk * 32;
          if constexpr (EPI == EPI_BF16 || EPI == EPI_BF16_BIAS) {
            __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(args.out) + (size_t)m * args.ldo + n0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 w;
              uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int c = q * 8 + e * 2;
                float a0 = __uint_as_float(r[c]), a1 = __uint_as_float(r[c + 1]);
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
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              float4 x = *reinterpret_cast<float4*>(out + q * 4);
              x.x += __uint_as_float(r[q * 4 + 0]);
              x.y += __uint_as_float(r[q * 4 + 1]);
              x.z += __uint_as_float(r[q * 4 + 2]);
              x.w += __uint_as_float(r[q * 4 + 3]);
              *reinterpret_cast<float4*>(out + q * 4) = x;
            }
          } else {  // EPI_F32 / EPI_PARTIAL_F32
            float* out = reinterpret_cast<float*>(args.out);
            if constexpr (EPI == EPI_PARTIAL_F32) out += (size_t)ks * args.M * args.ldo;
            out += (size_t)m * args.ldo + n0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              st_global_v4(out + q * 4, make_uint4(r[q * 4], r[q * 4 + 1], r[q * 4 + 2], r[q * 4 + 3]));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
    }
  }

  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
}

// Split-K reduction + the deferred epilogue: sums `splits` fp32 partial slabs.
template <int EPI>
__global__ void gemm_splitk_reduce(const float* __restrict__ ws, int splits, int M, int N, void* out, int ldo,
                                   const __nv_bfloat16* __restrict__ bias) {
  const int cols_per_thread = 4;
  const size_t total = (size_t)M * (EPI == EPI_SWIGLU ? N / 2 : N) / cols_per_thread;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    if constexpr (EPI == EPI_SWIGLU) {
      const int half_n = N / 2;
      const int m = (int)(i * 4 / half_n);
      const int j = (int)(i * 4 % half_n);  // output column
      const int blk = j / 64, within = j % 64;
      const int gcol = blk * 128 + within, ucol = gcol + 64;
      float4 g = make_float4(0, 0, 0, 0), u = make_float4(0, 0, 0, 0);
      for (int s = 0; s < splits; ++s) {
        const float* base = ws + (size_t)s * M * N + (size_t)m * N;
        const float4 gg = *reinterpret_cast<const float4*>(base + gcol);
        const float4 uu = *reinterpret_cast<const float4*>(base + ucol);
        g.x += gg.x; g.y += gg.y; g.z += gg.z; g.w += gg.w;
        u.x += uu.x; u.y += uu.y; u.z += uu.z; u.w += uu.w;
      }
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out) + (size_t)m * ldo + j;
      uint2 w;
      w.x = pack_bf16(silu(g.x) * u.x, silu(g.y) * u.y);
      w.y = pack_bf16(silu(g.z) * u.z, silu(g.w) * u.w);
      *reinterpret_cast<uint2*>(o) = w;
    } else {
      const int m = (int)(i * 4 / N);
      const int n = (int)(i * 4 % N);
      float4 a = make_float4(0, 0, 0, 0);
      for (int s = 0; s < splits; ++s) {
        const float4 p = *reinterpret_cast<const float4*>(ws + (size_t)s * M * N + (size_t)m * N + n);
        a.x += p.x; a.y += p.y; a.z += p.z; a.w += p.w;
      }
      if constexpr (EPI == EPI_RESID_F32) {
        float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + (size_t)m * ldo + n);
        float4 x = *o;
        x.x += a.x; x.y += a.y; x.z += a.z; x.w += a.w;
        *o = x;
      } else if constexpr (EPI == EPI_F32) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + (size_t)m * ldo + n) = a;
      } else {
        if constexpr (EPI == EPI_BF16_BIAS) {
          a.x += __bfloat162float(bias[n]); a.y += __bfloat162float(bias[n + 1]);
          a.z += __bfloat162float(bias[n + 2]); a.w += __bfloat162float(bias[n + 3]);
        }
        uint2 w;
        w.x = pack_bf16(a.x, a.y);
        w.y = pack_bf16(a.z, a.w);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + (size_t)m * ldo + n) = w;
      }
    }
  }
}

}  // namespace tc
