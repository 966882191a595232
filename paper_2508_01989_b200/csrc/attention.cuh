// Paged attention for the hybrid step (SURVEY.md 2, K1 + K2).
//
// KV pool layout (page-major so one request's KV migrates as whole pages):
//   pool[page][layer][kv_head][k|v][slot 0..PS-1][head_dim]   (bf16, PS = 16)
// The K block and the V block of one (page, layer, kv_head) are adjacent: 32 rows x head_dim,
// 8 KiB contiguous at head_dim 128, fetched by ONE TMA instruction through a 3-D tensor map
// {64 dims, pool rows, head_dim/64 halves} (strides 256 B, 128 B) with 128 B swizzle: each
// 64-dim half lands as its own 32-line slab (K rows 0-15, V rows 16-31; the K-major SW128
// layout), so the 8 keys of an ldmatrix phase hit 8 distinct bank groups
// (address = half*4096 + row*128 + ((chunk ^ row) & 7) * 16). Completion is tracked with
// mbarrier transaction counts, so no thread computes per-chunk gather addresses.
//
//  * attn_prefill_tc2 -- chunked-prefill queries attend causally to the paged prefix + in-chunk
//    keys on tcgen05 (S and O in TMEM), two q tiles per CTA, see its section below.
//  * attn_decode   -- balanced page stream: every SM gets the same number of page-heads
//    (contiguous range over all (request, kv head) segments); a producer warp streams
//    K/V pages through a 24-stage TMA ring, 4 consumer warps split the pages and merge
//    in shared memory; only segments cut by a CTA boundary merge through global memory.
#pragma once

#include "common.cuh"

namespace tc {

struct AttnParams {
  const __nv_bfloat16* qkv;  // [T, (H + 2 Hkv) * DH], RoPE already applied to q and k
  __nv_bfloat16* out;        // [T, H * DH]
  int layer, n_layers, n_heads, n_kv_heads, page_size;
  float scale_log2;          // log2(e) / sqrt(DH)
  const int* seq_q_start;    // first packed row
  const int* seq_q_len;      // rows (1 for decode)
  const int* seq_pos0;       // position of the first row
  const int* seq_bt_off;     // offset into block_tables
  const int* block_tables;   // flat page ids
  const int* qblk_seq;       // prefill work list
  const int* qblk_off;
  // decode work (see attn_decode): segments = (decode request, kv head)
  const int4* dec_seg_a;     // [seg] (block-table offset, kv_len, q row, kv head)
  const int4* dec_seg_b;     // [seg] (parts = CTAs covering the segment, first ws slot, 0, 0)
  const int4* dec_entries;   // per-CTA entry lists: (seg, page0, page1, part)
  const int* dec_cta_off;    // [grid + 1] entry offsets
  float* ws_o;               // [slot][G][DH] partial o of segments cut by CTA boundaries
  float* ws_ml;              // [slot][G][2]
  int* dec_cnt;              // [seg] arrival counters (zero; the last arriver resets)
  unsigned long long* pf_trace;  // tools only (TC_PF_TRACE): %globaltimer stamps of one attn_prefill_tc2 CTA
};

TC_DEVICE unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

TC_DEVICE void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
TC_DEVICE void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
TC_DEVICE void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
TC_DEVICE void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
TC_DEVICE void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

constexpr int kPage = 16;  // tokens per KV page (tc_instance_desc.page_size)

template <int DH>
struct KvBlock {
  static constexpr int kBytes = kPage * DH * 2;  // one (page, k|v, head) block
  static constexpr int kPairBytes = 2 * kBytes;  // K block + V block: one TMA box
  static constexpr int kHalves = DH / 64;
};

// Swizzled smem address of (key, col) of K (v = 0) or V (v = 1) inside consecutive page pairs
// starting at base.
template <int DH>
TC_DEVICE uint32_t kv_addr(uint32_t base, int key, int col, int v) {
  const int row = (key & (kPage - 1)) + v * kPage;
  return base + (uint32_t)((key >> 4) * KvBlock<DH>::kPairBytes + (col >> 6) * (2 * kPage * 128) + row * 128 +
                           ((((col & 63) >> 3) ^ (row & 7)) << 4));
}
// TMA coordinates (dim0, dim1, dim2) of the K/V pair starting at pool row `row`
#define KV_COORD(row) 0, (row), 0

// Pool row of (page, layer, head, K, slot 0) for the 3-D tensor map.
TC_DEVICE int kv_row(const AttnParams& p, int page, int head) {
  return (((page * p.n_layers + p.layer) * p.n_kv_heads + head) * 2) * kPage;
}

// ============================================================== chunked prefill (tcgen05)
// attn_prefill_tc2: one CTA = TWO consecutive 128-row q tiles of one slice and kv head (2 * TT
// tokens; a q row = (token r / G, head r % G), so the GQA group shares every K/V byte), FA4-style
// ping-pong. Both tiles share the K/V tiles the CTA stages (half the L2->SMEM traffic per query of
// round 1's one-tile kernel), and while one softmax group works on its S tile the tensor core
// computes the other tile's PV and next S:
//   MMA warp   per key tile j:  PV0_{j-1}, S0_j, PV1_{j-1}, S1_j   (tcgen05 executes in issue order,
//              so S_t,j overwrites P_t,j-1 in TMEM only after PV_t,j-1 has read it, and "S_t,j
//              complete" implies "PV_t,j-1 complete": the lazy O rescale needs no extra wait)
//   softmax    group t = warps 4t..4t+3, ONE thread per row: pass 1 row max over the 128 scores,
//              lazy base (O / l move only when the max grows by > 2^8), pass 2 re-reads S from TMEM
//              32 keys at a time (few live registers: 106 per thread, no spills) and writes P as
//              bf16 pairs over S columns 0-63. The mask decision is warp-uniform (round 1 let the
//              3 idle rows of a G = 5 tile drag their warp through the masked path on every tile:
//              that warp ran ~2x longer and the MMA waited for it).
// TMEM: S0 @0, S1 @128, O0 @256, O1 @256 + DH. The rows of tile 1 beyond the slice are skipped when
// the slice ends inside tile 0 (`two` false).
// Measured (Qwen2.5-14B config 5, %globaltimer trace TC_PF_TRACE=1): ~2.3 us per 128-key tile for
// both q tiles (tensor pipe busy ~1.5 us of it); round 1's one-tile kernel: ~4 us per q tile.
// Tried and dropped: FA4's polynomial exp2 on the FMA pipe for 1/2 or 3/4 of the scores (slower:
// the polynomial costs ~10 issue slots against MUFU.EX2's 8-cycle pipe occupancy, tools/xu_bench.cu),
// and issuing PV per 32-key chunk as the softmax publishes it (slower: a tcgen05.wait::st per chunk).
constexpr int kPfKeys = 128;     // keys per S tile
constexpr int kPfThreads = 352;  // warps 0-7 softmax / epilogue, 8 Q + K producer, 9 V producer,
                                 // 10 MMA issuer + TMEM owner
constexpr int kPf2KStages = 2;
constexpr int kPf2VStages = 2;

template <int DH, int G>
struct Pf2Cfg {
  static constexpr int TT = 128 / G;
  static constexpr int kHalves = DH / 64;
  static constexpr int kSlab = 128 * 128;          // 128 rows x 128 B
  static constexpr int kQBytes = kHalves * kSlab;  // one q tile [128 rows][DH]
  static constexpr int kKBytes = kHalves * kSlab;  // one K or V tile [128 keys][DH]
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = 2 * kQBytes;
  static constexpr int kOffV = kOffK + kPf2KStages * kKBytes;
  static constexpr int kBytes = kOffV + kPf2VStages * kKBytes + 1024;
  static constexpr uint32_t kQTx = kHalves * TT * G * 128;  // bytes the Q boxes of one tile deliver
  static_assert(kBytes <= 227 * 1024, "prefill smem");
};

template <int DH, int G>
__global__ void __launch_bounds__(kPfThreads, 1)
    attn_prefill_tc2(const __grid_constant__ CUtensorMap kv2_map, const __grid_constant__ CUtensorMap q_map, AttnParams p) {
  using C = Pf2Cfg<DH, G>;
  constexpr int TT = C::TT;
  constexpr int KS = kPf2KStages, VS = kPf2VStages;
  extern __shared__ uint8_t attn_smem_raw[];
  __shared__ uint64_t q_full, k_full[KS], k_empty[KS], v_full[VS], v_empty[VS];
  __shared__ uint64_t s_full[2], p_full[2], o_full[2];
  __shared__ uint32_t tmem_slot;
  const uint32_t sbase = (smem_u32(attn_smem_raw) + 1023u) & ~1023u;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int seq = p.qblk_seq[blockIdx.y];
  const int qoff = p.qblk_off[blockIdx.y];
  const int kvh = blockIdx.x;
  const int q_start = p.seq_q_start[seq], q_len = p.seq_q_len[seq], pos0 = p.seq_pos0[seq];
  const int* bt = p.block_tables + p.seq_bt_off[seq];
  const bool two = qoff + TT < q_len;
  const int nq = two ? 2 : 1;
  const int kv_end = pos0 + min(qoff + nq * TT, q_len);
  const int n_tiles = (kv_end + kPfKeys - 1) / kPfKeys;
  const int n_pages = (kv_end + kPage - 1) / kPage;
  // tools only: CTA (0, 1) (a full two-tile work item; the longest-first order puts a tail first)
  unsigned long long* trc = (p.pf_trace && blockIdx.x == 0 && blockIdx.y == min(1, (int)gridDim.y - 1)) ? p.pf_trace : nullptr;
  auto stamp = [&](int j, int k) {  // trace slot [key tile j < 64][k < 16]
    if (trc && j < 64) trc[j * 16 + k] = gtimer();
  };

  if (threadIdx.x == 0) {
    mbar_init(&q_full, 1);
    for (int s = 0; s < KS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < VS; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 128);
      mbar_init(&o_full[t], 1);
    }
    mbar_fence_init();
  }
  if (warp == 10) tmem_alloc(&tmem_slot, 512);
  if constexpr (TT * G < 128) {
    // q rows TT*G..127 of both tiles are never loaded: zero them so their S rows stay finite and
    // every row of a warp can take the unmasked softmax path (no per-lane divergence)
    for (int i = threadIdx.x; i < 2 * C::kHalves * (128 - TT * G) * 8; i += blockDim.x) {
      const int chunk = i % 8, row = TT * G + (i / 8) % (128 - TT * G), slab = i / (8 * (128 - TT * G));
      *reinterpret_cast<uint4*>(attn_smem_raw + (sbase - smem_u32(attn_smem_raw)) + C::kOffQ + slab * C::kSlab + row * 128 +
                                chunk * 16) = make_uint4(0u, 0u, 0u, 0u);
    }
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();  // q / K / V written by the QKV GEMM
  pdl_trigger();

  if (warp == 8 || warp == 9) {
    // ------------------------------------------------------------ TMA producers: warp 8 Q + K, warp 9 V
    const bool is_v = warp == 9;
    if (lane == 0 && !is_v) {
      tma_prefetch_desc(&kv2_map);
      tma_prefetch_desc(&q_map);
      mbar_arrive_expect_tx(&q_full, nq * C::kQTx);
      for (int t = 0; t < nq; ++t)
#pragma unroll
        for (int h = 0; h < C::kHalves; ++h)
          tma_load_3d(sbase + C::kOffQ + t * C::kQBytes + h * C::kSlab, &q_map, &q_full, h * 64, kvh * G,
                      q_start + qoff + t * TT);
    }
    auto page_id = [&](int gp) { return bt[gp < n_pages ? gp : 0]; };  // beyond the sequence: masked
    int cur = lane < 8 ? page_id(lane) : 0;
    const int depth = is_v ? VS : KS;
    uint64_t* fullb = is_v ? v_full : k_full;
    uint64_t* emptyb = is_v ? v_empty : k_empty;
    const uint32_t ring = sbase + (is_v ? C::kOffV : C::kOffK);
    for (int j = 0; j < n_tiles; ++j) {
      const int row = kv_row(p, cur, kvh) + (is_v ? kPage : 0);  // lanes 0-7: page 8j + lane
      if (lane < 8 && j + 1 < n_tiles) cur = page_id((j + 1) * 8 + lane);
      int rows[8];
#pragma unroll
      for (int pg = 0; pg < 8; ++pg) rows[pg] = __shfl_sync(0xffffffffu, row, pg);
      if (lane == 0) {
        const int st = j % depth;
        mbar_wait(&emptyb[st], ((j / depth) & 1) ^ 1);
        mbar_arrive_expect_tx(&fullb[st], C::kKBytes);
        const uint32_t d = ring + st * C::kKBytes;
#pragma unroll
        for (int pg = 0; pg < 8; ++pg)
#pragma unroll
          for (int h = 0; h < C::kHalves; ++h)
            tma_load_2d_u32(d + h * C::kSlab + pg * 2048, &kv2_map, &fullb[st], h * 64, rows[pg]);
      }
      __syncwarp();
    }
  } else if (warp == 10) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = umma_idesc_bf16(128, kPfKeys);
    constexpr uint32_t idesc_o = umma_idesc_bf16_bmn(128, DH);
    auto issue_s = [&](int t, int j) {
      const int st = j % KS;
      if (elect_one()) {
        const uint32_t kb = sbase + C::kOffK + st * C::kKBytes;
        const uint32_t qb = sbase + C::kOffQ + t * C::kQBytes;
#pragma unroll
        for (int h = 0; h < C::kHalves; ++h)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tmem + t * 128, umma_smem_desc<128>(qb + h * C::kSlab + k * 32),
                      umma_smem_desc<128>(kb + h * C::kSlab + k * 32), idesc_s, (h | k) ? 1u : 0u);
        umma_commit(&s_full[t]);
        if (t == nq - 1) umma_commit(&k_empty[st]);
      }
      __syncwarp();
    };
    // (measured: issuing PV per 32-key chunk as the softmax publishes it was slower -- the extra
    // tcgen05.wait::st per chunk lengthens the softmax more than the early PV start saves)
    auto issue_pv = [&](int t, int i) {
      const int st = i % VS;
      mbar_wait(&p_full[t], i & 1);
      if (t == 0) mbar_wait(&v_full[st], (i / VS) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t vb = sbase + C::kOffV + st * C::kKBytes;
#pragma unroll
        for (int kk = 0; kk < kPfKeys / 16; ++kk)
          umma_bf16_tmem_a(tmem + 256 + t * DH, tmem + t * 128 + kk * 8, umma_smem_desc_mn128(vb + kk * 2048, C::kSlab, 1024),
                           idesc_o, (i | kk) ? 1u : 0u);
        umma_commit(&o_full[t]);
        if (t == nq - 1) umma_commit(&v_empty[st]);
      }
      __syncwarp();
    };
    mbar_wait(&q_full, 0);
    for (int j = 0; j < n_tiles; ++j) {
      for (int t = 0; t < nq; ++t) {
        if (j >= 1) issue_pv(t, j - 1);

        if (t == 0) {
          mbar_wait(&k_full[j % KS], (j / KS) & 1);
          tc_fence_after();

        }
        issue_s(t, j);
      }
    }
    for (int t = 0; t < nq; ++t) issue_pv(t, n_tiles - 1);
  } else if ((warp >> 2) < nq) {
    // ------------------------------------------------------------ softmax / epilogue of q tile t
    const int t = warp >> 2, quarter = warp & 3;
    const int r = quarter * 32 + lane;  // row == TMEM lane
    const int tok = qoff + t * TT + r / G, g = r % G;
    const bool valid = r < TT * G && tok < q_len;
    // causal: keys < lim. Rows outside the slice are never stored; they take every key (finite
    // scores of zero / foreign q rows) so a warp's mask decision stays uniform.
    const int lim = valid ? pos0 + tok + 1 : 0x7fffffff;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t s_addr = tmem + lane_off + t * 128;
    const uint32_t o_addr = tmem + lane_off + 256 + t * DH;
    constexpr float kRescale = 8.f;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      if (lane == 0) stamp(j, 8 + warp);  // S_t,j seen by this warp
      const int key0 = j * kPfKeys;
      const bool full = __all_sync(0xffffffffu, key0 + kPfKeys - 1 < lim);  // warp-uniform
      // pass 1: row max over the 128 scores (two 64-column loads, 8 independent max chains)
      float mx8[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) mx8[e] = -INFINITY;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t v[64];
        tmem_ld_32x32b_x32(s_addr + hh * 64, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
        tmem_ld_32x32b_x32(s_addr + hh * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
        tmem_ld_wait();
        if (full) {
#pragma unroll
          for (int x = 0; x < 64; ++x) mx8[x & 7] = fmaxf(mx8[x & 7], __uint_as_float(v[x]));
        } else {
#pragma unroll
          for (int x = 0; x < 64; ++x)
            if (key0 + hh * 64 + x < lim) mx8[x & 7] = fmaxf(mx8[x & 7], __uint_as_float(v[x]));
        }
      }
      const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                             fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * p.scale_log2;
      const bool need = mx > m_used + kRescale;  // (also the first tile with a valid key: m_used = -inf)
      if (j > 0 && __any_sync(0xffffffffu, need && m_used != -INFINITY)) {
        // O holds PV_0..PV_{j-1}, complete: S_j completed after them (in-order tensor pipe)
        const float corr = (need && m_used != -INFINITY) ? fast_exp2(m_used - mx) : 1.f;
#pragma unroll
        for (int c = 0; c < DH / 32; ++c) {
          uint32_t ov[32];
          tmem_ld_32x32b_x32(o_addr + c * 32, ov);
          tmem_ld_wait();
#pragma unroll
          for (int x = 0; x < 32; ++x) ov[x] = __float_as_uint(__uint_as_float(ov[x]) * corr);
          tmem_st_32x32b_x16(o_addr + c * 32, *reinterpret_cast<const uint32_t(*)[16]>(&ov[0]));
          tmem_st_32x32b_x16(o_addr + c * 32 + 16, *reinterpret_cast<const uint32_t(*)[16]>(&ov[16]));
        }
        l *= corr;
      }
      if (need) m_used = mx;
      const float base = m_used == -INFINITY ? 0.f : m_used;
      float sum4[4] = {0.f, 0.f, 0.f, 0.f};
      // pass 2, 32 keys at a time (TMEM reloads are cheap; few live registers leave the scheduler
      // room to overlap the MUFU latency): P as bf16 pairs over S columns 16c .. 16c + 15, i.e.
      // over scores this thread has already consumed
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(s_addr + c * 32, v);
        tmem_ld_wait();
        uint32_t pk[16];
        if (full) {
#pragma unroll
          for (int x = 0; x < 16; ++x) {
            const float a0 = fmaf(__uint_as_float(v[2 * x]), p.scale_log2, -base);
            const float a1 = fmaf(__uint_as_float(v[2 * x + 1]), p.scale_log2, -base);
            const float p0 = fast_exp2(a0), p1 = fast_exp2(a1);
            sum4[x & 3] += p0 + p1;
            pk[x] = pack_bf16(p0, p1);
          }
        } else {
          const int k0 = key0 + c * 32;
#pragma unroll
          for (int x = 0; x < 16; ++x) {
            const float p0 = k0 + 2 * x < lim ? fast_exp2(fmaf(__uint_as_float(v[2 * x]), p.scale_log2, -base)) : 0.f;
            const float p1 =
                k0 + 2 * x + 1 < lim ? fast_exp2(fmaf(__uint_as_float(v[2 * x + 1]), p.scale_log2, -base)) : 0.f;
            sum4[x & 3] += p0 + p1;
            pk[x] = pack_bf16(p0, p1);
          }
        }
        tmem_st_32x32b_x16(s_addr + c * 16, pk);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[t]);
      if (lane == 0) stamp(j, warp);  // P_t,j written by this warp
      l += (sum4[0] + sum4[1]) + (sum4[2] + sum4[3]);
    }
    // O final once the last PV completes (S_{n-1} complete => PV_{n-2} complete)
    mbar_wait(&o_full[t], (n_tiles - 1) & 1);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* dst = p.out + (long long)(q_start + tok) * p.n_heads * DH + (kvh * G + g) * DH;
#pragma unroll
    for (int c = 0; c < DH / 32; ++c) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(o_addr + c * 32, o);
      tmem_ld_wait();
      if (valid) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(o[q * 8 + 0]) * inv, __uint_as_float(o[q * 8 + 1]) * inv);
          w.y = pack_bf16(__uint_as_float(o[q * 8 + 2]) * inv, __uint_as_float(o[q * 8 + 3]) * inv);
          w.z = pack_bf16(__uint_as_float(o[q * 8 + 4]) * inv, __uint_as_float(o[q * 8 + 5]) * inv);
          w.w = pack_bf16(__uint_as_float(o[q * 8 + 6]) * inv, __uint_as_float(o[q * 8 + 7]) * inv);
          st_global_v4(dst + c * 32 + q * 8, w);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 10) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ============================================================== decode
// Work decomposition (host, step_launch): a SEGMENT is (decode request, kv head) and covers
// that request's KV pages 0..ceil(kv_len/16)-1. All segments' pages, laid end to end, form one
// page stream of W page-heads; CTA c (one per SM, persistent) takes the contiguous range
// [W*c/NC, W*(c+1)/NC), so every SM streams the same number of bytes whatever the context
// mix. A CTA's range is a list of ENTRIES (segment, page0, page1, part).
//
// Warp roles inside a CTA:
//   consumers (NC warps)  warp w takes ring stages w, w+NC, ... of the page stream and keeps its
//                         own online-softmax state per entry; at the end of an entry it publishes
//                         the state into the entry's partial buffer (double-buffered, mbarriers)
//                         and goes straight on to the next entry's pages.
//   producer              streams each page's K and V blocks (one TMA box, 8 KiB at head_dim
//                         128) into the ring and the segment's q rows (one bulk copy per entry)
//                         into a double-buffered q slot; it waits only on a full ring.
//   merger                combines the NC partial states of each entry and writes the output
//                         row; only segments cut by a CTA boundary (at most 2 per CTA) go through
//                         global memory (the CTA that arrives last on the segment's counter
//                         combines the parts).
// Round 1 merged in a consumer warp behind a consumer-wide barrier: the ring stages owned by the
// merging warp stalled the in-order producer at every entry boundary.
// A page costs a consumer ~110 instructions: 16 + 16 mma.sync, 16 ldmatrix, the key mask only on
// a segment's last page, and a lazy softmax base (the base -- and with it l and o -- moves only
// when a row's max grows by more than 2^8, which after the first page is rare).
constexpr int kDecRingBytes = 192 * 1024;  // default ring (RING template parameter: A/B)
constexpr float kDecRescaleLog2 = 8.f;  // lazy base: p = 2^(s - base) <= 2^8, P stays in bf16 range
__host__ __device__ constexpr int dec_threads(int nc, int np) { return (nc + np + 1) * 32; }

template <int DH, int G, int NC, int RING = kDecRingBytes>
struct DecodeSmem {
  static constexpr int kStageBytes = KvBlock<DH>::kPairBytes;  // one page-head: K block then V block
  static constexpr int kStages = RING / kStageBytes;
  static constexpr int kQBytes = G * DH * 2;
  static constexpr int kPartFloats = NC * G * DH;  // per buffer
  static constexpr int kOffQ = RING;
  static constexpr int kOffPart = kOffQ + 2 * ((kQBytes + 127) / 128 * 128);
  static constexpr int kOffMl = kOffPart + 2 * kPartFloats * 4;
  static constexpr int kBytes = kOffMl + 2 * NC * G * 2 * 4 + 1024;
  // Stage g is consumed by warp g % NC. With S a multiple of NC every slot has ONE owner warp,
  // which waits for use k+1 only after finishing use k; otherwise a warp running a lap ahead
  // could pass a parity wait on a phase that has not landed yet (mbarrier parity ABA).
  static_assert(kStages % NC == 0, "decode ring: stages must be a multiple of the consumer warps");
  static_assert(kBytes <= 227 * 1024, "decode smem");
};

TC_DEVICE void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Merge n partial states (m, l in the log2 domain; o unnormalised) for G rows; lane handles
// dims lane*V .. lane*V+V-1. load_ml(j, r) -> float2(m, l); load_o(j, r, dst[V]).
template <int DH, int G, typename LoadMl, typename LoadO>
TC_DEVICE void merge_partials(int n, LoadMl&& load_ml, LoadO&& load_o, float (&acc)[G][DH / 32], float (&mm)[G],
                              float (&ll)[G]) {
  constexpr int V = DH / 32;
#pragma unroll
  for (int r = 0; r < G; ++r) {
    float mx = -INFINITY;
    for (int j = 0; j < n; ++j) mx = fmaxf(mx, load_ml(j, r).x);
    mm[r] = mx;
    ll[r] = 0.f;
#pragma unroll
    for (int e = 0; e < V; ++e) acc[r][e] = 0.f;
  }
  for (int j = 0; j < n; ++j) {
#pragma unroll
    for (int r = 0; r < G; ++r) {
      const float2 ml = load_ml(j, r);
      const float w = ml.x == -INFINITY ? 0.f : exp2f(ml.x - mm[r]);
      ll[r] += w * ml.y;
      float o[V];
      load_o(j, r, o);
#pragma unroll
      for (int e = 0; e < V; ++e) acc[r][e] += w * o[e];
    }
  }
}

template <int DH, int G>
TC_DEVICE void store_out_row(__nv_bfloat16* out_row, const float (&acc)[G][DH / 32], const float (&ll)[G]) {
  constexpr int V = DH / 32;
  const int lane = threadIdx.x % 32;
#pragma unroll
  for (int r = 0; r < G; ++r) {
    const float inv = ll[r] > 0.f ? 1.f / ll[r] : 0.f;
    __nv_bfloat16* dst = out_row + r * DH + lane * V;
    if constexpr (V == 4) {
      uint2 w;
      w.x = pack_bf16(acc[r][0] * inv, acc[r][1] * inv);
      w.y = pack_bf16(acc[r][2] * inv, acc[r][3] * inv);
      *reinterpret_cast<uint2*>(dst) = w;
    } else {
      *reinterpret_cast<uint32_t*>(dst) = pack_bf16(acc[r][0] * inv, acc[r][1] * inv);
    }
  }
}

TC_DEVICE uint32_t movmatrix_trans(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}

// One page of one consumer warp, in the TRANSPOSED formulation: the page's 16 keys are the MMA's M
// and the GQA group's heads its N (m16n8k16; G <= 8 heads, the rest zero), so a page costs
// 8 + 8 mma.sync instead of the 16 + 16 of a 16-row q fragment with G of 16 rows live.
//   S^T[16 keys x 8 heads] = K[16 x DH] . Q^T      (A = K via ldmatrix, B = q from registers)
//   online softmax per head column (lanes with equal lane % 4 share a head pair), lazy base
//   O^T[DH x 8 heads] += V^T[DH x 16 keys] . P^T   (A = V^T via ldmatrix.trans, B = P^T: the
//                                                  S^T fragment transposed in registers by movmatrix)
// Lane l holds keys l/4 and l/4 + 8 of heads 2(l%4) and 2(l%4) + 1: m[h], l[h], o[mt][h | 2 + h].
template <int DH>
TC_DEVICE void dec_page_t(const uint32_t (&qb)[DH / 16][2], uint32_t kv_smem, int key0, int kv_len, float scale_log2,
                          float (&m)[2], float (&l)[2], float (&o)[DH / 16][4]) {
  const int lane = threadIdx.x % 32;
  const int g = lane / 4;
  float s[4] = {0.f, 0.f, 0.f, 0.f};
  {
    // A fragment rows (keys) / column blocks of ldmatrix.x4: lane i -> key (i % 8) + 8 ((i / 8) % 2),
    // dims 8 (i / 16) of the k-step
    const int key = (lane % 8) + ((lane / 8) % 2) * 8, cb = (lane / 16) * 8;
#pragma unroll
    for (int ks = 0; ks < DH / 16; ++ks) {
      uint32_t a[4];
      ldsm_x4(kv_addr<DH>(kv_smem, key, ks * 16 + cb, 0), a[0], a[1], a[2], a[3]);
      mma_bf16_16816(s, a, qb[ks][0], qb[ks][1]);
    }
  }
  if (key0 + kPage > kv_len) {  // the segment's last page (warp-uniform)
    if (key0 + g >= kv_len) s[0] = s[1] = -INFINITY;
    if (key0 + g + 8 >= kv_len) s[2] = s[3] = -INFINITY;
  }
  float mx[2] = {fmaxf(s[0], s[2]), fmaxf(s[1], s[3])};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], off));
    mx[h] *= scale_log2;  // scale > 0: the max commutes with it
  }
  // every page holds at least one valid key, so mx is finite; m == -inf only before the first page
  const bool grow = mx[0] > m[0] + kDecRescaleLog2 || mx[1] > m[1] + kDecRescaleLog2;
  if (__any_sync(0xffffffffu, grow)) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float nb = fmaxf(m[h], mx[h]);
      const float corr = exp2f(m[h] - nb);  // m == -inf -> 0
      m[h] = nb;
      l[h] *= corr;
#pragma unroll
      for (int mt = 0; mt < DH / 16; ++mt) {
        o[mt][h] *= corr;
        o[mt][2 + h] *= corr;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    s[i] = exp2f(fmaf(s[i], scale_log2, -m[i & 1]));
    l[i & 1] += s[i];
  }
  // P^T as the B operand: rows (keys 0-7 | 8-15) x heads, transposed by movmatrix
  const uint32_t b0 = movmatrix_trans(pack_bf16(s[0], s[1])), b1 = movmatrix_trans(pack_bf16(s[2], s[3]));
  // V^T A fragments by ldmatrix.trans: lane i -> key 8 (i / 16) + i % 8, dims 16 mt + 8 ((i / 8) % 2)
  const int vkey = (lane / 16) * 8 + (lane % 8), vcb = ((lane / 8) % 2) * 8;
#pragma unroll
  for (int mt = 0; mt < DH / 16; ++mt) {
    uint32_t a[4];
    ldsm_x4_t(kv_addr<DH>(kv_smem, vkey, mt * 16 + vcb, 1), a[0], a[1], a[2], a[3]);
    mma_bf16_16816(o[mt], a, b0, b1);
  }
}

template <int DH, int G, int NC, int NP, int RING = kDecRingBytes>
__global__ void __launch_bounds__(dec_threads(NC, NP), 1) attn_decode(const __grid_constant__ CUtensorMap kv_map, AttnParams p) {
  using SM = DecodeSmem<DH, G, NC, RING>;
  constexpr int S = SM::kStages;
  static_assert(S % NP == 0, "decode ring: every stage must belong to one producer warp");
  constexpr int V = DH / 32;
  extern __shared__ uint8_t attn_smem_raw[];
  __shared__ uint64_t full[S], empty[S], qfull[2], qempty[2], pfull[2], pempty[2];
  const uint32_t sbase = (smem_u32(attn_smem_raw) + 1023u) & ~1023u;
  uint8_t* gbase = attn_smem_raw + (sbase - smem_u32(attn_smem_raw));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int e_begin = p.dec_cta_off[blockIdx.x], e_end = p.dec_cta_off[blockIdx.x + 1];
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&qfull[b], 1);
      // every lane arrives on the hand-off barriers, so each lane's own shared-memory accesses are
      // ordered by its own arrival (compute-sanitizer racecheck clean)
      mbar_init(&qempty[b], NC * 32);
      mbar_init(&pfull[b], NC * 32);
      mbar_init(&pempty[b], 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  pdl_wait();  // q / K / V written by the QKV GEMM (dec_cta_off above came from a memcpy)
  pdl_trigger();
  const int qkv_ld = (p.n_heads + 2 * p.n_kv_heads) * DH;
  float* part_o = reinterpret_cast<float*>(gbase + SM::kOffPart);
  float* part_ml = reinterpret_cast<float*>(gbase + SM::kOffMl);

  if (warp >= NC && warp < NC + NP) {
    // ------------------------------------------------------------ producers
    // NP warps issue the page stream together: warp NC + j issues stages g with g % NP == j. One
    // issuing thread sustains only ~14 GB/s of random 8 KiB bulk copies (tools/stream_bench.cu:
    // 2.1 / 4.1 / 6.9 TB/s chip-wide with 1 / 2 / 4 issuing warps per SM), so the round-1 single
    // producer, not the ring depth, capped the stream at ~5.2 TB/s.
    const int pj = warp - NC;
    if (lane == 0 && pj == 0) tma_prefetch_desc(&kv_map);
    int g = 0;  // stages of the stream so far
    for (int e0 = e_begin; e0 < e_end; e0 += 32) {
      // lane j holds entry e0 + j and its segment descriptor
      int4 ent = make_int4(0, 0, 0, 0), sa = make_int4(0, 0, 0, 0);
      if (e0 + lane < e_end) {
        ent = p.dec_entries[e0 + lane];
        sa = p.dec_seg_a[ent.x];
      }
      const int ne = min(32, e_end - e0);
      // lane j: block-table entry of page c + j of the chunk being issued. Loaded one chunk ahead --
      // the next chunk of this entry, or the first chunk of the next entry -- so the global-load
      // latency stays off the issue path (round 1 stalled the stream on it at every entry)
      auto first_chunk = [&](int k) {
        const int pg0 = __shfl_sync(0xffffffffu, ent.y, k), pg1 = __shfl_sync(0xffffffffu, ent.z, k);
        const int bt_off = __shfl_sync(0xffffffffu, sa.x, k);
        return pg0 + lane < pg1 ? __ldg(p.block_tables + bt_off + pg0 + lane) : 0;
      };
      int bt_first = first_chunk(0);
      for (int k = 0; k < ne; ++k) {
        const int e = e0 + k - e_begin;  // local entry index
        const int pg0 = __shfl_sync(0xffffffffu, ent.y, k), pg1 = __shfl_sync(0xffffffffu, ent.z, k);
        const int bt_off = __shfl_sync(0xffffffffu, sa.x, k), q_row = __shfl_sync(0xffffffffu, sa.z, k);
        const int kvh = __shfl_sync(0xffffffffu, sa.w, k);
        int bt_next = bt_first;
        if (k + 1 < ne) bt_first = first_chunk(k + 1);
        if (lane == 0 && pj == 0) {
          const int b = e & 1;
          mbar_wait(&qempty[b], ((e >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&qfull[b], SM::kQBytes);
          bulk_load(sbase + SM::kOffQ + b * ((SM::kQBytes + 127) / 128 * 128),
                    p.qkv + (long long)q_row * qkv_ld + kvh * G * DH, SM::kQBytes, &qfull[b]);
        }
        for (int c = pg0; c < pg1; c += 32) {
          const int row = c + lane < pg1 ? kv_row(p, bt_next, kvh) : 0;
          if (c + 32 + lane < pg1) bt_next = __ldg(p.block_tables + bt_off + c + 32 + lane);
          const int n = min(32, pg1 - c);
          for (int j = 0; j < n; ++j, ++g) {
            const int rj = __shfl_sync(0xffffffffu, row, j);
            if (lane == 0 && g % NP == pj) {
              const int st = g % S;
              mbar_wait(&empty[st], ((g / S) & 1) ^ 1);
              mbar_arrive_expect_tx(&full[st], SM::kStageBytes);
              tma_load_3d(sbase + st * SM::kStageBytes, &kv_map, &full[st], KV_COORD(rj));
            }
          }
        }
      }
    }
    return;
  }

  if (warp == NC + NP) {
    // ------------------------------------------------------------ merger
    for (int e0 = e_begin; e0 < e_end; e0 += 32) {
      int4 ent = make_int4(0, 0, 0, 0), sa = make_int4(0, 0, 0, 0), sb = make_int4(0, 0, 0, 0);
      if (e0 + lane < e_end) {
        ent = p.dec_entries[e0 + lane];
        sa = p.dec_seg_a[ent.x];
        sb = p.dec_seg_b[ent.x];
      }
      const int ne = min(32, e_end - e0);
      for (int k = 0; k < ne; ++k) {
        const int e = e0 + k - e_begin;
        const int seg = __shfl_sync(0xffffffffu, ent.x, k), part = __shfl_sync(0xffffffffu, ent.w, k);
        const int q_row = __shfl_sync(0xffffffffu, sa.z, k), kvh = __shfl_sync(0xffffffffu, sa.w, k);
        const int n_parts = __shfl_sync(0xffffffffu, sb.x, k), ws_base = __shfl_sync(0xffffffffu, sb.y, k);
        const int b = e & 1;
        mbar_wait(&pfull[b], (e >> 1) & 1);
        const float* bo = part_o + (b * NC * G) * DH;
        const float* bml = part_ml + (b * NC * G) * 2;
        float acc[G][V], mm[G], ll[G];
        merge_partials<DH, G>(
            NC, [&](int j, int r) { return *reinterpret_cast<const float2*>(bml + (j * G + r) * 2); },
            [&](int j, int r, float* d) {
              const float* src = bo + (j * G + r) * DH + lane * V;
#pragma unroll
              for (int x = 0; x < V; ++x) d[x] = src[x];
            },
            acc, mm, ll);
        __syncwarp();
        mbar_arrive(&pempty[b]);  // buffer b free for entry e + 2
        __nv_bfloat16* out_row = p.out + (long long)q_row * p.n_heads * DH + (long long)kvh * G * DH;
        if (n_parts == 1) {
          store_out_row<DH, G>(out_row, acc, ll);
          continue;
        }
        // segment cut by a CTA boundary: publish the CTA's part; the last arriver combines
        const int slot = ws_base + part;
#pragma unroll
        for (int r = 0; r < G; ++r) {
          float* dst = p.ws_o + ((long long)slot * G + r) * DH + lane * V;
#pragma unroll
          for (int x = 0; x < V; ++x) dst[x] = acc[r][x];
          if (lane == 0) *reinterpret_cast<float2*>(p.ws_ml + ((long long)slot * G + r) * 2) = make_float2(mm[r], ll[r]);
        }
        __syncwarp();
        int last = 0;
        if (lane == 0) {
          __threadfence();
          int* cnt = p.dec_cnt + seg;
          last = atomicAdd(cnt, 1) == n_parts - 1;
          if (last) *cnt = 0;  // ready for the next layer / step
        }
        if (!__shfl_sync(0xffffffffu, last, 0)) continue;
        __threadfence();
        merge_partials<DH, G>(
            n_parts,
            [&](int j, int r) { return __ldcg(reinterpret_cast<const float2*>(p.ws_ml + ((long long)(ws_base + j) * G + r) * 2)); },
            [&](int j, int r, float* d) {
              const float* src = p.ws_o + ((long long)(ws_base + j) * G + r) * DH + lane * V;
              if constexpr (V == 4) {
                const float4 t = __ldcg(reinterpret_cast<const float4*>(src));
                d[0] = t.x; d[1] = t.y; d[2] = t.z; d[3] = t.w;
              } else {
                const float2 t = __ldcg(reinterpret_cast<const float2*>(src));
                d[0] = t.x; d[1] = t.y;
              }
            },
            acc, mm, ll);
        store_out_row<DH, G>(out_row, acc, ll);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int g = lane / 4, c = lane % 4;  // key row / head pair of the transposed fragments
  int g_base = 0;  // stages before the current entry
  for (int e0 = e_begin; e0 < e_end; e0 += 32) {
    int4 ent = make_int4(0, 0, 0, 0), sa = make_int4(0, 0, 0, 0);
    if (e0 + lane < e_end) {
      ent = p.dec_entries[e0 + lane];
      sa = p.dec_seg_a[ent.x];
    }
    const int ne = min(32, e_end - e0);
    for (int k = 0; k < ne; ++k) {
      const int e = e0 + k - e_begin;
      const int pg0 = __shfl_sync(0xffffffffu, ent.y, k), pg1 = __shfl_sync(0xffffffffu, ent.z, k);
      const int kv_len = __shfl_sync(0xffffffffu, sa.y, k);
      const int b = e & 1;
      // Q^T B fragments (heads >= G are zero): lane holds q[head g][16 ks + 2c .. +1] and [.. + 8 ..]
      uint32_t qb[DH / 16][2];
      mbar_wait(&qfull[b], (e >> 1) & 1);
      {
        const __nv_bfloat16* qs = reinterpret_cast<const __nv_bfloat16*>(gbase + SM::kOffQ +
                                                                         b * ((SM::kQBytes + 127) / 128 * 128)) +
                                  (g < G ? g : 0) * DH + c * 2;
#pragma unroll
        for (int ks = 0; ks < DH / 16; ++ks) {
          qb[ks][0] = g < G ? *reinterpret_cast<const uint32_t*>(qs + ks * 16) : 0u;
          qb[ks][1] = g < G ? *reinterpret_cast<const uint32_t*>(qs + ks * 16 + 8) : 0u;
        }
      }
      __syncwarp();
      mbar_arrive(&qempty[b]);
      float o[DH / 16][4];
#pragma unroll
      for (int mt = 0; mt < DH / 16; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
      float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
      const int n = pg1 - pg0;
      // this warp's stages of the entry: g_base + i with (g_base + i) % NC == warp
      for (int i = (warp - g_base % NC + NC) % NC; i < n; i += NC) {
        const int gi = g_base + i;
        const int st = gi % S;
        mbar_wait(&full[st], (gi / S) & 1);
        dec_page_t<DH>(qb, sbase + st * SM::kStageBytes, (pg0 + i) * kPage, kv_len, p.scale_log2, m, l, o);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
      g_base += n;
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) l[h] += __shfl_xor_sync(0xffffffffu, l[h], off);
      // publish this warp's partial state (a warp without pages publishes m = -inf, l = 0, o = 0)
      mbar_wait(&pempty[b], ((e >> 1) & 1) ^ 1);  // the merger is done with entry e - 2
      float* po = part_o + ((b * NC + warp) * G) * DH;
      float* pml = part_ml + ((b * NC + warp) * G) * 2;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int hd = 2 * c + h;
        if (hd < G) {
#pragma unroll
          for (int mt = 0; mt < DH / 16; ++mt) {
            po[hd * DH + mt * 16 + g] = o[mt][h];
            po[hd * DH + mt * 16 + g + 8] = o[mt][2 + h];
          }
          if (g == 0) *reinterpret_cast<float2*>(pml + hd * 2) = make_float2(m[h], l[h]);
        }
      }
      __syncwarp();
      mbar_arrive(&pfull[b]);  // release: the partial's stores precede the arrival
    }
  }
}

// Compiled decode variants: (consumer warps, producer warps) at the 192 KiB ring; the first is the
// default (TC_DEC_CFG selects another for A/B).
template <int DH, int G, typename F>
void for_each_decode_variant_of(F&& f) {
  // the default (4 consumer, 4 producer warps) and one A/B alternative; 4:2 / 4:1 / 6:2 were
  // measured (fewer issuing warps cap the page stream, tools/stream_bench.cu) and dropped
  f(attn_decode<DH, G, 4, 4>, DecodeSmem<DH, G, 4>::kBytes, 4, 4);
  f(attn_decode<DH, G, 6, 4>, DecodeSmem<DH, G, 6>::kBytes, 6, 4);
}
template <typename F>
void for_each_decode_variant(F&& f) {
  auto g = [&](auto kern, int smem, int, int) { f(kern, smem); };
  for_each_decode_variant_of<64, 2>(g);
  for_each_decode_variant_of<128, 4>(g);
  for_each_decode_variant_of<128, 5>(g);
}

}  // namespace tc
