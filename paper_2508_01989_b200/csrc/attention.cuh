// Paged attention for the hybrid step (SURVEY.md 2, K1 + K2).
//
// KV pool layout (page-major so one request's KV migrates as whole pages):
//   pool[page][layer][k|v][kv_head][slot 0..PS-1][head_dim]   (bf16, PS = 16)
// One (page, layer, k|v, kv_head) block is 16 rows x head_dim, 4 KiB contiguous for
// head_dim 128. It is fetched by ONE TMA instruction through a 3-D tensor map
// {64 dims, pool rows, head_dim/64 halves} (strides 256 B, 128 B) with 128 B swizzle:
// each 64-dim half lands as its own 16-line slab (the K-major SW128 layout), so the
// 8 keys of an ldmatrix phase hit 8 distinct bank groups
// (address = half*2048 + key*128 + ((chunk ^ key) & 7) * 16). Completion is tracked with mbarrier transaction
// counts, so no thread computes per-chunk gather addresses.
//
//  * attn_prefill  -- chunked-prefill queries (a chunk may span prompts; each slice
//    is a sequence) attend causally to the paged prefix + in-chunk keys. CTA =
//    (16/G tokens x G heads) x 4 consumer warps of one GQA group + 1 TMA producer
//    warp; 64-key tiles (4 pages) in a 3-stage full/empty mbarrier ring. QK^T and
//    PV on tensor cores (mma.sync m16n8k16 bf16, fp32 accumulate), online softmax.
//  * attn_decode   -- split-KV at warp granularity: a work item is (request,
//    kv_head, run of pages); a persistent grid of independent warps walks its
//    items with a private 4-stage page ring (each warp issues its own TMA loads
//    S-1 pages ahead, across item boundaries). For requests split into several items
//    the warp that finishes an item LAST (atomic counter per request and kv head)
//    merges the partials -- no separate combine launch, no waiting.
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
  const int4* dec_items;     // decode work: (block-table offset, kvh | decode index << 8, page0, page1)
  int n_items;
  const int* dec_seq;        // decode index -> sequence
  const int* dec_item_base;  // decode index -> first item; items (d, kvh, j) at base + kvh * chunks + j
  const int* dec_chunks;     // decode index -> items per kv head
  float* ws_o;               // [item][G][DH]
  float* ws_ml;              // [item][G][2]
  int* dec_cnt;              // [decode][kv head] arrival counters (zero; the last arriver resets)
};

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
  static constexpr int kHalves = DH / 64;
};

#ifndef TC_KV_SLAB
#define TC_KV_SLAB 1  // 1: {64, rows, halves} box (one slab per half); 0: {64, halves, rows} (interleaved)
#endif
// Swizzled smem address of (key, col) inside consecutive page blocks starting at base.
template <int DH>
TC_DEVICE uint32_t kv_addr(uint32_t base, int key, int col) {
  const int row = key & (kPage - 1);
#if TC_KV_SLAB
  return base + (uint32_t)((key >> 4) * KvBlock<DH>::kBytes + (col >> 6) * (kPage * 128) + row * 128 +
                           ((((col & 63) >> 3) ^ (row & 7)) << 4));
#else
  const int line = row * KvBlock<DH>::kHalves + (col >> 6);
  return base + (uint32_t)((key >> 4) * KvBlock<DH>::kBytes + line * 128 + ((((col & 63) >> 3) ^ (line & 7)) << 4));
#endif
}
// TMA coordinates of a block: (dim0, dim1, dim2)
#if TC_KV_SLAB
#define KV_COORD(row) 0, (row), 0
#else
#define KV_COORD(row) 0, 0, (row)
#endif

// Pool row of (page, layer, k|v, head, slot 0) for the 3-D tensor map.
TC_DEVICE int kv_row(const AttnParams& p, int page, int kv, int head) {
  return (((page * p.n_layers + p.layer) * 2 + kv) * p.n_kv_heads + head) * kPage;
}

// Q fragment (A operand) of 16 rows: rows lo / hi -> (token, head).
template <int DH>
TC_DEVICE void attn_load_q(const AttnParams& p, int tok_lo, int head_lo, bool ok_lo, int tok_hi, int head_hi,
                           bool ok_hi, uint32_t (&qf)[DH / 16][4]) {
  const int qkv_ld = (p.n_heads + 2 * p.n_kv_heads) * DH;
  const int lane = threadIdx.x % 32;
  const __nv_bfloat16* qlo = p.qkv + (long long)tok_lo * qkv_ld + head_lo * DH + (lane % 4) * 2;
  const __nv_bfloat16* qhi = p.qkv + (long long)tok_hi * qkv_ld + head_hi * DH + (lane % 4) * 2;
#pragma unroll
  for (int ks = 0; ks < DH / 16; ++ks) {
    qf[ks][0] = ok_lo ? *reinterpret_cast<const uint32_t*>(qlo + ks * 16) : 0u;
    qf[ks][1] = ok_hi ? *reinterpret_cast<const uint32_t*>(qhi + ks * 16) : 0u;
    qf[ks][2] = ok_lo ? *reinterpret_cast<const uint32_t*>(qlo + ks * 16 + 8) : 0u;
    qf[ks][3] = ok_hi ? *reinterpret_cast<const uint32_t*>(qhi + ks * 16 + 8) : 0u;
  }
}

// S[16 x 8*NT] = Q K^T for keys [kbase, kbase + 8*NT) of the staged K blocks.
template <int DH, int NT>
TC_DEVICE void attn_qk(const uint32_t (&qf)[DH / 16][4], uint32_t k_smem, int kbase, float (&s)[NT][4]) {
  const int lane = threadIdx.x % 32;
  const int j = lane / 8, r = lane % 8;
#pragma unroll
  for (int t = 0; t < NT; ++t) s[t][0] = s[t][1] = s[t][2] = s[t][3] = 0.f;
#pragma unroll
  for (int ks = 0; ks < DH / 16; ++ks) {
#pragma unroll
    for (int t = 0; t < NT; t += 2) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4(kv_addr<DH>(k_smem, kbase + t * 8 + (j / 2) * 8 + r, ks * 16 + (j % 2) * 8), b0, b1, b2, b3);
      mma_bf16_16816(s[t], qf[ks], b0, b1);
      mma_bf16_16816(s[t + 1], qf[ks], b2, b3);
    }
  }
}

// O[16 x DH] += P[16 x 8*NT] V[keys kbase.., DH]
template <int DH, int NT>
TC_DEVICE void attn_pv(const float (&pr)[NT][4], uint32_t v_smem, int kbase, float (&o)[DH / 8][4]) {
  const int lane = threadIdx.x % 32;
  const int j = lane / 8, r = lane % 8;
#pragma unroll
  for (int kk = 0; kk < NT / 2; ++kk) {
    uint32_t a[4];
    a[0] = pack_bf16(pr[2 * kk][0], pr[2 * kk][1]);
    a[1] = pack_bf16(pr[2 * kk][2], pr[2 * kk][3]);
    a[2] = pack_bf16(pr[2 * kk + 1][0], pr[2 * kk + 1][1]);
    a[3] = pack_bf16(pr[2 * kk + 1][2], pr[2 * kk + 1][3]);
#pragma unroll
    for (int n = 0; n < DH / 8; n += 2) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(kv_addr<DH>(v_smem, kbase + kk * 16 + (j % 2) * 8 + r, n * 8 + (j / 2) * 8), b0, b1, b2, b3);
      mma_bf16_16816(o[n], a, b0, b1);
      mma_bf16_16816(o[n + 1], a, b2, b3);
    }
  }
}

// Online-softmax update for one tile. Rows lane/4 (c0,c1) and lane/4+8 (c2,c3).
// key_lim_lo/hi: exclusive key bound (absolute) for the two rows.
template <int DH, int NT>
TC_DEVICE void attn_softmax_step(float (&s)[NT][4], int key0, int key_lim_lo, int key_lim_hi, float scale_log2,
                                 float (&m)[2], float (&l)[2], float (&o)[DH / 8][4]) {
  const int lane = threadIdx.x % 32;
  float mx[2] = {m[0], m[1]};
#pragma unroll
  for (int t = 0; t < NT; ++t) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int key = key0 + t * 8 + (lane % 4) * 2 + (e & 1);
      const int lim = (e < 2) ? key_lim_lo : key_lim_hi;
      float v = s[t][e] * scale_log2;
      v = key < lim ? v : -INFINITY;
      s[t][e] = v;
      mx[e >> 1] = fmaxf(mx[e >> 1], v);
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 1));
    mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 2));
  }
  float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float base = mx[h] == -INFINITY ? 0.f : mx[h];
    corr[h] = exp2f(m[h] - base);  // m == -inf -> 0
    m[h] = mx[h];
    mx[h] = base;
  }
#pragma unroll
  for (int t = 0; t < NT; ++t) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float pe = exp2f(s[t][e] - mx[e >> 1]);
      s[t][e] = pe;
      rs[e >> 1] += pe;
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) l[h] = l[h] * corr[h] + rs[h];
#pragma unroll
  for (int n = 0; n < DH / 8; ++n) {
    o[n][0] *= corr[0];
    o[n][1] *= corr[0];
    o[n][2] *= corr[1];
    o[n][3] *= corr[1];
  }
}

// ============================================================== chunked prefill
constexpr int kPrefillStages = 3;
constexpr int kPrefillThreads = 160;  // 4 consumer warps + 1 TMA producer warp
constexpr int kTilePages = 4;         // 64 keys per tile

template <int DH>
struct PrefillSmem {
  static constexpr int kStageBytes = 2 * kTilePages * KvBlock<DH>::kBytes;  // K pages then V pages
  static constexpr int kBytes = kPrefillStages * kStageBytes + 1024;
};

template <int DH, int G>
__global__ void __launch_bounds__(kPrefillThreads, 2) attn_prefill(const __grid_constant__ CUtensorMap kv_map, AttnParams p) {
  constexpr int TPW = 16 / G;  // tokens per warp
  constexpr int TPC = 4 * TPW;
  constexpr int kKeys = kTilePages * kPage;
  extern __shared__ uint8_t attn_smem_raw[];
  __shared__ uint64_t full_bar[kPrefillStages], empty_bar[kPrefillStages];
  const uint32_t sbase = (smem_u32(attn_smem_raw) + 1023u) & ~1023u;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int seq = p.qblk_seq[blockIdx.x];
  const int qoff = p.qblk_off[blockIdx.x];
  const int kvh = blockIdx.y;
  const int q_start = p.seq_q_start[seq], q_len = p.seq_q_len[seq], pos0 = p.seq_pos0[seq];
  const int* bt = p.block_tables + p.seq_bt_off[seq];
  const int kv_end = pos0 + min(qoff + TPC, q_len);
  const int n_tiles = (kv_end + kKeys - 1) / kKeys;
  const int n_pages = (kv_end + kPage - 1) / kPage;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kPrefillStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 4);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == 4) {
    // ---------------- TMA producer: 4 K blocks + 4 V blocks per tile. Lanes 0-3 fetch the
    // next tile's page ids while lane 0 issues the current tile, so block-table latency never
    // sits between two TMA issues.
    auto page_id = [&](int gp) { return bt[gp < n_pages ? gp : 0]; };  // beyond the sequence: any page, masked
    int cur = lane < kTilePages ? page_id(lane) : 0;
    if (lane == 0) tma_prefetch_desc(&kv_map);
    for (int t = 0; t < n_tiles; ++t) {
      int ids[kTilePages];
#pragma unroll
      for (int pg = 0; pg < kTilePages; ++pg) ids[pg] = __shfl_sync(0xffffffffu, cur, pg);
      if (lane < kTilePages && t + 1 < n_tiles) cur = page_id((t + 1) * kTilePages + lane);
      if (lane == 0) {
        const int st = t % kPrefillStages;
        mbar_wait(&empty_bar[st], ((t / kPrefillStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&full_bar[st], PrefillSmem<DH>::kStageBytes);
        const uint32_t dst = sbase + st * PrefillSmem<DH>::kStageBytes;
#pragma unroll
        for (int pg = 0; pg < kTilePages; ++pg) {
          tma_load_3d(dst + pg * KvBlock<DH>::kBytes, &kv_map, &full_bar[st], KV_COORD(kv_row(p, ids[pg], 0, kvh)));
          tma_load_3d(dst + (kTilePages + pg) * KvBlock<DH>::kBytes, &kv_map, &full_bar[st],
                      KV_COORD(kv_row(p, ids[pg], 1, kvh)));
        }
      }
      __syncwarp();
    }
    return;
  }

  // ---------------- consumers: rows of this warp: r -> token r / G, head r % G
  const int r_lo = lane / 4, r_hi = lane / 4 + 8;
  const int tl_lo = qoff + warp * TPW + r_lo / G, tl_hi = qoff + warp * TPW + r_hi / G;
  const bool ok_lo = r_lo < TPW * G && tl_lo < q_len;
  const bool ok_hi = r_hi < TPW * G && tl_hi < q_len;
  const int head_lo = kvh * G + r_lo % G, head_hi = kvh * G + r_hi % G;
  uint32_t qf[DH / 16][4];
  attn_load_q<DH>(p, q_start + (ok_lo ? tl_lo : 0), head_lo, ok_lo, q_start + (ok_hi ? tl_hi : 0), head_hi, ok_hi, qf);
  const int lim_lo = ok_lo ? pos0 + tl_lo + 1 : 0;  // causal: query at pos0+tl sees keys <= pos0+tl
  const int lim_hi = ok_hi ? pos0 + tl_hi + 1 : 0;

  float o[DH / 8][4];
#pragma unroll
  for (int n = 0; n < DH / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};

  for (int t = 0; t < n_tiles; ++t) {
    const int st = t % kPrefillStages;
    mbar_wait(&full_bar[st], (t / kPrefillStages) & 1);
    const uint32_t k_smem = sbase + st * PrefillSmem<DH>::kStageBytes;
    const uint32_t v_smem = k_smem + kTilePages * KvBlock<DH>::kBytes;
    float s[8][4];
    attn_qk<DH, 8>(qf, k_smem, 0, s);
    attn_softmax_step<DH, 8>(s, t * kKeys, lim_lo, lim_hi, p.scale_log2, m, l, o);
    attn_pv<DH, 8>(s, v_smem, 0, o);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[st]);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    l[h] += __shfl_xor_sync(0xffffffffu, l[h], 1);
    l[h] += __shfl_xor_sync(0xffffffffu, l[h], 2);
  }
  const int out_ld = p.n_heads * DH;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const bool ok = h ? ok_hi : ok_lo;
    if (!ok) continue;
    const int tok = q_start + (h ? tl_hi : tl_lo);
    const int head = h ? head_hi : head_lo;
    const float inv = 1.f / l[h];
    __nv_bfloat16* dst = p.out + (long long)tok * out_ld + head * DH + (lane % 4) * 2;
#pragma unroll
    for (int n = 0; n < DH / 8; ++n)
      *reinterpret_cast<uint32_t*>(dst + n * 8) = pack_bf16(o[n][2 * h] * inv, o[n][2 * h + 1] * inv);
  }
}

// ============================================================== decode
constexpr int kDecodeStages = 3;
#ifndef TC_DECODE_FUSED_MERGE
#define TC_DECODE_FUSED_MERGE 1  // 1: last-arriving warp merges split items; 0: attn_decode_combine kernel
#endif
constexpr int kDecodeWarps = 4;

template <int DH>
struct DecodeSmem {
  static constexpr int kStageBytes = 2 * KvBlock<DH>::kBytes;  // one page: K block then V block
  static constexpr int kWarpBytes = kDecodeStages * kStageBytes;
  static constexpr int kBytes = kDecodeWarps * kWarpBytes + 1024;
};

template <int DH, int G>
__global__ void __launch_bounds__(kDecodeWarps * 32, 2) attn_decode(const __grid_constant__ CUtensorMap kv_map, AttnParams p) {
  extern __shared__ uint8_t attn_smem_raw[];
  __shared__ uint64_t bars[kDecodeWarps][kDecodeStages];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t wbase = ((smem_u32(attn_smem_raw) + 1023u) & ~1023u) + warp * DecodeSmem<DH>::kWarpBytes;
  uint64_t* full = bars[warp];
  if (lane == 0) {
    for (int s = 0; s < kDecodeStages; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
    tma_prefetch_desc(&kv_map);
  }
  __syncwarp();
  const int n_warps = gridDim.x * kDecodeWarps;
  const int gw = blockIdx.x * kDecodeWarps + warp;

  // load cursor (lane 0): walks this warp's (item, page) stream S-1 pages ahead. The page id
  // of the NEXT load is fetched right after an issue, so its latency overlaps a whole page of
  // compute instead of sitting in front of the TMA.
  int l_item = gw, l_page = -1, issued = 0;
  int4 l_it = make_int4(0, 0, 0, 0);  // cached current item of the load cursor
  int nx_kvh = 0, nx_page = -1;        // prefetched next (kv head, page id)
  auto advance = [&]() {  // move the cursor to the next (item, page) and start fetching its id
    while (l_item < p.n_items) {
      if (l_page < 0) {
        l_it = p.dec_items[l_item];
        l_page = l_it.z;
      }
      if (l_page < l_it.w) {
        nx_kvh = l_it.y & 0xff;
        nx_page = p.block_tables[l_it.x + l_page];
        ++l_page;
        return;
      }
      l_item += n_warps;
      l_page = -1;
    }
    nx_page = -1;
  };
  auto issue_next = [&]() {
    if (nx_page < 0) return;
    const int st = issued % kDecodeStages;
    const uint32_t dst = wbase + st * DecodeSmem<DH>::kStageBytes;
    fence_proxy_async();
    mbar_arrive_expect_tx(&full[st], DecodeSmem<DH>::kStageBytes);
    tma_load_3d(dst, &kv_map, &full[st], KV_COORD(kv_row(p, nx_page, 0, nx_kvh)));
    tma_load_3d(dst + KvBlock<DH>::kBytes, &kv_map, &full[st], KV_COORD(kv_row(p, nx_page, 1, nx_kvh)));
    ++issued;
    advance();
  };
  if (lane == 0) {
    advance();
    for (int k = 0; k < kDecodeStages - 1; ++k) issue_next();
  }

  const int r_lo = lane / 4, r_hi = lane / 4 + 8;
  const bool ok_lo = r_lo < G, ok_hi = r_hi < G;
  int n = 0;  // pages consumed by this warp
  for (int item = gw; item < p.n_items; item += n_warps) {
    const int4 it = p.dec_items[item];
    const int kvh = it.y & 0xff, d = it.y >> 8;
    const int seq = p.dec_seq[d];
    const int chunks = p.dec_chunks[d];
    const int q_row = p.seq_q_start[seq];
    const int kv_len = p.seq_pos0[seq] + 1;
    uint32_t qf[DH / 16][4];
    attn_load_q<DH>(p, q_row, kvh * G + (ok_lo ? r_lo : 0), ok_lo, q_row, kvh * G + (ok_hi ? r_hi : 0), ok_hi, qf);
    float o[DH / 8][4];
#pragma unroll
    for (int c = 0; c < DH / 8; ++c) o[c][0] = o[c][1] = o[c][2] = o[c][3] = 0.f;
    float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
    for (int pg = it.z; pg < it.w; ++pg, ++n) {
      if (lane == 0) issue_next();
      const int st = n % kDecodeStages;
      mbar_wait(&full[st], (n / kDecodeStages) & 1);
      const uint32_t k_smem = wbase + st * DecodeSmem<DH>::kStageBytes;
      float s[2][4];
      attn_qk<DH, 2>(qf, k_smem, 0, s);
      attn_softmax_step<DH, 2>(s, pg * kPage, kv_len, kv_len, p.scale_log2, m, l, o);
      attn_pv<DH, 2>(s, k_smem + KvBlock<DH>::kBytes, 0, o);
      __syncwarp();
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      l[h] += __shfl_xor_sync(0xffffffffu, l[h], 1);
      l[h] += __shfl_xor_sync(0xffffffffu, l[h], 2);
    }
    const int c0 = (lane % 4) * 2;
    __nv_bfloat16* out_row = p.out + (long long)q_row * p.n_heads * DH + (long long)kvh * G * DH;
    if (chunks == 1) {
      if (ok_lo) {  // only rows < G (lanes 0 .. 4G-1) carry results
        const float inv = 1.f / l[0];
#pragma unroll
        for (int c = 0; c < DH / 8; ++c)
          *reinterpret_cast<uint32_t*>(out_row + r_lo * DH + c * 8 + c0) = pack_bf16(o[c][0] * inv, o[c][1] * inv);
      }
      continue;
    }
    if (ok_lo) {
      float* wo = p.ws_o + ((long long)item * G + r_lo) * DH + c0;
#pragma unroll
      for (int c = 0; c < DH / 8; ++c) *reinterpret_cast<float2*>(wo + c * 8) = make_float2(o[c][0], o[c][1]);
      if (lane % 4 == 0) *reinterpret_cast<float2*>(p.ws_ml + ((long long)item * G + r_lo) * 2) = make_float2(m[0], l[0]);
    }
#if !TC_DECODE_FUSED_MERGE
    continue;  // merged by attn_decode_combine
#endif
    __threadfence();
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      int* cnt = p.dec_cnt + d * p.n_kv_heads + kvh;
      last = atomicAdd(cnt, 1) == chunks - 1;
      if (last) *cnt = 0;  // ready for the next layer / step
    }
    if (!__shfl_sync(0xffffffffu, last, 0)) continue;
    __threadfence();
    // last arriver: merge the request's chunks (<= 32, host-guaranteed) for this kv head.
    // lane j loads (m, l) of chunk j for all G rows in one round trip; the per-row max and the
    // chunk weights go through shuffles; then every lane accumulates DH/32 dims of all G rows,
    // two chunks of vector loads in flight at a time.
    const int base = p.dec_item_base[d] + kvh * chunks;
    float wj[G];  // lane j: weight of chunk j for row r (before normalisation)
    float mj[G], lj[G];
#pragma unroll
    for (int r = 0; r < G; ++r) {
      const float2 ml = lane < chunks ? __ldcg(reinterpret_cast<const float2*>(p.ws_ml + ((long long)(base + lane) * G + r) * 2))
                                      : make_float2(-INFINITY, 0.f);
      mj[r] = ml.x;
      lj[r] = ml.y;
    }
    float inv_l[G];
#pragma unroll
    for (int r = 0; r < G; ++r) {
      const float mm = warp_max(mj[r]);
      wj[r] = (mj[r] == -INFINITY || mm == -INFINITY) ? 0.f : exp2f(mj[r] - mm);
      const float ll = warp_sum(wj[r] * lj[r]);
      inv_l[r] = ll > 0.f ? 1.f / ll : 0.f;
    }
    constexpr int V = DH / 32;  // dims per lane
    float acc[G][V];
#pragma unroll
    for (int r = 0; r < G; ++r)
#pragma unroll
      for (int e = 0; e < V; ++e) acc[r][e] = 0.f;
    for (int j = 0; j < chunks; j += 2) {
      float oa[2][G][V];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int r = 0; r < G; ++r) {
          const int jj = min(j + u, chunks - 1);
          const float* src = p.ws_o + ((long long)(base + jj) * G + r) * DH + lane * V;
          if constexpr (V == 4) {
            const float4 t = __ldcg(reinterpret_cast<const float4*>(src));
            oa[u][r][0] = t.x; oa[u][r][1] = t.y; oa[u][r][2] = t.z; oa[u][r][3] = t.w;
          } else {
            const float2 t = __ldcg(reinterpret_cast<const float2*>(src));
            oa[u][r][0] = t.x; oa[u][r][1] = t.y;
          }
        }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (j + u >= chunks) break;
#pragma unroll
        for (int r = 0; r < G; ++r) {
          const float f = __shfl_sync(0xffffffffu, wj[r], j + u);
#pragma unroll
          for (int e = 0; e < V; ++e) acc[r][e] += f * oa[u][r][e];
        }
      }
    }
#pragma unroll
    for (int r = 0; r < G; ++r) {
      __nv_bfloat16* dst = out_row + r * DH + lane * V;
      if constexpr (V == 4) {
        uint2 w;
        w.x = pack_bf16(acc[r][0] * inv_l[r], acc[r][1] * inv_l[r]);
        w.y = pack_bf16(acc[r][2] * inv_l[r], acc[r][3] * inv_l[r]);
        *reinterpret_cast<uint2*>(dst) = w;
      } else {
        *reinterpret_cast<uint32_t*>(dst) = pack_bf16(acc[r][0] * inv_l[r], acc[r][1] * inv_l[r]);
      }
    }
  }
}

// Separate merge of split decode items (TC_DECODE_FUSED_MERGE = 0): one warp per (request,
// kv head), same vectorised merge as the fused path.
template <int DH, int G>
__global__ void attn_decode_combine(AttnParams p, int n_dec) {
  const int lane = threadIdx.x % 32;
  const int wid = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (wid >= n_dec * p.n_kv_heads) return;
  const int d = wid / p.n_kv_heads, kvh = wid % p.n_kv_heads;
  const int chunks = p.dec_chunks[d];
  if (chunks <= 1) return;
  const int base = p.dec_item_base[d] + kvh * chunks;
  const int q_row = p.seq_q_start[p.dec_seq[d]];
  __nv_bfloat16* out_row = p.out + (long long)q_row * p.n_heads * DH + (long long)kvh * G * DH;
  float wj[G], mj[G], lj[G], inv_l[G];
#pragma unroll
  for (int r = 0; r < G; ++r) {
    const float2 ml = lane < chunks ? __ldcg(reinterpret_cast<const float2*>(p.ws_ml + ((long long)(base + lane) * G + r) * 2))
                                    : make_float2(-INFINITY, 0.f);
    mj[r] = ml.x;
    lj[r] = ml.y;
  }
#pragma unroll
  for (int r = 0; r < G; ++r) {
    const float mm = warp_max(mj[r]);
    wj[r] = (mj[r] == -INFINITY || mm == -INFINITY) ? 0.f : exp2f(mj[r] - mm);
    const float ll = warp_sum(wj[r] * lj[r]);
    inv_l[r] = ll > 0.f ? 1.f / ll : 0.f;
  }
  constexpr int V = DH / 32;
  float acc[G][V] = {};
  for (int j = 0; j < chunks; ++j) {
#pragma unroll
    for (int r = 0; r < G; ++r) {
      const float f = __shfl_sync(0xffffffffu, wj[r], j);
      const float* src = p.ws_o + ((long long)(base + j) * G + r) * DH + lane * V;
#pragma unroll
      for (int e = 0; e < V; ++e) acc[r][e] += f * __ldcg(src + e);
    }
  }
#pragma unroll
  for (int r = 0; r < G; ++r)
#pragma unroll
    for (int e = 0; e < V; ++e) out_row[r * DH + lane * V + e] = __float2bfloat16(acc[r][e] * inv_l[r]);
}

}  // namespace tc
