// Paged attention for the hybrid step (SURVEY.md 2, K1 + K2).
//
// KV pool layout (page-major so one request's KV migrates as whole pages):
//   pool[page][layer][k|v][kv_head][slot 0..PS-1][head_dim]   (bf16)
// One page of Llama-3-8B = 32 x 2 x 8 x 16 x 128 x 2 B = 2 MiB; the K (or V)
// rows of one (page, layer, kv_head) are 4 KiB contiguous, read with 16 B
// cp.async into padded shared-memory tiles of 64 keys (4 pages).
//
//  * attn_prefill  -- chunked-prefill queries (a chunk may span prompts; each
//    slice is a sequence) attend causally to the paged prefix + in-chunk keys.
//    CTA = (16/G tokens x G heads) x 4 warps of one GQA group; QK^T and PV on
//    tensor cores (mma.sync m16n8k16 bf16, fp32 accumulate), online softmax.
//  * attn_decode   -- one query token per request; CTA = (request, kv_head,
//    KV split); the 4 warps take interleaved 16-key pages of each 64-key tile,
//    merged in shared memory, then across splits by attn_decode_combine.
#pragma once

#include "common.cuh"

namespace tc {

struct AttnParams {
  const __nv_bfloat16* qkv;  // [T, (H + 2 Hkv) * DH], RoPE already applied to q and k
  __nv_bfloat16* out;        // [T, H * DH]
  const __nv_bfloat16* kv;   // pool base (bf16)
  long long page_stride;     // elements per page
  int layer, n_layers, n_heads, n_kv_heads, page_size;
  float scale_log2;          // log2(e) / sqrt(DH)
  // sequences of this step
  const int* seq_q_start;    // first packed row
  const int* seq_q_len;      // rows (1 for decode)
  const int* seq_pos0;       // position of the first row
  const int* seq_bt_off;     // offset into block_tables
  const int* block_tables;   // flat page ids
  // prefill work list
  const int* qblk_seq;
  const int* qblk_off;
  // decode work list
  const int* dec_seq;        // decode index -> sequence index
  int n_splits, tiles_per_split;
  float* ws_o;               // [n_dec, Hkv, splits, G, DH]
  float* ws_ml;              // [n_dec, Hkv, splits, G, 2]
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
TC_DEVICE void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int bytes = valid ? 16 : 0;  // zero-fill when invalid
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
TC_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
TC_DEVICE void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr int kAttnKeys = 64;  // keys per shared-memory tile
constexpr int kAttnThreads = 128;

template <int DH>
struct AttnTile {
  static constexpr int LD = DH + 8;                      // padded row: conflict-free ldmatrix
  static constexpr int kHalfElems = kAttnKeys * LD;      // K or V
  static constexpr int kStageElems = 2 * kHalfElems;
  static constexpr int kChunksPerRow = DH / 8;           // 16 B chunks
};

// Stage keys [key0, key0 + 64) of (layer, kv_head) into smem K|V; keys >= kv_len are zero-filled.
template <int DH>
TC_DEVICE void attn_load_tile(const AttnParams& p, const int* bt, int kvh, int key0, int kv_len, uint32_t smem_stage) {
  using T = AttnTile<DH>;
  const long long head_off = ((long long)(p.layer * 2) * p.n_kv_heads + kvh) * p.page_size * DH;
  const long long v_off = (long long)p.n_kv_heads * p.page_size * DH;
  constexpr int kChunks = kAttnKeys * T::kChunksPerRow;
#pragma unroll
  for (int i = threadIdx.x; i < kChunks; i += kAttnThreads) {
    const int key = i / T::kChunksPerRow;
    const int part = i % T::kChunksPerRow;
    const int gk = key0 + key;
    const bool valid = gk < kv_len;
    const int page = valid ? bt[gk / p.page_size] : 0;
    const __nv_bfloat16* src = p.kv + (long long)page * p.page_stride + head_off +
                               (long long)(gk % p.page_size) * DH + part * 8;
    const uint32_t dst = smem_stage + (uint32_t)(key * T::LD + part * 8) * 2;
    cp_async16(dst, src, valid);
    cp_async16(dst + T::kHalfElems * 2, src + v_off, valid);
  }
}

// Q fragment (A operand) for the warp's 16 rows: row r -> (token row_tok[r], head row_head[r]).
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

// S[16 x 8*NT] = Q K^T for keys [kbase, kbase + 8*NT) of the staged tile.
template <int DH, int NT>
TC_DEVICE void attn_qk(const uint32_t (&qf)[DH / 16][4], uint32_t k_smem, int kbase, float (&s)[NT][4]) {
  using T = AttnTile<DH>;
  const int lane = threadIdx.x % 32;
#pragma unroll
  for (int t = 0; t < NT; ++t) s[t][0] = s[t][1] = s[t][2] = s[t][3] = 0.f;
#pragma unroll
  for (int ks = 0; ks < DH / 16; ++ks) {
#pragma unroll
    for (int t = 0; t < NT; t += 2) {
      const int j = lane / 8, r = lane % 8;
      const int key = kbase + t * 8 + (j / 2) * 8 + r;
      const int dim = ks * 16 + (j % 2) * 8;
      uint32_t b0, b1, b2, b3;
      ldsm_x4(k_smem + (uint32_t)(key * T::LD + dim) * 2, b0, b1, b2, b3);
      mma_bf16_16816(s[t], qf[ks], b0, b1);
      mma_bf16_16816(s[t + 1], qf[ks], b2, b3);
    }
  }
}

// O[16 x DH] += P[16 x 8*NT] V[keys kbase.., DH]
template <int DH, int NT>
TC_DEVICE void attn_pv(const float (&pr)[NT][4], uint32_t v_smem, int kbase, float (&o)[DH / 8][4]) {
  using T = AttnTile<DH>;
  const int lane = threadIdx.x % 32;
#pragma unroll
  for (int kk = 0; kk < NT / 2; ++kk) {
    uint32_t a[4];
    a[0] = pack_bf16(pr[2 * kk][0], pr[2 * kk][1]);
    a[1] = pack_bf16(pr[2 * kk][2], pr[2 * kk][3]);
    a[2] = pack_bf16(pr[2 * kk + 1][0], pr[2 * kk + 1][1]);
    a[3] = pack_bf16(pr[2 * kk + 1][2], pr[2 * kk + 1][3]);
#pragma unroll
    for (int n = 0; n < DH / 8; n += 2) {
      const int j = lane / 8, r = lane % 8;
      const int key = kbase + kk * 16 + (j % 2) * 8 + r;
      const int dim = n * 8 + (j / 2) * 8;
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(v_smem + (uint32_t)(key * T::LD + dim) * 2, b0, b1, b2, b3);
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

template <int DH, int G>
__global__ void __launch_bounds__(kAttnThreads) attn_prefill(AttnParams p) {
  using T = AttnTile<DH>;
  constexpr int TPW = 16 / G;  // tokens per warp
  constexpr int TPC = 4 * TPW;
  extern __shared__ __align__(16) uint8_t attn_smem[];
  const uint32_t sbase = smem_u32(attn_smem);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int seq = p.qblk_seq[blockIdx.x];
  const int qoff = p.qblk_off[blockIdx.x];
  const int kvh = blockIdx.y;
  const int q_start = p.seq_q_start[seq], q_len = p.seq_q_len[seq], pos0 = p.seq_pos0[seq];
  const int* bt = p.block_tables + p.seq_bt_off[seq];
  const int kv_end = pos0 + min(qoff + TPC, q_len);

  // rows of this warp: r -> token r / G, head r % G
  const int r_lo = lane / 4, r_hi = lane / 4 + 8;
  const int tl_lo = qoff + warp * TPW + r_lo / G, tl_hi = qoff + warp * TPW + r_hi / G;
  const bool ok_lo = r_lo < TPW * G && tl_lo < q_len;
  const bool ok_hi = r_hi < TPW * G && tl_hi < q_len;
  const int head_lo = kvh * G + r_lo % G, head_hi = kvh * G + r_hi % G;
  uint32_t qf[DH / 16][4];
  attn_load_q<DH>(p, q_start + (ok_lo ? tl_lo : 0), head_lo, ok_lo, q_start + (ok_hi ? tl_hi : 0), head_hi, ok_hi, qf);
  // causal bound (exclusive): query at position pos0 + tl sees keys <= pos0 + tl
  const int lim_lo = ok_lo ? pos0 + tl_lo + 1 : 0;
  const int lim_hi = ok_hi ? pos0 + tl_hi + 1 : 0;

  float o[DH / 8][4];
#pragma unroll
  for (int n = 0; n < DH / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};

  const int n_tiles = (kv_end + kAttnKeys - 1) / kAttnKeys;
  attn_load_tile<DH>(p, bt, kvh, 0, kv_end, sbase);
  cp_async_commit();
  for (int t = 0; t < n_tiles; ++t) {
    const uint32_t stage = sbase + (uint32_t)((t & 1) * T::kStageElems) * 2;
    if (t + 1 < n_tiles)
      attn_load_tile<DH>(p, bt, kvh, (t + 1) * kAttnKeys, kv_end, sbase + (uint32_t)(((t + 1) & 1) * T::kStageElems) * 2);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    float s[8][4];
    attn_qk<DH, 8>(qf, stage, 0, s);
    attn_softmax_step<DH, 8>(s, t * kAttnKeys, lim_lo, lim_hi, p.scale_log2, m, l, o);
    attn_pv<DH, 8>(s, stage + T::kHalfElems * 2, 0, o);
    __syncthreads();
  }
  // normalise and store
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

template <int DH, int G>
__global__ void __launch_bounds__(kAttnThreads) attn_decode(AttnParams p) {
  using T = AttnTile<DH>;
  extern __shared__ __align__(16) uint8_t attn_smem[];
  const uint32_t sbase = smem_u32(attn_smem);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int d = blockIdx.x, kvh = blockIdx.y, split = blockIdx.z;
  const int seq = p.dec_seq[d];
  const int q_row = p.seq_q_start[seq];
  const int kv_len = p.seq_pos0[seq] + 1;
  const int* bt = p.block_tables + p.seq_bt_off[seq];
  const int n_tiles_all = (kv_len + kAttnKeys - 1) / kAttnKeys;
  const int t0 = split * p.tiles_per_split;
  const int t1 = min(n_tiles_all, t0 + p.tiles_per_split);

  const int r_lo = lane / 4, r_hi = lane / 4 + 8;
  const bool ok_lo = r_lo < G, ok_hi = r_hi < G;
  uint32_t qf[DH / 16][4];
  attn_load_q<DH>(p, q_row, kvh * G + (ok_lo ? r_lo : 0), ok_lo, q_row, kvh * G + (ok_hi ? r_hi : 0), ok_hi, qf);

  float o[DH / 8][4];
#pragma unroll
  for (int n = 0; n < DH / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};

  // 3-stage ring of 64-key tiles; warp w consumes keys [16w, 16w+16) of each tile
  constexpr int kStages = 3;
  for (int s = 0; s < kStages - 1; ++s) {
    if (t0 + s < t1) attn_load_tile<DH>(p, bt, kvh, (t0 + s) * kAttnKeys, kv_len, sbase + (uint32_t)(s * T::kStageElems) * 2);
    cp_async_commit();
  }
  for (int t = t0; t < t1; ++t) {
    const int i = t - t0;
    const int pf = t + kStages - 1;
    if (pf < t1) attn_load_tile<DH>(p, bt, kvh, pf * kAttnKeys, kv_len, sbase + (uint32_t)(((i + kStages - 1) % kStages) * T::kStageElems) * 2);
    cp_async_commit();
    cp_async_wait<kStages - 1>();
    __syncthreads();
    const uint32_t stage = sbase + (uint32_t)((i % kStages) * T::kStageElems) * 2;
    const int kb = warp * 16;
    float s[2][4];
    attn_qk<DH, 2>(qf, stage, kb, s);
    attn_softmax_step<DH, 2>(s, t * kAttnKeys + kb, kv_len, kv_len, p.scale_log2, m, l, o);
    attn_pv<DH, 2>(s, stage + T::kHalfElems * 2, kb, o);
    __syncthreads();
  }
  cp_async_wait<0>();
  // reduce the row sums across the quad
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    l[h] += __shfl_xor_sync(0xffffffffu, l[h], 1);
    l[h] += __shfl_xor_sync(0xffffffffu, l[h], 2);
  }
  // cross-warp merge through shared memory (reuses the tile buffers)
  __syncthreads();
  float* sm_o = reinterpret_cast<float*>(attn_smem);     // [4 warps][G][DH]
  float* sm_ml = sm_o + 4 * G * DH;                      // [4 warps][G][2]
  if (lane % 4 == 0) {
    if (ok_lo) { sm_ml[(warp * G + r_lo) * 2] = m[0]; sm_ml[(warp * G + r_lo) * 2 + 1] = l[0]; }
    if (ok_hi) { sm_ml[(warp * G + r_hi) * 2] = m[1]; sm_ml[(warp * G + r_hi) * 2 + 1] = l[1]; }
  }
#pragma unroll
  for (int n = 0; n < DH / 8; ++n) {
    const int c = n * 8 + (lane % 4) * 2;
    if (ok_lo) { sm_o[(warp * G + r_lo) * DH + c] = o[n][0]; sm_o[(warp * G + r_lo) * DH + c + 1] = o[n][1]; }
    if (ok_hi) { sm_o[(warp * G + r_hi) * DH + c] = o[n][2]; sm_o[(warp * G + r_hi) * DH + c + 1] = o[n][3]; }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < G * DH; idx += kAttnThreads) {
    const int r = idx / DH, c = idx % DH;
    float mm = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) mm = fmaxf(mm, sm_ml[(w * G + r) * 2]);
    float acc = 0.f, ll = 0.f;
    if (mm != -INFINITY) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float f = exp2f(sm_ml[(w * G + r) * 2] - mm);
        acc += f * sm_o[(w * G + r) * DH + c];
        ll += f * sm_ml[(w * G + r) * 2 + 1];
      }
    }
    if (p.n_splits == 1) {
      const int head = kvh * G + r;
      p.out[(long long)q_row * p.n_heads * DH + head * DH + c] = __float2bfloat16(ll > 0.f ? acc / ll : 0.f);
    } else {
      const long long slot = (((long long)d * p.n_kv_heads + kvh) * p.n_splits + split) * G + r;
      p.ws_o[slot * DH + c] = acc;
      if (c == 0) {
        p.ws_ml[slot * 2] = mm;
        p.ws_ml[slot * 2 + 1] = ll;
      }
    }
  }
}

// Merge split-KV partials: grid (n_dec, H), DH threads.
template <int DH, int G>
__global__ void attn_decode_combine(AttnParams p) {
  const int d = blockIdx.x, head = blockIdx.y, c = threadIdx.x;
  const int kvh = head / G, r = head % G;
  const int q_row = p.seq_q_start[p.dec_seq[d]];
  float mm = -INFINITY;
  for (int s = 0; s < p.n_splits; ++s) {
    const long long slot = (((long long)d * p.n_kv_heads + kvh) * p.n_splits + s) * G + r;
    mm = fmaxf(mm, p.ws_ml[slot * 2]);
  }
  float acc = 0.f, ll = 0.f;
  if (mm != -INFINITY) {
    for (int s = 0; s < p.n_splits; ++s) {
      const long long slot = (((long long)d * p.n_kv_heads + kvh) * p.n_splits + s) * G + r;
      const float f = exp2f(p.ws_ml[slot * 2] - mm);
      acc += f * p.ws_o[slot * DH + c];
      ll += f * p.ws_ml[slot * 2 + 1];
    }
  }
  p.out[(long long)q_row * p.n_heads * DH + head * DH + c] = __float2bfloat16(ll > 0.f ? acc / ll : 0.f);
}

}  // namespace tc
