// Memory-bound kernels of the hybrid step:
// embedding gather, RMSNorm (fp32 residual stream -> bf16), greedy argmax
// sampling, deterministic weight init and the KV page migration copy. (RoPE and
// the paged KV append are fused into the QKV GEMM epilogue, gemm.cuh.) All use 16 B vector accesses and warp-shuffle reductions.
#pragma once

#include "common.cuh"

namespace tc {

// ---------------------------------------------------------------- weight init
// value = ((u24 * 2^-24) * 2 - 1) * scale + offset, u24 = top 24 bits of
// splitmix64(splitmix64(seed ^ splitmix64(tensor_id)) + logical_index), computed
// with explicitly rounded fp32 ops so the numpy oracle reproduces every bit.
__host__ __device__ inline uint64_t sm64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// interleave64 != 0: physical row p of a [2*F, K] gate|up matrix stores logical
// row (p/128)*64 + p%64 of gate (p%128 < 64) or of up (tensor_id + 1).
__global__ void init_weights(__nv_bfloat16* dst, long long rows, long long cols, uint64_t seed, uint64_t tensor_id,
                             float scale, float offset, int interleave64) {
  const long long n = rows * cols;
  const uint64_t key_a = sm64(seed ^ sm64(tensor_id));
  const uint64_t key_b = sm64(seed ^ sm64(tensor_id + 1));
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long prow = i / cols, col = i % cols;
    long long lrow = prow;
    uint64_t key = key_a;
    if (interleave64) {
      const long long blk = prow / 128, within = prow % 128;
      lrow = blk * 64 + (within % 64);
      key = within < 64 ? key_a : key_b;
    }
    const uint64_t h = sm64(key + (uint64_t)(lrow * cols + col));
    const float u = (float)(uint32_t)(h >> 40) * 5.9604644775390625e-08f;  // exact
    const float c = u * 2.0f - 1.0f;                                          // exact
    const float v = __fadd_rn(__fmul_rn(c, scale), offset);
    dst[i] = __float2bfloat16_rn(v);
  }
}

// ---------------------------------------------------------------- embedding
// resid[t, :] = float(embed[tokens[t], :])
__global__ void embed_rows(const int* __restrict__ tokens, const __nv_bfloat16* __restrict__ embed,
                           float* __restrict__ resid, int d) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x;
  const __nv_bfloat16* src = embed + (long long)tokens[t] * d;
  float* dst = resid + (long long)t * d;
  for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
    const uint4 v = *reinterpret_cast<const uint4*>(src + c);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = unpack_bf16(w[e]);
      dst[c + 2 * e] = f.x;
      dst[c + 2 * e + 1] = f.y;
    }
  }
}

// ---------------------------------------------------------------- RMSNorm
// out[r, :] = bf16(x[src_row(r), :] * rsqrt(mean(x^2) + eps) * w), fp32 math.
// rows == nullptr: identity row map; otherwise gathers rows (sampled-row LM head).
// The row is read once into registers (<= kMaxVec float4 per thread: d <= 8192).
template <int THREADS>
__global__ void __launch_bounds__(THREADS) rmsnorm_rows(const float* __restrict__ x, const int* __restrict__ rows,
                                                        const __nv_bfloat16* __restrict__ w,
                                                        __nv_bfloat16* __restrict__ out, int d, float eps) {
  constexpr int kMaxVec = 8192 / (4 * THREADS);
  // the norm weights do not depend on the predecessor kernel: fetch them before the PDL wait
  uint2 wv[kMaxVec];
#pragma unroll
  for (int i = 0; i < kMaxVec; ++i) {
    const int c = (i * THREADS + threadIdx.x) * 4;
    if (c < d) wv[i] = __ldg(reinterpret_cast<const uint2*>(w + c));
  }
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  const int src = rows ? rows[r] : r;
  const float* xr = x + (long long)src * d;
  float4 v[kMaxVec];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxVec; ++i) {
    const int c = (i * THREADS + threadIdx.x) * 4;
    if (c < d) {
      v[i] = __ldg(reinterpret_cast<const float4*>(xr + c));
      ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    }
  }
  __shared__ float red[THREADS / 32];
  ss = warp_sum(ss);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int i = 0; i < THREADS / 32; ++i) tot += red[i];
  const float inv = rsqrtf(tot / (float)d + eps);
  __nv_bfloat16* o = out + (long long)r * d;
#pragma unroll
  for (int i = 0; i < kMaxVec; ++i) {
    const int c = (i * THREADS + threadIdx.x) * 4;
    if (c < d) {
      const float2 w01 = unpack_bf16(wv[i].x), w23 = unpack_bf16(wv[i].y);
      uint2 pk;
      pk.x = pack_bf16(v[i].x * inv * w01.x, v[i].y * inv * w01.y);
      pk.y = pack_bf16(v[i].z * inv * w23.x, v[i].w * inv * w23.y);
      *reinterpret_cast<uint2*>(o + c) = pk;
    }
  }
}

// ---------------------------------------------------------------- greedy sampling
// ids[r] = argmax_v logits[r, v], lowest index on ties.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) argmax_rows(const float* __restrict__ logits, int vocab, int* __restrict__ ids) {
  pdl_wait();
  pdl_trigger();
  const float* row = logits + (long long)blockIdx.x * vocab;
  float best = -INFINITY;
  int best_i = 0x7fffffff;
  for (int c = threadIdx.x * 4; c < vocab; c += THREADS * 4) {
    const float4 v = *reinterpret_cast<const float4*>(row + c);
    const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (e[k] > best) {  // strictly greater keeps the lowest index within a thread
        best = e[k];
        best_i = c + k;
      }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
    if (ob > best || (ob == best && oi < best_i)) {
      best = ob;
      best_i = oi;
    }
  }
  __shared__ float sb[THREADS / 32];
  __shared__ int si[THREADS / 32];
  if (threadIdx.x % 32 == 0) {
    sb[threadIdx.x / 32] = best;
    si[threadIdx.x / 32] = best_i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < THREADS / 32; ++w)
      if (sb[w] > best || (sb[w] == best && si[w] < best_i)) {
        best = sb[w];
        best_i = si[w];
      }
    ids[blockIdx.x] = best_i;
  }
}

// ---------------------------------------------------------------- KV migration
// Whole-page copies of one request's KV (all layers): dst_pool[dst_page[i]] = src_pool[src_page[i]].
// Pools may live on different GPUs (peer pointers over NVLink, UVA). Work unit = one 64 KiB slice
// of a page per block iteration (512 threads x 8 x 16 B loads in flight, then the stores): 32-bit
// index math once per slice (round 1 divided a 64-bit element index by the page size per 16 B).
constexpr int kCopyThreads = 512;
constexpr int kCopySliceVec = kCopyThreads * 8;  // 16 B vectors per slice (64 KiB)

template <typename SrcPage, typename DstPage>
__device__ __forceinline__ void copy_page_slices(const uint4* __restrict__ src_pool, uint4* __restrict__ dst_pool,
                                                 SrcPage&& src_page, DstPage&& dst_page, int n_pages, long long page_vec) {
  const int spp = (int)((page_vec + kCopySliceVec - 1) / kCopySliceVec);  // slices per page
  for (int b = blockIdx.x; b < n_pages * spp; b += gridDim.x) {
    const int pg = b / spp;
    const long long off = (long long)(b - pg * spp) * kCopySliceVec;
    const uint4* s = src_pool + (long long)src_page(pg) * page_vec + off;
    uint4* d = dst_pool + (long long)dst_page(pg) * page_vec + off;
    const int n = (int)min((long long)kCopySliceVec, page_vec - off);
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = threadIdx.x + u * kCopyThreads;
      if (i < n) v[u] = ld_nc_v4(s + i);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = threadIdx.x + u * kCopyThreads;
      if (i < n) st_global_v4(d + i, v[u]);
    }
  }
}

// page lists in device memory (tc_copy_pages)
__global__ void __launch_bounds__(kCopyThreads) kv_copy_pages(const uint4* __restrict__ src_pool, uint4* __restrict__ dst_pool,
                                                              const int* __restrict__ src_pages,
                                                              const int* __restrict__ dst_pages, int n_pages,
                                                              long long page_vec) {
  copy_page_slices(src_pool, dst_pool, [&](int i) { return src_pages[i]; }, [&](int i) { return dst_pages[i]; }, n_pages,
                   page_vec);
}

// Page lists of one asynchronous migration travel in the kernel's parameter space (16 KB of the
// 32 KB limit): no staging buffer, no H2D copy on the copy stream, any number of migrations in
// flight. Requests longer than kMigPagesPerLaunch pages take several launches.
constexpr int kMigPagesPerLaunch = 2040;
struct MigPages {
  int n;
  int32_t src[kMigPagesPerLaunch];
  int32_t dst[kMigPagesPerLaunch];
};

__global__ void __launch_bounds__(kCopyThreads) kv_migrate_pages(const uint4* __restrict__ src_pool, uint4* __restrict__ dst_pool,
                                                                 const __grid_constant__ MigPages pl, long long page_vec) {
  copy_page_slices(src_pool, dst_pool, [&](int i) { return pl.src[i]; }, [&](int i) { return pl.dst[i]; }, pl.n, page_vec);
}

}  // namespace tc
