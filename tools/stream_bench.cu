// Read-stream microbenchmark (tools only): what HBM read rate does each way of streaming bytes
// into an SM reach on this B200, as a function of bytes in flight per SM? Informs the decode
// attention page stream (8 KiB TMA boxes through a smem ring) and the decode-only weight-streaming
// GEMMs (16 KiB TMA boxes), both of which plateau near 5.2 TB/s.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/stream_bench tools/stream_bench.cu -lcuda
//   tools/stream_bench            -> one JSON line per configuration
//
// Kernels: ldg (LDG.128, U loads in flight per thread), bulk (cp.async.bulk 1-D copies of B bytes
// into an S-stage ring, one issuing thread, consumers release at once), tensor (cp.async.bulk.tensor
// 2-D boxes of 64 cols x R rows, 128 B swizzle, like the GEMM weight stream). Chunks are visited
// in a pseudo-random order (like KV pages) or sequentially.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(smem_u32(b)),
      "r"(par)
      : "memory");
}

__device__ __forceinline__ uint64_t chunk_of(uint64_t i, uint64_t n, int random) {
  return random ? (i * 2654435761ull) % n : i;  // n odd-ish prime-free: a permutation when gcd = 1
}

__global__ void ldg_stream(const uint4* __restrict__ p, uint64_t n_vec, uint64_t* sink) {
  constexpr int U = 8;
  uint32_t acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_vec; i += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = i + u * stride < n_vec ? __ldcs(p + i + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// cp.async.bulk of `chunk` bytes per stage; chunks assigned round-robin to CTAs. P producer warps
// (lane 0 each) issue interleaved stages (stage k by producer k % P); `region` chunks bound the
// random walk (TLB reach test: random over 4 GiB vs inside a few hundred MiB).
__global__ void bulk_stream(const uint8_t* __restrict__ base, uint64_t n_chunks, int chunk, int stages, int random,
                            int producers, uint64_t region, int lanes) {
  extern __shared__ __align__(1024) uint8_t ring[];
  __shared__ uint64_t full[64], empty[64];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t mine = (n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp < producers) {
    // lanes 0..lanes-1 of each producer warp issue one chunk each per round (SIMT issue)
    if (lane < lanes)
      for (uint64_t k = (uint64_t)warp * lanes + lane; k < mine; k += (uint64_t)producers * lanes) {
        const int st = (int)(k % stages);
        mbar_wait(&empty[st], (uint32_t)((k / stages) & 1) ^ 1);
        mbar_expect(&full[st], chunk);
        const uint64_t idx = blockIdx.x + k * gridDim.x;
        // random 1: pseudo-random over the whole buffer; 2: inside the first `region` chunks only (L2-resident)
        const uint64_t c = random == 2 ? chunk_of(idx, region, 1) : random ? (idx / region) * region + chunk_of(idx % region, region, 1) : idx;
        const uint8_t* src = base + (c % n_chunks) * chunk;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(ring + st * chunk)),
                     "l"(src), "r"(chunk), "r"(smem_u32(&full[st]))
                     : "memory");
      }
  } else if (warp == producers && lane == 0) {
    for (uint64_t k = 0; k < mine; ++k) {
      const int st = (int)(k % stages);
      mbar_wait(&full[st], (uint32_t)((k / stages) & 1));
      mbar_arrive(&empty[st]);
    }
  }
}

// 2-D tensor boxes (64 bf16 columns x rows), 128 B swizzle: the GEMM weight stream's access shape
__global__ void tensor_stream(const __grid_constant__ CUtensorMap map, uint64_t n_boxes, int box_rows, int stages,
                              int random, int rows_per_col_block) {
  extern __shared__ __align__(1024) uint8_t ring_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ring_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[64], empty[64];
  const int bytes = box_rows * 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t mine = (n_boxes - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (uint64_t k = 0; k < mine; ++k) {
      const int st = (int)(k % stages);
      mbar_wait(&empty[st], (uint32_t)((k / stages) & 1) ^ 1);
      mbar_expect(&full[st], bytes);
      const uint64_t b = chunk_of(blockIdx.x + k * gridDim.x, n_boxes, random);
      const int c0 = (int)(b / rows_per_col_block) * 64, c1 = (int)(b % rows_per_col_block) * box_rows;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(ring + st * bytes)),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(c0), "r"(c1), "r"(smem_u32(&full[st]))
          : "memory");
    }
  } else if (threadIdx.x == 32) {
    for (uint64_t k = 0; k < mine; ++k) {
      const int st = (int)(k % stages);
      mbar_wait(&full[st], (uint32_t)((k / stages) & 1));
      mbar_arrive(&empty[st]);
    }
  }
}

// 3-D boxes exactly like the decode KV stream (kv_map): {64 dims, 32 rows, 2 halves}, 128 B swizzle,
// one 8 KiB (K, V) page-head block per box, random blocks; P producer warps
__global__ void tensor3d_stream(const __grid_constant__ CUtensorMap map, uint64_t n_blocks, int stages, int producers) {
  extern __shared__ __align__(1024) uint8_t ring_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ring_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[64], empty[64];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t mine = (n_blocks - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp < producers) {
    if (lane == 0)
      for (uint64_t k = warp; k < mine; k += producers) {
        const int st = (int)(k % stages);
        mbar_wait(&empty[st], (uint32_t)((k / stages) & 1) ^ 1);
        mbar_expect(&full[st], 8192);
        const int row = (int)(chunk_of(blockIdx.x + k * gridDim.x, n_blocks, 1) * 32);
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                smem_u32(ring + st * 8192)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(row), "r"(0), "r"(smem_u32(&full[st]))
            : "memory");
      }
  } else if (warp == producers && lane == 0) {
    for (uint64_t k = 0; k < mine; ++k) {
      const int st = (int)(k % stages);
      mbar_wait(&full[st], (uint32_t)((k / stages) & 1));
      mbar_arrive(&empty[st]);
    }
  }
}

int main() {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t bytes = (size_t)4 << 30;  // 4 GiB: far beyond L2
  uint8_t* buf = nullptr;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 1, bytes));
  uint64_t* sink = nullptr;
  CK(cudaMalloc(&sink, 8));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto time_it = [&](auto&& launch) {
    launch();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      CK(cudaEventRecord(a));
      launch();
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = ms < best ? ms : best;
    }
    CK(cudaGetLastError());
    return best;
  };
  for (int per_sm : {2}) {
    for (int thr : {512}) {
      const int grid = sms * per_sm;
      if (per_sm * thr > 2048) continue;
      const float ms = time_it([&] { ldg_stream<<<grid, thr>>>((const uint4*)buf, bytes / 16, sink); });
      std::printf("{\"kernel\": \"ldg_u8\", \"grid\": %d, \"threads\": %d, \"inflight_per_sm_kb\": %d, \"gb_s\": %.1f}\n",
                  grid, thr, per_sm * thr * 8 * 16 / 1024, bytes / ms / 1e6);
    }
  }
  {
    PFN_cuTensorMapEncodeTiled_v12000 enc3 = nullptr;
    cudaDriverEntryPointQueryResult q3;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc3), cudaEnableDefault, &q3));
    const uint64_t rows = bytes / 256;  // rows of 128 dims (256 B), viewed {64 dims, rows, 2 halves}
    CUtensorMap map;
    cuuint64_t dims[3] = {64, rows, 2};
    cuuint64_t strides[2] = {256, 128};
    cuuint32_t box[3] = {64, 32, 2};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc3(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 1;
    const uint64_t n_blocks = rows / 32 - 1;
    for (int producers : {1, 2, 4, 8}) {
      const int stages = 24;
      CK(cudaFuncSetAttribute(tensor3d_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024 + 1024));
      const float ms = time_it([&] { tensor3d_stream<<<sms, 32 * (producers + 1), 192 * 1024 + 1024>>>(map, n_blocks, stages, producers); });
      std::printf("{\"kernel\": \"tensor3d_kv\", \"random\": 1, \"box_bytes\": 8192, \"producers\": %d, \"gb_s\": %.1f}\n",
                  producers, (double)n_blocks * 8192 / ms / 1e6);
    }
  }
  for (int random : {1, 2})
  for (int chunk : {2048, 8192, 16384})
    for (int producers : {1, 2, 4})
      for (int lanes : {1, 4, 8}) {
        const int ring = 192 * 1024;
        const int stages = ring / chunk;
        if (stages % (producers * lanes)) continue;
        CK(cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, ring));
        const uint64_t n = (bytes / 4) / chunk - 1;  // 1 GiB per timing
        const uint64_t region = ((random == 2 ? 32ull : 4096ull) << 20) / chunk - 1;
        const float ms = time_it([&] {
          bulk_stream<<<sms, 32 * (producers + 1), ring>>>(buf, n, chunk, stages, random, producers, region, lanes);
        });
        std::printf("{\"kernel\": \"bulk\", \"random\": %d, \"chunk\": %d, \"producers\": %d, \"lanes\": %d, "
                    "\"gb_s\": %.1f}\n", random, chunk, producers, lanes, (double)n * chunk / ms / 1e6);
      }
  // tensor map over the buffer as [rows, 8192 cols] bf16 (16 KiB rows), boxes 64 cols x R rows
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q));
  const uint64_t cols = 8192, rows = bytes / (cols * 2);
  for (int box_rows : {64, 128})
    for (int ring_kb : {192})
      for (int random : {0, 1}) {
        CUtensorMap map;
        cuuint64_t dims[2] = {cols, rows};
        cuuint64_t strides[1] = {cols * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
        cuuint32_t es[2] = {1, 1};
        if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS) {
          std::fprintf(stderr, "encode failed\n");
          return 1;
        }
        const int bb = box_rows * 128, stages = ring_kb * 1024 / bb;
        if (stages < 2 || stages > 64) continue;
        const int rpcb = (int)(rows / box_rows);
        const uint64_t n = (uint64_t)(cols / 64) * rpcb - 1;
        CK(cudaFuncSetAttribute(tensor_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, ring_kb * 1024 + 1024));
        const float ms = time_it([&] { tensor_stream<<<sms, 64, ring_kb * 1024 + 1024>>>(map, n, box_rows, stages, random, rpcb); });
        std::printf("{\"kernel\": \"tensor2d\", \"random\": %d, \"box_bytes\": %d, \"ring_kb_per_sm\": %d, \"gb_s\": %.1f}\n",
                    random, bb, ring_kb, (double)n * bb / ms / 1e6);
      }
  return 0;
}
