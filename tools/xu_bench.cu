// Pipe-throughput microbenchmark (tools only): warp instructions per cycle per SM for the ops the
// prefill softmax issues -- MUFU.EX2, F2FP (cvt.rn.bf16x2.f32), the exp2 polynomial, FFMA -- with
// 8 independent chains per thread and 1..16 warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/xu_bench tools/xu_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t cvt2(float a, float b) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ float exp2_poly(float x) {
  x = fmaxf(x, -127.f);
  const float t = __fadd_rn(x, 12582912.f);
  const float f = __fsub_rn(x, __fsub_rn(t, 12582912.f));
  const float q = fmaf(fmaf(fmaf(0.05502927f, f, 0.24225698f), f, 0.69325305f), f, 0.99995134f);
  return __int_as_float(__float_as_int(q) + (__float_as_int(t) << 23));
}

template <int OP>
__global__ void bench(float* out, int iters, long long* cycles) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = -0.001f * (threadIdx.x + i);
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) v[i] = ex2(v[i]) - 1.5f;          // MUFU + FADD
      if (OP == 1) acc += cvt2(v[i], v[i] + 1.f), v[i] += 1e-7f;  // F2FP (+ FADD, IADD)
      if (OP == 2) v[i] = exp2_poly(v[i]) - 1.5f;    // poly
      if (OP == 3) v[i] = fmaf(v[i], 0.999f, 1e-3f); // FFMA
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)acc;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const char* names[4] = {"mufu_ex2(+fadd)", "f2fp_bf16x2(+fadd,iadd)", "exp2_poly", "ffma"};
  const int iters = 4096;
  for (int op = 0; op < 4; ++op)
    for (int warps : {1, 2, 4, 8, 16}) {
      auto k = op == 0 ? bench<0> : op == 1 ? bench<1> : op == 2 ? bench<2> : bench<3>;
      k<<<148, warps * 32>>>(out, iters, cyc);
      k<<<148, warps * 32>>>(out, iters, cyc);
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double ops = (double)iters * 8 * warps;  // warp-level op instances per SM
      std::printf("{\"op\": \"%s\", \"warps_per_sm\": %d, \"cycles\": %lld, \"warp_ops_per_clk_per_sm\": %.3f}\n",
                  names[op], warps, c, ops / (double)c);
    }
  return 0;
}
