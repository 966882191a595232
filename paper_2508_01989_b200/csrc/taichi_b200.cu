// libtaichi_b200 -- implementation of include/taichi_b200.h.
//
// One tc_instance = one TaiChi instance = one GPU stream holding a full model
// replica (no tensor parallelism: Llama-3-8B / Qwen2.5-14B fit one B200), a
// page-major paged KV pool and the step workspaces. A hybrid step (the GPU
// form of BatchPlan) is packed as [prefill slice rows | decode rows] and runs:
//   embed -> L x [RMSNorm -> QKV GEMM (+bias) -> RoPE + paged KV append ->
//   chunked-prefill attention | split-KV decode attention -> O GEMM (+resid) ->
//   RMSNorm -> gate_up GEMM (+SwiGLU) -> down GEMM (+resid)] ->
//   RMSNorm on sampled rows only -> LM-head GEMM -> argmax.
#include <cudaTypedefs.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <list>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "attention.cuh"
#include "common.cuh"
#include "elementwise.cuh"
#include "gemm.cuh"
#include "gemm_ws.cuh"
#include "taichi_b200.h"

namespace {

thread_local std::string g_last_error;

struct TcFail {
  tc_status code;
  std::string msg;
};

#define TC_CUDA(x)                                                                                     \
  do {                                                                                                 \
    cudaError_t e_ = (x);                                                                              \
    if (e_ != cudaSuccess)                                                                             \
      throw TcFail{TC_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_) + " @" + std::to_string(__LINE__)}; \
  } while (0)
#define TC_REQUIRE(cond, msg)                       \
  do {                                              \
    if (!(cond)) throw TcFail{TC_ERR_INVALID, msg}; \
  } while (0)

template <typename F>
tc_status guarded(F&& f) {
  try {
    f();
    return TC_OK;
  } catch (const TcFail& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return TC_ERR_INVALID;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// ------------------------------------------------------------------ TMA maps
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw TcFail{TC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable"};
  return fn;
}

// Row-major bf16 [rows, cols] GEMM operand, box = kGemmBK (K) x box_rows, swizzle = row bytes.
CUtensorMap make_kmajor_map(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {(cuuint32_t)tc::kGemmBK, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          tc::kGemmBK == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw TcFail{TC_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r)};
  return m;
}

// fp32 [rows, cols] row-major, box 128 cols x 32 rows, no swizzle: the target of the
// weight-stationary GEMM's TMA bulk residual add (one 32-token x 128-feature chunk per box).
CUtensorMap make_resid_map(void* base, uint64_t rows, uint64_t cols) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 4};
  const cuuint32_t box[2] = {128, 32};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw TcFail{TC_ERR_CUDA, "cuTensorMapEncodeTiled (resid) failed: " + std::to_string((int)r)};
  return m;
}

CUtensorMap encode_map(void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box) {
  CUtensorMap m;
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, base, dims, strides, box, estr,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw TcFail{TC_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r)};
  return m;
}

// Step kernels launch with programmatic stream serialization (PDL): each kernel's prologue
// overlaps its predecessor's tail; the kernels order their memory accesses with
// griddepcontrol.wait (common.cuh pdl_wait). TC_PDL=0 disables it (A/B switch).
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TC_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  TC_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

// ------------------------------------------------------------------ GEMM dispatch
int device_sms(int dev) {
  static std::mutex mu;
  static std::unordered_map<int, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  TC_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  cache[dev] = n;
  return n;
}

template <int BN, int EPI>
void set_gemm_smem() {
  TC_CUDA(cudaFuncSetAttribute(tc::gemm_bf16_tcgen05<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               tc::GemmCfg<BN>::kSmemBytes));
}

void init_kernel_attrs(int dev) {
  static std::mutex mu;
  static std::set<int> done;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(dev)) return;
  DeviceGuard g(dev);
  set_gemm_smem<128, 0>(); set_gemm_smem<128, 1>(); set_gemm_smem<128, 2>(); set_gemm_smem<128, 3>(); set_gemm_smem<128, 4>(); set_gemm_smem<128, 5>();
  set_gemm_smem<256, 0>(); set_gemm_smem<256, 1>(); set_gemm_smem<256, 2>(); set_gemm_smem<256, 3>(); set_gemm_smem<256, 4>(); set_gemm_smem<256, 5>();
  TC_CUDA(cudaFuncSetAttribute(tc::gemm_ws_2sm<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::kWsSmemBytes));
  TC_CUDA(cudaFuncSetAttribute(tc::gemm_ws_2sm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::kWsSmemBytes));
  TC_CUDA(cudaFuncSetAttribute(tc::gemm_ws_2sm<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::kWsSmemBytes));
  TC_CUDA(cudaFuncSetAttribute(tc::gemm_ws_2sm<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::kWsSmemBytes));
  TC_CUDA(cudaFuncSetAttribute(tc::gemm_ws_2sm<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::kWsSmemBytes));
  TC_CUDA(cudaFuncSetAttribute(tc::gemm_ws_2sm<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::kWsSmemBytes));
  // attention kernels: maximum shared-memory carveout (the driver's default split is smaller)
  auto attr = [](const void* fn, int bytes) {
    TC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    TC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared));
  };
  attr((const void*)tc::attn_prefill_tc2<64, 2>, tc::Pf2Cfg<64, 2>::kBytes);
  attr((const void*)tc::attn_prefill_tc2<128, 4>, tc::Pf2Cfg<128, 4>::kBytes);
  attr((const void*)tc::attn_prefill_tc2<128, 5>, tc::Pf2Cfg<128, 5>::kBytes);
  tc::for_each_decode_variant([&](auto k, int bytes) { attr((const void*)k, bytes); });
  done.insert(dev);
}

// Split-K workspace: one fp32 partial tile per unit of split GEMMs + per-tile arrival counters.
constexpr size_t kSkWsBytes = (size_t)96 << 20;
constexpr int kSkMaxTiles = 1 << 15;

struct GemmChoice {
  int bn, m_tiles, n_tiles, kb, splits, grid;
  double est_us;
};

// Tile width / split-K choice, from tools/gemm_bench.py on B200 (profiles/r01/gemm_bench*.json):
//  * M > 128 (mixed / prefill steps): data-parallel 128x256 tiles. Split-K loses at M = 576
//    (down: 98 us unsplit vs 125 us with 3 splits) because the partial round trip and the
//    last-arriver reduction land in the tail of the wave.
//  * M <= 128: 128-wide tiles split 3 ways when fewer than half the SMs would get a tile
//    (qkv 23 -> 21 us, down 66 -> 41 us at M = 64).
GemmChoice choose_gemm(int M, int N, int K, int epi, int sms, int force_bn, int force_splits) {
  GemmChoice c{};
  c.m_tiles = (M + tc::kGemmBM - 1) / tc::kGemmBM;
  c.kb = K / tc::kGemmBK;
  if (force_bn) c.bn = force_bn;
  else if (epi != tc::EPI_RESID_F32 && M <= tc::kGemmBM && (long long)c.m_tiles * (N / 128) < sms / 2) c.bn = 128;
  else c.bn = (N % 256 == 0) ? 256 : 128;
  TC_REQUIRE(N % c.bn == 0, "gemm: N not divisible by tile width");
  c.n_tiles = N / c.bn;
  const long long tiles = (long long)c.m_tiles * c.n_tiles;
  int sp = 1;
  if (force_splits > 0) {
    sp = force_splits;
  } else if (epi == tc::EPI_RESID_F32 && tiles < sms) {
    // red.add split-K: minimise waves * (k-blocks per split + per-unit overhead). The overhead of
    // ~8 k-blocks (pipeline fill + epilogue) reproduces the measured optima (o: 3 splits, 27 us
    // vs 35 unsplit; down: 5 splits, 68 vs 97; M = 64: 9 splits, o 35 -> 13 us, down 99 -> 27 us).
    double best = 1e30;
    for (int cand = 1; cand <= std::min(16, std::max(1, c.kb / 4)); ++cand) {
      const long long waves = (tiles * cand + sms - 1) / sms;
      const double t = (double)waves * ((c.kb + cand - 1) / cand + 8);
      if (t < best - 1e-9) {
        best = t;
        sp = cand;
      }
    }
  } else if (M <= tc::kGemmBM && tiles < sms / 2) {
    sp = (int)std::min<long long>(3, std::max<long long>(1, sms / tiles));
  }
  sp = std::max(1, std::min(sp, c.kb));
  while (epi != tc::EPI_RESID_F32 && sp > 1 && (size_t)tiles * sp * tc::kGemmBM * c.bn * 4 > kSkWsBytes) --sp;
  c.splits = sp;
  c.grid = (int)std::min<long long>(sms, tiles * sp);
  c.est_us = 0;
  return c;
}

template <int BN>
void launch_gemm_bn(const CUtensorMap& ma, const CUtensorMap& mb, const tc::GemmArgs& args, int epi, int grid,
                    cudaStream_t s) {
  const int smem = tc::GemmCfg<BN>::kSmemBytes;
  switch (epi) {
    case tc::EPI_BF16: launch_k(tc::gemm_bf16_tcgen05<BN, tc::EPI_BF16>, grid, tc::kGemmThreads, smem, s, ma, mb, args); break;
    case tc::EPI_BF16_BIAS: launch_k(tc::gemm_bf16_tcgen05<BN, tc::EPI_BF16_BIAS>, grid, tc::kGemmThreads, smem, s, ma, mb, args); break;
    case tc::EPI_RESID_F32: launch_k(tc::gemm_bf16_tcgen05<BN, tc::EPI_RESID_F32>, grid, tc::kGemmThreads, smem, s, ma, mb, args); break;
    case tc::EPI_SWIGLU: launch_k(tc::gemm_bf16_tcgen05<BN, tc::EPI_SWIGLU>, grid, tc::kGemmThreads, smem, s, ma, mb, args); break;
    case tc::EPI_F32: launch_k(tc::gemm_bf16_tcgen05<BN, tc::EPI_F32>, grid, tc::kGemmThreads, smem, s, ma, mb, args); break;
    case tc::EPI_QKV_ROPE: launch_k(tc::gemm_bf16_tcgen05<BN, tc::EPI_QKV_ROPE>, grid, tc::kGemmThreads, smem, s, ma, mb, args); break;
    default: throw TcFail{TC_ERR_INVALID, "unsupported gemm epilogue"};
  }
}

// Weight matrix with TMA maps for each tile width.
struct WMat {
  __nv_bfloat16* ptr = nullptr;
  int64_t rows = 0, cols = 0;
  CUtensorMap map128, map256;
  void make_maps() {
    if (rows % 128 == 0) map128 = make_kmajor_map(ptr, rows, cols, 128);
    if (rows % 256 == 0) map256 = make_kmajor_map(ptr, rows, cols, 256);
  }
  const CUtensorMap& map(int bn) const { return bn == 128 ? map128 : map256; }
};

// Activation operand [rows, cols] of the projections: the 128-row map of the token-major
// kernels plus lazily encoded maps with box heights 16..128 (half token tiles of gemm_ws_2sm).
struct ActMap {
  const void* base = nullptr;
  uint64_t rows = 0, cols = 0;
  CUtensorMap m128;
  std::array<CUtensorMap, 9> by16;
  std::array<bool, 9> have{};
  void init(const void* p, uint64_t r, uint64_t c) {
    base = p;
    rows = r;
    cols = c;
    m128 = make_kmajor_map(p, r, c, 128);
    have.fill(false);
  }
  const CUtensorMap& box(int box_rows) {
    TC_REQUIRE(box_rows % 16 == 0 && box_rows >= 16 && box_rows <= 128, "gemm: bad activation box");
    const int i = box_rows / 16;
    if (!have[i]) {
      by16[i] = make_kmajor_map(base, rows, cols, (uint32_t)box_rows);
      have[i] = true;
    }
    return by16[i];
  }
};

struct SkWorkspace {
  float* ws = nullptr;
  int* cnt = nullptr;
};

// Weight-stationary pair kernel (gemm_ws.cuh) for mixed / prefill steps: T > kWsMinRows rows,
// weight rows a multiple of 256. TC_GEMM_WS=0 in the environment falls back to the token-major
// kernels (A/B switch for measurement).
constexpr int kWsMinRows = 128;
bool ws_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TC_GEMM_WS");
    return !(e && e[0] == '0');
  }();
  return on;
}

void launch_gemm_ws(const CUtensorMap& mw, const CUtensorMap& mx, const CUtensorMap& mo, const tc::GemmArgs& args, int epi,
                    int grid, cudaStream_t s) {
  const int smem = tc::kWsSmemBytes;
  switch (epi) {
    case tc::EPI_BF16: launch_k(tc::gemm_ws_2sm<tc::EPI_BF16>, grid, tc::kWsThreads, smem, s, mw, mx, mo, args); break;
    case tc::EPI_BF16_BIAS: launch_k(tc::gemm_ws_2sm<tc::EPI_BF16_BIAS>, grid, tc::kWsThreads, smem, s, mw, mx, mo, args); break;
    case tc::EPI_RESID_F32: launch_k(tc::gemm_ws_2sm<tc::EPI_RESID_F32>, grid, tc::kWsThreads, smem, s, mw, mx, mo, args); break;
    case tc::EPI_SWIGLU: launch_k(tc::gemm_ws_2sm<tc::EPI_SWIGLU>, grid, tc::kWsThreads, smem, s, mw, mx, mo, args); break;
    case tc::EPI_F32: launch_k(tc::gemm_ws_2sm<tc::EPI_F32>, grid, tc::kWsThreads, smem, s, mw, mx, mo, args); break;
    case tc::EPI_QKV_ROPE: launch_k(tc::gemm_ws_2sm<tc::EPI_QKV_ROPE>, grid, tc::kWsThreads, smem, s, mw, mx, mo, args); break;
    default: throw TcFail{TC_ERR_INVALID, "unsupported gemm epilogue"};
  }
}

// Tiling / split / stream-K plan of a weight-stationary GEMM.
tc::GemmArgs plan_gemm_ws(int M, int N, int K, int epi, int sms, int force_splits) {
  tc::GemmArgs args{};
  // token tiles: the fewest that keep TN <= 256 (each extra tile re-reads the weights)
  const int n_tt = (M + 255) / 256;
  args.tn = ((M + n_tt - 1) / n_tt + 31) / 32 * 32;
  args.stages = tc::ws_stages(args.tn);
  args.M = M;
  args.N = N;
  args.K = K;
  args.m_tiles = n_tt;
  args.n_tiles = N / 256;
  args.kb = K / tc::kGemmBK;
  const long long tiles = (long long)args.m_tiles * args.n_tiles;
  const int pairs = sms / 2;
  // Residual epilogue (O / down): every partial is a TMA
  // bulk add, so the k-blocks are spread by GROUPED stream-K -- pair groups of n_tt siblings (one
  // per token tile) walk the weight-tile-major (tile, k-block) stream in lockstep, group g taking
  // [W g / G, W (g+1) / G) (W = weight tiles * kb), cut at tile boundaries. Every pair gets the same
  // k-blocks whatever the tile count (O at T = 576: 16 weight tiles x 3 token tiles = 48 units on
  // 74 pairs left a third of the pairs idle), and siblings read each weight k-block together, so
  // it leaves DRAM once. TC_WS_STREAMK=0: k-split units instead (A/B).
  static const int streamk_mode = [] {
    const char* e = std::getenv("TC_WS_STREAMK");
    return e ? std::atoi(e) : 1;
  }();
  int sp = 1;
  if (epi == tc::EPI_RESID_F32) {
    if (force_splits > 0) {
      sp = force_splits;
    } else if (tiles < pairs) {
      // k-split units: minimise waves * (k-blocks per split + per-unit overhead of ~8 k-blocks)
      double best = 1e30;
      for (int cand = 1; cand <= std::min(16, std::max(1, args.kb / 4)); ++cand) {
        const long long waves = (tiles * cand + pairs - 1) / pairs;
        const double t = (double)waves * ((args.kb + cand - 1) / cand + 8);
        if (t < best - 1e-9) {
          best = t;
          sp = cand;
        }
      }
    }
  }
  args.splits = std::max(1, std::min(sp, args.kb));
  args.units = (int)(tiles * args.splits);
  args.streamk = (epi == tc::EPI_RESID_F32 && force_splits == 0 && streamk_mode != 0 && n_tt <= pairs) ? 1 : 0;
  if (args.streamk) {
    args.splits = 1;
    args.groups = (int)std::min<long long>(pairs / n_tt, (long long)args.n_tiles * args.kb);
    args.units = args.groups * n_tt;  // pairs launched
  }
  return args;
}

int run_gemm_ws(ActMap& a, const WMat& w, int M, void* out, int ldo, const __nv_bfloat16* bias, int epi, int sms,
                cudaStream_t s, int force_splits, const tc::QkvRopeArgs* rope, const CUtensorMap* out_map) {
  const int N = (int)w.rows;
  TC_REQUIRE(N % 256 == 0, "gemm_ws: weight rows must be a multiple of 256");
  const int pairs = sms / 2;
  static const int env_splits = [] {
    const char* e = std::getenv("TC_WS_SPLITS");
    return e ? std::atoi(e) : 0;
  }();
  if (force_splits == 0 && env_splits > 0) force_splits = env_splits;
  tc::GemmArgs args = plan_gemm_ws(M, N, (int)w.cols, epi, sms, force_splits);
  args.out = out;
  args.ldo = ldo;
  args.bias = bias;
  if (epi == tc::EPI_QKV_ROPE) {
    TC_REQUIRE(rope != nullptr, "gemm: fused QKV epilogue needs RoPE / KV metadata");
    TC_REQUIRE(128 % rope->head_dim == 0, "gemm_ws: a 128-row half tile must cover whole heads");
    args.rope = *rope;
  }
  // Data-parallel units over the fewest pairs that keep the round count (decode-only gate_up:
  // 112 units as 2 rounds of 56 pairs instead of 74 + 38; mixed gate_up: 5 rounds of 68): the
  // weight stream of every round runs on equal SM counts. Measured: decode-only 5.145-5.149 vs
  // 5.168-5.171 ms (three same-box rounds), config 2 61.4-61.8k vs 61.3k, config 5 neutral.
  // TC_WS_BALANCE=0: min(pairs, units) (A/B).
  static const bool balance = [] {
    const char* e = std::getenv("TC_WS_BALANCE");
    return !(e && e[0] == '0');
  }();
  long long used = std::min<long long>(pairs, args.units);
  if (balance && !args.streamk && args.units > pairs) {
    const long long rounds = (args.units + pairs - 1) / pairs;
    used = (args.units + rounds - 1) / rounds;
  }
  const int grid = 2 * (int)used;
  // TC_WS_TRACE=1 (tools only): per-CTA %globaltimer timeline of this launch printed to stderr
  static const bool trace = std::getenv("TC_WS_TRACE") != nullptr;
  unsigned long long* trace_dev = nullptr;
  if (trace) {
    TC_CUDA(cudaMalloc(&trace_dev, (size_t)grid * 16 * 8));
    TC_CUDA(cudaMemsetAsync(trace_dev, 0, (size_t)grid * 16 * 8, s));
    args.trace = trace_dev;
  }
  CUtensorMap resid_map;
  if (epi == tc::EPI_RESID_F32) {
    // the residual's TMA map: the instance's (built once) or, for tc_gemm, one over `out`
    TC_REQUIRE(ldo == N, "gemm_ws: residual output must be dense [M, N]");
    resid_map = out_map ? *out_map : make_resid_map(out, (uint64_t)M, (uint64_t)N);
  }
  launch_gemm_ws(w.map(128), a.box(args.tn / 2), epi == tc::EPI_RESID_F32 ? resid_map : w.map(128), args, epi, grid, s);
  TC_CUDA(cudaGetLastError());
  if (trace) {
    std::vector<unsigned long long> h((size_t)grid * 16);
    TC_CUDA(cudaMemcpyAsync(h.data(), trace_dev, h.size() * 8, cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    cudaFree(trace_dev);
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < grid; ++b)
      if (h[b * 16]) t0 = std::min(t0, h[b * 16]);
    std::fprintf(stderr, "ws_trace M=%d N=%d K=%d epi=%d tn=%d units=%d splits=%d grid=%d (us from first entry: min/med/max)\n",
                 M, N, args.K, epi, args.tn, args.units, args.splits, grid);
    const char* names[14] = {"entry", "prologue", "first_stage", "last_mma", "epi_first", "epi_last", "exit",
                             "epi_start_last", "c0_tmem", "c0_done", "c2_tmem", "c2_done", "c4_tmem", "c4_done"};
    for (int e = 0; e < 14; ++e) {
      std::vector<double> v;
      for (int b = 0; b < grid; ++b)
        if (h[b * 16 + e]) v.push_back((h[b * 16 + e] - t0) / 1e3);
      if (v.empty()) continue;
      std::sort(v.begin(), v.end());
      std::fprintf(stderr, "  %-12s %8.2f %8.2f %8.2f  (n=%zu)\n", names[e], v.front(), v[v.size() / 2], v.back(), v.size());
    }
  }
  return 1;
}

// out = epi(A[M,K] * W[N,K]^T). a: the activation buffer's maps.
int run_gemm(ActMap& a, const WMat& w, int M, void* out, int ldo, const __nv_bfloat16* bias, int epi,
             int sms, const SkWorkspace& sk, cudaStream_t s, int force_bn = 0, int force_splits = 0,
             const tc::QkvRopeArgs* rope = nullptr, const CUtensorMap* out_map = nullptr) {
  const int N = (int)w.rows, K = (int)w.cols;
  TC_REQUIRE(K % 64 == 0, "gemm: K must be a multiple of 64");
  TC_REQUIRE(N % 128 == 0, "gemm: N must be a multiple of 128");
  TC_REQUIRE(force_bn == 0 || force_bn == 128 || force_bn == 256 || force_bn == 1024,
             "gemm: tile width must be 128, 256 or 1024 (= weight-stationary pair)");
  static const bool ws_small = [] {
    const char* e = std::getenv("TC_WS_SMALL");
    return !(e && e[0] == '0');
  }();
  if (N % 256 == 0 &&
      (force_bn == 1024 || (force_bn == 0 && ws_enabled() && epi != tc::EPI_F32 && (M > kWsMinRows || ws_small)))) {
    return run_gemm_ws(a, w, M, out, ldo, bias, epi, sms, s, force_splits, rope, out_map);
  }
  const CUtensorMap& a_map = a.m128;
  const GemmChoice c = choose_gemm(M, N, K, epi, sms, force_bn, force_splits);
  TC_REQUIRE((long long)c.m_tiles * c.n_tiles <= kSkMaxTiles, "gemm: too many tiles");
  tc::GemmArgs args{};
  args.M = M;
  args.N = N;
  args.K = K;
  args.m_tiles = c.m_tiles;
  args.n_tiles = c.n_tiles;
  args.kb = c.kb;
  args.splits = c.splits;
  args.units = c.m_tiles * c.n_tiles * c.splits;
  args.out = out;
  args.ldo = ldo;
  args.bias = bias;
  args.ws = sk.ws;
  args.tile_cnt = sk.cnt;
  if (epi == tc::EPI_QKV_ROPE) {
    TC_REQUIRE(rope != nullptr, "gemm: fused QKV epilogue needs RoPE / KV metadata");
    TC_REQUIRE(c.bn % rope->head_dim == 0, "gemm: tile width must cover whole heads");
    args.rope = *rope;
  }
  if (c.bn == 128) launch_gemm_bn<128>(a_map, w.map(128), args, epi, c.grid, s);
  else launch_gemm_bn<256>(a_map, w.map(256), args, epi, c.grid, s);
  TC_CUDA(cudaGetLastError());
  return 1;
}

// ------------------------------------------------------------------ instance
struct LayerW {
  WMat qkv, o, gate_up, down;
  __nv_bfloat16 *qkv_bias = nullptr, *attn_norm = nullptr, *mlp_norm = nullptr;
};

constexpr int kMaxDecodeItems = 16384;

constexpr uint64_t kTidEmbed = 1, kTidLmHead = 2, kTidFinalNorm = 3;
inline uint64_t tid_layer(int l, int j) { return 16 + 16ull * l + j; }
constexpr float kLinScale = 0.034641016f;  // uniform(-a, a) with std 0.02
constexpr float kBiasScale = 0.1f;
constexpr float kNormScale = 0.1f;

struct PhaseTimer {
  bool on = false;
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  cudaEvent_t get() {
    if (used == pool.size()) {
      cudaEvent_t e;
      TC_CUDA(cudaEventCreate(&e));
      pool.push_back(e);
    }
    return pool[used++];
  }
  void reset() {
    marks.clear();
    used = 0;
  }
};

// ------------------------------------------------------------------ KV pool
// A CUDA event shared by everyone who must order against it (a migration's copy-done event is
// referenced by its tc_event, by the destination's inbound list and by the source pool's quarantine).
struct SharedEvent {
  cudaEvent_t e = nullptr;
  int device = 0;
  SharedEvent(int dev, bool timing) : device(dev) {
    DeviceGuard g(dev);
    TC_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  }
  ~SharedEvent() {
    DeviceGuard g(device);
    if (e) cudaEventDestroy(e);
  }
  bool done() const { return cudaEventQuery(e) == cudaSuccess; }
};
using EvPtr = std::shared_ptr<SharedEvent>;

// Page-major KV pool of one GPU. Several instances on one GPU may share it (tc_instance_desc.
// share_kv_pool): one allocator, so co-located instances draw on the whole HBM budget instead of
// fixed per-instance slices. Pages an in-flight copy still reads (the source side of a migration)
// or writes (the destination of a migration whose request is released early) sit in quarantine
// until that copy's event completes; allocation reclaims them, blocking on the oldest only when the
// free list alone cannot serve the request.
struct KvPool {
  int device = 0;
  __nv_bfloat16* kv = nullptr;
  int64_t page_elems = 0, n_pages = 0;
  std::mutex mu;
  std::vector<int32_t> free_pages;
  struct Held {
    EvPtr ev;
    std::vector<int32_t> pages;
  };
  std::deque<Held> quarantine;
  int64_t quarantined = 0;
  ~KvPool() {
    DeviceGuard g(device);
    if (kv) cudaFree(kv);
  }
  // caller holds mu
  void reclaim(bool block_until, int64_t want) {
    while (!quarantine.empty()) {
      Held& h = quarantine.front();
      if (!h.ev->done()) {
        if (!block_until || (int64_t)free_pages.size() >= want) break;
        DeviceGuard g(device);
        TC_CUDA(cudaEventSynchronize(h.ev->e));
      }
      for (auto p = h.pages.rbegin(); p != h.pages.rend(); ++p) free_pages.push_back(*p);
      quarantined -= (int64_t)h.pages.size();
      quarantine.pop_front();
    }
  }
  void take(std::vector<int32_t>& t, int64_t need, int64_t req) {
    std::lock_guard<std::mutex> lk(mu);
    const int64_t more = need - (int64_t)t.size();
    if ((int64_t)free_pages.size() < more) reclaim(false, more);
    if ((int64_t)free_pages.size() < more) reclaim(true, more);
    if ((int64_t)free_pages.size() < more)
      throw TcFail{TC_ERR_OOM, "KV pool exhausted (req " + std::to_string(req) + ", need " + std::to_string(more) +
                                   " more pages, free " + std::to_string(free_pages.size()) + " of " +
                                   std::to_string(n_pages) + ")"};
    while ((int64_t)t.size() < need) {
      t.push_back(free_pages.back());
      free_pages.pop_back();
    }
  }
  void give(std::vector<int32_t>&& pages, const EvPtr& busy_until) {
    std::lock_guard<std::mutex> lk(mu);
    if (busy_until && !busy_until->done()) {
      quarantined += (int64_t)pages.size();
      quarantine.push_back(Held{busy_until, std::move(pages)});
      return;
    }
    for (auto p = pages.rbegin(); p != pages.rend(); ++p) free_pages.push_back(*p);
  }
  int64_t free_count() {
    std::lock_guard<std::mutex> lk(mu);
    reclaim(false, 0);
    return (int64_t)free_pages.size();
  }
};

}  // namespace

// Launch shape of a step: everything its kernel launches depend on besides the metadata contents.
struct GraphKey {
  int T, n_seq, n_qblk, n_logit, n_bt, n_seg, max_entries, dec_grid, pf_sms, meta_ints;
  bool operator==(const GraphKey& o) const { return std::memcmp(this, &o, sizeof(GraphKey)) == 0; }
};

// Instantiated step graphs by launch shape (LRU), plus the shapes seen once: a shape is captured
// on its second occurrence, so one-off shapes never pay for instantiation.
struct GraphCache {
  struct Entry {
    GraphKey key;
    cudaGraphExec_t exec;
    int launches;
  };
  static constexpr size_t kCap = 24, kSeenCap = 256;
  std::list<Entry> lru;
  std::deque<GraphKey> seen_once;
  const Entry* find(const GraphKey& k) {
    for (auto it = lru.begin(); it != lru.end(); ++it)
      if (it->key == k) {
        lru.splice(lru.begin(), lru, it);
        return &lru.front();
      }
    return nullptr;
  }
  bool seen(const GraphKey& k) {
    for (const GraphKey& x : seen_once)
      if (x == k) return true;
    seen_once.push_back(k);
    if (seen_once.size() > kSeenCap) seen_once.pop_front();
    return false;
  }
  void put(const GraphKey& k, cudaGraphExec_t ex, int launches) {
    lru.push_front(Entry{k, ex, launches});
    if (lru.size() > kCap) {
      cudaGraphExecDestroy(lru.back().exec);
      lru.pop_back();
    }
  }
  void clear() {
    for (Entry& e : lru) cudaGraphExecDestroy(e.exec);
    lru.clear();
  }
};

bool graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TC_GRAPH");
    return !(e && e[0] == '0') && std::getenv("TC_WS_TRACE") == nullptr && std::getenv("TC_PF_TRACE") == nullptr;
  }();
  return on;
}

// An asynchronous KV migration (tc_kv_migrate_async): copy-done event + timing.
struct tc_event {
  EvPtr done;                       // copy finished (destination pages valid, source pages reusable)
  cudaEvent_t t0 = nullptr;         // copy start on the migration stream (timing)
  int device = 0;
  int64_t bytes = 0, pages = 0;
  int32_t peer = 0;                 // 1 if source and destination are on different GPUs
};

// Another process's KV pool mapped into this one (CUDA IPC).
struct tc_remote_pool {
  int device = 0;        // device the mapping was opened on (the importer's)
  void* base = nullptr;  // peer (or same-GPU) pointer to the exporter's pool
  int64_t page_bytes = 0, n_pages = 0;
};

struct tc_instance {
  tc_instance_desc desc{};
  tc_model_dims d{};
  int sms = 0;
  cudaStream_t stream = nullptr;
  // weights (shared_ptr: instances on one GPU may share one replica)
  std::shared_ptr<void> weight_owner;
  __nv_bfloat16 *embed = nullptr, *final_norm = nullptr;
  WMat lm_head;
  std::vector<LayerW> layers;
  // KV pool (possibly shared with other instances on this GPU) and this instance's page tables
  std::shared_ptr<KvPool> pool;
  __nv_bfloat16* kv = nullptr;  // == pool->kv
  int64_t page_elems = 0, n_pages = 0;
  CUtensorMap kv_map;  // 3-D view {64 dims, pool rows, head_dim/64 halves}; box = one (K, V) page pair
  CUtensorMap kv2_map;  // 2-D view {head_dim, pool rows}; box = one 64-dim half of one K or V block
  CUtensorMap q_map;    // 3-D view of the q heads of the qkv buffer {head_dim, q heads, rows}
  std::unordered_map<int64_t, std::vector<int32_t>> tables;
  // requests whose pages here are still being written by an inbound migration copy: steps,
  // outbound copies and releases of the request order after the event
  std::unordered_map<int64_t, EvPtr> inbound;
  // activations
  int qkv_n = 0;
  float* resid = nullptr;
  __nv_bfloat16 *xnorm = nullptr, *qkv = nullptr, *attn_out = nullptr, *act = nullptr, *lm_in = nullptr;
  float* logits = nullptr;
  int* ids_dev = nullptr;
  int* ids_host = nullptr;
  ActMap map_xnorm, map_attn, map_act, map_lm_in;
  CUtensorMap map_resid;  // fp32 residual stream, target of the GEMMs' TMA bulk adds
  SkWorkspace sk;
  float *attn_ws_o = nullptr, *attn_ws_ml = nullptr;
  int* attn_cnt = nullptr;
  size_t attn_ws_floats = 0;
  float2* rope = nullptr;
  // per-step metadata
  int32_t* meta_host = nullptr;
  int32_t* meta_dev = nullptr;
  size_t meta_ints = 0;
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
  // concurrent attention: prefill attention runs on stream_pf beside decode attention, on the
  // SMs the (narrowed) decode grid leaves free
  cudaStream_t stream_pf = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int pf_sms = 0;  // SMs left to prefill attention in this step (0 = serial)
  bool step_pending = false;
  int last_sampled = 0;
  int launches = 0;       // kernels launched by the last step
  int64_t h2d_bytes = 0;  // bytes copied H2D by the last step

  // migration: one high-priority copy stream per destination (copies to different destinations
  // overlap each other and this instance's steps); tail = this instance's step stream position a
  // copy must follow (a step in flight may still write the request's newest row)
  std::unordered_map<const void*, cudaStream_t> mig_streams;  // key: destination instance / remote pool
  cudaEvent_t mig_tail = nullptr;
  tc_event* last_mig = nullptr;  // tc_kv_migrate / tc_kv_migrate_wait (synchronous form)
  int mig_ctas = 0;              // copy kernel grid (0 = 2 x SMs)
  PhaseTimer prof;
  GraphCache graphs;
};

namespace {

tc_model_dims preset(const std::string& full) {
  std::string name = full;
  int layers_override = -1;
  auto colon = full.find(":L");
  if (colon != std::string::npos) {
    name = full.substr(0, colon);
    layers_override = std::stoi(full.substr(colon + 2));
  }
  tc_model_dims m{};
  if (name == "tiny") {
    m = {2, 256, 4, 2, 64, 512, 1024, 0, 1.0e4f, 1e-5f};
  } else if (name == "llama3_8b") {
    m = {32, 4096, 32, 8, 128, 14336, 128256, 0, 5.0e5f, 1e-5f};
  } else if (name == "qwen2_5_14b") {
    m = {48, 5120, 40, 8, 128, 13824, 152064, 1, 1.0e6f, 1e-6f};
  } else {
    throw TcFail{TC_ERR_INVALID, "unknown model preset " + name};
  }
  if (layers_override > 0) m.n_layers = layers_override;
  return m;
}

void check_dims(const tc_model_dims& m) {
  TC_REQUIRE(m.n_layers >= 1 && m.d_model >= 64, "dims: bad sizes");
  TC_REQUIRE(m.head_dim == 64 || m.head_dim == 128, "dims: head_dim must be 64 or 128");
  TC_REQUIRE(m.n_heads % m.n_kv_heads == 0, "dims: n_heads % n_kv_heads");
  const int g = m.n_heads / m.n_kv_heads;
  TC_REQUIRE((m.head_dim == 64 && g == 2) || (m.head_dim == 128 && (g == 4 || g == 5)),
             "dims: supported (head_dim, group) = (64,2), (128,4), (128,5)");
  TC_REQUIRE(m.d_model % 128 == 0 && m.ffn_dim % 64 == 0 && m.vocab % 128 == 0, "dims: alignment");
}

void init_tensor(__nv_bfloat16* p, int64_t rows, int64_t cols, uint64_t seed, uint64_t tid, float scale, float offset,
                 int interleave, cudaStream_t s) {
  const int64_t n = rows * cols;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 65536);
  tc::init_weights<<<blocks, 256, 0, s>>>(p, rows, cols, seed, tid, scale, offset, interleave);
  TC_CUDA(cudaGetLastError());
}

void* carve(uint8_t*& cur, size_t bytes) {
  void* p = cur;
  cur += (bytes + 255) & ~size_t(255);
  return p;
}

void alloc_weights(tc_instance* I) {
  const tc_model_dims& m = I->d;
  const int64_t dm = m.d_model, H = m.n_heads, Hk = m.n_kv_heads, dh = m.head_dim, F = m.ffn_dim, V = m.vocab;
  I->qkv_n = (int)((H + 2 * Hk) * dh);
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  size_t per_layer = al(I->qkv_n * dm * 2) + al(dm * H * dh * 2) + al(2 * F * dm * 2) + al(dm * F * 2) +
                     al(I->qkv_n * 2) + 2 * al(dm * 2);
  size_t total = 2 * al(V * dm * 2) + al(dm * 2) + per_layer * m.n_layers;
  void* block = nullptr;
  TC_CUDA(cudaMalloc(&block, total));
  const int dev = I->desc.device;
  I->weight_owner = std::shared_ptr<void>(block, [dev](void* p) {
    DeviceGuard g(dev);
    cudaFree(p);
  });
  uint8_t* cur = static_cast<uint8_t*>(block);
  cudaStream_t s = I->stream;
  const uint64_t seed = I->desc.weight_seed;
  I->embed = (__nv_bfloat16*)carve(cur, V * dm * 2);
  init_tensor(I->embed, V, dm, seed, kTidEmbed, 1.0f, 0.f, 0, s);
  I->lm_head.ptr = (__nv_bfloat16*)carve(cur, V * dm * 2);
  I->lm_head.rows = V;
  I->lm_head.cols = dm;
  init_tensor(I->lm_head.ptr, V, dm, seed, kTidLmHead, kLinScale, 0.f, 0, s);
  I->final_norm = (__nv_bfloat16*)carve(cur, dm * 2);
  init_tensor(I->final_norm, 1, dm, seed, kTidFinalNorm, kNormScale, 1.f, 0, s);
  I->layers.resize(m.n_layers);
  for (int l = 0; l < m.n_layers; ++l) {
    LayerW& L = I->layers[l];
    L.qkv = {(__nv_bfloat16*)carve(cur, I->qkv_n * dm * 2), I->qkv_n, dm};
    init_tensor(L.qkv.ptr, I->qkv_n, dm, seed, tid_layer(l, 0), kLinScale, 0.f, 0, s);
    L.o = {(__nv_bfloat16*)carve(cur, dm * H * dh * 2), dm, H * dh};
    init_tensor(L.o.ptr, dm, H * dh, seed, tid_layer(l, 1), kLinScale, 0.f, 0, s);
    L.gate_up = {(__nv_bfloat16*)carve(cur, 2 * F * dm * 2), 2 * F, dm};
    init_tensor(L.gate_up.ptr, 2 * F, dm, seed, tid_layer(l, 2), kLinScale, 0.f, 1, s);
    L.down = {(__nv_bfloat16*)carve(cur, dm * F * 2), dm, F};
    init_tensor(L.down.ptr, dm, F, seed, tid_layer(l, 4), kLinScale, 0.f, 0, s);
    L.qkv_bias = (__nv_bfloat16*)carve(cur, I->qkv_n * 2);
    init_tensor(L.qkv_bias, 1, I->qkv_n, seed, tid_layer(l, 7), m.qkv_bias ? kBiasScale : 0.f, 0.f, 0, s);
    L.attn_norm = (__nv_bfloat16*)carve(cur, dm * 2);
    init_tensor(L.attn_norm, 1, dm, seed, tid_layer(l, 5), kNormScale, 1.f, 0, s);
    L.mlp_norm = (__nv_bfloat16*)carve(cur, dm * 2);
    init_tensor(L.mlp_norm, 1, dm, seed, tid_layer(l, 6), kNormScale, 1.f, 0, s);
    L.qkv.make_maps();
    L.o.make_maps();
    L.gate_up.make_maps();
    L.down.make_maps();
  }
  I->lm_head.make_maps();
}

void alloc_buffers(tc_instance* I) {
  const tc_model_dims& m = I->d;
  const int T = I->desc.max_step_tokens, S = I->desc.max_seqs;
  const int64_t dm = m.d_model;
  // round row counts up to the GEMM M tile so TMA boxes never leave the buffer
  const int Tp = (T + 127) / 128 * 128, Sp = (S + 127) / 128 * 128;
  TC_CUDA(cudaMalloc(&I->resid, (size_t)Tp * dm * 4));
  TC_CUDA(cudaMalloc(&I->xnorm, (size_t)Tp * dm * 2));
  TC_CUDA(cudaMalloc(&I->qkv, (size_t)Tp * I->qkv_n * 2));
  TC_CUDA(cudaMalloc(&I->attn_out, (size_t)Tp * m.n_heads * m.head_dim * 2));
  TC_CUDA(cudaMalloc(&I->act, (size_t)Tp * m.ffn_dim * 2));
  TC_CUDA(cudaMalloc(&I->lm_in, (size_t)Sp * dm * 2));
  TC_CUDA(cudaMalloc(&I->logits, (size_t)S * m.vocab * 4));
  TC_CUDA(cudaMalloc(&I->ids_dev, (size_t)S * 4));
  TC_CUDA(cudaMallocHost(&I->ids_host, (size_t)S * 4));
  TC_CUDA(cudaMemset(I->xnorm, 0, (size_t)Tp * dm * 2));
  TC_CUDA(cudaMemset(I->attn_out, 0, (size_t)Tp * m.n_heads * m.head_dim * 2));
  TC_CUDA(cudaMemset(I->act, 0, (size_t)Tp * m.ffn_dim * 2));
  TC_CUDA(cudaMemset(I->lm_in, 0, (size_t)Sp * dm * 2));
  I->map_xnorm.init(I->xnorm, Tp, dm);
  I->map_resid = make_resid_map(I->resid, Tp, dm);
  I->map_attn.init(I->attn_out, Tp, (uint64_t)m.n_heads * m.head_dim);
  I->map_act.init(I->act, Tp, m.ffn_dim);
  I->map_lm_in.init(I->lm_in, Sp, dm);
  {
    const int G = m.n_heads / m.n_kv_heads;
    const cuuint64_t dims[3] = {(cuuint64_t)m.head_dim, (cuuint64_t)m.n_heads, (cuuint64_t)Tp};
    const cuuint64_t strides[2] = {(cuuint64_t)m.head_dim * 2, (cuuint64_t)I->qkv_n * 2};
    const cuuint32_t box[3] = {64, (cuuint32_t)G, (cuuint32_t)(128 / G)};
    I->q_map = encode_map(I->qkv, 3, dims, strides, box);
  }
  // stream-K partial slots + tile counters (counters must start at zero)
  TC_CUDA(cudaMalloc(&I->sk.ws, kSkWsBytes));
  TC_CUDA(cudaMalloc(&I->sk.cnt, (size_t)kSkMaxTiles * 4));
  TC_CUDA(cudaMemset(I->sk.cnt, 0, (size_t)kSkMaxTiles * 4));
  // decode split-KV partials (one slot per work item)
  const int G = m.n_heads / m.n_kv_heads;
  I->attn_ws_floats = (size_t)kMaxDecodeItems * G * m.head_dim;
  TC_CUDA(cudaMalloc(&I->attn_ws_o, I->attn_ws_floats * 4));
  TC_CUDA(cudaMalloc(&I->attn_ws_ml, (size_t)kMaxDecodeItems * G * 2 * 4));
  TC_CUDA(cudaMalloc(&I->attn_cnt, (size_t)S * m.n_kv_heads * 4));
  TC_CUDA(cudaMemset(I->attn_cnt, 0, (size_t)S * m.n_kv_heads * 4));
  // RoPE table in fp64 -> fp32
  const int half = m.head_dim / 2;
  std::vector<float2> cs((size_t)I->desc.max_context * half);
  for (int pos = 0; pos < I->desc.max_context; ++pos)
    for (int j = 0; j < half; ++j) {
      const double inv = std::pow((double)m.rope_theta, -2.0 * j / (double)m.head_dim);
      const double a = (double)pos * inv;
      cs[(size_t)pos * half + j] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
  TC_CUDA(cudaMalloc(&I->rope, cs.size() * sizeof(float2)));
  TC_CUDA(cudaMemcpy(I->rope, cs.data(), cs.size() * sizeof(float2), cudaMemcpyHostToDevice));
  // metadata: 4T + 4S + qblocks(<= T + S) * 2 + S (dec) + S (logit rows) + block tables
  const int64_t max_pages_per_seq = (I->desc.max_context + I->desc.page_size - 1) / I->desc.page_size;
  I->meta_ints = 4 * (size_t)T + 4 * (size_t)S + 2 * (size_t)(T + S) + 4 * (size_t)S +
                 12 * (size_t)S * m.n_kv_heads + 4 * 1024 + 1024 + (size_t)S * max_pages_per_seq + 128;
  TC_CUDA(cudaMallocHost(&I->meta_host, I->meta_ints * 4));
  TC_CUDA(cudaMalloc(&I->meta_dev, I->meta_ints * 4));
  TC_CUDA(cudaEventCreate(&I->ev_start));
  TC_CUDA(cudaEventCreateWithFlags(&I->ev_fork, cudaEventDisableTiming));
  TC_CUDA(cudaEventCreateWithFlags(&I->ev_join, cudaEventDisableTiming));
  TC_CUDA(cudaEventCreate(&I->ev_stop));
  TC_CUDA(cudaEventCreateWithFlags(&I->mig_tail, cudaEventDisableTiming));
}

void ensure_pages(tc_instance* I, int64_t req, int64_t n_tokens) {
  const int ps = I->desc.page_size;
  const int64_t need = (n_tokens + ps - 1) / ps;
  std::vector<int32_t>& t = I->tables[req];
  if ((int64_t)t.size() >= need) return;
  I->pool->take(t, need, req);
}

// Inbound copy of req still running? (drops the entry once its event completed)
EvPtr inbound_pending(tc_instance* I, int64_t req) {
  auto it = I->inbound.find(req);
  if (it == I->inbound.end()) return nullptr;
  if (it->second->done()) {
    I->inbound.erase(it);
    return nullptr;
  }
  return it->second;
}

// busy_until: the pages stay quarantined until this event (an outbound copy still reading them)
void release_pages(tc_instance* I, int64_t req, EvPtr busy_until = nullptr) {
  auto it = I->tables.find(req);
  if (it == I->tables.end()) return;
  if (!busy_until) busy_until = inbound_pending(I, req);  // an inbound copy may still write them
  I->inbound.erase(req);
  I->pool->give(std::move(it->second), busy_until);
  I->tables.erase(it);
}

struct ProfScope {
  tc_instance* I;
  cudaEvent_t b = nullptr;
  const char* name;
  ProfScope(tc_instance* inst, const char* n) : I(inst), name(n) {
    if (I->prof.on) {
      b = I->prof.get();
      cudaEventRecord(b, I->stream);
    }
  }
  ~ProfScope() {
    if (I->prof.on) {
      cudaEvent_t e = I->prof.get();
      cudaEventRecord(e, I->stream);
      I->prof.marks.push_back({name, {b, e}});
    }
  }
};

// decode attention variant (A/B): TC_DEC_CFG="<consumer warps>:<producer warps>" (default 4:4;
// tc::for_each_decode_variant_of lists the compiled ones); TC_DEC_GRID caps the grid
std::pair<int, int> dec_cfg() {
  static const std::pair<int, int> c = [] {
    int nc = 4, np = 4;
    if (const char* e = std::getenv("TC_DEC_CFG")) std::sscanf(e, "%d:%d", &nc, &np);
    return std::make_pair(nc, np);
  }();
  return c;
}

template <int DH, int G>
void launch_decode(tc_instance* I, const tc::AttnParams& p, int dec_grid) {
  const auto c = dec_cfg();
  bool done = false;
  tc::for_each_decode_variant_of<DH, G>([&](auto kern, int smem, int nc, int np) {
    if (done || nc != c.first || np != c.second) return;
    launch_k(kern, dec_grid, tc::dec_threads(nc, np), smem, I->stream, I->kv_map, p);
    done = true;
  });
  TC_REQUIRE(done, "decode attention: TC_DEC_CFG names a variant that is not compiled");
}

template <int DH, int G>
void launch_prefill(tc_instance* I, const tc::AttnParams& p, int n_qblk, cudaStream_t s) {
  const dim3 grid(I->d.n_kv_heads, n_qblk);
  static const bool trace = std::getenv("TC_PF_TRACE") != nullptr;
  if (trace) {  // tools only: %globaltimer timeline of CTA (0, 1), printed to stderr
    tc::AttnParams q = p;
    TC_CUDA(cudaMalloc(&q.pf_trace, 64 * 16 * 8));
    TC_CUDA(cudaMemsetAsync(q.pf_trace, 0, 64 * 16 * 8, s));
    launch_k(tc::attn_prefill_tc2<DH, G>, grid, tc::kPfThreads, tc::Pf2Cfg<DH, G>::kBytes, s, I->kv2_map, I->q_map, q);
    std::vector<unsigned long long> h(64 * 16);
    TC_CUDA(cudaMemcpyAsync(h.data(), q.pf_trace, h.size() * 8, cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    cudaFree(q.pf_trace);
    const unsigned long long t0 = h[8];
    std::fprintf(stderr, "pf_trace (ns): key tile j | P written by softmax warps 0-7 | S seen by warps 0-7\n");
    for (int j = 0; j < 64; ++j) {
      if (!h[j * 16 + 8]) break;
      std::fprintf(stderr, "pf_trace %3d", j);
      for (int k = 0; k < 16; ++k) std::fprintf(stderr, " %6lld", h[j * 16 + k] ? (long long)(h[j * 16 + k] - t0) : -1ll);
      std::fprintf(stderr, "\n");
    }
    return;
  }
  launch_k(tc::attn_prefill_tc2<DH, G>, grid, tc::kPfThreads, tc::Pf2Cfg<DH, G>::kBytes, s, I->kv2_map, I->q_map, p);
}

template <int DH, int G>
void launch_attention(tc_instance* I, const tc::AttnParams& p, int n_qblk, int n_dec, int dec_grid) {
  if (n_qblk > 0 && n_dec > 0 && I->pf_sms > 0) {
    // decode on the main stream over sms - pf_sms CTAs (launched first, so its persistent CTAs
    // take their SMs), prefill beside it on stream_pf over whatever SMs remain; join before O
    TC_CUDA(cudaEventRecord(I->ev_fork, I->stream));
    launch_decode<DH, G>(I, p, dec_grid);
    TC_CUDA(cudaStreamWaitEvent(I->stream_pf, I->ev_fork, 0));
    launch_prefill<DH, G>(I, p, n_qblk, I->stream_pf);
    TC_CUDA(cudaEventRecord(I->ev_join, I->stream_pf));
    TC_CUDA(cudaStreamWaitEvent(I->stream, I->ev_join, 0));
    I->launches += 2;
    TC_CUDA(cudaGetLastError());
    return;
  }
  if (n_qblk > 0) {
    launch_prefill<DH, G>(I, p, n_qblk, I->stream);
    ++I->launches;
  }
  if (n_dec > 0) {
    launch_decode<DH, G>(I, p, dec_grid);
    ++I->launches;
  }
  TC_CUDA(cudaGetLastError());
}

void dispatch_attention(tc_instance* I, const tc::AttnParams& p, int n_qblk, int n_dec, int dec_grid) {
  const int G = I->d.n_heads / I->d.n_kv_heads;
  if (I->d.head_dim == 64 && G == 2) launch_attention<64, 2>(I, p, n_qblk, n_dec, dec_grid);
  else if (I->d.head_dim == 128 && G == 4) launch_attention<128, 4>(I, p, n_qblk, n_dec, dec_grid);
  else if (I->d.head_dim == 128 && G == 5) launch_attention<128, 5>(I, p, n_qblk, n_dec, dec_grid);
  else throw TcFail{TC_ERR_INVALID, "unsupported attention shape"};
}

void step_launch(tc_instance* I, const tc_step_desc* st) {
  TC_REQUIRE(st != nullptr, "step: null descriptor");
  TC_REQUIRE(!I->step_pending, "step: previous step not waited");
  const tc_model_dims& m = I->d;
  const int ps = I->desc.page_size;
  const int n_pf = st->n_prefill, n_dec = st->n_decode;
  TC_REQUIRE(n_pf >= 0 && n_dec >= 0 && n_pf + n_dec > 0, "step: empty step");
  const int n_seq = n_pf + n_dec;
  TC_REQUIRE(n_seq <= I->desc.max_seqs, "step: too many sequences");
  int T = n_dec;
  for (int i = 0; i < n_pf; ++i) {
    TC_REQUIRE(st->prefill[i].n_tokens >= 1 && st->prefill[i].pos0 >= 0, "step: bad prefill slice");
    TC_REQUIRE(st->prefill[i].pos0 + st->prefill[i].n_tokens <= I->desc.max_context, "step: slice beyond max_context");
    T += st->prefill[i].n_tokens;
  }
  TC_REQUIRE(T <= I->desc.max_step_tokens, "step: too many tokens");
  for (int i = 0; i < n_dec; ++i) {
    TC_REQUIRE(st->decode[i].pos >= 0 && st->decode[i].pos < I->desc.max_context, "step: bad decode position");
    TC_REQUIRE(st->decode[i].token_id >= 0 && st->decode[i].token_id < m.vocab, "step: token id out of range");
  }
  // every argument is checked before any page is allocated (a rejected step changes nothing)
  for (int i = 0; i < n_pf; ++i) {
    TC_REQUIRE(st->prefill[i].token_ids != nullptr, "step: null token ids");
    for (int k = 0; k < st->prefill[i].n_tokens; ++k)
      TC_REQUIRE(st->prefill[i].token_ids[k] >= 0 && st->prefill[i].token_ids[k] < m.vocab, "step: token id out of range");
  }
  // physical pages for every new position
  for (int i = 0; i < n_pf; ++i) ensure_pages(I, st->prefill[i].req_id, st->prefill[i].pos0 + st->prefill[i].n_tokens);
  for (int i = 0; i < n_dec; ++i) ensure_pages(I, st->decode[i].req_id, st->decode[i].pos + 1);
  // requests whose KV is still arriving from another instance: the step orders after the copy
  std::vector<EvPtr> waits;
  for (int i = 0; i < n_pf; ++i)
    if (EvPtr e = inbound_pending(I, st->prefill[i].req_id)) waits.push_back(e);
  for (int i = 0; i < n_dec; ++i)
    if (EvPtr e = inbound_pending(I, st->decode[i].req_id)) waits.push_back(e);

  const int G = m.n_heads / m.n_kv_heads;
  const int tpc = 2 * (128 / G);  // prefill tokens per attention CTA (two 128-row q tiles)
  int n_qblk = 0, n_logit = 0, n_bt = 0;
  for (int i = 0; i < n_pf; ++i) {
    n_qblk += (st->prefill[i].n_tokens + tpc - 1) / tpc;
    n_logit += st->prefill[i].want_logits ? 1 : 0;
    n_bt += (st->prefill[i].pos0 + st->prefill[i].n_tokens + ps - 1) / ps;
  }
  n_logit += n_dec;
  for (int i = 0; i < n_dec; ++i) n_bt += st->decode[i].pos / ps + 1;
  // decode work (attn_decode): segments (decode j, kv head h) = seg j * Hk + h, laid end to end
  // as one stream of page-heads; CTA c takes pages [W*c/NC, W*(c+1)/NC).
  const int n_seg = n_dec * m.n_kv_heads;
  long long W = 0;
  for (int i = 0; i < n_dec; ++i) W += (long long)(st->decode[i].pos / ps + 1) * m.n_kv_heads;
  // Mixed steps run prefill attention beside decode attention (pf_sms SMs left to prefill; the
  // prefill CTAs spill onto every SM once the persistent decode CTAs finish). Model: decode moves
  // its K/V at ~50 GB/s per SM up to ~5.6 TB/s; prefill costs ~3 us per 128-key tile + 8 us per CTA;
  // step attention time(P) = T_dec(sms - P) + max(0, W_pf - P * T_dec) / sms. The curve is flat
  // near its minimum; take the smallest P within 0.5% of it, plus 4 (measured optima, round 2:
  // Llama-3-8B P=512 over 512 + 64 decodes @1k: 32-48; Qwen2.5-14B 1024 over 4096 + 32 @8k: 24-56, flat).
  // TC_PF_SMS overrides (0 = serial).
  I->pf_sms = 0;
  if (n_dec > 0 && n_qblk > 0) {
    long long pf_tiles = 0;
    for (int i = 0; i < n_pf; ++i) {
      const tc_prefill_slice& sl = st->prefill[i];
      for (int q = 0; q < sl.n_tokens; q += tpc) pf_tiles += (sl.pos0 + std::min(q + tpc, sl.n_tokens) + 127) / 128;
    }
    pf_tiles *= m.n_kv_heads;
    // CTA-us: ~3 us per 128-key tile (both q tiles of attn_prefill_tc2; measured 2.3-2.8 us in the
    // %globaltimer trace, TC_PF_TRACE) plus ~8 us fixed per CTA (Q load, TMEM, epilogue, tail)
    const double w_pf = (3.0 * (double)pf_tiles + 8.0 * n_qblk * m.n_kv_heads) * (m.head_dim / 128.0);
    const double dec_bytes = (double)W * ps * m.head_dim * 2 * 2;
    // decode page-stream rate per SM and its HBM cap (bytes per us); TC_DEC_RATE="per_sm:cap" (GB/s)
    static const std::pair<double, double> dec_rate = [] {
      double a = 50.0, b = 5600.0;  // (4 producer warps: 5.6 TB/s on 124 SMs, ncu)
      if (const char* e = std::getenv("TC_DEC_RATE")) std::sscanf(e, "%lf:%lf", &a, &b);
      return std::make_pair(a * 1e3, b * 1e3);
    }();
    auto t_of = [&](int P) {
      const double t_dec = dec_bytes / std::min((I->sms - P) * dec_rate.first, dec_rate.second);  // us
      return t_dec + std::max(0.0, w_pf - P * t_dec) / I->sms;
    };
    const int p_max = std::min(n_qblk * m.n_kv_heads, I->sms / 2);
    double t_min = 1e30;
    for (int P = 4; P <= p_max; P += 4) t_min = std::min(t_min, t_of(P));
    int want = 0;
    for (int P = 4; P <= p_max; P += 4)
      if (t_of(P) <= 1.005 * t_min) {
        want = std::min(P + 4, p_max);
        break;
      }
    static const int env_pf = [] {
      const char* e = std::getenv("TC_PF_SMS");
      return e ? std::atoi(e) : -1;
    }();
    if (env_pf >= 0) want = env_pf;
    I->pf_sms = std::max(0, std::min({want, n_qblk * m.n_kv_heads, I->sms / 2}));
  }
  const int dec_sms = I->sms - I->pf_sms;
  static const int env_dec_grid = [] {
    const char* e = std::getenv("TC_DEC_GRID");
    return e ? std::atoi(e) : 0;
  }();
  const int dec_cap = env_dec_grid > 0 ? std::min(env_dec_grid, dec_sms) : dec_sms;
  const int dec_grid = n_dec ? (int)std::max<long long>(1, std::min<long long>(dec_cap, (W + 7) / 8)) : 0;
  // entries: one per (CTA, segment overlap); at most n_seg + dec_grid
  const int max_entries = n_seg + dec_grid;
  // layout of the metadata block
  int32_t* h = I->meta_host;
  size_t off = 0;
  auto take = [&](size_t n) {
    const size_t o = off;
    off += (n + 3) & ~size_t(3);
    return o;
  };
  const size_t o_tok = take(T), o_pos = take(T), o_rseq = take(T), o_kvrow = take(T), o_qs = take(n_seq), o_ql = take(n_seq),
               o_p0 = take(n_seq), o_bo = take(n_seq), o_qbs = take(n_qblk), o_qbo = take(n_qblk),
               o_lrow = take(n_logit), o_bt = take(n_bt), o_sega = take(4 * (size_t)n_seg), o_segb = take(4 * (size_t)n_seg),
               o_ent = take(4 * (size_t)max_entries), o_ctaoff = take((size_t)dec_grid + 1);
  TC_REQUIRE(off <= I->meta_ints, "step: metadata overflow");
  int row = 0, qb = 0, lr = 0, bt = 0;
  for (int i = 0; i < n_pf; ++i) {
    const tc_prefill_slice& sl = st->prefill[i];
    const std::vector<int32_t>& pages = I->tables[sl.req_id];
    h[o_qs + i] = row;
    h[o_ql + i] = sl.n_tokens;
    h[o_p0 + i] = sl.pos0;
    h[o_bo + i] = bt;
    const int np = (sl.pos0 + sl.n_tokens + ps - 1) / ps;
    for (int k = 0; k < np; ++k) h[o_bt + bt++] = pages[k];
    for (int k = 0; k < sl.n_tokens; ++k) {
      h[o_tok + row + k] = sl.token_ids[k];
      h[o_pos + row + k] = sl.pos0 + k;
      h[o_rseq + row + k] = i;
      h[o_kvrow + row + k] = pages[(sl.pos0 + k) / ps] * ps + (sl.pos0 + k) % ps;
    }
    for (int q = 0; q < sl.n_tokens; q += tpc) {
      h[o_qbs + qb] = i;
      h[o_qbo + qb] = q;
      ++qb;
    }
    row += sl.n_tokens;
    if (sl.want_logits) h[o_lrow + lr++] = row - 1;
  }
  if (qb > 1) {
    // longest-first prefill work list (causal: later q blocks see more keys) so the CTAs that
    // run on the few SMs left beside decode attention finish together
    std::vector<std::pair<int, int>> order(qb);
    for (int q = 0; q < qb; ++q) {
      const tc_prefill_slice& sl = st->prefill[h[o_qbs + q]];
      order[q] = {-(sl.pos0 + std::min(h[o_qbo + q] + tpc, sl.n_tokens)), q};
    }
    std::stable_sort(order.begin(), order.end());
    std::vector<int32_t> qs(qb), qo(qb);
    for (int q = 0; q < qb; ++q) {
      qs[q] = h[o_qbs + order[q].second];
      qo[q] = h[o_qbo + order[q].second];
    }
    std::copy(qs.begin(), qs.end(), h + o_qbs);
    std::copy(qo.begin(), qo.end(), h + o_qbo);
  }
  for (int j = 0; j < n_dec; ++j) {
    const tc_decode_item& di = st->decode[j];
    const int s = n_pf + j;
    const std::vector<int32_t>& pages = I->tables[di.req_id];
    h[o_qs + s] = row;
    h[o_ql + s] = 1;
    h[o_p0 + s] = di.pos;
    h[o_bo + s] = bt;
    const int np = di.pos / ps + 1;
    for (int k = 0; k < np; ++k) h[o_bt + bt++] = pages[k];
    h[o_tok + row] = di.token_id;
    h[o_pos + row] = di.pos;
    h[o_rseq + row] = s;
    h[o_kvrow + row] = pages[di.pos / ps] * ps + di.pos % ps;
    h[o_lrow + lr++] = row;
    ++row;
  }
  if (n_dec) {
    // segment descriptors
    int32_t* sa = h + o_sega;
    int32_t* sb = h + o_segb;
    for (int j = 0; j < n_dec; ++j)
      for (int kh = 0; kh < m.n_kv_heads; ++kh) {
        const int sg = j * m.n_kv_heads + kh;
        sa[4 * sg + 0] = h[o_bo + n_pf + j];
        sa[4 * sg + 1] = st->decode[j].pos + 1;
        sa[4 * sg + 2] = h[o_qs + n_pf + j];
        sa[4 * sg + 3] = kh;
        sb[4 * sg + 0] = 0;
        sb[4 * sg + 1] = 0;
        sb[4 * sg + 2] = sb[4 * sg + 3] = 0;
      }
    // walk the page stream, cutting it at CTA boundaries
    int32_t* ent = h + o_ent;
    int ne = 0, sg = 0, pg = 0;  // cursor: segment, page within it
    auto seg_pages = [&](int g) { return st->decode[g / m.n_kv_heads].pos / ps + 1; };
    for (int c = 0; c < dec_grid; ++c) {
      h[o_ctaoff + c] = ne;
      long long left = W * (c + 1) / dec_grid - W * c / dec_grid;
      while (left > 0) {
        const int np = seg_pages(sg);
        const int take_n = (int)std::min<long long>(left, np - pg);
        ent[4 * ne + 0] = sg;
        ent[4 * ne + 1] = pg;
        ent[4 * ne + 2] = pg + take_n;
        ent[4 * ne + 3] = sb[4 * sg + 0]++;  // part index; the count becomes the segment's parts
        ++ne;
        pg += take_n;
        left -= take_n;
        if (pg == np) {
          ++sg;
          pg = 0;
        }
      }
    }
    h[o_ctaoff + dec_grid] = ne;
    TC_REQUIRE(ne <= max_entries, "step: decode entry overflow");
    int slots = 0;
    for (int g = 0; g < n_seg; ++g) {
      if (sb[4 * g + 0] > 1) {
        sb[4 * g + 1] = slots;
        slots += sb[4 * g + 0];
      }
    }
    TC_REQUIRE(slots <= kMaxDecodeItems, "step: decode partial slots overflow");
  }
  cudaStream_t s = I->stream;
  DeviceGuard dg(I->desc.device);
  if (I->prof.on) I->prof.reset();
  I->launches = 0;
  I->h2d_bytes = (int64_t)off * 4;
  for (const EvPtr& e : waits) TC_CUDA(cudaStreamWaitEvent(s, e->e, 0));
  TC_CUDA(cudaEventRecord(I->ev_start, s));
  // The step's ~230 launches go out as one CUDA graph when this launch shape has been seen before
  // (the metadata block is re-read from pinned host memory by the graph's memcpy node, so only the
  // shape -- grids and metadata offsets -- has to match). TC_GRAPH=0 disables it.
  const GraphKey gkey{T, n_seq, n_qblk, n_logit, n_bt, n_seg, max_entries, dec_grid, I->pf_sms, (int)off};
  const bool graph_ok = graphs_enabled() && !I->prof.on && waits.empty();
  if (graph_ok) {
    if (const GraphCache::Entry* ge = I->graphs.find(gkey)) {
      TC_CUDA(cudaGraphLaunch(ge->exec, s));
      I->launches = ge->launches;
      TC_CUDA(cudaEventRecord(I->ev_stop, s));
      I->step_pending = true;
      I->last_sampled = n_logit;
      return;
    }
  }
  const bool capture = graph_ok && I->graphs.seen(gkey);
  if (capture) TC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  TC_CUDA(cudaMemcpyAsync(I->meta_dev, h, off * 4, cudaMemcpyHostToDevice, s));
  const int32_t* dm = I->meta_dev;


  {
    ProfScope ps_(I, "embed");
    launch_k(tc::embed_rows, T, 256, 0, s, dm + o_tok, I->embed, I->resid, m.d_model);
    ++I->launches;
  }
  tc::AttnParams ap{};
  ap.qkv = I->qkv;
  ap.out = I->attn_out;
  ap.n_layers = m.n_layers;
  ap.n_heads = m.n_heads;
  ap.n_kv_heads = m.n_kv_heads;
  ap.page_size = ps;
  ap.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)m.head_dim));
  ap.seq_q_start = dm + o_qs;
  ap.seq_q_len = dm + o_ql;
  ap.seq_pos0 = dm + o_p0;
  ap.seq_bt_off = dm + o_bo;
  ap.block_tables = dm + o_bt;
  ap.qblk_seq = dm + o_qbs;
  ap.qblk_off = dm + o_qbo;
  ap.dec_seg_a = reinterpret_cast<const int4*>(dm + o_sega);
  ap.dec_seg_b = reinterpret_cast<const int4*>(dm + o_segb);
  ap.dec_entries = reinterpret_cast<const int4*>(dm + o_ent);
  ap.dec_cta_off = dm + o_ctaoff;
  ap.ws_o = I->attn_ws_o;
  ap.dec_cnt = I->attn_cnt;
  ap.ws_ml = I->attn_ws_ml;
  ap.pf_trace = nullptr;
  tc::QkvRopeArgs rp{};
  rp.kv = I->kv;
  rp.rope_cs = I->rope;
  rp.positions = dm + o_pos;
  rp.row_seq = dm + o_rseq;
  rp.row_kv = dm + o_kvrow;
  rp.seq_bt_off = dm + o_bo;
  rp.block_tables = dm + o_bt;
  rp.page_stride = I->page_elems;
  rp.n_heads = m.n_heads;
  rp.n_kv_heads = m.n_kv_heads;
  rp.head_dim = m.head_dim;
  rp.page_size = ps;
  constexpr int rms_threads = 256;
  // Every step, decode-only ones included, runs each projection as direct weight-stationary units
  // with its fused epilogue. (Round 2 measured the alternative for T <= 128 -- stream-K partials
  // into a zeroed fp32 scratch plus RoPE / SwiGLU finish kernels -- at 5.44 vs 5.22 ms per
  // decode-only step: the finish kernels and the scratch round trip cost more than the direct
  // units' 1.5-wave imbalance on gate_up and QKV's 24 busy pairs.)
  for (int l = 0; l < m.n_layers; ++l) {
    const LayerW& L = I->layers[l];
    {
      ProfScope p_(I, "norm");
      launch_k(tc::rmsnorm_rows<rms_threads>, T, rms_threads, 0, s, I->resid, nullptr, L.attn_norm, I->xnorm, m.d_model, m.rms_eps);
      ++I->launches;
    }
    {
      // QKV projection with fused bias, RoPE and paged KV append (q stays in I->qkv)
      ProfScope p_(I, "gemm_qkv");
      rp.layer = l;
      I->launches += run_gemm(I->map_xnorm, L.qkv, T, I->qkv, I->qkv_n, m.qkv_bias ? L.qkv_bias : nullptr,
                              tc::EPI_QKV_ROPE, I->sms, I->sk, s, 0, 0, &rp, nullptr);
    }
    {
      ProfScope p_(I, "attn");
      ap.layer = l;
      dispatch_attention(I, ap, n_qblk, n_dec, dec_grid);
    }
    {
      ProfScope p_(I, "gemm_o");
      I->launches += run_gemm(I->map_attn, L.o, T, I->resid, m.d_model, nullptr, tc::EPI_RESID_F32, I->sms, I->sk, s, 0, 0,
                              nullptr, &I->map_resid);
    }
    {
      ProfScope p_(I, "norm");
      launch_k(tc::rmsnorm_rows<rms_threads>, T, rms_threads, 0, s, I->resid, nullptr, L.mlp_norm, I->xnorm, m.d_model, m.rms_eps);
      ++I->launches;
    }
    {
      ProfScope p_(I, "gemm_gate_up");
      I->launches += run_gemm(I->map_xnorm, L.gate_up, T, I->act, m.ffn_dim, nullptr, tc::EPI_SWIGLU, I->sms, I->sk, s);
    }
    {
      ProfScope p_(I, "gemm_down");
      I->launches += run_gemm(I->map_act, L.down, T, I->resid, m.d_model, nullptr, tc::EPI_RESID_F32, I->sms, I->sk, s, 0, 0,
                              nullptr, &I->map_resid);
    }
  }
  if (n_logit > 0) {
    ProfScope p_(I, "lm_head");
    launch_k(tc::rmsnorm_rows<rms_threads>, n_logit, rms_threads, 0, s, I->resid, dm + o_lrow, I->final_norm, I->lm_in,
             m.d_model, m.rms_eps);
    I->launches += 2;  // gathered RMSNorm + argmax
    I->launches += run_gemm(I->map_lm_in, I->lm_head, n_logit, I->logits, m.vocab, nullptr, tc::EPI_F32, I->sms, I->sk, s);
    launch_k(tc::argmax_rows<1024>, n_logit, 1024, 0, s, I->logits, m.vocab, I->ids_dev);
    TC_CUDA(cudaMemcpyAsync(I->ids_host, I->ids_dev, (size_t)n_logit * 4, cudaMemcpyDeviceToHost, s));
  }
  TC_CUDA(cudaGetLastError());
  if (capture) {
    cudaGraph_t g = nullptr;
    TC_CUDA(cudaStreamEndCapture(s, &g));
    cudaGraphExec_t ex = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    TC_CUDA(e);
    I->graphs.put(gkey, ex, I->launches);
    TC_CUDA(cudaGraphLaunch(ex, s));
  }
  TC_CUDA(cudaEventRecord(I->ev_stop, s));
  I->step_pending = true;
  I->last_sampled = n_logit;
}

void step_wait(tc_instance* I, tc_step_result* r) {
  TC_REQUIRE(I->step_pending, "wait: no step in flight");
  DeviceGuard dg(I->desc.device);
  TC_CUDA(cudaEventSynchronize(I->ev_stop));
  I->step_pending = false;
  if (!r) return;
  r->n_sampled = I->last_sampled;
  r->launches = I->launches;
  r->h2d_bytes = I->h2d_bytes;
  r->d2h_bytes = (int64_t)I->last_sampled * 4 + (r->logits ? (int64_t)I->last_sampled * I->d.vocab * 4 : 0);
  if (r->sampled_ids) std::memcpy(r->sampled_ids, I->ids_host, (size_t)I->last_sampled * 4);
  if (r->logits && I->last_sampled > 0)
    TC_CUDA(cudaMemcpy(r->logits, I->logits, (size_t)I->last_sampled * I->d.vocab * 4, cudaMemcpyDeviceToHost));
  float ms = 0.f;
  TC_CUDA(cudaEventElapsedTime(&ms, I->ev_start, I->ev_stop));
  r->gpu_ms = ms;
  r->attn_pf_sms = I->pf_sms;
}

void event_destroy(tc_event* ev);

void destroy(tc_instance* I) {
  DeviceGuard dg(I->desc.device);
  if (I->stream) cudaStreamSynchronize(I->stream);
  I->graphs.clear();
  for (auto& kv : I->mig_streams) {
    cudaStreamSynchronize(kv.second);
    cudaStreamDestroy(kv.second);
  }
  if (I->last_mig) event_destroy(I->last_mig);
  // pages go back to the (possibly shared) pool; copies into them have finished (streams synced
  // above for outbound; inbound copies are ordered by their events in the pool's quarantine)
  if (I->pool) {
    std::vector<int64_t> reqs;
    for (auto& t : I->tables) reqs.push_back(t.first);
    for (int64_t r : reqs) release_pages(I, r);
  }
  auto f = [](void* p) {
    if (p) cudaFree(p);
  };
  I->weight_owner.reset();
  I->pool.reset();
  f(I->resid); f(I->xnorm); f(I->qkv); f(I->attn_out); f(I->act); f(I->lm_in);
  f(I->logits); f(I->ids_dev); f(I->sk.ws); f(I->sk.cnt); f(I->attn_ws_o); f(I->attn_ws_ml); f(I->attn_cnt); f(I->rope); f(I->meta_dev);
  if (I->ids_host) cudaFreeHost(I->ids_host);
  if (I->meta_host) cudaFreeHost(I->meta_host);
  for (cudaEvent_t e : {I->ev_start, I->ev_stop, I->mig_tail, I->ev_fork, I->ev_join})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : I->prof.pool) cudaEventDestroy(e);
  if (I->stream) cudaStreamDestroy(I->stream);
  if (I->stream_pf) cudaStreamDestroy(I->stream_pf);
  delete I;
}

void enable_peer(int a, int b) {
  if (a == b) return;
  static std::mutex mu;
  static std::set<std::pair<int, int>> done;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({a, b})) return;
  int can = 0;
  TC_CUDA(cudaDeviceCanAccessPeer(&can, a, b));
  TC_REQUIRE(can, "peer access unavailable between GPUs " + std::to_string(a) + " and " + std::to_string(b));
  DeviceGuard g(a);
  const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
  if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) TC_CUDA(e);
  cudaGetLastError();
  done.insert({a, b});
}

// Launch the page-copy kernel on src's copy stream toward dst_key (ordered after src's in-flight
// step); returns the event (t0 recorded before the first launch, done after the last).
tc_event* launch_page_copy(tc_instance* src, const void* dst_key, void* dst_base, const int32_t* sp, const int32_t* dp,
                           int64_t np, bool peer, cudaEvent_t after = nullptr) {
  std::unique_ptr<tc_event> ev(new tc_event());
  ev->device = src->desc.device;
  ev->pages = np;
  ev->bytes = np * src->page_elems * 2;
  ev->peer = peer;
  ev->done = std::make_shared<SharedEvent>(src->desc.device, true);
  DeviceGuard dg(src->desc.device);
  TC_CUDA(cudaEventCreate(&ev->t0));
  cudaStream_t& cs = src->mig_streams[dst_key];
  if (!cs) {
    int lo = 0, hi = 0;
    TC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    TC_CUDA(cudaStreamCreateWithPriority(&cs, cudaStreamNonBlocking, hi));
  }
  TC_CUDA(cudaEventRecord(src->mig_tail, src->stream));
  TC_CUDA(cudaStreamWaitEvent(cs, src->mig_tail, 0));
  if (after) TC_CUDA(cudaStreamWaitEvent(cs, after, 0));
  TC_CUDA(cudaEventRecord(ev->t0, cs));
  const int64_t page_vec = src->page_elems * 2 / 16;
  const int cap = src->mig_ctas > 0 ? src->mig_ctas : 4 * src->sms;
  for (int64_t b0 = 0; b0 < np; b0 += tc::kMigPagesPerLaunch) {
    tc::MigPages pl;
    pl.n = (int)std::min<int64_t>(tc::kMigPagesPerLaunch, np - b0);
    for (int i = 0; i < pl.n; ++i) {
      pl.src[i] = sp[b0 + i];
      pl.dst[i] = dp[b0 + i];
    }
    const int64_t slices = (int64_t)pl.n * ((page_vec + tc::kCopySliceVec - 1) / tc::kCopySliceVec);
    const int blocks = (int)std::min<int64_t>(cap, std::max<int64_t>(1, slices));
    tc::kv_migrate_pages<<<blocks, tc::kCopyThreads, 0, cs>>>(reinterpret_cast<const uint4*>(src->kv), reinterpret_cast<uint4*>(dst_base),
                                                 pl, page_vec);
    TC_CUDA(cudaGetLastError());
  }
  TC_CUDA(cudaEventRecord(ev->done->e, cs));
  return ev.release();
}

// Asynchronous KV migration (K11): every page src holds for req (at least the first n_tokens rows;
// a step in flight on src may have written one more row, which must travel too -- a request that
// flows away and back within that step brings it home, engine.hpp:461-493) is pushed into freshly
// allocated pages of dst by kv_migrate_pages on src's high-priority copy stream for dst, after
// src's in-flight step. Nothing blocks the host: src's pages return to its pool once the copy's
// event completes (quarantine), and dst's next step / outbound copy / release of req orders
// after that event. Across GPUs the kernel's stores go over NVLink (peer access, UVA).
tc_event* migrate_async(tc_instance* src, tc_instance* dst, int64_t req, int64_t n_tokens) {
  TC_REQUIRE(src && dst && src != dst, "migrate: need two distinct instances");
  TC_REQUIRE(src->page_elems == dst->page_elems && src->desc.page_size == dst->desc.page_size,
             "migrate: instances differ in KV geometry");
  auto it = src->tables.find(req);
  TC_REQUIRE(it != src->tables.end(), "migrate: request has no KV on source");
  TC_REQUIRE(dst->tables.find(req) == dst->tables.end() || dst->tables[req].empty(),
             "migrate: request already has KV on destination");
  const int ps = src->desc.page_size;
  TC_REQUIRE(n_tokens >= 0 && (n_tokens + ps - 1) / ps <= (int64_t)it->second.size(),
             "migrate: source holds fewer pages than requested");
  const int64_t np = (int64_t)it->second.size();
  ensure_pages(dst, req, np * ps);
  enable_peer(src->desc.device, dst->desc.device);
  // after any inbound copy of req (and, inside launch_page_copy, after src's in-flight step); dst
  // pages may be quarantined pages of an earlier copy: reclaim only hands them out once their
  // event completed, so no ordering is needed on the destination side
  EvPtr in = inbound_pending(src, req);
  std::unique_ptr<tc_event> ev(launch_page_copy(src, dst, dst->kv, it->second.data(), dst->tables[req].data(), np,
                                                src->desc.device != dst->desc.device, in ? in->e : nullptr));
  dst->inbound[req] = ev->done;
  // source pages return to the pool once the copy has read them
  release_pages(src, req, ev->done);
  return ev.release();
}

tc_event* push_pages(tc_instance* src, tc_remote_pool* dst, const int32_t* sp, const int32_t* dp, int32_t np) {
  TC_REQUIRE(src && dst && dst->base, "push: null instance or pool");
  TC_REQUIRE(dst->device == src->desc.device, "push: pool was imported on another device than the source's");
  TC_REQUIRE(dst->page_bytes == src->page_elems * 2, "push: pools differ in page geometry");
  TC_REQUIRE(np >= 0 && (np == 0 || (sp && dp)), "push: null page list");
  for (int32_t i = 0; i < np; ++i) {
    TC_REQUIRE(sp[i] >= 0 && sp[i] < src->n_pages, "push: source page out of range");
    TC_REQUIRE(dp[i] >= 0 && dp[i] < dst->n_pages, "push: destination page out of range");
  }
  return launch_page_copy(src, dst, dst->base, sp, dp, np, true);
}

void event_wait(tc_event* ev, float* copy_ms, int64_t* bytes) {
  TC_REQUIRE(ev, "event: null");
  DeviceGuard dg(ev->device);
  TC_CUDA(cudaEventSynchronize(ev->done->e));
  float ms = 0.f;
  TC_CUDA(cudaEventElapsedTime(&ms, ev->t0, ev->done->e));
  if (copy_ms) *copy_ms = ms;
  if (bytes) *bytes = ev->bytes;
}

void event_destroy(tc_event* ev) {
  if (!ev) return;
  DeviceGuard dg(ev->device);
  if (ev->t0) cudaEventDestroy(ev->t0);
  delete ev;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* tc_last_error(void) { return g_last_error.c_str(); }
const char* tc_version(void) { return "taichi_b200 0.1 (sm_100a)"; }

tc_status tc_model_preset(const char* name, tc_model_dims* out) {
  return guarded([&] {
    TC_REQUIRE(name && out, "preset: null argument");
    *out = preset(name);
  });
}

uint16_t tc_weight_value(uint64_t seed, uint64_t tensor_id, int64_t index, float scale, float offset) {
  const uint64_t key = tc::sm64(seed ^ tc::sm64(tensor_id));
  const uint64_t h = tc::sm64(key + (uint64_t)index);
  const float u = (float)(uint32_t)(h >> 40) * 5.9604644775390625e-08f;
  const float c = u * 2.0f - 1.0f;
  volatile float prod = c * scale;  // keep the two roundings separate
  const float v = prod + offset;
  uint32_t bits;
  std::memcpy(&bits, &v, 4);
  const uint32_t lsb = (bits >> 16) & 1u;
  return (uint16_t)((bits + 0x7FFFu + lsb) >> 16);
}

tc_status tc_instance_create(const tc_instance_desc* desc, tc_instance** out) {
  tc_instance* I = nullptr;
  const tc_status st = guarded([&] {
    TC_REQUIRE(desc && out, "create: null argument");
    check_dims(desc->dims);
    TC_REQUIRE(desc->page_size == 16, "create: page_size must be 16");
    TC_REQUIRE(desc->max_step_tokens >= 1 && desc->max_seqs >= 1 && desc->max_context >= 16, "create: bad limits");
    TC_REQUIRE(desc->kv_pool_tokens <= 0 || desc->kv_pool_tokens >= desc->page_size, "create: KV pool too small");
    I = new tc_instance();
    I->desc = *desc;
    I->d = desc->dims;
    int n_dev = 0;
    TC_CUDA(cudaGetDeviceCount(&n_dev));
    TC_REQUIRE(desc->device >= 0 && desc->device < n_dev, "create: no such CUDA device");
    DeviceGuard dg(desc->device);
    int major = 0, minor = 0;
    TC_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, desc->device));
    TC_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, desc->device));
    TC_REQUIRE(major == 10 && minor == 0, "create: libtaichi_b200 is built for sm_100a (B200) only");
    I->sms = device_sms(desc->device);
    init_kernel_attrs(desc->device);
    TC_CUDA(cudaStreamCreateWithFlags(&I->stream, cudaStreamNonBlocking));
    TC_CUDA(cudaStreamCreateWithFlags(&I->stream_pf, cudaStreamNonBlocking));
    if (desc->share_weights) {
      const tc_instance* o = desc->share_weights;
      TC_REQUIRE(o->desc.device == desc->device, "create: share_weights needs the same device");
      TC_REQUIRE(std::memcmp(&o->d, &desc->dims, sizeof(tc_model_dims)) == 0 && o->desc.weight_seed == desc->weight_seed,
                 "create: share_weights needs identical dims and seed");
      I->weight_owner = o->weight_owner;
      I->embed = o->embed;
      I->final_norm = o->final_norm;
      I->lm_head = o->lm_head;
      I->layers = o->layers;
      I->qkv_n = o->qkv_n;
    } else {
      alloc_weights(I);
    }
    alloc_buffers(I);
    const tc_model_dims& m = I->d;
    I->page_elems = (int64_t)m.n_layers * 2 * m.n_kv_heads * desc->page_size * m.head_dim;
    if (desc->share_kv_pool) {
      const tc_instance* o = desc->share_kv_pool;
      TC_REQUIRE(o->desc.device == desc->device && o->page_elems == I->page_elems,
                 "create: share_kv_pool needs the same device and KV geometry");
      I->pool = o->pool;
    } else {
      I->pool = std::make_shared<KvPool>();
      I->pool->device = desc->device;
      I->pool->page_elems = I->page_elems;
      int64_t tokens = desc->kv_pool_tokens;
      if (tokens <= 0) {
        // auto: every free byte of HBM but a reserve of max(4 GiB, 12% of HBM) -- room for the step
        // workspaces (~0.8 GB each at Llama-3-8B) of up to ~20 instances that share this GPU and
        // this pool (share_kv_pool), e.g. the 8 instances of config 3 time-shared on one B200
        size_t free_b = 0, total_b = 0;
        TC_CUDA(cudaMemGetInfo(&free_b, &total_b));
        const int64_t usable = (int64_t)free_b - std::max<int64_t>((int64_t)4 << 30, (int64_t)(0.12 * (double)total_b));
        TC_REQUIRE(usable > I->page_elems * 2, "create: no HBM left for a KV pool");
        tokens = usable / (I->page_elems * 2) * desc->page_size;
      }
      I->pool->n_pages = (tokens + desc->page_size - 1) / desc->page_size;
      TC_CUDA(cudaMalloc(&I->pool->kv, (size_t)I->pool->n_pages * I->page_elems * 2));
      TC_CUDA(cudaMemsetAsync(I->pool->kv, 0, (size_t)I->pool->n_pages * I->page_elems * 2, I->stream));
      I->pool->free_pages.resize(I->pool->n_pages);
      for (int64_t i = 0; i < I->pool->n_pages; ++i) I->pool->free_pages[i] = (int32_t)(I->pool->n_pages - 1 - i);  // pop_back -> 0,1,..
    }
    I->kv = I->pool->kv;
    I->n_pages = I->pool->n_pages;
    {
      const uint64_t rows = (uint64_t)I->n_pages * m.n_layers * 2 * m.n_kv_heads * desc->page_size;
      TC_REQUIRE(rows < (1ull << 31), "create: KV pool too large for 32-bit TMA row coordinates");
      // dims {64 dims, pool rows, head_dim/64 halves}: one box = the adjacent K and V blocks of a
      // (page, layer, kv head); each 64-dim half lands as a separate 32-line 128 B-swizzled slab
      // (bank-conflict-free ldmatrix, K-major SW128 layout)
      const cuuint64_t dims[3] = {64, rows, (cuuint64_t)(m.head_dim / 64)};
      const cuuint64_t strides[2] = {(cuuint64_t)m.head_dim * 2, 128};
      const cuuint32_t box[3] = {64, (cuuint32_t)(2 * desc->page_size), (cuuint32_t)(m.head_dim / 64)};
      const cuuint32_t estr[3] = {1, 1, 1};
      const CUresult r = tensor_map_encoder()(&I->kv_map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, I->kv, dims, strides, box,
                                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw TcFail{TC_ERR_CUDA, "KV tensor map encode failed: " + std::to_string((int)r)};
    }
    {
      const uint64_t rows = (uint64_t)I->n_pages * m.n_layers * 2 * m.n_kv_heads * desc->page_size;
      const cuuint64_t dims[2] = {(cuuint64_t)m.head_dim, rows};
      const cuuint64_t strides[1] = {(cuuint64_t)m.head_dim * 2};
      const cuuint32_t box[2] = {64, (cuuint32_t)desc->page_size};
      I->kv2_map = encode_map(I->kv, 2, dims, strides, box);
    }
    TC_CUDA(cudaStreamSynchronize(I->stream));
  });
  if (st != TC_OK) {
    if (I) destroy(I);
    return st;
  }
  *out = I;
  return TC_OK;
}

tc_status tc_instance_destroy(tc_instance* inst) {
  return guarded([&] {
    if (inst) destroy(inst);
  });
}

tc_status tc_step_launch(tc_instance* inst, const tc_step_desc* step) {
  return guarded([&] {
    TC_REQUIRE(inst, "step: null instance");
    step_launch(inst, step);
  });
}

tc_status tc_step_wait(tc_instance* inst, tc_step_result* result) {
  return guarded([&] {
    TC_REQUIRE(inst, "wait: null instance");
    step_wait(inst, result);
  });
}

tc_status tc_kv_reserve(tc_instance* inst, int64_t req_id, int64_t n_tokens) {
  return guarded([&] {
    TC_REQUIRE(inst && n_tokens >= 0, "reserve: bad argument");
    ensure_pages(inst, req_id, n_tokens);
  });
}

tc_status tc_kv_release(tc_instance* inst, int64_t req_id) {
  return guarded([&] {
    TC_REQUIRE(inst, "release: null instance");
    release_pages(inst, req_id);
  });
}

tc_status tc_kv_stats(tc_instance* inst, int64_t req_id, int64_t* req_pages, int64_t* free_pages) {
  return guarded([&] {
    TC_REQUIRE(inst, "stats: null instance");
    auto it = inst->tables.find(req_id);
    if (req_pages) *req_pages = it == inst->tables.end() ? 0 : (int64_t)it->second.size();
    if (free_pages) *free_pages = inst->pool->free_count();
  });
}

tc_status tc_kv_migrate_async(tc_instance* src, tc_instance* dst, int64_t req_id, int64_t n_tokens, tc_event** ev) {
  return guarded([&] {
    TC_REQUIRE(ev, "migrate_async: null event out-pointer");
    *ev = migrate_async(src, dst, req_id, n_tokens);
  });
}

tc_status tc_event_query(tc_event* ev, int32_t* done) {
  return guarded([&] {
    TC_REQUIRE(ev && done, "event_query: null argument");
    const cudaError_t e = cudaEventQuery(ev->done->e);
    if (e != cudaSuccess && e != cudaErrorNotReady) TC_CUDA(e);
    *done = e == cudaSuccess;
  });
}

tc_status tc_event_wait(tc_event* ev, float* copy_ms, int64_t* bytes) {
  return guarded([&] { event_wait(ev, copy_ms, bytes); });
}

tc_status tc_event_destroy(tc_event* ev) {
  return guarded([&] { event_destroy(ev); });
}

tc_status tc_kv_migrate(tc_instance* src, tc_instance* dst, int64_t req_id, int64_t n_tokens) {
  return guarded([&] {
    TC_REQUIRE(src, "migrate: null source");
    TC_REQUIRE(!src->last_mig, "migrate: previous migration on this source not waited");
    src->last_mig = migrate_async(src, dst, req_id, n_tokens);
  });
}

tc_status tc_kv_migrate_wait(tc_instance* src, float* copy_ms, int64_t* bytes) {
  return guarded([&] {
    TC_REQUIRE(src && src->last_mig, "migrate_wait: no migration in flight");
    tc_event* ev = src->last_mig;
    src->last_mig = nullptr;
    std::unique_ptr<tc_event, void (*)(tc_event*)> hold(ev, event_destroy);
    event_wait(ev, copy_ms, bytes);
  });
}

tc_status tc_kv_pool_export(tc_instance* inst, void* handle, int64_t* page_bytes, int64_t* n_pages) {
  return guarded([&] {
    TC_REQUIRE(inst && handle, "export: null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == TC_IPC_HANDLE_BYTES, "IPC handle size");
    DeviceGuard dg(inst->desc.device);
    cudaIpcMemHandle_t h;
    TC_CUDA(cudaIpcGetMemHandle(&h, inst->kv));
    std::memcpy(handle, &h, sizeof(h));
    if (page_bytes) *page_bytes = inst->page_elems * 2;
    if (n_pages) *n_pages = inst->n_pages;
  });
}

tc_status tc_kv_pool_import(int32_t device, const void* handle, int64_t page_bytes, int64_t n_pages, tc_remote_pool** out) {
  return guarded([&] {
    TC_REQUIRE(handle && out && page_bytes > 0 && n_pages > 0, "import: bad argument");
    DeviceGuard dg(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    std::unique_ptr<tc_remote_pool> p(new tc_remote_pool());
    p->device = device;
    p->page_bytes = page_bytes;
    p->n_pages = n_pages;
    TC_CUDA(cudaIpcOpenMemHandle(&p->base, h, cudaIpcMemLazyEnablePeerAccess));
    *out = p.release();
  });
}

tc_status tc_remote_pool_close(tc_remote_pool* pool) {
  return guarded([&] {
    if (!pool) return;
    DeviceGuard dg(pool->device);
    cudaDeviceSynchronize();  // no copy may still target the mapping
    const cudaError_t e = cudaIpcCloseMemHandle(pool->base);
    delete pool;
    TC_CUDA(e);
  });
}

tc_status tc_kv_push_pages(tc_instance* src, tc_remote_pool* dst, const int32_t* src_pages, const int32_t* dst_pages,
                           int32_t n_pages, tc_event** ev) {
  return guarded([&] {
    TC_REQUIRE(ev, "push: null event out");
    *ev = push_pages(src, dst, src_pages, dst_pages, n_pages);
  });
}

tc_status tc_set_migration_ctas(tc_instance* inst, int32_t ctas) {
  return guarded([&] {
    TC_REQUIRE(inst && ctas >= 0, "migration_ctas: bad argument");
    inst->mig_ctas = ctas;
  });
}

tc_status tc_kv_pool_info(tc_instance* inst, void** base, int64_t* page_bytes, int64_t* n_pages) {
  return guarded([&] {
    TC_REQUIRE(inst, "pool_info: null instance");
    if (base) *base = inst->kv;
    if (page_bytes) *page_bytes = inst->page_elems * 2;
    if (n_pages) *n_pages = inst->n_pages;
  });
}

tc_status tc_kv_pages(tc_instance* inst, int64_t req_id, int32_t* pages, int32_t max_pages, int32_t* n_pages) {
  return guarded([&] {
    TC_REQUIRE(inst, "pages: null instance");
    auto it = inst->tables.find(req_id);
    const int32_t n = it == inst->tables.end() ? 0 : (int32_t)it->second.size();
    if (n_pages) *n_pages = n;
    for (int32_t i = 0; i < n && i < max_pages && pages; ++i) pages[i] = it->second[i];
  });
}

tc_status tc_weight_ptr(tc_instance* inst, const char* name, void** ptr, int64_t* rows, int64_t* cols) {
  return guarded([&] {
    TC_REQUIRE(inst && name && ptr, "weight_ptr: null argument");
    const tc_model_dims& m = inst->d;
    const std::string n = name;
    auto put = [&](void* p, int64_t r, int64_t c) {
      *ptr = p;
      if (rows) *rows = r;
      if (cols) *cols = c;
    };
    if (n == "embed") return put(inst->embed, m.vocab, m.d_model);
    if (n == "lm_head") return put(inst->lm_head.ptr, m.vocab, m.d_model);
    if (n == "final_norm") return put(inst->final_norm, 1, m.d_model);
    TC_REQUIRE(n.size() > 1 && n[0] == 'L' && n.find('.') != std::string::npos, "weight_ptr: unknown weight " + n);
    const int l = std::stoi(n.substr(1, n.find('.') - 1));
    TC_REQUIRE(l >= 0 && l < m.n_layers, "weight_ptr: layer out of range");
    const std::string f = n.substr(n.find('.') + 1);
    const LayerW& L = inst->layers[l];
    if (f == "qkv") return put(L.qkv.ptr, L.qkv.rows, L.qkv.cols);
    if (f == "o") return put(L.o.ptr, L.o.rows, L.o.cols);
    if (f == "gate_up") return put(L.gate_up.ptr, L.gate_up.rows, L.gate_up.cols);
    if (f == "down") return put(L.down.ptr, L.down.rows, L.down.cols);
    if (f == "qkv_bias") return put(L.qkv_bias, 1, inst->qkv_n);
    if (f == "attn_norm") return put(L.attn_norm, 1, m.d_model);
    if (f == "mlp_norm") return put(L.mlp_norm, 1, m.d_model);
    throw TcFail{TC_ERR_INVALID, "weight_ptr: unknown weight " + n};
  });
}

tc_status tc_gemm(int32_t device, const void* a, const void* b, void* out, const void* bias, int32_t m, int32_t n,
                  int32_t k, int32_t epilogue, int32_t bn, int32_t k_splits, void* stream) {
  return guarded([&] {
    TC_REQUIRE(a && b && out && m > 0 && n > 0 && k > 0, "gemm: bad argument");
    TC_REQUIRE(epilogue >= 0 && epilogue <= 4, "gemm: bad epilogue");
    TC_REQUIRE(k_splits >= 0, "gemm: bad k_splits");
    DeviceGuard dg(device);
    init_kernel_attrs(device);
    const int sms = device_sms(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    WMat w;
    w.ptr = (__nv_bfloat16*)b;
    w.rows = n;
    w.cols = k;
    w.make_maps();
    ActMap am;
    am.init(a, m, k);
    const int ldo = epilogue == tc::EPI_SWIGLU ? n / 2 : n;
    // one persistent split-K workspace per device (the tile counters self-reset: the last
    // arriver of every split tile zeroes its counter), so calls on one stream reuse it
    static std::mutex mu;
    static std::unordered_map<int, SkWorkspace> per_dev;
    SkWorkspace sk;
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = per_dev.find(device);
      if (it == per_dev.end()) {
        SkWorkspace w_;
        TC_CUDA(cudaMalloc(&w_.ws, kSkWsBytes));
        TC_CUDA(cudaMalloc(&w_.cnt, (size_t)kSkMaxTiles * 4));
        TC_CUDA(cudaMemset(w_.cnt, 0, (size_t)kSkMaxTiles * 4));
        it = per_dev.emplace(device, w_).first;
      }
      sk = it->second;
    }
    run_gemm(am, w, m, out, ldo, (const __nv_bfloat16*)bias, epilogue, sms, sk, s, bn, k_splits);
  });
}

tc_status tc_copy_pages(const void* src_pool, void* dst_pool, const int32_t* src_pages_dev,
                        const int32_t* dst_pages_dev, int32_t n_pages, int64_t page_bytes, void* stream) {
  return guarded([&] {
    TC_REQUIRE(src_pool && dst_pool && n_pages >= 0 && page_bytes % 16 == 0, "copy_pages: bad argument");
    if (n_pages == 0) return;
    int dev = 0;
    TC_CUDA(cudaGetDevice(&dev));
    const int sms = device_sms(dev);
    const int64_t page_vec = page_bytes / 16;
    const int64_t slices = (int64_t)n_pages * ((page_vec + tc::kCopySliceVec - 1) / tc::kCopySliceVec);
    const int blocks = (int)std::min<int64_t>(4 * sms, std::max<int64_t>(1, slices));
    tc::kv_copy_pages<<<blocks, tc::kCopyThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const uint4*>(src_pool), reinterpret_cast<uint4*>(dst_pool), src_pages_dev, dst_pages_dev,
        n_pages, page_vec);
    TC_CUDA(cudaGetLastError());
  });
}

tc_status tc_read_device(void* host_dst, const void* dev_src, size_t bytes) {
  return guarded([&] {
    TC_REQUIRE(host_dst && dev_src, "read_device: null argument");
    TC_CUDA(cudaMemcpy(host_dst, dev_src, bytes, cudaMemcpyDeviceToHost));
  });
}

tc_status tc_set_profiling(tc_instance* inst, int32_t on) {
  return guarded([&] {
    TC_REQUIRE(inst, "profiling: null instance");
    inst->prof.on = on != 0;
  });
}

tc_status tc_phase_ms(tc_instance* inst, const char* phase, float* ms) {
  return guarded([&] {
    TC_REQUIRE(inst && phase && ms, "phase_ms: null argument");
    DeviceGuard dg(inst->desc.device);
    TC_CUDA(cudaEventSynchronize(inst->ev_stop));
    float total = 0.f;
    for (auto& mk : inst->prof.marks) {
      if (mk.first != phase) continue;
      float t = 0.f;
      TC_CUDA(cudaEventElapsedTime(&t, mk.second.first, mk.second.second));
      total += t;
    }
    *ms = total;
  });
}

}  // extern "C"
