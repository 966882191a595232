/* taichi_b200.h -- C ABI of the B200 hybrid-iteration library (libtaichi_b200.so).
 *
 * The reference (/root/reference/proj, a header-only C++ simulator) has no GPU
 * code and no FFI: its hybrid step and KV migration are two cost-model calls.
 * These entry points replace exactly those seams:
 *
 *   tc_step_launch / tc_step_wait   replace iteration_time_ms at its call site
 *                                   engine.hpp:324-325 (launch) and the
 *                                   IterationComplete handler engine.hpp:461
 *                                   (wait + read back sampled token ids);
 *                                   cost_model.hpp:43-53.
 *   tc_kv_migrate(_async)           replaces transfer_time_ms at engine.hpp:402
 *                                   (degrade/backflow, full footprint) and
 *                                   engine.hpp:516 (init, prompt_len tokens);
 *                                   cost_model.hpp:81-85.
 *   tc_kv_reserve / tc_kv_release   physical mirror of the logical KV slot
 *                                   accounting of cluster.hpp:130-181.
 *
 * Conventions: plain C types only; every call returns tc_status (0 = ok) and
 * never throws; tc_last_error() returns this thread's last message. The library
 * owns all device memory (weights, KV pool, block tables, workspaces); caller
 * buffers are borrowed only for the duration of a call. One instance = one GPU
 * stream; calls on one instance must come from one host thread at a time.
 */
#ifndef TAICHI_B200_H_
#define TAICHI_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t tc_status;
enum {
  TC_OK = 0,
  TC_ERR_INVALID = 1,     /* bad argument / descriptor (ConfigError on the C++ side) */
  TC_ERR_CUDA = 2,        /* CUDA runtime / driver failure */
  TC_ERR_OOM = 3,         /* KV pool or device memory exhausted */
  TC_ERR_STATE = 4        /* call out of order (e.g. wait without launch) (EngineError) */
};

/* Decoder shape (Llama-3 / Qwen2 family). */
typedef struct {
  int32_t n_layers;
  int32_t d_model;
  int32_t n_heads;
  int32_t n_kv_heads;
  int32_t head_dim;   /* 64 or 128 */
  int32_t ffn_dim;
  int32_t vocab;
  int32_t qkv_bias;   /* 1 for Qwen2 */
  float rope_theta;
  float rms_eps;
} tc_model_dims;

typedef struct tc_instance tc_instance;

/* Presets: "tiny", "llama3_8b", "qwen2_5_14b".
 * Optional suffix ":L<n>" overrides the layer count (layer-reduced oracle runs). */
tc_status tc_model_preset(const char* name, tc_model_dims* out);

typedef struct {
  int32_t device;            /* CUDA ordinal; one instance per GPU in production */
  tc_model_dims dims;
  uint64_t weight_seed;      /* deterministic random init (see tc_weight_value) */
  int32_t page_size;         /* tokens per KV page (16) */
  int64_t kv_pool_tokens;    /* physical KV capacity in tokens (rounded up to pages); <= 0: every
                                free byte of HBM but a 4 GiB reserve */
  int32_t max_step_tokens;   /* max packed rows per step (prefill + decode) */
  int32_t max_seqs;          /* max sequences (slices + decodes) per step */
  int32_t max_context;       /* max position + 1 (RoPE table size) */
  const struct tc_instance* share_weights; /* optional: reuse this instance's weights (same device,
                                              dims and seed) -- several instances on one GPU */
  const struct tc_instance* share_kv_pool; /* optional: draw KV pages from this instance's pool (same
                                              device and KV geometry; kv_pool_tokens is then ignored):
                                              co-located instances share one HBM budget */
} tc_instance_desc;

tc_status tc_instance_create(const tc_instance_desc* desc, tc_instance** out);
tc_status tc_instance_destroy(tc_instance* inst);

/* One prompt slice of a chunked prefill: tokens [pos0, pos0 + n_tokens) of
 * request req_id. want_logits = 1 when this slice finishes the prompt (the next
 * token is sampled from its last row). */
typedef struct {
  int64_t req_id;
  int32_t pos0;
  int32_t n_tokens;
  const int32_t* token_ids;
  int32_t want_logits;
} tc_prefill_slice;

/* One decode row: feed token_id at position pos (KV grows to pos + 1). */
typedef struct {
  int64_t req_id;
  int32_t pos;
  int32_t token_id;
} tc_decode_item;

enum { TC_STEP_KEEP_LOGITS = 1 }; /* copy fp32 logits of sampled rows to the result */

/* A hybrid step: the GPU form of BatchPlan (cluster.hpp:41-46). */
typedef struct {
  int32_t n_prefill;
  const tc_prefill_slice* prefill;
  int32_t n_decode;
  const tc_decode_item* decode;
  int32_t flags;
} tc_step_desc;

/* Sampled ids are ordered: prefill slices with want_logits (in order), then decodes. */
typedef struct {
  int32_t n_sampled;
  int32_t* sampled_ids;   /* caller buffer, capacity >= n_decode + n_prefill */
  float* logits;          /* optional caller buffer [n_sampled * vocab] (TC_STEP_KEEP_LOGITS) */
  float gpu_ms;           /* device time of the step (CUDA events on the instance stream) */
  int32_t launches;       /* kernels this library launched for the step */
  int64_t h2d_bytes;      /* host->device bytes copied for the step (token ids + metadata) */
  int64_t d2h_bytes;      /* device->host bytes read back (sampled ids [+ logits]) */
  int32_t attn_pf_sms;    /* SMs given to prefill attention beside decode attention (0 = serial) */
} tc_step_result;

/* Enqueue a step (asynchronous); pages for new positions are allocated here. */
tc_status tc_step_launch(tc_instance* inst, const tc_step_desc* step);
/* Wait for the last launched step and read back its sampled token ids. */
tc_status tc_step_wait(tc_instance* inst, tc_step_result* result);

/* Ensure pages for positions [0, n_tokens) of req_id; tc_kv_release frees them. */
tc_status tc_kv_reserve(tc_instance* inst, int64_t req_id, int64_t n_tokens);
tc_status tc_kv_release(tc_instance* inst, int64_t req_id);
/* Pages currently held by req_id (0 if none) and free pages in the pool. */
tc_status tc_kv_stats(tc_instance* inst, int64_t req_id, int64_t* req_pages, int64_t* free_pages);

/* KV migration -- replaces transfer_time_ms at engine.hpp:402 (degrade / backflow) and
 * engine.hpp:516 (init); cost_model.hpp:81-85.
 *
 * tc_kv_migrate_async moves the KV of req_id from src to dst: every page src holds for it (at
 * least the first n_tokens rows; a step in flight on src may have written one more row). Pages on
 * dst are allocated now; the copy kernel runs on src's high-priority copy stream for dst, after
 * src's in-flight step, and pushes over NVLink when the instances are on different GPUs. The call
 * never blocks: src's pages return to its pool when the copy completes, and dst's next step that
 * touches req_id (and any later migration or release of it) orders after the copy on the GPU.
 * Several migrations may be in flight from and to one instance. The returned event reports
 * completion and the copy's device time; destroy it when done (the copy is unaffected). */
typedef struct tc_event tc_event;
tc_status tc_kv_migrate_async(tc_instance* src, tc_instance* dst, int64_t req_id, int64_t n_tokens, tc_event** ev);
tc_status tc_event_query(tc_event* ev, int32_t* done);                      /* non-blocking */
tc_status tc_event_wait(tc_event* ev, float* copy_ms, int64_t* bytes);      /* blocks until the copy is done */
tc_status tc_event_destroy(tc_event* ev);
/* Synchronous form (one migration per source at a time): tc_kv_migrate, then tc_kv_migrate_wait
 * returns the copy's device time and bytes. */
tc_status tc_kv_migrate(tc_instance* src, tc_instance* dst, int64_t req_id, int64_t n_tokens);
tc_status tc_kv_migrate_wait(tc_instance* src, float* copy_ms, int64_t* bytes);
/* Grid of the copy kernel (0 = 2 x SMs, full bandwidth; fewer CTAs leave SMs to the steps). */
tc_status tc_set_migration_ctas(tc_instance* inst, int32_t ctas);

/* Cross-process KV migration (one process per GPU, the deployment bench.py --gpus N uses).
 * The destination process exports its KV pool (CUDA IPC handle, TC_IPC_HANDLE_BYTES opaque bytes)
 * and reserves pages for the request (tc_kv_reserve + tc_kv_pages); the source process imports the
 * pool once and pushes pages with tc_kv_push_pages: the same copy kernel as tc_kv_migrate_async,
 * on src's copy stream after its in-flight step, its stores going over NVLink to the peer GPU.
 * Page bookkeeping stays with each owner: the destination's page list travels with the control
 * message (the reference engine's Migration record, engine.hpp:388-413), the source releases its
 * pages (tc_kv_release) once the event completed. Same-GPU imports (two processes on one GPU)
 * work too; they are what the single-GPU tests exercise. */
#define TC_IPC_HANDLE_BYTES 64
typedef struct tc_remote_pool tc_remote_pool;
tc_status tc_kv_pool_export(tc_instance* inst, void* handle /* TC_IPC_HANDLE_BYTES */, int64_t* page_bytes,
                            int64_t* n_pages);
tc_status tc_kv_pool_import(int32_t device, const void* handle, int64_t page_bytes, int64_t n_pages,
                            tc_remote_pool** out);
tc_status tc_remote_pool_close(tc_remote_pool* pool);
tc_status tc_kv_push_pages(tc_instance* src, tc_remote_pool* dst, const int32_t* src_pages, const int32_t* dst_pages,
                           int32_t n_pages, tc_event** ev);

/* Device pointer of the KV pool and its geometry (tests / tools). */
tc_status tc_kv_pool_info(tc_instance* inst, void** base, int64_t* page_bytes, int64_t* n_pages);
/* Page list of req_id (caller buffer of capacity max_pages). */
tc_status tc_kv_pages(tc_instance* inst, int64_t req_id, int32_t* pages, int32_t max_pages, int32_t* n_pages);
/* Device pointer of a named weight ("embed", "lm_head", "final_norm", "L<i>.qkv",
 * "L<i>.qkv_bias", "L<i>.o", "L<i>.gate_up", "L<i>.down", "L<i>.attn_norm", "L<i>.mlp_norm"). */
tc_status tc_weight_ptr(tc_instance* inst, const char* name, void** ptr, int64_t* rows, int64_t* cols);
/* Synchronous device -> host copy of `bytes` at a library-owned device pointer (tools/tests). */
tc_status tc_read_device(void* host_dst, const void* dev_src, size_t bytes);
/* The deterministic init: bf16 bits of element (row, col) of logical tensor tensor_id. */
uint16_t tc_weight_value(uint64_t seed, uint64_t tensor_id, int64_t index, float scale, float offset);

/* Kernel-level entry points on caller device pointers (parity tests, microbench).
 * epilogue: 0 bf16, 1 bf16+bias, 2 fp32 residual add, 3 SwiGLU (64-interleaved), 4 fp32.
 * bn = 0 picks the tile width; k_splits = 0 picks split-K automatically. */
tc_status tc_gemm(int32_t device, const void* a, const void* b, void* out, const void* bias, int32_t m, int32_t n,
                  int32_t k, int32_t epilogue, int32_t bn, int32_t k_splits, void* stream);
tc_status tc_copy_pages(const void* src_pool, void* dst_pool, const int32_t* src_pages_dev,
                        const int32_t* dst_pages_dev, int32_t n_pages, int64_t page_bytes, void* stream);

/* Per-kernel device time of the last step (ms) for the named phase, e.g.
 * "gemm_qkv", "attn", "gemm_o", "gemm_gate_up", "gemm_down", "lm_head" (summed
 * over layers). Enabled by tc_set_profiling(inst, 1) (adds events per kernel). */
tc_status tc_set_profiling(tc_instance* inst, int32_t on);
tc_status tc_phase_ms(tc_instance* inst, const char* phase, float* ms);

const char* tc_last_error(void);
const char* tc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TAICHI_B200_H_ */
