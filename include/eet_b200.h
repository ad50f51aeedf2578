/*
 * eet_b200.h — C ABI of the B200-native EET decoder-layer path.
 *
 * Plain pointers, sizes and a CUDA stream handle (passed as void*); no torch
 * types. Every entry point returns an eet_status (0 = OK); eet_last_error()
 * gives the message of the last failure on the calling thread. All compute
 * entry points are stream-ordered and asynchronous.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/maskfold/<file>:<line>). The Python host package
 * (paper_2104_12470_b200) binds this ABI with ctypes and mirrors the
 * reference's operator names, argument meaning and error behaviour.
 *
 * Conventions
 *   - dtype: EET_F32 (reference "fp32 mode"), EET_BF16, EET_F16.
 *   - Weights are stored K-major ("[out, in]", i.e. the reference's x @ W with
 *     W transposed once on upload); the fused QKV weight is [3h, h] = [Wq;Wk;Wv]^T.
 *   - Hidden state x is float32 [b, t, h] with batch stride x_sb and slot
 *     stride x_ss (elements), so the reference's strided activation view
 *     acts.hidden[:b, :t] (runtime.py:407) is accepted as-is.
 *   - Left padding (core.py:98-123): pads[b] in [0, seq_len); sequence b's
 *     real tokens occupy slots [pads[b], seq_len).
 *   - KV cache per layer: K and V each [b_max, heads, s_max, hd] in the layer
 *     dtype (memory.py:237-307).
 */
#ifndef EET_B200_H
#define EET_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  EET_OK = 0,
  EET_ERR_SHAPE = 1,     /* maps to ValueError          */
  EET_ERR_OVERFLOW = 2,  /* maps to CacheOverflowError  */
  EET_ERR_CUDA = 3,      /* maps to RuntimeError        */
  EET_ERR_POOL = 4,      /* maps to PoolError           */
  EET_ERR_ARG = 5,       /* maps to ValueError          */
  EET_ERR_UNSUPPORTED = 6
} eet_status;

typedef enum { EET_F32 = 0, EET_BF16 = 1, EET_F16 = 2 } eet_dtype;

typedef enum { EET_SCOPE_WITHIN = 0, EET_SCOPE_ACROSS = 1 } eet_scope;

typedef enum { EET_PHASE_PROMPT = 0, EET_PHASE_INCREMENTAL = 1 } eet_phase;

/* ---------------------------------------------------------------- library */
const char* eet_last_error(void);
int eet_abi_version(void);

/* Number of kernel launches issued by this library since load (the bench's
 * gpu_launches evidence). */
uint64_t eet_launch_count(void);

/* Per-launch profiler (bench.py's roofline numbers): while enabled, each
 * launch outside graph capture is bracketed by CUDA events on its own
 * stream and tagged with its algorithmic bytes / flops. enable(1) resets.
 * summary(kind): launches, summed device ms, bytes and flops of that kind. */
int eet_profile_enable(int on);
int eet_profile_kinds(void);
const char* eet_profile_kind_name(int kind);
int eet_profile_summary(int kind, uint64_t* count, double* total_ms,
                        double* bytes, double* flops);

/* ------------------------------------------------------------- folding plan
 * Replaces folding.py:30-54 (plan_folding). Pure host arithmetic; the row
 * kernels take their launch shape from it. */
int eet_plan_folding(int logical_size, int unit_cap, int* fold_count,
                     int* sub_block_count, int* threads_per_block);

/* ------------------------------------------------------------ buffer pool
 * Device arena with the reference's two-scope reuse policy and ledger
 * (memory.py:136-214 BufferPool, :44-87 AllocationLog). Sizes are BYTES.
 * WITHIN reuses an idle buffer only on exact capacity match; ACROSS reuses
 * the first idle buffer (creation order) with capacity >= size; otherwise
 * cudaMalloc. Buffers are never freed before eet_pool_destroy. */
typedef struct eet_pool eet_pool;
int eet_pool_create(eet_pool** out);
/* device_backed = 0: an accounting-only arena (host allocations, same
 * policy and ledger) for planning and CPU-side policy checks. */
int eet_pool_create_ex(eet_pool** out, int device_backed);
int eet_pool_destroy(eet_pool* pool);
int eet_pool_request(eet_pool* pool, size_t bytes, int scope, const char* tag,
                     int* handle, void** dptr, size_t* capacity, int* reused);
/* bytes: the size the claim requested (recorded in the ledger). */
int eet_pool_release(eet_pool* pool, int handle, size_t bytes);
/* stats[0..3] = total_capacity, peak_in_use, malloc_count, reuse_count */
int eet_pool_stats(eet_pool* pool, uint64_t stats[4]);
int eet_pool_ledger_size(eet_pool* pool, size_t* n);
/* buffer i in creation order: capacity (bytes) and whether it is idle */
int eet_pool_buffer_count(eet_pool* pool, size_t* n);
int eet_pool_buffer_info(eet_pool* pool, size_t i, uint64_t* capacity, int* idle);
/* Debug poisoning: fill every idle buffer with the byte `value` (0xFF makes
 * every fp32 / fp16 / bf16 element a NaN), synchronously. A later request
 * that reuses the buffer sees the pattern, so a kernel that reads scratch it
 * never wrote shows up as non-finite output. No reference counterpart
 * (the reference's numpy buffers come zeroed or written). */
int eet_pool_debug_fill(eet_pool* pool, int value);
/* event: 0 request, 1 release; decision: 0 malloc, 1 reuse, 2 idle */
int eet_pool_ledger_get(eet_pool* pool, size_t i, int* event, uint64_t* bytes,
                        int* decision, char* tag, size_t tag_cap);

/* ------------------------------------------------ operator-level kernels */
/* In-place mask-fused softmax over [batch*heads, seq, seq] fp32 planes.
 * causal=1: fused_causal_softmax (attention.py:73-104);
 * causal=0: fused_padding_softmax (attention.py:107-135).
 * d_pads: device int32[batch]. fold_cap: unit cap of the folding plan
 * (folding.py:30-54; 0 = default 1024). */
int eet_masked_softmax(float* scores, const int* d_pads, int batch, int heads,
                       int seq, int causal, int fold_cap, void* stream);

/* In-place decode-step softmax over [batch, heads, len] fp32, window
 * [pads[b], len) (attention.py:138-163). */
int eet_step_softmax(float* scores, const int* d_pads, int batch, int heads,
                     int len, int fold_cap, void* stream);

/* Row layer norm (runtime.py:83-94), fp32 in/out: y = LN(x)*g + b. */
int eet_layer_norm(const float* x, const float* gamma, const float* beta,
                   float* y, int rows, int hidden, int fold_cap, void* stream);

/* Mask-fused multi-head attention, fp32 q/k/v/out [b, s, h]
 * (mha_forward, attention.py:172-217). Pad-query rows come out zero; keys
 * below pads[b] are never read. */
int eet_mha_forward(const float* q, const float* k, const float* v, float* out,
                    const int* d_pads, int batch, int seq, int hidden,
                    int heads, int causal, void* stream);

/* Dense C[M,N] = A[M,K] * B[N,K]^T (+bias) in the given dtype (fp32 accum);
 * C is float32 [M, ldc]. Used by tests and the LM head. */
int eet_gemm(int dtype, const void* A, const void* B, const float* bias,
             float* C, int M, int N, int K, int ldc, void* stream);

/* Weight packing on the device: dst[c][r] = (dtype) src[r][c] for a
 * row-major float32 src [rows, cols]. Turns the reference's [in, out]
 * matrices (weights.py:31-51; MFW1 payload, weights.py:142-204) into the
 * K-major [out, in] compute layout without a host-side transpose. */
int eet_transpose_cast(int dtype, const float* src, int rows, int cols, void* dst, void* stream);

/* Decode projection kernel of the incremental phase (gemv_cl.cu; the
 * per-token halves of runtime.py:131-136, :188, :206-213) as a test /
 * micro-benchmark entry: W [N, K] K-major 16-bit, M <= 16 token rows.
 * x == NULL: input X [M, K] 16-bit (ld K); x != NULL: input LayerNorm(x)
 * of fp32 rows x [M, K] (ld K) with g, b [K] (runtime.py:83-94).
 * mode 0: out = fp32 [M, N]; mode 2: out = 16-bit GELU(.) [M, N];
 * mode 3: out (fp32 [M, N]) += result (residual). EET_ERR_UNSUPPORTED for
 * shapes the kernel does not take (K % 64, M > 16, ...). */
int eet_gemv_decode(int dtype, const void* w, int N, int K, const void* X, const float* x, const float* g,
                    const float* b, int M, int mode, void* out, void* stream);

/* In-graph ablation for timing: comma list of decode launches to leave out
 * of eet_generate's decode steps ("qkv,attn,o,w1,w2,head"; "" = none).
 * Results are wrong while set; bench.py derives per-kernel in-graph times
 * from the step-time deltas (programmatic dependent launch intact). */
int eet_debug_skip(const char* spec);

/* Calibration: microseconds per grid-wide barrier of a persistent kernel
 * with `ctas` CTAs (mode 0: flat arrival counter, 1: cluster-hierarchical). */
int eet_debug_grid_barrier(int n, int ctas, int mode, float* us_per_barrier);

/* Calibration: n dependent launches of an empty kernel (ctas CTAs), with or
 * without programmatic dependent launch; counter may be NULL. */
int eet_debug_launch_chain(int n, int ctas, int pdl, int* counter, void* stream);

/* Development trace of the split-K cluster decode GEMV / LM head
 * (gemv_cl.cu): on = 1 resets and enables it; on = 0 disables it and copies
 * out <= 8192 records of 24 int64 [(N << 32) | (K << 1) | ln, block, start,
 * wait passed, X staged, weights landed, partials sent, end (globaltimer),
 * then clock64 offsets of the phase ends of CTA 0]. */
int eet_debug_cltrace(int on, long long* out, int* n);
/* Development trace of the fused decode kernels: on = 1 resets and
 * enables, on = 0 disables and copies out (out: 8192 x 8 int64, n: 2 ints)
 * up to 4096 attn_o.cu records [sequence, head, start, wait passed,
 * attention done, contexts gathered, end] and, from row 4096, up to 4096
 * qkv_attn_o.cu records [sequence << 16 | head, start, wait passed, LN
 * staged, q/k/v reduced, attention done, contexts gathered, end]
 * (globaltimer ns, one per CTA). */
int eet_debug_aotrace(int on, long long* out, int* n);

/* ------------------------------------------------------------ layer path */
typedef struct {
  const float* ln1_g; const float* ln1_b;      /* [h]                   */
  const void*  wqkv;                           /* [3h, h]  layer dtype  */
  const void*  wo;                             /* [h, h]                */
  const float* ln2_g; const float* ln2_b;      /* [h]                   */
  const void*  w1;                             /* [4h, h]               */
  const void*  w2;                             /* [h, 4h]               */
  const float* b_qkv; const float* b_o;        /* optional biases (NULL) */
  const float* b_1;   const float* b_2;
} eet_layer_weights;

typedef struct eet_runtime eet_runtime;

/* One runtime per (device, dtype, capacities). Owns device scratch for row
 * maps and split-K partials; activation scratch comes from `pool`. */
int eet_runtime_create(eet_runtime** out, int dtype, int hidden, int heads,
                       int max_batch, int max_sequence, eet_pool* pool);
int eet_runtime_destroy(eet_runtime* rt);

/* decoder_layer_forward (runtime.py:217-263), in place on x.
 *   phase PROMPT: t == seq_len, attends causally within the prompt and writes
 *                 K/V for slots [kv_filled, kv_filled+t);
 *   phase INCREMENTAL: t == 1, appends slot kv_filled and attends over
 *                 [pads[b], kv_filled]. The caller advances the cursor.
 * kcache/vcache: this layer's [b_max, heads, s_max, hd] tensors.
 * h_pads: HOST int32[b]. Pad rows of x are neither read nor written. */
int eet_decoder_layer_forward(eet_runtime* rt, float* x, long long x_sb,
                              long long x_ss, int batch, int t,
                              const eet_layer_weights* w, void* kcache,
                              void* vcache, int kv_filled, const int* h_pads,
                              int seq_len, int phase, void* stream);

/* Windowed prompt pass (new; SURVEY App. B.1 — the reference is left-pad
 * only): sequence b's valid slots are [h_start[b], h_end[b]) of the t-slot
 * rows of x, e.g. right padding = start 0, end len_b. Same layout, cache and
 * kernels as eet_decoder_layer_forward with phase PROMPT (kv cursor 0); slots
 * outside the window are skipped, not masked, and K/V is written only for
 * the window. Incremental steps need one common cursor: left-pad batches. */
int eet_decoder_layer_forward_window(eet_runtime* rt, float* x, long long x_sb,
                                     long long x_ss, int batch, int t,
                                     const eet_layer_weights* w, void* kcache,
                                     void* vcache, const int* h_start,
                                     const int* h_end, void* stream);
int eet_encoder_layer_forward_window(eet_runtime* rt, float* x, long long x_sb,
                                     long long x_ss, int batch, int t,
                                     const eet_layer_weights* w,
                                     const int* h_start, const int* h_end,
                                     void* stream);

/* encoder_layer_forward (runtime.py:266-301): bidirectional, no cache. */
int eet_encoder_layer_forward(eet_runtime* rt, float* x, long long x_sb,
                              long long x_ss, int batch, int t,
                              const eet_layer_weights* w, const int* h_pads,
                              void* stream);

/* ------------------------------------------------------- tensor parallel
 * Megatron split for h >= 4096: each rank holds heads/tp
 * heads (wqkv [3*h/tp, h], wo [h, h/tp]) and 4h/tp FFN columns (w1
 * [4h/tp, h], w2 [h, 4h/tp]); LN parameters and x are replicated. A layer is
 *   p = attention_partial(x); all_reduce(p); residual_add(x, p);
 *   p = ffn_partial(x);       all_reduce(p); residual_add(x, p);
 * with the all-reduce (sum over ranks of [rows, h]) done by the caller's
 * communicator (NCCL over NVLink). Partials are fp32 for EET_F32 and the
 * layer dtype for EET_BF16 / EET_F16 (half the NVLink bytes). `rows`
 * returns the packed valid-token count.
 * Row-chunked form (the all-reduce of one chunk overlaps the GEMM of the
 * next): attention_core (LN1, QKV, attention; context kept by the runtime)
 * then attention_out(r0, r1) per chunk of packed rows; ffn_mid (LN2, W1,
 * GELU; intermediate kept) then ffn_out(r0, r1); partial_rows points at row
 * r0 of the caller's partial. The reference has no TP; these
 * stages are new. */
int eet_runtime_create_tp(eet_runtime** out, int dtype, int hidden,
                          int heads_total, int tp_rank, int tp_size,
                          int max_batch, int max_sequence, eet_pool* pool);
int eet_tp_attention_partial(eet_runtime* rt, const float* x, long long x_sb,
                             long long x_ss, int batch, int t,
                             const eet_layer_weights* w, void* kcache,
                             void* vcache, int kv_filled, const int* h_pads,
                             int seq_len, int phase, void* partial, int* rows,
                             void* stream);
int eet_tp_attention_core(eet_runtime* rt, const float* x, long long x_sb,
                          long long x_ss, int batch, int t,
                          const eet_layer_weights* w, void* kcache,
                          void* vcache, int kv_filled, const int* h_pads,
                          int seq_len, int phase, int* rows, void* stream);
int eet_tp_attention_out(eet_runtime* rt, const eet_layer_weights* w, int r0,
                         int r1, void* partial_rows, void* stream);
int eet_tp_ffn_partial(eet_runtime* rt, const float* x, long long x_sb,
                       long long x_ss, const eet_layer_weights* w,
                       void* partial, void* stream);
int eet_tp_ffn_mid(eet_runtime* rt, const float* x, long long x_sb,
                   long long x_ss, const eet_layer_weights* w, void* stream);
int eet_tp_ffn_out(eet_runtime* rt, const eet_layer_weights* w, int r0,
                   int r1, void* partial_rows, void* stream);
int eet_tp_residual_add(eet_runtime* rt, float* x, long long x_sb, long long x_ss,
                        const void* reduced, void* stream);

/* ------------------------------------------------------------- generation */
typedef struct {
  int layers, vocab, max_sequence;
  const void* tok_emb;       /* [vocab, h]  layer dtype      */
  const void* pos_emb;       /* [s_max, h]  layer dtype      */
  const eet_layer_weights* layer;   /* [layers]              */
  const float* lnf_g; const float* lnf_b;
  const void* head;          /* [vocab, h] K-major (output_head^T) */
  void* const* kcache;       /* [layers] device pointers     */
  void* const* vcache;
  float* hidden;             /* activation cache [b_max, max_prompt, h] fp32 */
  int max_prompt;
} eet_model;

/* generate (runtime.py:372-437): one prompt pass, then `steps` incremental
 * steps captured once into a CUDA graph and replayed. In 16-bit modes a
 * decode step is embed -> per layer [LN1 + QKV + attention + out-projection
 * in one kernel, LN2 + W1, W2] -> LN + LM head + argmax (where the shapes
 * allow; the five-launch layer otherwise). Deterministic: repeated calls
 * give bit-identical tokens and logits. Greedy argmax with the lowest id on
 * ties. h_prompts: HOST int32 [batch, max_len] padded with
 * anything past each length; h_lengths: HOST int32[batch].
 * h_tokens: HOST int64 [batch, steps] (written on return).
 * d_logits: optional DEVICE fp32 [steps, batch, vocab] (may be NULL).
 * use_graph: 0 runs the decode step eagerly (debug). */
int eet_generate(eet_runtime* rt, const eet_model* model,
                 const int* h_prompts, const int* h_lengths, int batch,
                 int max_len, int steps, long long* h_tokens, float* d_logits,
                 int use_graph, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EET_B200_H */
