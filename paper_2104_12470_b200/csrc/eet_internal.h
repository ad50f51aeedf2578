// Internal declarations shared by the CUDA translation units of libeet_b200.
// Not part of the public ABI (include/eet_b200.h is).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <string>
#include <atomic>
#include <utility>

#include "../../include/eet_b200.h"

namespace eet {

// ----------------------------------------------------------- error plumbing
void set_error(const std::string& msg);
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Per-launch profiler (eet_profile_*): when enabled and the stream is not
// capturing, each launch is bracketed by CUDA events on its own stream and
// tagged with its algorithmic bytes / flops. Also counts every launch.
enum KernelKind : int {
  K_LAYERNORM = 0, K_SOFTMAX, K_EMBED, K_ARGMAX, K_ADVANCE, K_GEMM_F32, K_GEMV,
  K_GEMM_TC, K_ATTN_PREFILL, K_ATTN_DECODE, K_DECODE_STEP, K_KIND_COUNT
};
struct ProfScope {
  int slot = -1;
  bool graph = false;
  cudaStream_t st;
  // bytes/flops: fixed part; *_per_key: scaled by the attended key count of
  // the replay when the launch sits in a captured decode graph (keys unknown
  // at capture time), see prof_after_replay()
  ProfScope(int kind, cudaStream_t st, double bytes, double flops, double bytes_per_key = 0,
            double flops_per_key = 0);
  ~ProfScope();
};
bool prof_on();
// after a graph replay: sync `st`, fold the captured launches in (keys = the
// replay's attended keys summed over the batch)
void prof_after_replay(cudaStream_t st, double keys);
void prof_graph_reset();

struct Fail {
  int code;
};

#define EET_CHECK_CUDA(expr)                                                   \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::eet::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));    \
      throw ::eet::Fail{EET_ERR_CUDA};                                         \
    }                                                                          \
  } while (0)

#define EET_REQUIRE(cond, code, msg)                                           \
  do {                                                                         \
    if (!(cond)) {                                                             \
      ::eet::set_error(msg);                                                   \
      throw ::eet::Fail{code};                                                 \
    }                                                                          \
  } while (0)

// EET_SYNC_DEBUG=1: synchronise after every launch and name it on stderr
// (locates a hanging or faulting kernel; never set during timing).
bool sync_debug();
void sync_debug_after(const char* file, int line);
#define EET_LAUNCH_CHECK()                                                     \
  do {                                                                         \
    EET_CHECK_CUDA(cudaGetLastError());                                        \
    if (::eet::sync_debug()) ::eet::sync_debug_after(__FILE__, __LINE__);      \
  } while (0)

// ------------------------------------------------------------ folding plan
// folding.py:30-54: minimal k with ceil(n / 2^k) <= cap.
struct FoldPlan {
  int fold_count, sub_blocks, threads;
};
FoldPlan plan_folding(int logical, int cap);

// --------------------------------------------------------------- epilogue
// What a GEMM-like kernel does with accumulator element (m, n).
enum EpiMode : int {
  EPI_STORE_F32 = 0,  // out_f32[m*ldo + n] = acc + bias
  EPI_STORE_T = 1,    // out_T[m*ldo + n]   = acc + bias          (layer dtype)
  EPI_GELU_T = 2,     // out_T[m*ldo + n]   = gelu(acc + bias)
  EPI_RESID = 3,      // x[b*x_sb + t*x_ss + n] += acc + bias      (row map)
  EPI_QKV = 4,        // n<hq: q_T[m*hq+n]; else K/V cache scatter (row map)
  EPI_ARGMAX = 5,     // LM head: greedy token per row (lm_head_argmax only), optional logits
};

// Pending residual in 2^-32 fixed point (decode out-projection, attn_o.cu):
// contributions are added with integer atomics, so their sum does not
// depend on arrival order; consumers read x + pend(acc) and the W2 epilogue
// folds it into x and re-zeroes it.
constexpr float kAccScale = 4294967296.0f;            // 2^32
constexpr float kAccInv = 2.3283064365386963e-10f;    // 2^-32
__device__ __forceinline__ float acc_to_f(long long a) { return __ll2float_rn(a) * kAccInv; }

struct Epi {
  int mode = EPI_STORE_F32;
  long long* acc = nullptr;       // EPI_RESID (decode GEMV): pending fixed-point residual rows, ld acc_sb
  long long acc_sb = 0;
  const float* bias = nullptr;
  void* out = nullptr;
  int ldo = 0;
  // residual (EPI_RESID) / cache scatter (EPI_QKV): packed row m -> (b, t)
  float* x = nullptr;
  long long x_sb = 0, x_ss = 0;
  const int2* rinfo = nullptr;
  // EPI_QKV
  void* kc = nullptr;
  void* vc = nullptr;
  int heads = 0, hd = 0, hq = 0, smax = 0;
  const int* kv_start = nullptr;  // device scalar (may be null) ...
  int kv_base = 0;                // ... plus this: first cache slot of the step
  // EPI_ARGMAX (runtime.py:425: lowest id on ties); out = optional logits
  // [steps, batch, vocab] written at step *d_step
  int2* cand = nullptr;           // [rtiles * 16] (value bits, id) per tile and row
  int* ticket = nullptr;          // zero on entry, left zero
  int* cur = nullptr;             // [batch] next token
  long long* toks = nullptr;      // [batch, steps]
  const int* d_step = nullptr;
  int steps = 0, batch = 0;
};

// ---------------------------------------------------------------- launchers
// Row ops (rowops.cu)
void launch_layer_norm(const float* x, long long x_sb, long long x_ss,
                       const int2* rinfo, int rows, const float* g,
                       const float* b, void* y, int y_dtype, int ldy, int h,
                       int fold_cap, cudaStream_t st);
void launch_masked_softmax(float* s, const int* pads, int batch, int heads,
                           int seq, int causal, int fold_cap, cudaStream_t st);
void launch_step_softmax(float* s, const int* pads, int batch, int heads,
                         int len, int fold_cap, cudaStream_t st);
void launch_embed_prompt(int dtype, const void* tok, const void* pos,
                         const int* prompts, int max_len, const int* pads,
                         float* x, long long x_sb, int batch, int t, int h,
                         cudaStream_t st);
void launch_embed_step(int dtype, const void* tok, const void* pos,
                       const int* cur_tok, const int* pads,
                       const int* d_filled, float* x, long long x_sb,
                       int batch, int h, cudaStream_t st);
void launch_argmax(const float* logits, int batch, int vocab, int* cur_tok,
                   long long* tokens_out, int steps, const int* d_step,
                   float* logits_all, cudaStream_t st);
void launch_advance(int* d_filled, int* d_step, cudaStream_t st);
void launch_residual_add(float* x, long long x_sb, long long x_ss, const int2* rinfo,
                         const void* reduced, int dtype, int rows, int h, cudaStream_t st);

// GEMMs (gemm_simt.cu / gemm_tc.cu). C = A[M,K] * B[N,K]^T, fp32 accumulate.
void gemm_f32_simt(const float* A, int lda, const float* B, int ldb, int M,
                   int N, int K, const Epi& e, cudaStream_t st);
void gemv_small_m(int dtype, const void* A, int lda, const void* B, int ldb,
                  int M, int N, int K, const Epi& e, cudaStream_t st);
void gemm_tc_sm100(int dtype, const void* A, int lda, const void* B, int ldb,
                   int M, int N, int K, const Epi& e, cudaStream_t st);
void gemv_tc_sm100(int dtype, const void* A, int lda, const void* B, int ldb,
                   int M, int N, int K, const Epi& e, cudaStream_t st);
// decode GEMV with the LayerNorm of its input rows fused into the prologue;
// false when the shape is not eligible (caller runs LN + gemm instead)
bool gemv_tc_ln_sm100(int dtype, const float* x, long long x_sb, long long x_ss,
                      const int2* rinfo, const float* g, const float* b, const void* B,
                      int ldb, int M, int N, int K, const Epi& e, cudaStream_t st);
// fp32 GEMM as 3xTF32 on tcgen05 (gemm_tf32.cu); false when not eligible
bool gemm_tf32x3(const float* A, int lda, const float* B, int ldb, int M, int N, int K, const Epi& e,
                 cudaStream_t st);
// deterministic split-K second stage (partials summed in split order) + epilogue
void launch_splitk_reduce(const float* part, int splits, int M, int N, const Epi& e, cudaStream_t st);
// Dispatch by dtype and M (the one GEMM entry the runtime uses).
void gemm(int dtype, const void* A, int lda, const void* B, int ldb, int M,
          int N, int K, const Epi& e, cudaStream_t st);

// Attention (attention.cu)
struct PrefillArgs {
  int dtype;
  const void* q; int ldq; const int* q_rowbase;   // q row = q_rowbase[b] + slot
  const void* k; const void* v;                   // (b,head,slot,d) strides
  long long k_sb, k_sh, k_ss;
  void* o; int ldo; const int* o_rowbase;
  const int* pads;
  const int* h_pads;   // host copy for byte/flop accounting (may be null)
  int batch, seq, heads, hd;
  float scale;
  int causal;
  int zero_pad_rows;   // padded layout: write zero rows for pad queries
  int q_rows;          // rows of the packed q buffer (TMA extent)
  const int* ends = nullptr;     // [b] valid end per sequence (windows); nullptr: seq
  const int* h_ends = nullptr;   // host copy (work list, accounting)
};
void launch_attn_prefill(const PrefillArgs& a, cudaStream_t st);
bool attn_prefill_tc(const PrefillArgs& a, int q_rows, cudaStream_t st, double bytes, double flops);

struct DecodeArgs {
  int dtype;
  const void* q; int ldq;              // row b
  const void* kc; const void* vc;      // [b, heads, smax, hd]
  int batch, heads, hd, smax;
  const int* pads;
  const int* kv_start;                 // keys [pad_b, (*kv_start) + kv_base + 1)
  int kv_base;
  const int* h_pads;                   // host copies for byte accounting only
  int L_host;                          // (-1: unknown, e.g. inside a graph)
  float scale;
  float* part;                         // [b, heads, splits, hd + 2]
  int* counters;                       // [b * heads], zero on entry, left zero
  void* o; int ldo;                    // row b
  int splits;
  unsigned long long kv_policy = 0;    // L2 cache hint of the K/V bulk copies (0: none)
};
void launch_attn_decode(const DecodeArgs& a, cudaStream_t st);
// decode attention fused with the out-projection + residual (attn_o.cu);
// false when not eligible (16-bit, hd 64/128, one CTA per (sequence, head))
bool launch_attn_o(const DecodeArgs& a, const void* wo, int h, long long* acc, long long acc_sb,
                   const float* bias, cudaStream_t st);

// ---- decode projections / LM head straight from the K-major weights (gemv_cl.cu)
// acc (LayerNorm source only): pending fixed-point residual rows added to x
bool gemv_cl(int dtype, const void* W, int M, int N, int K, const void* X, int ldx, const float* x,
             long long x_sb, long long x_ss, const int2* rinfo, const float* g, const float* b, const Epi& e,
             cudaStream_t st, const long long* acc = nullptr, long long acc_sb = 0);
// decode LN1 + QKV + attention + out-projection in one kernel (qkv_attn_o.cu)
bool qkv_attn_o_ok(int dtype, int batch, int h, int heads, int hd, int hq, const float* x, long long x_sb,
                   const void* kc, const void* vc, const void* wqkv, const void* wo);
bool launch_qkv_attn_o(int dtype, int batch, int h, int heads, int smax, const float* x, long long x_sb,
                       const float* g, const float* bl, const void* wqkv, const float* bqkv, void* kc, void* vc,
                       const int* pads, const int* kv_start, int kv_base, const void* wo, const float* bo,
                       long long* acc, long long acc_sb, int L_host, const int* h_pads, cudaStream_t st);
// would gemv_cl take this projection (same checks, no launch)
bool gemv_cl_ok(int dtype, const void* W, int M, int N, int K, const void* X, int ldx, const float* x,
                long long x_sb, const float* g, const float* b, int mode);
bool lm_head_argmax(int dtype, const void* W, int M, int N, int K, const float* x, long long x_sb, long long x_ss,
                    const int2* rinfo, const float* g, const float* b, const Epi& e, cudaStream_t st);
// decode attention split plan (attention.cu)
int decode_splits(int batch, int heads, int smax, int hd, int es);

// cudaLaunchKernelEx with optional programmatic-dependent-launch edge and
// cluster shape. Kernels launched with pdl=true must execute
// griddepcontrol.wait before touching memory written by earlier kernels.
bool pdl_enabled();                    // EET_NO_PDL=1 turns the PDL edges off (A/B, debugging)
template <typename... KArgs, typename... Args>
inline void launch_cfg(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       bool pdl, dim3 cluster, bool cluster_attr, Args&&... args) {
  pdl = pdl && pdl_enabled();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  int n = 0;
  if (pdl) {
    attrs[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_attr) {
    attrs[n].id = cudaLaunchAttributeClusterDimension;
    attrs[n].val.clusterDim.x = cluster.x;
    attrs[n].val.clusterDim.y = cluster.y;
    attrs[n].val.clusterDim.z = cluster.z;
    ++n;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = n;
  EET_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}
template <typename... KArgs, typename... Args>
inline void launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      bool pdl, dim3 cluster, Args&&... args) {
  launch_cfg(kernel, grid, block, smem, st, pdl, cluster, cluster.x * cluster.y * cluster.z > 1,
             std::forward<Args>(args)...);
}
// kernels that use cluster instructions (barrier.cluster, mapa, st.async):
// launched as a cluster even when it has one CTA
template <typename... KArgs, typename... Args>
inline void launch_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                           bool pdl, dim3 cluster, Args&&... args) {
  launch_cfg(kernel, grid, block, smem, st, pdl, cluster, true, std::forward<Args>(args)...);
}

// dtype helpers
inline size_t dtype_size(int dt) { return dt == EET_F32 ? 4 : 2; }

}  // namespace eet
