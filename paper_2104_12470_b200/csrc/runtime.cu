// C-ABI implementation (include/eet_b200.h): device buffer pool, operator
// entry points, the decoder/encoder layer orchestration and the two-phase
// generate loop with a CUDA-graph-captured decode step.
#include "common.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <mutex>
#include <vector>

namespace eet {

static thread_local std::string t_err;
std::atomic<uint64_t> g_launches{0};
void set_error(const std::string& msg) { t_err = msg; }

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("EET_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

bool sync_debug() {
  static const bool on = [] {
    const char* e = std::getenv("EET_SYNC_DEBUG");
    return e && e[0] == '1';
  }();
  return on;
}
void sync_debug_after(const char* file, int line) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(nullptr, &cs);
  std::fprintf(stderr, "[eet] launch %s:%d ... ", file, line);
  std::fflush(stderr);
  if (cs == cudaStreamCaptureStatusNone) {
    const cudaError_t e = cudaDeviceSynchronize();
    std::fprintf(stderr, "%s\n", cudaGetErrorString(e));
  } else {
    std::fprintf(stderr, "(capturing)\n");
  }
  std::fflush(stderr);
}

// ------------------------------------------------------------ profiler
namespace {
struct ProfRec {
  int kind;
  cudaEvent_t ev0, ev1;
  double bytes, flops, bytes_per_key, flops_per_key;
};
struct ProfAcc {
  uint64_t n = 0;
  double ms = 0, bytes = 0, flops = 0;
};
struct Profiler {
  bool on = false;
  std::vector<ProfRec> eager, graph;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> spare;
  size_t used = 0;
  ProfAcc acc[K_KIND_COUNT];
  std::pair<cudaEvent_t, cudaEvent_t> events() {
    if (used == spare.size()) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      spare.push_back({a, b});
    }
    return spare[used++];
  }
} g_prof;

const char* kKindNames[K_KIND_COUNT] = {"layernorm", "softmax", "embed", "argmax", "advance",
                                        "gemm_f32", "gemv", "gemm_tc", "attn_prefill",
                                        "attn_decode", "decode_step"};

void fold(const ProfRec& r, double keys) {
  float e = 0.f;
  EET_CHECK_CUDA(cudaEventElapsedTime(&e, r.ev0, r.ev1));
  ProfAcc& a = g_prof.acc[r.kind];
  a.n += 1;
  a.ms += e;
  a.bytes += r.bytes + r.bytes_per_key * keys;
  a.flops += r.flops + r.flops_per_key * keys;
}
}  // namespace

bool prof_on() { return g_prof.on; }

ProfScope::ProfScope(int kind, cudaStream_t s, double bytes, double flops, double bpk, double fpk)
    : st(s) {
  count_launch();
  if (!g_prof.on) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) return;
  auto ev = g_prof.events();
  graph = cs == cudaStreamCaptureStatusActive;
  if (graph) {   // an event-record node inside the captured graph
    cudaEventRecordWithFlags(ev.first, st, cudaEventRecordExternal);
    slot = (int)g_prof.graph.size();
    g_prof.graph.push_back(ProfRec{kind, ev.first, ev.second, bytes, flops, bpk, fpk});
  } else {
    cudaEventRecord(ev.first, st);
    slot = (int)g_prof.eager.size();
    g_prof.eager.push_back(ProfRec{kind, ev.first, ev.second, bytes, flops, 0, 0});
  }
}

ProfScope::~ProfScope() {
  if (slot < 0) return;
  if (graph) cudaEventRecordWithFlags(g_prof.graph[slot].ev1, st, cudaEventRecordExternal);
  else cudaEventRecord(g_prof.eager[slot].ev1, st);
}

void prof_after_replay(cudaStream_t st, double keys) {
  if (!g_prof.on || g_prof.graph.empty()) return;
  EET_CHECK_CUDA(cudaStreamSynchronize(st));
  for (const auto& r : g_prof.graph) fold(r, keys);
}

void prof_graph_reset() { g_prof.graph.clear(); }

}  // namespace eet

using namespace eet;

#define EET_API_BEGIN try {
#define EET_API_END                                                         \
  }                                                                          \
  catch (const Fail& f) {                                                    \
    return f.code;                                                           \
  }                                                                          \
  catch (const std::exception& ex) {                                         \
    set_error(ex.what());                                                    \
    return EET_ERR_CUDA;                                                     \
  }                                                                          \
  return EET_OK;

static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Ablation for in-graph timing (bench.py roofline, tools/decode_step_time.py):
// EET_SKIP or eet_debug_skip("qkv,attn,o,w1,w2,head") leaves those decode
// launches out of the step (results become wrong; only their in-graph cost
// is measured this way, with programmatic dependent launch intact).
static std::mutex g_skip_mu;
static std::string g_skip = [] {
  const char* e = std::getenv("EET_SKIP");
  return std::string(e ? e : "");
}();
static bool skip_decode(const char* what) {
  std::lock_guard<std::mutex> lk(g_skip_mu);
  if (g_skip.empty()) return false;
  return ("," + g_skip + ",").find("," + std::string(what) + ",") != std::string::npos;
}

extern "C" {

const char* eet_last_error(void) { return t_err.c_str(); }
int eet_abi_version(void) { return 1; }

uint64_t eet_launch_count(void) { return g_launches.load(); }

int eet_debug_skip(const char* spec) {
  std::lock_guard<std::mutex> lk(g_skip_mu);
  g_skip = spec ? spec : "";
  return EET_OK;
}

int eet_profile_enable(int on) {
  EET_API_BEGIN
  EET_CHECK_CUDA(cudaDeviceSynchronize());
  g_prof.on = on != 0;
  g_prof.eager.clear();
  g_prof.graph.clear();
  g_prof.used = 0;
  for (auto& a : g_prof.acc) a = ProfAcc{};
  EET_API_END
}

int eet_profile_kinds(void) { return K_KIND_COUNT; }

const char* eet_profile_kind_name(int kind) {
  return (kind >= 0 && kind < K_KIND_COUNT) ? kKindNames[kind] : "";
}

int eet_profile_summary(int kind, uint64_t* count, double* total_ms, double* bytes,
                        double* flops) {
  EET_API_BEGIN
  EET_REQUIRE(kind >= 0 && kind < K_KIND_COUNT, EET_ERR_ARG, "bad kernel kind");
  EET_CHECK_CUDA(cudaDeviceSynchronize());
  for (const auto& r : g_prof.eager) fold(r, 0);   // resolve pending eager launches
  g_prof.eager.clear();
  const ProfAcc& a = g_prof.acc[kind];
  *count = a.n;
  *total_ms = a.ms;
  *bytes = a.bytes;
  *flops = a.flops;
  EET_API_END
}

int eet_plan_folding(int logical, int cap, int* k, int* t, int* n) {
  EET_API_BEGIN
  EET_REQUIRE(cap >= 1, EET_ERR_ARG, "unit_cap must be >= 1");
  EET_REQUIRE(logical >= 1 && logical <= 16384, EET_ERR_ARG,
              "logical_size outside supported range [1, 16384]");
  FoldPlan p = plan_folding(logical, cap);
  *k = p.fold_count;
  *t = p.sub_blocks;
  *n = p.threads;
  EET_API_END
}

}  // extern "C"

// ================================================================ pool
// memory.py:136-214 policy on device memory; ledger mirrors AllocationLog.
struct eet_pool {
  struct Buf {
    void* ptr;
    size_t cap;
    bool idle;
    std::string tag;
  };
  struct Rec {
    int event;      // 0 request, 1 release
    uint64_t bytes;
    int decision;   // 0 malloc, 1 reuse, 2 idle
    std::string tag;
  };
  std::vector<Buf> bufs;
  std::vector<Rec> ledger;
  uint64_t in_use = 0, peak = 0, mallocs = 0, reuses = 0;
  bool device = true;

  ~eet_pool() {
    for (auto& b : bufs) device ? (void)cudaFree(b.ptr) : std::free(b.ptr);
  }

  // returns handle index
  int request(size_t bytes, int scope, const char* tag, void** ptr, bool* reused) {
    EET_REQUIRE(bytes >= 1, EET_ERR_ARG, "buffer size must be >= 1");
    EET_REQUIRE(scope == EET_SCOPE_WITHIN || scope == EET_SCOPE_ACROSS, EET_ERR_ARG,
                "scope must be within or across");
    int idx = -1;
    for (size_t i = 0; i < bufs.size(); ++i) {
      if (!bufs[i].idle) continue;
      if (scope == EET_SCOPE_WITHIN ? bufs[i].cap == bytes : bufs[i].cap >= bytes) {
        idx = (int)i;
        break;
      }
    }
    std::string t = tag ? tag : "";
    if (idx < 0) {
      void* p = nullptr;
      if (device) {
        EET_CHECK_CUDA(cudaMalloc(&p, bytes));
      } else {
        p = std::malloc(bytes);
        EET_REQUIRE(p != nullptr, EET_ERR_CUDA, "host allocation failed");
      }
      bufs.push_back(Buf{p, bytes, false, t});
      idx = (int)bufs.size() - 1;
      ++mallocs;
      ledger.push_back(Rec{0, bytes, 0, t});
      *reused = false;
    } else {
      bufs[idx].idle = false;
      bufs[idx].tag = t;
      ++reuses;
      ledger.push_back(Rec{0, bytes, 1, t});
      *reused = true;
    }
    in_use += bufs[idx].cap;
    peak = std::max(peak, in_use);
    *ptr = bufs[idx].ptr;
    return idx;
  }

  void release(int idx, size_t bytes) {
    EET_REQUIRE(idx >= 0 && idx < (int)bufs.size(), EET_ERR_POOL, "unknown buffer handle");
    EET_REQUIRE(!bufs[idx].idle, EET_ERR_POOL, "buffer handle released twice");
    bufs[idx].idle = true;
    in_use -= bufs[idx].cap;
    ledger.push_back(Rec{1, bytes, 2, bufs[idx].tag});
  }

  uint64_t total() const {
    uint64_t s = 0;
    for (auto& b : bufs) s += b.cap;
    return s;
  }
};

// RAII claim used inside the layer orchestration.
struct Claim {
  eet_pool* pool;
  int idx = -1;
  size_t bytes = 0;
  void* ptr = nullptr;
  Claim(eet_pool* p, size_t b, int scope, const char* tag) : pool(p), bytes(b) {
    bool r;
    idx = pool->request(std::max<size_t>(b, 1), scope, tag, &ptr, &r);
  }
  void release() {
    if (idx >= 0) pool->release(idx, bytes);
    idx = -1;
  }
  ~Claim() {
    if (idx >= 0) {
      try { pool->release(idx, bytes); } catch (...) {}
    }
  }
  template <typename P> P* as() const { return reinterpret_cast<P*>(ptr); }
};

extern "C" {

int eet_pool_create(eet_pool** out) {
  EET_API_BEGIN
  *out = new eet_pool();
  EET_API_END
}

int eet_pool_create_ex(eet_pool** out, int device_backed) {
  EET_API_BEGIN
  *out = new eet_pool();
  (*out)->device = device_backed != 0;
  EET_API_END
}

int eet_pool_destroy(eet_pool* pool) {
  EET_API_BEGIN
  delete pool;
  EET_API_END
}

int eet_pool_request(eet_pool* pool, size_t bytes, int scope, const char* tag, int* handle,
                     void** dptr, size_t* capacity, int* reused) {
  EET_API_BEGIN
  bool r = false;
  int idx = pool->request(bytes, scope, tag, dptr, &r);
  *handle = idx;
  if (capacity) *capacity = pool->bufs[idx].cap;
  if (reused) *reused = r ? 1 : 0;
  EET_API_END
}

int eet_pool_release(eet_pool* pool, int handle, size_t bytes) {
  EET_API_BEGIN
  pool->release(handle, bytes);
  EET_API_END
}

int eet_pool_stats(eet_pool* pool, uint64_t stats[4]) {
  EET_API_BEGIN
  stats[0] = pool->total();
  stats[1] = pool->peak;
  stats[2] = pool->mallocs;
  stats[3] = pool->reuses;
  EET_API_END
}

int eet_pool_debug_fill(eet_pool* pool, int value) {
  EET_API_BEGIN
  EET_CHECK_CUDA(cudaDeviceSynchronize());
  for (auto& b : pool->bufs) {
    if (!b.idle) continue;
    if (pool->device) EET_CHECK_CUDA(cudaMemset(b.ptr, value & 0xFF, b.cap));
    else std::memset(b.ptr, value & 0xFF, b.cap);
  }
  EET_CHECK_CUDA(cudaDeviceSynchronize());
  EET_API_END
}

int eet_pool_ledger_size(eet_pool* pool, size_t* n) {
  EET_API_BEGIN
  *n = pool->ledger.size();
  EET_API_END
}

int eet_pool_buffer_count(eet_pool* pool, size_t* n) {
  EET_API_BEGIN
  *n = pool->bufs.size();
  EET_API_END
}

int eet_pool_buffer_info(eet_pool* pool, size_t i, uint64_t* capacity, int* idle) {
  EET_API_BEGIN
  EET_REQUIRE(i < pool->bufs.size(), EET_ERR_ARG, "buffer index out of range");
  *capacity = pool->bufs[i].cap;
  *idle = pool->bufs[i].idle ? 1 : 0;
  EET_API_END
}

int eet_pool_ledger_get(eet_pool* pool, size_t i, int* event, uint64_t* bytes, int* decision,
                        char* tag, size_t tag_cap) {
  EET_API_BEGIN
  EET_REQUIRE(i < pool->ledger.size(), EET_ERR_ARG, "ledger index out of range");
  const auto& r = pool->ledger[i];
  *event = r.event;
  *bytes = r.bytes;
  *decision = r.decision;
  if (tag && tag_cap) {
    std::strncpy(tag, r.tag.c_str(), tag_cap - 1);
    tag[tag_cap - 1] = 0;
  }
  EET_API_END
}

// ============================================================ operators
int eet_masked_softmax(float* scores, const int* d_pads, int batch, int heads, int seq, int causal,
                       int fold_cap, void* stream) {
  EET_API_BEGIN
  EET_REQUIRE(batch >= 1 && heads >= 1 && seq >= 1, EET_ERR_SHAPE, "softmax: empty shape");
  launch_masked_softmax(scores, d_pads, batch, heads, seq, causal, fold_cap, S(stream));
  EET_API_END
}

int eet_step_softmax(float* scores, const int* d_pads, int batch, int heads, int len, int fold_cap,
                     void* stream) {
  EET_API_BEGIN
  EET_REQUIRE(batch >= 1 && heads >= 1 && len >= 1, EET_ERR_SHAPE, "step softmax: empty shape");
  launch_step_softmax(scores, d_pads, batch, heads, len, fold_cap, S(stream));
  EET_API_END
}

int eet_layer_norm(const float* x, const float* g, const float* b, float* y, int rows, int h,
                   int fold_cap, void* stream) {
  EET_API_BEGIN
  launch_layer_norm(x, h, h, nullptr, rows, g, b, y, EET_F32, h, h, fold_cap, S(stream));
  EET_API_END
}

int eet_mha_forward(const float* q, const float* k, const float* v, float* out, const int* d_pads,
                    int batch, int seq, int hidden, int heads, int causal, void* stream) {
  EET_API_BEGIN
  EET_REQUIRE(heads >= 1 && hidden % heads == 0, EET_ERR_SHAPE, "hidden not divisible by heads");
  PrefillArgs a{};
  a.dtype = EET_F32;
  a.q = q; a.ldq = hidden; a.q_rowbase = nullptr;
  a.k = k; a.v = v;
  a.k_sb = (long long)seq * hidden; a.k_sh = hidden / heads; a.k_ss = hidden;
  a.o = out; a.ldo = hidden; a.o_rowbase = nullptr;
  a.pads = d_pads;
  a.batch = batch; a.seq = seq; a.heads = heads; a.hd = hidden / heads;
  a.scale = 1.0f / std::sqrt((float)a.hd);
  a.causal = causal;
  a.zero_pad_rows = 1;
  launch_attn_prefill(a, S(stream));
  EET_API_END
}

int eet_gemm(int dtype, const void* A, const void* B, const float* bias, float* C, int M, int N,
             int K, int ldc, void* stream) {
  EET_API_BEGIN
  Epi e;
  e.mode = EPI_STORE_F32;
  e.out = C;
  e.ldo = ldc;
  e.bias = bias;
  gemm(dtype, A, K, B, K, M, N, K, e, S(stream));
  EET_API_END
}

}  // extern "C"

// ============================================================= runtime
struct StepPlan {
  int T = 0;               // packed (valid) rows
  int batch = 0, t = 0;    // x is [batch, t, h]
  int seq = 0;             // prompt length (prefill window)
  int phase = EET_PHASE_PROMPT;
  bool valid = false;
  std::vector<int> h_pads; // host copy: uploads are skipped when unchanged
  int2* rinfo = nullptr;   // [T] (b, t_local)
  int* rowbase = nullptr;  // [b] packed row of slot s = rowbase[b] + s
  int* pads = nullptr;     // [b] first valid slot
  // per-sequence valid end (right padding / explicit windows, prompt phase):
  // empty = every sequence ends at seq
  std::vector<int> h_ends;
  int* ends = nullptr;     // [b] device copy, nullptr when h_ends is empty
  int* ends_buf = nullptr;
};

struct eet_runtime {
  int dtype, h, heads, hd, bmax, smax, splits;
  int hq, ffn;                        // local Q/K/V width and FFN width (tensor-parallel shard)
  int tp_rank = 0, tp_size = 1;
  eet_pool* pool;
  cudaStream_t cs = nullptr;          // private stream for graph capture
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  StepPlan plans[3];                  // 0: layer API, 1: generate prompt, 2: generate step
  std::vector<void*> owned;
  float* part = nullptr;              // decode split partials
  int* counters = nullptr;
  int* d_prompts = nullptr;           // [bmax * smax]
  int* d_filled = nullptr;
  int* d_step = nullptr;
  int* d_cur = nullptr;               // [bmax]
  int* h_prompts = nullptr;           // pinned staging: prompts in, tokens out
  long long* h_tokens = nullptr;
  float* xdec = nullptr;              // decode residual stream [bmax, h]
  long long* oacc = nullptr;          // pending out-projection [bmax, h], 2^-32 fixed point, zero between layers
  void* tp_ctx = nullptr;             // tensor parallel: attention context kept for the row-chunked out-proj
  void* tp_mid = nullptr;             // tensor parallel: FFN intermediate kept for the row-chunked W2
  int2* cand = nullptr;               // fused LM-head argmax candidates
  int* cand_ticket = nullptr;
  int cand_cap = 0;

  void* dev(size_t bytes) {
    void* p = nullptr;
    EET_CHECK_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    owned.push_back(p);
    return p;
  }
  ~eet_runtime() {
    for (void* p : owned) cudaFree(p);
    if (h_prompts) cudaFreeHost(h_prompts);
    if (h_tokens) cudaFreeHost(h_tokens);
    if (cs) cudaStreamDestroy(cs);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
  }
};

static void plan_alloc(eet_runtime* rt, StepPlan& p) {
  p.rinfo = (int2*)rt->dev(sizeof(int2) * (size_t)rt->bmax * rt->smax);
  p.rowbase = (int*)rt->dev(sizeof(int) * rt->bmax);
  p.pads = (int*)rt->dev(sizeof(int) * rt->bmax);
  p.ends_buf = (int*)rt->dev(sizeof(int) * rt->bmax);
}

// Host-side packing of the valid tokens (pad skipping): prompt rows are the
// slots [pad_b, t) of each sequence, incremental rows are every sequence.
// The device copies are refreshed only when the batch layout changes.
// ends (optional, prompt phase): sequence b's valid slots are [pads[b],
// ends[b]) instead of [pads[b], seq) — right-padded / windowed batches
// (the reference itself is left-pad only)
static void plan_fill(StepPlan& p, int batch, int t, const int* pads, int seq, int phase,
                      cudaStream_t st, const int* ends = nullptr) {
  const bool same_ends = ends ? (p.h_ends.size() == (size_t)batch && std::equal(ends, ends + batch, p.h_ends.begin()))
                              : p.h_ends.empty();
  if (p.valid && p.batch == batch && p.t == t && p.seq == seq && p.phase == phase && same_ends &&
      std::equal(pads, pads + batch, p.h_pads.begin()))
    return;
  std::vector<int2> ri;
  std::vector<int> rb(batch);
  ri.reserve((size_t)batch * t);
  for (int b = 0; b < batch; ++b) {
    int first = (phase == EET_PHASE_PROMPT) ? pads[b] : 0;
    const int last = (ends && phase == EET_PHASE_PROMPT) ? ends[b] : t;
    rb[b] = (int)ri.size() - first;
    for (int s = first; s < last; ++s) ri.push_back(make_int2(b, s));
  }
  p.T = (int)ri.size();
  p.batch = batch;
  p.t = t;
  p.seq = seq;
  p.phase = phase;
  p.h_pads.assign(pads, pads + batch);
  // pageable-source async copies return once the source is staged
  if (!ri.empty())
    EET_CHECK_CUDA(cudaMemcpyAsync(p.rinfo, ri.data(), sizeof(int2) * ri.size(),
                                   cudaMemcpyHostToDevice, st));
  EET_CHECK_CUDA(cudaMemcpyAsync(p.rowbase, rb.data(), sizeof(int) * batch, cudaMemcpyHostToDevice, st));
  EET_CHECK_CUDA(cudaMemcpyAsync(p.pads, pads, sizeof(int) * batch, cudaMemcpyHostToDevice, st));
  if (ends) {
    p.h_ends.assign(ends, ends + batch);
    EET_CHECK_CUDA(cudaMemcpyAsync(p.ends_buf, ends, sizeof(int) * batch, cudaMemcpyHostToDevice, st));
    p.ends = p.ends_buf;
  } else {
    p.h_ends.clear();
    p.ends = nullptr;
  }
  p.valid = true;
}

// Attention half of a pre-norm layer over a prepared plan (runtime.py:106-189):
//   LN1 (gather valid rows) -> QKV GEMM (epilogue: Q packed, K/V -> cache)
//   -> mask-fused attention -> out-proj GEMM.
// The out-proj epilogue adds into x (single GPU) or, for a tensor-parallel
// shard, stores this rank's partial sum into `partial` ([T, h] fp32) for the
// all-reduce. Cache slot of local position 0 = (kv_dev ? *kv_dev : 0) +
// kv_base; the device form lets a captured decode step advance without
// re-capture.
// Tensor-parallel epilogue of the row-split projections: this rank's partial
// sum in fp32 (fp32 mode) or the layer dtype (16-bit modes: half the bytes
// on NVLink), rows [r0, r1) of the packed plan.
static Epi tp_partial_epi(const eet_runtime* rt, void* partial, const float* bias) {
  Epi e;
  e.bias = bias;
  e.mode = rt->dtype == EET_F32 ? EPI_STORE_F32 : EPI_STORE_T;
  e.out = partial;
  e.ldo = rt->h;
  return e;
}

// Returns true when the out-projection was fused into the decode attention
// (attn_o.cu): its result is then pending in rt->oacc and the FFN's LN2 + W1
// and W2 GEMVs consume it.
static bool attn_block(eet_runtime* rt, const StepPlan& p, float* x, long long x_sb, long long x_ss,
                       const eet_layer_weights* w, void* kc, void* vc, const int* kv_dev,
                       int kv_base, bool causal, int L_host, void* partial, cudaStream_t st,
                       bool keep_ctx = false) {
  const int h = rt->h, hq = rt->hq, T = p.T, dt = rt->dtype;
  const size_t es = dtype_size(dt);
  const int scope = (p.phase == EET_PHASE_PROMPT) ? EET_SCOPE_WITHIN : EET_SCOPE_ACROSS;
  if (T == 0) return false;

  // decode: the whole attention half in one kernel (qkv_attn_o.cu), or the
  // attention + out-projection in one (attn_o.cu), when the FFN GEMVs that
  // consume the pending out-projection take this shape
  const bool inc = p.phase == EET_PHASE_INCREMENTAL;
  const bool pend_ok = inc && !keep_ctx && !partial && (x_ss & 3) == 0 && !skip_decode("o") &&
                       gemv_cl_ok(dt, w->w1, T, rt->ffn, h, nullptr, 0, x, x_sb, w->ln2_g, w->ln2_b, EPI_GELU_T) &&
                       gemv_cl_ok(dt, w->w2, T, h, rt->ffn, nullptr, rt->ffn, nullptr, 0, nullptr, nullptr, EPI_RESID);
  const bool fuse_all = pend_ok && rt->splits == 1 && T == p.batch && !skip_decode("qkv") && !skip_decode("attn") &&
                        qkv_attn_o_ok(dt, T, h, rt->heads, rt->hd, hq, x, x_sb, kc, vc, w->wqkv, w->wo);
  if (pend_ok && !rt->oacc) {
    rt->oacc = (long long*)rt->dev(sizeof(long long) * (size_t)rt->bmax * h);
    EET_CHECK_CUDA(cudaMemsetAsync(rt->oacc, 0, sizeof(long long) * (size_t)rt->bmax * h, st));
  }
  Claim q(rt->pool, (size_t)T * hq * es, scope, "attention.query");
  if (fuse_all) {
    Claim ctx(rt->pool, (size_t)T * hq * es, scope, "attention.context");
    const bool ok = launch_qkv_attn_o(dt, T, h, rt->heads, rt->smax, x, x_sb, w->ln1_g, w->ln1_b, w->wqkv, w->b_qkv,
                                      kc, vc, p.pads, kv_dev, kv_base, w->wo, w->b_o, rt->oacc, h, L_host,
                                      p.h_pads.data(), st);
    EET_REQUIRE(ok, EET_ERR_UNSUPPORTED, "fused decode attention rejected an eligible shape");
    ctx.release();
    q.release();
    return true;
  }
  {
    Epi e;
    e.mode = EPI_QKV;
    e.bias = w->b_qkv;
    e.out = q.ptr;
    e.rinfo = p.rinfo;
    e.kc = kc;
    e.vc = vc;
    e.heads = rt->heads;
    e.hd = rt->hd;
    e.hq = hq;
    e.smax = rt->smax;
    e.kv_start = kv_dev;
    e.kv_base = kv_base;
    // decode rows: LN1 runs inside the GEMV prologue; otherwise LN -> GEMM
    if (inc && skip_decode("qkv")) {
    } else if (inc && gemv_cl(dt, w->wqkv, T, 3 * hq, h, nullptr, 0, x, x_sb, x_ss, p.rinfo, w->ln1_g, w->ln1_b,
                              e, st)) {
      // split-K cluster GEMV straight from the K-major weight, LayerNorm fused (gemv_cl.cu)
    } else if (!(T <= 32 && gemv_tc_ln_sm100(dt, x, x_sb, x_ss, p.rinfo, w->ln1_g, w->ln1_b, w->wqkv, h,
                                             T, 3 * hq, h, e, st))) {
      Claim ln(rt->pool, (size_t)T * h * es, scope, "attention.layernorm");
      launch_layer_norm(x, x_sb, x_ss, p.rinfo, T, w->ln1_g, w->ln1_b, ln.ptr, dt, h, h, 0, st);
      gemm(dt, ln.ptr, h, w->wqkv, h, T, 3 * hq, h, e, st);
    }
  }

  Claim ctx(rt->pool, keep_ctx ? 0 : (size_t)T * hq * es, scope, "attention.context");
  if (keep_ctx) {                     // tensor parallel, row-chunked out-proj later (eet_tp_attention_out)
    if (!rt->tp_ctx) rt->tp_ctx = rt->dev((size_t)rt->bmax * rt->smax * hq * es);
    ctx.ptr = rt->tp_ctx;
  }
  const float scale = 1.0f / std::sqrt((float)rt->hd);
  if (p.phase == EET_PHASE_PROMPT) {
    PrefillArgs a{};
    a.dtype = dt;
    a.q = q.ptr; a.ldq = hq; a.q_rowbase = p.rowbase;
    a.k = kc; a.v = vc;
    a.k_sb = (long long)rt->heads * rt->smax * rt->hd;
    a.k_sh = (long long)rt->smax * rt->hd;
    a.k_ss = rt->hd;
    a.o = ctx.ptr; a.ldo = hq; a.o_rowbase = p.rowbase;
    a.pads = p.pads;
    a.h_pads = p.h_pads.data();
    a.ends = p.ends;
    a.h_ends = p.h_ends.empty() ? nullptr : p.h_ends.data();
    a.batch = p.batch; a.seq = p.seq; a.heads = rt->heads; a.hd = rt->hd;
    a.scale = scale;
    a.causal = causal ? 1 : 0;
    a.zero_pad_rows = 0;
    a.q_rows = p.T;
    launch_attn_prefill(a, st);
  } else {
    DecodeArgs a{};
    a.dtype = dt;
    a.q = q.ptr; a.ldq = hq;
    a.kc = kc; a.vc = vc;
    a.batch = p.batch; a.heads = rt->heads; a.hd = rt->hd; a.smax = rt->smax;
    a.pads = p.pads;
    a.kv_start = kv_dev;
    a.kv_base = kv_base;
    a.h_pads = p.h_pads.data();
    a.L_host = L_host;
    a.scale = scale;
    a.part = rt->part;
    a.counters = rt->counters;
    a.o = ctx.ptr; a.ldo = hq;
    a.splits = rt->splits;
    if (!skip_decode("attn")) {
      if (pend_ok && launch_attn_o(a, w->wo, h, rt->oacc, h, w->b_o, st)) {
        q.release();
        ctx.release();
        return true;
      }
      launch_attn_decode(a, st);
    }
  }
  q.release();
  if (keep_ctx) return false;
  {
    Epi e;
    e.bias = w->b_o;
    if (partial) {
      e = tp_partial_epi(rt, partial, w->b_o);
    } else {
      e.mode = EPI_RESID;
      e.x = x; e.x_sb = x_sb; e.x_ss = x_ss;
      e.rinfo = p.rinfo;
    }
    if (p.phase == EET_PHASE_INCREMENTAL && skip_decode("o")) {
    } else if (!(p.phase == EET_PHASE_INCREMENTAL &&
                 gemv_cl(dt, w->wo, T, h, hq, ctx.ptr, hq, nullptr, 0, 0, nullptr, nullptr, nullptr, e, st)))
      gemm(dt, ctx.ptr, hq, w->wo, hq, T, h, hq, e, st);
  }
  ctx.release();
  return false;
}

// Feed-forward half (runtime.py:192-214): LN2 -> W1 GEMM (+GELU) -> W2 GEMM,
// residual into x or a tensor-parallel partial as above. Both pool requests
// use across-module scope like the reference (runtime.py:200-207).
// acc: pending out-projection rows (attn_block returned true): read by the
// LN2 prologue of W1, folded into x and re-zeroed by the W2 epilogue.
static void ffn_block(eet_runtime* rt, const StepPlan& p, float* x, long long x_sb, long long x_ss,
                      const eet_layer_weights* w, void* partial, cudaStream_t st, bool keep_mid = false,
                      long long* acc = nullptr) {
  const int h = rt->h, f = rt->ffn, T = p.T, dt = rt->dtype;
  const size_t es = dtype_size(dt);
  if (T == 0) return;
  // EET_FFN_CHUNKED=1 reproduces the reference's memory shape in fp32 mode:
  // the intermediate accumulated in two half-width chunks, live buffer
  // T x 2h (runtime.py:195-214). Default: one T x 4h intermediate (two
  // launches fewer: c1 0.119 vs 0.143 ms per layer); 16-bit layers hold
  // T x 4h in the bytes of the reference's fp32 T x 2h chunk either way.
  static const bool chunked = [] {
    const char* v = std::getenv("EET_FFN_CHUNKED");
    return v && v[0] == '1';
  }();
  if (chunked && dt == EET_F32 && !keep_mid && !partial && f % 8 == 0) {
    const int fc = f / 2;
    Claim ln2(rt->pool, (size_t)T * h * es, EET_SCOPE_ACROSS, "ffn.layernorm");
    launch_layer_norm(x, x_sb, x_ss, p.rinfo, T, w->ln2_g, w->ln2_b, ln2.ptr, dt, h, h, 0, st);
    Claim mid(rt->pool, (size_t)T * fc * es, EET_SCOPE_ACROSS, "ffn.intermediate");
    for (int c = 0; c < 2; ++c) {
      Epi e1;
      e1.mode = EPI_GELU_T;
      e1.bias = w->b_1 ? w->b_1 + (size_t)c * fc : nullptr;
      e1.out = mid.ptr;
      e1.ldo = fc;
      gemm(dt, ln2.ptr, h, static_cast<const float*>(w->w1) + (size_t)c * fc * h, h, T, fc, h, e1, st);
      Epi e2;
      e2.mode = EPI_RESID;
      e2.bias = c == 0 ? w->b_2 : nullptr;
      e2.x = x; e2.x_sb = x_sb; e2.x_ss = x_ss;
      e2.rinfo = p.rinfo;
      gemm(dt, mid.ptr, fc, static_cast<const float*>(w->w2) + (size_t)c * fc, f, T, h, fc, e2, st);
    }
    mid.release();
    ln2.release();
    return;
  }
  Claim mid(rt->pool, keep_mid ? 0 : (size_t)T * f * es, EET_SCOPE_ACROSS, "ffn.intermediate");
  if (keep_mid) {                     // tensor parallel, row-chunked W2 later (eet_tp_ffn_out)
    if (!rt->tp_mid) rt->tp_mid = rt->dev((size_t)rt->bmax * rt->smax * f * es);
    mid.ptr = rt->tp_mid;
  }
  {
    Epi e;
    e.mode = EPI_GELU_T;
    e.bias = w->b_1;
    e.out = mid.ptr;
    e.ldo = f;
    const bool inc = p.phase == EET_PHASE_INCREMENTAL;
    if (inc && skip_decode("w1")) {
    } else if (inc && gemv_cl(dt, w->w1, T, f, h, nullptr, 0, x, x_sb, x_ss, p.rinfo, w->ln2_g, w->ln2_b, e, st, acc,
                              h)) {
    } else {
      EET_REQUIRE(!acc, EET_ERR_UNSUPPORTED, "pending out-projection without its W1 GEMV");
      if (!(T <= 32 && gemv_tc_ln_sm100(dt, x, x_sb, x_ss, p.rinfo, w->ln2_g, w->ln2_b, w->w1, h, T, f, h, e, st))) {
        Claim ln2(rt->pool, (size_t)T * h * es, EET_SCOPE_ACROSS, "ffn.layernorm");
        launch_layer_norm(x, x_sb, x_ss, p.rinfo, T, w->ln2_g, w->ln2_b, ln2.ptr, dt, h, h, 0, st);
        gemm(dt, ln2.ptr, h, w->w1, h, T, f, h, e, st);
      }
    }
  }
  if (keep_mid) return;
  {
    Epi e;
    e.bias = w->b_2;
    if (partial) {
      e = tp_partial_epi(rt, partial, w->b_2);
    } else {
      e.mode = EPI_RESID;
      e.x = x; e.x_sb = x_sb; e.x_ss = x_ss;
      e.rinfo = p.rinfo;
      e.acc = acc;
      e.acc_sb = h;
    }
    if (p.phase == EET_PHASE_INCREMENTAL && skip_decode("w2")) {
    } else if (!(p.phase == EET_PHASE_INCREMENTAL &&
                 gemv_cl(dt, w->w2, T, h, f, mid.ptr, f, nullptr, 0, 0, nullptr, nullptr, nullptr, e, st))) {
      EET_REQUIRE(!acc, EET_ERR_UNSUPPORTED, "pending out-projection without its W2 GEMV");
      gemm(dt, mid.ptr, f, w->w2, f, T, h, f, e, st);
    }
  }
  mid.release();
}

// One whole pre-norm layer (runtime.py:217-263) on a single GPU.
static void layer_impl(eet_runtime* rt, const StepPlan& p, float* x, long long x_sb,
                       long long x_ss, const eet_layer_weights* w, void* kc, void* vc,
                       const int* kv_dev, int kv_base, bool causal, int L_host, cudaStream_t st) {
  const bool pending = attn_block(rt, p, x, x_sb, x_ss, w, kc, vc, kv_dev, kv_base, causal, L_host, nullptr, st);
  ffn_block(rt, p, x, x_sb, x_ss, w, nullptr, st, false, pending ? rt->oacc : nullptr);
}

extern "C" {

// heads: heads held by this runtime (all of them, or one tensor-parallel
// shard's); hd = hidden / heads_total.
static eet_runtime* runtime_new(int dtype, int hidden, int heads_total, int tp_rank, int tp_size,
                                int max_batch, int max_sequence, eet_pool* pool) {
  EET_REQUIRE(dtype == EET_F32 || dtype == EET_BF16 || dtype == EET_F16, EET_ERR_ARG, "bad dtype");
  EET_REQUIRE(heads_total >= 1 && hidden % heads_total == 0, EET_ERR_ARG, "hidden not divisible by heads");
  EET_REQUIRE(tp_size >= 1 && tp_rank >= 0 && tp_rank < tp_size, EET_ERR_ARG, "bad tensor-parallel rank");
  EET_REQUIRE(heads_total % tp_size == 0 && (4 * hidden) % tp_size == 0, EET_ERR_ARG,
              "heads and 4*hidden must divide by the tensor-parallel size");
  EET_REQUIRE(max_batch >= 1 && max_sequence >= 1, EET_ERR_ARG, "bad capacities");
  EET_REQUIRE(pool != nullptr && pool->device, EET_ERR_ARG, "runtime needs a device-backed buffer pool");
  std::unique_ptr<eet_runtime> rt(new eet_runtime());
  const int heads = heads_total / tp_size;
  rt->dtype = dtype;
  rt->h = hidden;
  rt->heads = heads;
  rt->hd = hidden / heads_total;
  rt->hq = heads * rt->hd;
  rt->ffn = 4 * hidden / tp_size;
  rt->tp_rank = tp_rank;
  rt->tp_size = tp_size;
  rt->bmax = max_batch;
  rt->smax = max_sequence;
  rt->pool = pool;
  rt->splits = decode_splits(max_batch, heads, max_sequence, rt->hd, (int)dtype_size(dtype));
  for (auto& p : rt->plans) plan_alloc(rt.get(), p);
  rt->part = (float*)rt->dev(sizeof(float) * (size_t)max_batch * heads * rt->splits * (rt->hd + 2));
  rt->counters = (int*)rt->dev(sizeof(int) * (size_t)max_batch * heads);
  EET_CHECK_CUDA(cudaMemset(rt->counters, 0, sizeof(int) * (size_t)max_batch * heads));
  rt->d_prompts = (int*)rt->dev(sizeof(int) * (size_t)max_batch * max_sequence);
  rt->d_filled = (int*)rt->dev(sizeof(int));
  rt->d_step = (int*)rt->dev(sizeof(int));
  rt->d_cur = (int*)rt->dev(sizeof(int) * max_batch);
  EET_CHECK_CUDA(cudaMallocHost(&rt->h_prompts, sizeof(int) * (size_t)max_batch * max_sequence));
  EET_CHECK_CUDA(cudaMallocHost(&rt->h_tokens, sizeof(long long) * (size_t)max_batch * max_sequence));
  EET_CHECK_CUDA(cudaStreamCreateWithFlags(&rt->cs, cudaStreamNonBlocking));
  EET_CHECK_CUDA(cudaEventCreateWithFlags(&rt->ev_in, cudaEventDisableTiming));
  EET_CHECK_CUDA(cudaEventCreateWithFlags(&rt->ev_out, cudaEventDisableTiming));
  EET_CHECK_CUDA(cudaDeviceSynchronize());
  return rt.release();
}

int eet_runtime_create(eet_runtime** out, int dtype, int hidden, int heads, int max_batch,
                       int max_sequence, eet_pool* pool) {
  EET_API_BEGIN
  *out = runtime_new(dtype, hidden, heads, 0, 1, max_batch, max_sequence, pool);
  EET_API_END
}

int eet_runtime_create_tp(eet_runtime** out, int dtype, int hidden, int heads_total, int tp_rank,
                          int tp_size, int max_batch, int max_sequence, eet_pool* pool) {
  EET_API_BEGIN
  *out = runtime_new(dtype, hidden, heads_total, tp_rank, tp_size, max_batch, max_sequence, pool);
  EET_API_END
}

int eet_runtime_destroy(eet_runtime* rt) {
  EET_API_BEGIN
  if (rt) cudaDeviceSynchronize();
  delete rt;
  EET_API_END
}

int eet_decoder_layer_forward(eet_runtime* rt, float* x, long long x_sb, long long x_ss, int batch,
                              int t, const eet_layer_weights* w, void* kc, void* vc,
                              int kv_filled, const int* h_pads, int seq_len, int phase,
                              void* stream) {
  EET_API_BEGIN
  EET_REQUIRE(batch >= 1 && batch <= rt->bmax, EET_ERR_SHAPE, "batch exceeds runtime capacity");
  if (phase == EET_PHASE_INCREMENTAL) {
    EET_REQUIRE(t == 1, EET_ERR_SHAPE, "incremental step takes 1 token");
    EET_REQUIRE(kv_filled >= seq_len, EET_ERR_SHAPE, "incremental phase before the prompt was cached");
  } else {
    EET_REQUIRE(t == seq_len, EET_ERR_SHAPE, "prompt pass length does not match seq_len");
    EET_REQUIRE(kv_filled == 0, EET_ERR_SHAPE, "prompt phase expects an empty cache");
  }
  EET_REQUIRE(kv_filled + t <= rt->smax, EET_ERR_OVERFLOW, "step would overflow the cache");
  for (int b = 0; b < batch; ++b)
    EET_REQUIRE(h_pads[b] >= 0 && h_pads[b] < seq_len, EET_ERR_SHAPE, "pad outside [0, seq_len)");
  StepPlan& p = rt->plans[0];
  plan_fill(p, batch, t, h_pads, seq_len, phase, S(stream));
  layer_impl(rt, p, x, x_sb, x_ss, w, kc, vc, nullptr, kv_filled, true, kv_filled + t, S(stream));
  EET_API_END
}

static void check_windows(const eet_runtime* rt, int batch, int t, const int* h_start, const int* h_end) {
  EET_REQUIRE(batch >= 1 && batch <= rt->bmax && t >= 1 && t <= rt->smax, EET_ERR_SHAPE,
              "batch / length exceed runtime capacity");
  for (int b = 0; b < batch; ++b)
    EET_REQUIRE(h_start[b] >= 0 && h_start[b] < h_end[b] && h_end[b] <= t, EET_ERR_SHAPE,
                "window outside [0, seq_len) or empty");
}

int eet_decoder_layer_forward_window(eet_runtime* rt, float* x, long long x_sb, long long x_ss, int batch,
                                     int t, const eet_layer_weights* w, void* kc, void* vc, const int* h_start,
                                     const int* h_end, void* stream) {
  EET_API_BEGIN
  check_windows(rt, batch, t, h_start, h_end);
  StepPlan& p = rt->plans[0];
  plan_fill(p, batch, t, h_start, t, EET_PHASE_PROMPT, S(stream), h_end);
  layer_impl(rt, p, x, x_sb, x_ss, w, kc, vc, nullptr, 0, true, t, S(stream));
  EET_API_END
}

int eet_encoder_layer_forward_window(eet_runtime* rt, float* x, long long x_sb, long long x_ss, int batch,
                                     int t, const eet_layer_weights* w, const int* h_start, const int* h_end,
                                     void* stream) {
  EET_API_BEGIN
  check_windows(rt, batch, t, h_start, h_end);
  StepPlan& p = rt->plans[0];
  plan_fill(p, batch, t, h_start, t, EET_PHASE_PROMPT, S(stream), h_end);
  const size_t kvb = (size_t)batch * rt->heads * rt->smax * rt->hd * dtype_size(rt->dtype);
  Claim kbuf(rt->pool, kvb, EET_SCOPE_WITHIN, "attention.key");
  Claim vbuf(rt->pool, kvb, EET_SCOPE_WITHIN, "attention.value");
  layer_impl(rt, p, x, x_sb, x_ss, w, kbuf.ptr, vbuf.ptr, nullptr, 0, false, t, S(stream));
  EET_API_END
}

int eet_encoder_layer_forward(eet_runtime* rt, float* x, long long x_sb, long long x_ss, int batch,
                              int t, const eet_layer_weights* w, const int* h_pads, void* stream) {
  EET_API_BEGIN
  EET_REQUIRE(batch >= 1 && batch <= rt->bmax && t <= rt->smax, EET_ERR_SHAPE,
              "encoder input exceeds runtime capacity");
  for (int b = 0; b < batch; ++b)
    EET_REQUIRE(h_pads[b] >= 0 && h_pads[b] < t, EET_ERR_SHAPE, "pad outside [0, seq_len)");
  StepPlan& p = rt->plans[0];
  plan_fill(p, batch, t, h_pads, t, EET_PHASE_PROMPT, S(stream));
  // bidirectional attention reads K/V scattered into scratch [b, heads, smax, hd]
  const size_t kvb = (size_t)batch * rt->heads * rt->smax * rt->hd * dtype_size(rt->dtype);
  Claim kbuf(rt->pool, kvb, EET_SCOPE_WITHIN, "attention.key");
  Claim vbuf(rt->pool, kvb, EET_SCOPE_WITHIN, "attention.value");
  layer_impl(rt, p, x, x_sb, x_ss, w, kbuf.ptr, vbuf.ptr, nullptr, 0, false, t, S(stream));
  EET_API_END
}

// ------------------------------------------------------- tensor parallel
static void check_layer_args(eet_runtime* rt, int batch, int t, int kv_filled, const int* h_pads,
                             int seq_len, int phase) {
  EET_REQUIRE(batch >= 1 && batch <= rt->bmax, EET_ERR_SHAPE, "batch exceeds runtime capacity");
  if (phase == EET_PHASE_INCREMENTAL) {
    EET_REQUIRE(t == 1, EET_ERR_SHAPE, "incremental step takes 1 token");
    EET_REQUIRE(kv_filled >= seq_len, EET_ERR_SHAPE, "incremental phase before the prompt was cached");
  } else {
    EET_REQUIRE(t == seq_len, EET_ERR_SHAPE, "prompt pass length does not match seq_len");
    EET_REQUIRE(kv_filled == 0, EET_ERR_SHAPE, "prompt phase expects an empty cache");
  }
  EET_REQUIRE(kv_filled + t <= rt->smax, EET_ERR_OVERFLOW, "step would overflow the cache");
  for (int b = 0; b < batch; ++b)
    EET_REQUIRE(h_pads[b] >= 0 && h_pads[b] < seq_len, EET_ERR_SHAPE, "pad outside [0, seq_len)");
}

int eet_tp_attention_partial(eet_runtime* rt, const float* x, long long x_sb, long long x_ss,
                             int batch, int t, const eet_layer_weights* w, void* kc, void* vc,
                             int kv_filled, const int* h_pads, int seq_len, int phase,
                             void* partial, int* rows, void* stream) {
  EET_API_BEGIN
  check_layer_args(rt, batch, t, kv_filled, h_pads, seq_len, phase);
  StepPlan& p = rt->plans[0];
  plan_fill(p, batch, t, h_pads, seq_len, phase, S(stream));
  if (rows) *rows = p.T;
  attn_block(rt, p, const_cast<float*>(x), x_sb, x_ss, w, kc, vc, nullptr, kv_filled, true,
             kv_filled + t, partial, S(stream));
  EET_API_END
}

int eet_tp_attention_core(eet_runtime* rt, const float* x, long long x_sb, long long x_ss,
                          int batch, int t, const eet_layer_weights* w, void* kc, void* vc,
                          int kv_filled, const int* h_pads, int seq_len, int phase, int* rows, void* stream) {
  EET_API_BEGIN
  check_layer_args(rt, batch, t, kv_filled, h_pads, seq_len, phase);
  StepPlan& p = rt->plans[0];
  plan_fill(p, batch, t, h_pads, seq_len, phase, S(stream));
  if (rows) *rows = p.T;
  attn_block(rt, p, const_cast<float*>(x), x_sb, x_ss, w, kc, vc, nullptr, kv_filled, true,
             kv_filled + t, nullptr, S(stream), /*keep_ctx=*/true);
  EET_API_END
}

// row-split projection of the kept activation (ctx / mid) for packed rows
// [r0, r1) into this rank's partial rows (ld h)
static void tp_out_rows(eet_runtime* rt, const void* act, int K, const void* W, const float* bias, int r0,
                        int r1, void* partial, cudaStream_t st) {
  const StepPlan& p = rt->plans[0];
  EET_REQUIRE(p.valid && act, EET_ERR_ARG, "tensor-parallel rows before their core stage");
  EET_REQUIRE(r0 >= 0 && r1 <= p.T && r0 <= r1, EET_ERR_ARG, "tensor-parallel rows out of range");
  if (r1 == r0) return;
  const size_t es = dtype_size(rt->dtype);
  const Epi e = tp_partial_epi(rt, partial, bias);
  gemm(rt->dtype, reinterpret_cast<const char*>(act) + (size_t)r0 * K * es, K, W, K, r1 - r0, rt->h, K, e, st);
}

int eet_tp_attention_out(eet_runtime* rt, const eet_layer_weights* w, int r0, int r1, void* partial_rows,
                         void* stream) {
  EET_API_BEGIN
  tp_out_rows(rt, rt->tp_ctx, rt->hq, w->wo, w->b_o, r0, r1, partial_rows, S(stream));
  EET_API_END
}

int eet_tp_ffn_partial(eet_runtime* rt, const float* x, long long x_sb, long long x_ss,
                       const eet_layer_weights* w, void* partial, void* stream) {
  EET_API_BEGIN
  EET_REQUIRE(rt->plans[0].valid, EET_ERR_ARG, "ffn partial before an attention partial");
  ffn_block(rt, rt->plans[0], const_cast<float*>(x), x_sb, x_ss, w, partial, S(stream));
  EET_API_END
}

int eet_tp_ffn_mid(eet_runtime* rt, const float* x, long long x_sb, long long x_ss,
                   const eet_layer_weights* w, void* stream) {
  EET_API_BEGIN
  EET_REQUIRE(rt->plans[0].valid, EET_ERR_ARG, "ffn partial before an attention partial");
  ffn_block(rt, rt->plans[0], const_cast<float*>(x), x_sb, x_ss, w, nullptr, S(stream), /*keep_mid=*/true);
  EET_API_END
}

int eet_tp_ffn_out(eet_runtime* rt, const eet_layer_weights* w, int r0, int r1, void* partial_rows,
                   void* stream) {
  EET_API_BEGIN
  tp_out_rows(rt, rt->tp_mid, rt->ffn, w->w2, w->b_2, r0, r1, partial_rows, S(stream));
  EET_API_END
}

int eet_tp_residual_add(eet_runtime* rt, float* x, long long x_sb, long long x_ss,
                        const void* reduced, void* stream) {
  EET_API_BEGIN
  EET_REQUIRE(rt->plans[0].valid, EET_ERR_ARG, "residual add before an attention partial");
  const StepPlan& p = rt->plans[0];
  launch_residual_add(x, x_sb, x_ss, p.rinfo, reduced, rt->dtype, p.T, rt->h, S(stream));
  EET_API_END
}

// ----------------------------------------------------------- generate
static void head_step(eet_runtime* rt, const eet_model* m, const float* x, long long x_sb,
                      int slot, int batch, int steps, long long* d_tokens, float* d_logits,
                      cudaStream_t st) {
  const int h = rt->h, dt = rt->dtype;
  const size_t es = dtype_size(dt);
  Claim lg(rt->pool, (size_t)batch * m->vocab * 4, EET_SCOPE_ACROSS, "output.logits");
  Epi e;
  e.mode = EPI_STORE_F32;
  e.out = lg.ptr;
  e.ldo = m->vocab;
  // rows (b, slot): the decode plan's row map (b, 0) over x shifted by `slot`
  const float* xs = x + (long long)slot * h;
  if (x == rt->xdec && skip_decode("head")) {         // ablation: decode-step head
    lg.release();
    return;
  }
  // packed head: argmax fused into the GEMV (no logits round trip)
  const int rtiles = (m->vocab + 15) / 16;
  if (rt->cand_cap < rtiles) {
    rt->cand = (int2*)rt->dev(sizeof(int2) * (size_t)rtiles * 16);
    rt->cand_ticket = (int*)rt->dev(sizeof(int));
    EET_CHECK_CUDA(cudaMemsetAsync(rt->cand_ticket, 0, sizeof(int), st));
    rt->cand_cap = rtiles;
  }
  Epi ea;
  ea.mode = EPI_ARGMAX;
  ea.out = d_logits;
  ea.ldo = m->vocab;
  ea.cand = rt->cand;
  ea.ticket = rt->cand_ticket;
  ea.cur = rt->d_cur;
  ea.toks = d_tokens;
  ea.d_step = rt->d_step;
  ea.steps = steps;
  ea.batch = batch;
  if (lm_head_argmax(dt, m->head, batch, m->vocab, h, xs, x_sb, h, rt->plans[2].rinfo, m->lnf_g, m->lnf_b, ea,
                     st)) {
    lg.release();
    return;
  } else if (!(batch <= 32 && gemv_tc_ln_sm100(dt, xs, x_sb, h, rt->plans[2].rinfo, m->lnf_g, m->lnf_b,
                                               m->head, h, batch, m->vocab, h, e, st))) {
    Claim ln(rt->pool, (size_t)batch * h * es, EET_SCOPE_ACROSS, "output.layernorm");
    launch_layer_norm(xs, x_sb, h, nullptr, batch, m->lnf_g, m->lnf_b, ln.ptr, dt, h, h, 0, st);
    gemm(dt, ln.ptr, h, m->head, h, batch, m->vocab, h, e, st);
  }
  launch_argmax(lg.as<float>(), batch, m->vocab, rt->d_cur, d_tokens, steps, rt->d_step, d_logits,
                st);
  lg.release();
}

// L_host: keys attended this step when known on the host (-1 under capture)
// The decode residual stream lives in a compact [b, h] buffer: the activation
// cache rows (max_prompt * h apart, one 2 MB page each at c2) cost every
// LN-fused GEMV a TLB walk per row.
static void decode_iteration(eet_runtime* rt, const eet_model* m, int batch, int steps,
                             long long* d_tokens, float* d_logits, int L_host, cudaStream_t st) {
  const int h = rt->h;
  if (!rt->xdec) rt->xdec = (float*)rt->dev(sizeof(float) * (size_t)rt->bmax * h);
  float* x = rt->xdec;
  const long long x_sb = h;
  StepPlan& p = rt->plans[2];
  launch_embed_step(rt->dtype, m->tok_emb, m->pos_emb, rt->d_cur, p.pads, rt->d_filled, x, x_sb,
                    batch, h, st);
  for (int l = 0; l < m->layers; ++l)
    layer_impl(rt, p, x, x_sb, h, &m->layer[l], m->kcache[l], m->vcache[l], rt->d_filled, 0, true,
               L_host, st);
  launch_advance(rt->d_filled, rt->d_step, st);
  head_step(rt, m, x, x_sb, 0, batch, steps, d_tokens, d_logits, st);
}

int eet_generate(eet_runtime* rt, const eet_model* m, const int* h_prompts, const int* h_lengths,
                 int batch, int max_len, int steps, long long* h_tokens, float* d_logits,
                 int use_graph, void* stream) {
  EET_API_BEGIN
  EET_REQUIRE(batch >= 1 && batch <= rt->bmax, EET_ERR_SHAPE, "batch exceeds configured maximum");
  EET_REQUIRE(max_len >= 1 && max_len <= m->max_prompt, EET_ERR_SHAPE, "prompt exceeds max prompt");
  EET_REQUIRE(max_len + steps <= rt->smax && max_len + steps <= m->max_sequence, EET_ERR_SHAPE,
              "prompt + steps exceeds max sequence");
  cudaStream_t caller = S(stream);
  cudaStream_t st = rt->cs;
  EET_CHECK_CUDA(cudaEventRecord(rt->ev_in, caller));
  EET_CHECK_CUDA(cudaStreamWaitEvent(st, rt->ev_in, 0));
  if (rt->oacc)                       // pending out-projection: zero between layers, reset per call
    EET_CHECK_CUDA(cudaMemsetAsync(rt->oacc, 0, sizeof(long long) * (size_t)rt->bmax * rt->h, st));

  std::vector<int> pads(batch);
  int t = 0;
  for (int b = 0; b < batch; ++b) t = std::max(t, h_lengths[b]);
  EET_REQUIRE(t == max_len, EET_ERR_ARG, "max_len must equal the longest prompt");
  for (int b = 0; b < batch; ++b) {
    EET_REQUIRE(h_lengths[b] >= 1, EET_ERR_ARG, "every prompt must have at least one token");
    pads[b] = t - h_lengths[b];
  }
  // inputs go host -> pinned staging -> device (async DMA)
  std::memcpy(rt->h_prompts, h_prompts, sizeof(int) * (size_t)batch * max_len);
  EET_CHECK_CUDA(cudaMemcpyAsync(rt->d_prompts, rt->h_prompts, sizeof(int) * (size_t)batch * max_len,
                                 cudaMemcpyHostToDevice, st));
  const int h = rt->h;
  const long long x_sb = (long long)m->max_prompt * h;

  // prompt pass (PROMPT_PARALLEL over all slots at once)
  StepPlan& pp = rt->plans[1];
  plan_fill(pp, batch, t, pads.data(), t, EET_PHASE_PROMPT, st);
  launch_embed_prompt(rt->dtype, m->tok_emb, m->pos_emb, rt->d_prompts, max_len, pp.pads,
                      m->hidden, x_sb, batch, t, h, st);
  for (int l = 0; l < m->layers; ++l)
    layer_impl(rt, pp, m->hidden, x_sb, h, &m->layer[l], m->kcache[l], m->vcache[l], nullptr, 0,
               true, t, st);

  Claim tok(rt->pool, sizeof(long long) * (size_t)batch * std::max(steps, 1), EET_SCOPE_ACROSS,
            "output.tokens");
  if (steps > 0) {
    int zero = 0;
    EET_CHECK_CUDA(cudaMemcpyAsync(rt->d_filled, &t, sizeof(int), cudaMemcpyHostToDevice, st));
    EET_CHECK_CUDA(cudaMemcpyAsync(rt->d_step, &zero, sizeof(int), cudaMemcpyHostToDevice, st));
    StepPlan& ps = rt->plans[2];
    plan_fill(ps, batch, 1, pads.data(), t, EET_PHASE_INCREMENTAL, st);
    head_step(rt, m, m->hidden, x_sb, t - 1, batch, steps, tok.as<long long>(), d_logits, st);
    // step 0 eagerly (settles every pool buffer), the rest replay one graph
    decode_iteration(rt, m, batch, steps, tok.as<long long>(), d_logits, t + 1, st);
    if (steps > 1) {
      if (use_graph) {
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        const uint64_t before = g_launches.load();
        EET_CHECK_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        try {
          decode_iteration(rt, m, batch, steps, tok.as<long long>(), d_logits, -1, st);
        } catch (...) {
          cudaStreamEndCapture(st, &g);
          if (g) cudaGraphDestroy(g);
          throw;
        }
        EET_CHECK_CUDA(cudaStreamEndCapture(st, &g));
        // captured launches run only when the graph replays: count them there
        const uint64_t nodes = g_launches.load() - before;
        g_launches.fetch_sub(nodes);
        EET_CHECK_CUDA(cudaGraphInstantiate(&ge, g, 0));
        for (int s = 1; s < steps; ++s) {
          EET_CHECK_CUDA(cudaGraphLaunch(ge, st));
          count_launch(nodes);
          if (prof_on()) {                 // keys attended by this replay
            double keys = 0;
            for (int b = 0; b < batch; ++b) keys += t + s + 1 - pads[b];
            prof_after_replay(st, keys);
          }
        }
        prof_graph_reset();
        EET_CHECK_CUDA(cudaGraphExecDestroy(ge));
        EET_CHECK_CUDA(cudaGraphDestroy(g));
      } else {
        for (int s = 1; s < steps; ++s)
          decode_iteration(rt, m, batch, steps, tok.as<long long>(), d_logits, t + s + 1, st);
      }
    }
    EET_CHECK_CUDA(cudaMemcpyAsync(rt->h_tokens, tok.ptr, sizeof(long long) * (size_t)batch * steps,
                                   cudaMemcpyDeviceToHost, st));
  }
  tok.release();
  EET_CHECK_CUDA(cudaEventRecord(rt->ev_out, st));
  EET_CHECK_CUDA(cudaStreamWaitEvent(caller, rt->ev_out, 0));
  EET_CHECK_CUDA(cudaStreamSynchronize(st));
  if (steps > 0) std::memcpy(h_tokens, rt->h_tokens, sizeof(long long) * (size_t)batch * steps);
  EET_API_END
}

}  // extern "C"
