// Mask-fused attention (§2.1 Algorithm 1; attention.py:73-217,
// runtime.py:106-189). Causal and padding bounds are derived from the
// query/key slot indices and each sequence's pad offset; no mask tensor is
// built or read, keys below the pad offset are never loaded, and tiles that
// lie wholly in the padding are skipped.
//
//  * attn_prefill_kernel — context phase: flash-style online softmax over
//    64x64 (query, key) tiles, fp32 accumulation, scores never reach HBM.
//  * attn_decode_kernel  — incremental phase: split-K flash-decoding over the
//    KV cache, one query per sequence; the last CTA of each (b, head) merges
//    the splits. HBM-bound on the K/V read.
#include "sm100.cuh"

#include <cstdlib>

namespace eet {

// =============================================================== prefill
namespace {
constexpr int PQ = 64, PK = 64, PTHREADS = 256;
}

template <typename T, int HD>
__global__ void __launch_bounds__(PTHREADS) attn_prefill_kernel(PrefillArgs a) {
  extern __shared__ __align__(16) float sm[];
  float* Qs = sm;                          // [PQ][HD+1]
  float* Ks = Qs + PQ * (HD + 1);          // [PK][HD+1]
  float* Vs = Ks + PK * (HD + 1);          // [PK][HD]
  float* Ps = Vs + PK * HD;                // [PQ][PK+1]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int b = blockIdx.z, head = blockIdx.y, q0 = blockIdx.x * PQ;
  const int pad = a.pads[b];
  // valid slots [pad, seq): seq = this sequence's end (right-padded windows) or the common length
  const int seq = a.ends ? a.ends[b] : a.seq, hd = a.hd;
  const int qhi = min(q0 + PQ, seq);
  const T* Q = reinterpret_cast<const T*>(a.q);
  const T* K = reinterpret_cast<const T*>(a.k);
  const T* V = reinterpret_cast<const T*>(a.v);
  T* O = reinterpret_cast<T*>(a.o);
  // packed layouts give a per-sequence row base; padded layouts use b * seq
  const long long qrb = a.q_rowbase ? a.q_rowbase[b] : (long long)b * a.seq;
  const long long orb = a.o_rowbase ? a.o_rowbase[b] : (long long)b * a.seq;

  if (a.zero_pad_rows) {                   // padded layout: pad-query rows are exact zeros
    int zend = min(pad, qhi);
    for (int idx = tid; idx < (zend - q0) * hd; idx += PTHREADS) {
      int r = q0 + idx / hd, d = idx % hd;
      O[(orb + r) * a.ldo + head * hd + d] = from_f<T>(0.f);
    }
  }
  if (qhi <= pad || q0 >= seq) return;    // whole tile is padding: skipped

  // Q tile (rows outside [pad, seq) and dims >= hd are zero)
  for (int idx = tid; idx < PQ * HD; idx += PTHREADS) {
    int r = idx / HD, d = idx % HD;
    int slot = q0 + r;
    float v = 0.f;
    if (slot >= pad && slot < seq && d < hd)
      v = to_f(Q[(qrb + slot) * a.ldq + head * hd + d]);
    Qs[r * (HD + 1) + d] = v;
  }

  float m_i[4], l_i[4], o[4][HD / 16];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    m_i[i] = -INFINITY;
    l_i[i] = 0.f;
#pragma unroll
    for (int dd = 0; dd < HD / 16; ++dd) o[i][dd] = 0.f;
  }
  const int kend = a.causal ? qhi : seq;   // keys [pad, kend)
  const long long kb = (long long)b * a.k_sb + (long long)head * a.k_sh;

  for (int kt = pad; kt < kend; kt += PK) {
    __syncthreads();
    for (int idx = tid; idx < PK * HD; idx += PTHREADS) {
      int r = idx / HD, d = idx % HD;
      int slot = kt + r;
      float kv = 0.f, vv = 0.f;
      if (slot < kend && d < hd) {
        long long off = kb + (long long)slot * a.k_ss + d;
        kv = to_f(K[off]);
        vv = to_f(V[off]);
      }
      Ks[r * (HD + 1) + d] = kv;
      Vs[r * HD + d] = vv;
    }
    __syncthreads();
    float s[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) s[i][j] = 0.f;
#pragma unroll 8
    for (int d = 0; d < HD; ++d) {
      float qv[4], kv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) qv[i] = Qs[(ty * 4 + i) * (HD + 1) + d];
#pragma unroll
      for (int j = 0; j < 4; ++j) kv[j] = Ks[(tx + 16 * j) * (HD + 1) + d];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s[i][j] = fmaf(qv[i], kv[j], s[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int qs = q0 + ty * 4 + i;
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ks = kt + tx + 16 * j;
        bool ok = ks < kend && qs >= pad && qs < seq && (!a.causal || ks <= qs);
        s[i][j] = ok ? s[i][j] * a.scale : -INFINITY;
        mx = fmaxf(mx, s[i][j]);
      }
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float mn = fmaxf(m_i[i], mx);
      float corr = 1.f, rs = 0.f;
      if (mn != -INFINITY) {
        corr = (m_i[i] == -INFINITY) ? 0.f : expf(m_i[i] - mn);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float p = (s[i][j] == -INFINITY) ? 0.f : expf(s[i][j] - mn);
          s[i][j] = p;
          rs += p;
        }
        m_i[i] = mn;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) s[i][j] = 0.f;
      }
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) rs += __shfl_xor_sync(0xffffffffu, rs, off);
      l_i[i] = l_i[i] * corr + rs;
#pragma unroll
      for (int dd = 0; dd < HD / 16; ++dd) o[i][dd] *= corr;
#pragma unroll
      for (int j = 0; j < 4; ++j) Ps[(ty * 4 + i) * (PK + 1) + tx + 16 * j] = s[i][j];
    }
    __syncthreads();
    const int kn = min(PK, kend - kt);
    for (int k = 0; k < kn; ++k) {
      float pv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) pv[i] = Ps[(ty * 4 + i) * (PK + 1) + k];
#pragma unroll
      for (int dd = 0; dd < HD / 16; ++dd) {
        float vv = Vs[k * HD + tx + 16 * dd];
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i][dd] = fmaf(pv[i], vv, o[i][dd]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int qs = q0 + ty * 4 + i;
    if (qs < pad || qs >= seq) continue;
    const float inv = l_i[i] > 0.f ? 1.0f / l_i[i] : 0.f;
    T* orow = O + (orb + qs) * a.ldo + head * hd;
#pragma unroll
    for (int dd = 0; dd < HD / 16; ++dd) {
      int d = tx + 16 * dd;
      if (d < hd) orow[d] = from_f<T>(o[i][dd] * inv);
    }
  }
}

template <typename T, int HD>
static void prefill_launch(const PrefillArgs& a, cudaStream_t st, double bytes, double flops) {
  size_t smem = sizeof(float) * (PQ * (HD + 1) + PK * (HD + 1) + PK * HD + PQ * (PK + 1));
  auto k = attn_prefill_kernel<T, HD>;
  EET_CHECK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((a.seq + PQ - 1) / PQ, a.heads, a.batch);
  ProfScope ps(K_ATTN_PREFILL, st, bytes, flops);
  k<<<grid, PTHREADS, smem, st>>>(a);
  EET_LAUNCH_CHECK();
}

template <typename T>
static void prefill_dispatch(const PrefillArgs& a, cudaStream_t st, double bytes, double flops) {
  if (a.hd <= 16) prefill_launch<T, 16>(a, st, bytes, flops);
  else if (a.hd <= 32) prefill_launch<T, 32>(a, st, bytes, flops);
  else if (a.hd <= 64) prefill_launch<T, 64>(a, st, bytes, flops);
  else if (a.hd <= 128) prefill_launch<T, 128>(a, st, bytes, flops);
  else EET_REQUIRE(false, EET_ERR_UNSUPPORTED, "attention: head_dim > 128 not supported");
}

// Right-padded / windowed prompt pass on the tensor-core path: the last
// 64-key K/V tile of sequence b may reach past its end into cache slots this
// pass never wrote (stale values, possibly NaN); their P is 0 but 0 * NaN is
// NaN in the PV MMA. Zero those slots [end_b, min(seq, pad_b + 64 *
// ceil((end_b - pad_b) / 64))) of every (b, head) plane first.
__global__ void kv_zero_tail_kernel(PrefillArgs a, int es) {
  const int b = blockIdx.y, head = blockIdx.x;
  const int pad = a.pads[b], end = a.ends[b];
  const int tail = min(a.seq, pad + ((end - pad + 63) / 64) * 64);
  const long long row_bytes = (long long)a.hd * es;
  char* kb = reinterpret_cast<char*>(const_cast<void*>(a.k)) + ((long long)b * a.k_sb + (long long)head * a.k_sh) * es;
  char* vb = reinterpret_cast<char*>(const_cast<void*>(a.v)) + ((long long)b * a.k_sb + (long long)head * a.k_sh) * es;
  const long long n = (long long)(tail - end) * row_bytes / 4;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    reinterpret_cast<int*>(kb + end * row_bytes)[i] = 0;
    reinterpret_cast<int*>(vb + end * row_bytes)[i] = 0;
  }
}

void launch_attn_prefill(const PrefillArgs& a, cudaStream_t st) {
  if (a.batch <= 0 || a.seq <= 0) return;
  if (a.ends && a.dtype != EET_F32 && a.k_ss == a.hd) {
    kv_zero_tail_kernel<<<dim3(a.heads, a.batch), 128, 0, st>>>(a, (int)dtype_size(a.dtype));
    count_launch();
    EET_LAUNCH_CHECK();
  }
  // algorithmic work: valid (query, key) pairs only (pads skipped)
  double pairs = 0, rows = 0;
  for (int b = 0; b < a.batch && a.h_pads; ++b) {
    double len = (a.h_ends ? a.h_ends[b] : a.seq) - a.h_pads[b];
    pairs += a.causal ? len * (len + 1) / 2 : len * len;
    rows += len;
  }
  if (!a.h_pads) { pairs = (double)a.batch * a.seq * (a.seq + 1) / 2; rows = (double)a.batch * a.seq; }
  const double es = (double)dtype_size(a.dtype);
  const double bytes = rows * a.heads * a.hd * es * 4;
  const double flops = pairs * a.heads * 4.0 * a.hd;
  if (attn_prefill_tc(a, a.q_rows, st, bytes, flops)) return;   // tcgen05 path (16-bit, hd 64/128)
  switch (a.dtype) {
    case EET_F32: prefill_dispatch<float>(a, st, bytes, flops); break;
    case EET_BF16: prefill_dispatch<__nv_bfloat16>(a, st, bytes, flops); break;
    default: prefill_dispatch<__half>(a, st, bytes, flops);
  }
}

// ================================================================ decode
// Lane layout: LPK lanes cooperate on one key row (E dims each); a warp
// scores 32/LPK keys per step; 4 warps per CTA; each CTA owns one split of
// the window [pad_b, L) of one (b, head).
namespace {
constexpr int DWARPS = 4;
}

template <typename T, int E, int LPK, bool VEC>
__global__ void __launch_bounds__(DWARPS * 32) attn_decode_kernel(DecodeArgs a) {
  constexpr int G = 32 / LPK;
  constexpr int U = 8;                    // key steps whose K/V loads are in flight together
  __shared__ float sm_m[DWARPS], sm_l[DWARPS];
  __shared__ float sm_acc[DWARPS][LPK * E];
  __shared__ int sm_last;
  sm100::griddep_wait();                  // K/V of this step were written by the QKV GEMV
  sm100::griddep_launch_dependents();
  const int split = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / LPK, sub = lane % LPK;
  const int hd = a.hd;
  const int pad = a.pads[b];
  const int L = (a.kv_start ? *a.kv_start : 0) + a.kv_base + 1;
  const int n = L - pad;
  const int chunk = (n + a.splits - 1) / a.splits;
  const int ks = pad + split * chunk, ke = min(ks + chunk, L);
  const T* Q = reinterpret_cast<const T*>(a.q) + (long long)b * a.ldq + head * hd;
  const long long base = ((long long)b * a.heads + head) * a.smax * hd;
  const T* Kc = reinterpret_cast<const T*>(a.kc) + base;
  const T* Vc = reinterpret_cast<const T*>(a.vc) + base;
  const int d0 = sub * E;

  float q[E];
  if constexpr (VEC) {
    if (d0 < hd) {
#pragma unroll
      for (int c = 0; c < E; c += 16 / (int)sizeof(T)) load16<T>(Q + d0 + c, q + c);
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) q[e] = 0.f;
    }
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) q[e] = (d0 + e < hd) ? to_f(Q[d0 + e]) : 0.f;
  }

  float m = -INFINITY, l = 0.f, acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;

  auto load_row = [&](const T* src, int j, float* dst) {
    const long long off = (long long)j * hd + d0;
    if constexpr (VEC) {
#pragma unroll
      for (int c = 0; c < E; c += 16 / (int)sizeof(T)) load16<T>(src + off + c, dst + c);
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) dst[e] = (d0 + e < hd) ? to_f(src[off + e]) : 0.f;
    }
  };

  constexpr int STEP = DWARPS * G;        // keys per CTA-wide step
  for (int jb = ks + warp * G; jb < ke; jb += STEP * U) {   // warp-uniform trip count
    float kv[U][E], vv[U][E];
#pragma unroll
    for (int u = 0; u < U; ++u) {         // issue every load of the batch first
      const int j = jb + u * STEP + g;
      if (j < ke && d0 < hd) {
        load_row(Kc, j, kv[u]);
        load_row(Vc, j, vv[u]);
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) kv[u][e] = vv[u][e] = 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = jb + u * STEP + g;
      float dot = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) dot = fmaf(q[e], kv[u][e], dot);
#pragma unroll
      for (int o = 1; o < LPK; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      if (j < ke) {
        const float s = dot * a.scale;
        const float mn = fmaxf(m, s);
        const float corr = (m == -INFINITY) ? 0.f : expf(m - mn);
        const float p = expf(s - mn);
        l = l * corr + p;
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = fmaf(p, vv[u][e], acc[e] * corr);
        m = mn;
      }
    }
  }
  // merge the key groups of this warp (lanes with equal `sub`)
#pragma unroll
  for (int o = LPK; o < 32; o <<= 1) {
    float mo = __shfl_xor_sync(0xffffffffu, m, o);
    float lo = __shfl_xor_sync(0xffffffffu, l, o);
    float mn = fmaxf(m, mo);
    float c1 = (m == -INFINITY) ? 0.f : expf(m - mn);
    float c2 = (mo == -INFINITY) ? 0.f : expf(mo - mn);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      float ao = __shfl_xor_sync(0xffffffffu, acc[e], o);
      acc[e] = acc[e] * c1 + ao * c2;
    }
    l = l * c1 + lo * c2;
    m = mn;
  }
  if (g == 0) {
    if (sub == 0) { sm_m[warp] = m; sm_l[warp] = l; }
#pragma unroll
    for (int e = 0; e < E; ++e) sm_acc[warp][d0 + e] = acc[e];
  }
  __syncthreads();
  // warp 0 merges the 4 warps and publishes this split
  float* part = a.part + (((long long)b * a.heads + head) * a.splits + split) * (hd + 2);
  if (warp == 0) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < DWARPS; ++w) M = fmaxf(M, sm_m[w]);
    float Lsum = 0.f;
    float cw[DWARPS];
#pragma unroll
    for (int w = 0; w < DWARPS; ++w) {
      cw[w] = (sm_m[w] == -INFINITY) ? 0.f : expf(sm_m[w] - M);
      Lsum += sm_l[w] * cw[w];
    }
    for (int d = lane; d < hd; d += 32) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < DWARPS; ++w) v += sm_acc[w][d] * cw[w];
      if (a.splits == 1) {
        reinterpret_cast<T*>(a.o)[(long long)b * a.ldo + head * hd + d] = from_f<T>(v / Lsum);
      } else {
        part[d] = v;
      }
    }
    if (lane == 0 && a.splits > 1) { part[hd] = M; part[hd + 1] = Lsum; }
  }
  if (a.splits == 1) return;
  // the last split to finish merges all splits (no second launch)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int prev = atomicAdd(&a.counters[b * a.heads + head], 1);
    sm_last = (prev == a.splits - 1);
  }
  __syncthreads();
  if (!sm_last) return;
  __threadfence();
  const float* p0 = a.part + ((long long)b * a.heads + head) * a.splits * (hd + 2);
  float M = -INFINITY;
  for (int s2 = 0; s2 < a.splits; ++s2) M = fmaxf(M, __ldcg(p0 + s2 * (hd + 2) + hd));
  float Lsum = 0.f;
  for (int s2 = 0; s2 < a.splits; ++s2) {
    float ms = __ldcg(p0 + s2 * (hd + 2) + hd);
    if (ms != -INFINITY) Lsum += __ldcg(p0 + s2 * (hd + 2) + hd + 1) * expf(ms - M);
  }
  for (int d = threadIdx.x; d < hd; d += blockDim.x) {
    float v = 0.f;
    for (int s2 = 0; s2 < a.splits; ++s2) {
      float ms = __ldcg(p0 + s2 * (hd + 2) + hd);
      if (ms != -INFINITY) v += __ldcg(p0 + s2 * (hd + 2) + d) * expf(ms - M);
    }
    reinterpret_cast<T*>(a.o)[(long long)b * a.ldo + head * hd + d] = from_f<T>(v / Lsum);
  }
  if (threadIdx.x == 0) a.counters[b * a.heads + head] = 0;
}

// Streaming variant: the K and V rows of a (sequence, head) are contiguous in
// the [b, heads, s_max, hd] cache, so a producer warp moves them into a
// shared-memory ring with TMA bulk copies (64 keys per chunk, full/empty
// mbarriers) while 8 compute warps consume earlier chunks. With enough
// (sequence, head) pairs to fill the GPU (c2: 16 x 16) each CTA owns a whole
// pair and there is nothing to combine; small batches split the key range
// and the last CTA of a pair merges the splits. Requires 16-byte key rows.
constexpr int DCHUNK = 64;
constexpr int CWARPS = 8;

template <typename T, int E, int LPK, int NBUF>
__global__ void __launch_bounds__((CWARPS + 1) * 32) attn_decode_bulk_kernel(DecodeArgs a) {
  constexpr int G = 32 / LPK;
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ __align__(8) uint64_t full[NBUF], empty[NBUF];
  __shared__ float sm_m[CWARPS], sm_l[CWARPS];
  __shared__ float sm_acc[CWARPS][LPK * E];
  __shared__ int sm_last;
  const int split = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / LPK, sub = lane % LPK;
  const int hd = a.hd;
  const size_t chunk_elems = (size_t)DCHUNK * hd;
  T* ring = reinterpret_cast<T*>(dsm);                    // [NBUF][K chunk | V chunk]
  if (threadIdx.x == 0) {
    for (int i = 0; i < NBUF; ++i) {
      sm100::mbar_init(&full[i], 1);
      sm100::mbar_init(&empty[i], CWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // The cursor and the pads were written long before the preceding kernel
  // and every cache slot but this step's (L-1, written by the QKV GEMV that
  // precedes us) by earlier steps: the producer streams those before
  // griddepcontrol.wait, so the first chunks land while the GEMV finishes.
  const int pad = a.pads[b];
  const int L = (a.kv_start ? *a.kv_start : 0) + a.kv_base + 1;
  const int n = L - pad;
  const int per = (n + a.splits - 1) / a.splits;
  const int ks = pad + split * per, ke = min(ks + per, L);
  const int nk = max(ke - ks, 0);
  const int nch = (nk + DCHUNK - 1) / DCHUNK;
  const long long base = ((long long)b * a.heads + head) * a.smax * hd;

  if (warp == CWARPS) {                   // ---- producer warp
    if (lane == 0) {
      const T* Kc = reinterpret_cast<const T*>(a.kc) + base + (long long)ks * hd;
      const T* Vc = reinterpret_cast<const T*>(a.vc) + base + (long long)ks * hd;
      bool waited = false;
      for (int c = 0; c < nch; ++c) {
        const int buf = c % NBUF;
        if (c >= NBUF) sm100::mbar_wait(&empty[buf], ((c / NBUF) - 1) & 1);
        const int kn = min(DCHUNK, nk - c * DCHUNK);
        if (!waited && ks + c * DCHUNK + kn == L) {   // chunk holds this step's slot
          sm100::griddep_wait();
          waited = true;
        }
        const uint32_t bytes = (uint32_t)(kn * hd * sizeof(T));
        T* dst = ring + buf * 2 * chunk_elems;
        sm100::mbar_expect_tx(&full[buf], 2 * bytes);
        if (a.kv_policy) {             // cached rows are read once per step: EVICT_FIRST
          sm100::bulk_load_hint(dst, Kc + (size_t)c * chunk_elems, bytes, &full[buf], a.kv_policy);
          sm100::bulk_load_hint(dst + chunk_elems, Vc + (size_t)c * chunk_elems, bytes, &full[buf], a.kv_policy);
        } else {
          sm100::bulk_load(dst, Kc + (size_t)c * chunk_elems, bytes, &full[buf]);
          sm100::bulk_load(dst + chunk_elems, Vc + (size_t)c * chunk_elems, bytes, &full[buf]);
        }
      }
    }
  } else {                                // ---- compute warps
    sm100::griddep_wait();                // q of this step comes from the QKV GEMV
    sm100::griddep_launch_dependents();
    const T* Q = reinterpret_cast<const T*>(a.q) + (long long)b * a.ldq + head * hd;
    const int d0 = sub * E;
    float q[E];
    if (d0 < hd) {
#pragma unroll
      for (int c = 0; c < E; c += 16 / (int)sizeof(T)) load16<T>(Q + d0 + c, q + c);
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) q[e] = 0.f;
    }
    float m = -INFINITY, l = 0.f, acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = 0.f;
    for (int c = 0; c < nch; ++c) {
      const int buf = c % NBUF;
      sm100::mbar_wait(&full[buf], (c / NBUF) & 1);
      const T* sK = ring + buf * 2 * chunk_elems;
      const T* sV = sK + chunk_elems;
      const int kn = min(DCHUNK, nk - c * DCHUNK);
      for (int jb = warp * G; jb < kn; jb += CWARPS * G) {     // warp-uniform
        const int j = jb + g;
        const bool ok = j < kn;
        float kv[E], vv[E];
        if (ok && d0 < hd) {
#pragma unroll
          for (int cc = 0; cc < E; cc += 16 / (int)sizeof(T)) {
            load16<T>(sK + (size_t)j * hd + d0 + cc, kv + cc);
            load16<T>(sV + (size_t)j * hd + d0 + cc, vv + cc);
          }
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e) kv[e] = vv[e] = 0.f;
        }
        float dot = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) dot = fmaf(q[e], kv[e], dot);
#pragma unroll
        for (int o = 1; o < LPK; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (ok) {
          const float s = dot * a.scale;
          const float mn = fmaxf(m, s);
          const float corr = (m == -INFINITY) ? 0.f : expf(m - mn);
          const float p = expf(s - mn);
          l = l * corr + p;
#pragma unroll
          for (int e = 0; e < E; ++e) acc[e] = fmaf(p, vv[e], acc[e] * corr);
          m = mn;
        }
      }
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&empty[buf]);
    }
#pragma unroll
    for (int o = LPK; o < 32; o <<= 1) {
      float mo = __shfl_xor_sync(0xffffffffu, m, o);
      float lo = __shfl_xor_sync(0xffffffffu, l, o);
      float mn = fmaxf(m, mo);
      float c1 = (m == -INFINITY) ? 0.f : expf(m - mn);
      float c2 = (mo == -INFINITY) ? 0.f : expf(mo - mn);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        float ao = __shfl_xor_sync(0xffffffffu, acc[e], o);
        acc[e] = acc[e] * c1 + ao * c2;
      }
      l = l * c1 + lo * c2;
      m = mn;
    }
    if (g == 0) {
      if (sub == 0) { sm_m[warp] = m; sm_l[warp] = l; }
#pragma unroll
      for (int e = 0; e < E; ++e) sm_acc[warp][d0 + e] = acc[e];
    }
  }
  __syncthreads();
  float* part = a.part + (((long long)b * a.heads + head) * a.splits + split) * (hd + 2);
  if (warp == 0) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < CWARPS; ++w) M = fmaxf(M, sm_m[w]);
    float Lsum = 0.f, cw[CWARPS];
#pragma unroll
    for (int w = 0; w < CWARPS; ++w) {
      cw[w] = (sm_m[w] == -INFINITY) ? 0.f : expf(sm_m[w] - M);
      Lsum += sm_l[w] * cw[w];
    }
    for (int d = lane; d < hd; d += 32) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < CWARPS; ++w) v += sm_acc[w][d] * cw[w];
      if (a.splits == 1) reinterpret_cast<T*>(a.o)[(long long)b * a.ldo + head * hd + d] = from_f<T>(v / Lsum);
      else part[d] = v;
    }
    if (lane == 0 && a.splits > 1) { part[hd] = M; part[hd + 1] = Lsum; }
  }
  if (a.splits == 1) return;
  // last split of the pair merges: the partial's writers (warp 0) fence it
  // to device scope, then a barrier and one acq_rel atomic (acquire of
  // everyone else's partials)
  if (warp == 0) __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int prev;
    asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(prev) : "l"(&a.counters[b * a.heads + head]) : "memory");
    sm_last = (prev == a.splits - 1);
  }
  __syncthreads();
  if (!sm_last) return;
  const float* p0 = a.part + ((long long)b * a.heads + head) * a.splits * (hd + 2);
  float M = -INFINITY;
  for (int s2 = 0; s2 < a.splits; ++s2) M = fmaxf(M, __ldcg(p0 + s2 * (hd + 2) + hd));
  float Lsum = 0.f;
  for (int s2 = 0; s2 < a.splits; ++s2) {
    float ms = __ldcg(p0 + s2 * (hd + 2) + hd);
    if (ms != -INFINITY) Lsum += __ldcg(p0 + s2 * (hd + 2) + hd + 1) * expf(ms - M);
  }
  for (int d = threadIdx.x; d < hd; d += blockDim.x) {
    float v = 0.f;
    for (int s2 = 0; s2 < a.splits; ++s2) {
      float ms = __ldcg(p0 + s2 * (hd + 2) + hd);
      if (ms != -INFINITY) v += __ldcg(p0 + s2 * (hd + 2) + d) * expf(ms - M);
    }
    reinterpret_cast<T*>(a.o)[(long long)b * a.ldo + head * hd + d] = from_f<T>(v / Lsum);
  }
  if (threadIdx.x == 0) a.counters[b * a.heads + head] = 0;
}

int decode_splits(int batch, int heads, int smax, int hd, int es) {
  (void)hd; (void)es;
  // one wave of the streaming kernel (3 CTAs of 64 KB ring per SM): a
  // second, partial wave of split CTAs costs more than the merge saves
  // (ncu r01: 512 CTAs = 1.15 waves, 22.6 us for 34 MB)
  const int pairs = std::max(1, batch * heads);
  const int slots = 3 * device_sm_count();
  const int by_sms = std::max(1, slots / pairs);
  const int cap = std::max(1, (smax + 63) / 64);       // >= 64 keys per split
  static const int forced = [] {                       // A/B switch
    const char* e = std::getenv("EET_DEC_SPLITS");
    return e ? atoi(e) : 0;
  }();
  if (forced > 0) return std::min(forced, cap);
  return std::max(1, std::min(by_sms, std::min(cap, 64)));
}

template <typename T, int E, int LPK, bool VEC>
static void decode_launch(const DecodeArgs& a, cudaStream_t st) {
  dim3 grid(a.splits, a.heads, a.batch);
  // algorithmic bytes: K and V rows of the window [pad_b, L) + q + out;
  // inside a captured graph L is device-side: the profiler scales per key
  const double es = (double)sizeof(T);
  const double per_key_b = (double)a.heads * a.hd * 2 * es, per_key_f = (double)a.heads * 4.0 * a.hd;
  double keys = 0;
  if (a.L_host >= 0)
    for (int b = 0; b < a.batch; ++b) keys += a.L_host - (a.h_pads ? a.h_pads[b] : 0);
  ProfScope ps(K_ATTN_DECODE, st, keys * per_key_b + 2.0 * a.batch * a.heads * a.hd * es,
               keys * per_key_f, a.L_host >= 0 ? 0.0 : per_key_b, a.L_host >= 0 ? 0.0 : per_key_f);
  launch_ex(attn_decode_kernel<T, E, LPK, VEC>, grid, dim3(DWARPS * 32), 0, st, true, dim3(1, 1, 1), a);
  EET_LAUNCH_CHECK();
}

template <typename T, int E, int LPK, int NBUF>
static void decode_bulk_launch_n(const DecodeArgs& a, cudaStream_t st);

template <typename T, int E, int LPK>
static void decode_bulk_launch(const DecodeArgs& a, cudaStream_t st) {
  // 4 x 16 KB ring (<= 64 KB): 2 CTAs per SM stay co-resident with the
  // neighbouring GEMVs under PDL (a 6-deep ring measured slower, r01)
  constexpr int NBUF = (E * LPK * sizeof(T) <= 128) ? 4 : 2;
  decode_bulk_launch_n<T, E, LPK, NBUF>(a, st);
}

template <typename T, int E, int LPK, int NBUF>
static void decode_bulk_launch_n(const DecodeArgs& a, cudaStream_t st) {
  dim3 grid(a.splits, a.heads, a.batch);
  double keys = 0;
  for (int b = 0; b < a.batch; ++b)
    keys += (a.L_host >= 0 ? a.L_host : a.smax) - (a.h_pads ? a.h_pads[b] : 0);
  const double es = (double)sizeof(T);
  const double per_key_b = (double)a.heads * a.hd * 2 * es, per_key_f = (double)a.heads * 4.0 * a.hd;
  if (a.L_host < 0) keys = 0;
  const size_t smem = (size_t)NBUF * 2 * DCHUNK * a.hd * sizeof(T);
  auto kern = attn_decode_bulk_kernel<T, E, LPK, NBUF>;
  EET_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ProfScope ps(K_ATTN_DECODE, st, keys * per_key_b + 2.0 * a.batch * a.heads * a.hd * es,
               keys * per_key_f, a.L_host >= 0 ? 0.0 : per_key_b, a.L_host >= 0 ? 0.0 : per_key_f);
  launch_ex(kern, grid, dim3((CWARPS + 1) * 32), smem, st, true, dim3(1, 1, 1), a);
  EET_LAUNCH_CHECK();
}

template <typename T>
static void decode_dispatch(const DecodeArgs& a, cudaStream_t st) {
  constexpr int VE = 16 / sizeof(T);
  const int hd = a.hd;
  {
    // streaming kernel: 16-byte key rows
    const bool ok = (hd * (int)sizeof(T)) % 16 == 0 && hd % VE == 0 && hd / VE <= 32 &&
                    hd * (int)sizeof(T) <= 512 && (a.ldq % VE) == 0 &&
                    ((reinterpret_cast<uintptr_t>(a.kc) | reinterpret_cast<uintptr_t>(a.vc) |
                      reinterpret_cast<uintptr_t>(a.q)) & 15) == 0;
    if (ok) {
      const int lanes = hd / VE;
      // 16-bit head_dim 64: 4 lanes x 16 elements per key, 8 keys per warp
      // step = one step per 64-key chunk (half the serial softmax chain of
      // 8 lanes x 8)
      static const int e16 = [] {
        const char* e = std::getenv("EET_ATTN_E8");
        return (e && e[0] == '1') ? 0 : 1;
      }();
      static const int nbuf = [] {                     // A/B switch: ring depth
        const char* e = std::getenv("EET_DEC_NBUF");
        return e ? atoi(e) : 4;
      }();
      if (sizeof(T) == 2 && hd == 64 && e16) {
        if (nbuf == 3) return decode_bulk_launch_n<T, 2 * VE, 4, 3>(a, st);
        if (nbuf == 2) return decode_bulk_launch_n<T, 2 * VE, 4, 2>(a, st);
        return decode_bulk_launch<T, 2 * VE, 4>(a, st);
      }
      if (lanes <= 1) return decode_bulk_launch<T, VE, 1>(a, st);
      if (lanes <= 2) return decode_bulk_launch<T, VE, 2>(a, st);
      if (lanes <= 4) return decode_bulk_launch<T, VE, 4>(a, st);
      if (lanes <= 8) return decode_bulk_launch<T, VE, 8>(a, st);
      if (lanes <= 16) return decode_bulk_launch<T, VE, 16>(a, st);
      return decode_bulk_launch<T, VE, 32>(a, st);
    }
  }
  EET_REQUIRE(hd <= 256, EET_ERR_UNSUPPORTED, "decode attention: head_dim > 256");
  const bool vec = (hd % VE == 0) && ((reinterpret_cast<uintptr_t>(a.kc) | reinterpret_cast<uintptr_t>(a.vc) | reinterpret_cast<uintptr_t>(a.q)) & 15) == 0 && (a.ldq % VE == 0);
  if (vec) {
    int lanes = hd / VE;
    if (lanes <= 1) return decode_launch<T, VE, 1, true>(a, st);
    if (lanes <= 2) return decode_launch<T, VE, 2, true>(a, st);
    if (lanes <= 4) return decode_launch<T, VE, 4, true>(a, st);
    if (lanes <= 8) return decode_launch<T, VE, 8, true>(a, st);
    if (lanes <= 16) return decode_launch<T, VE, 16, true>(a, st);
    if (lanes <= 32) return decode_launch<T, VE, 32, true>(a, st);
    return decode_launch<T, 2 * VE, 32, true>(a, st);
  }
  if (hd <= 1) return decode_launch<T, 1, 1, false>(a, st);
  if (hd <= 2) return decode_launch<T, 1, 2, false>(a, st);
  if (hd <= 4) return decode_launch<T, 1, 4, false>(a, st);
  if (hd <= 8) return decode_launch<T, 1, 8, false>(a, st);
  if (hd <= 16) return decode_launch<T, 1, 16, false>(a, st);
  if (hd <= 32) return decode_launch<T, 1, 32, false>(a, st);
  if (hd <= 64) return decode_launch<T, 2, 32, false>(a, st);
  if (hd <= 128) return decode_launch<T, 4, 32, false>(a, st);
  return decode_launch<T, 8, 32, false>(a, st);
}

void launch_attn_decode(const DecodeArgs& a_in, cudaStream_t st) {
  if (a_in.batch <= 0) return;
  static const unsigned long long pol = [] {     // A/B switch: EET_DEC_KV_EVICT_FIRST=0/1
    const char* e = std::getenv("EET_DEC_KV_EVICT_FIRST");
    return (e && e[0] == '1') ? 0x12F0000000000000ull : 0ull;
  }();
  DecodeArgs a = a_in;
  a.kv_policy = pol;
  switch (a.dtype) {
    case EET_F32: decode_dispatch<float>(a, st); break;
    case EET_BF16: decode_dispatch<__nv_bfloat16>(a, st); break;
    default: decode_dispatch<__half>(a, st);
  }
}

}  // namespace eet
