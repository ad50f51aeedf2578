// One decode-step kernel for the whole attention half of a layer:
// LayerNorm 1 + QKV projection (runtime.py:83-94, :131-136) fused with the
// attention over the cache (:160-178) and the out-projection (:186-188),
// for one new token per sequence (incremental phase).
//
// Unfused, this is two dependent launches (the QKV GEMV, then the attention +
// out-projection of attn_o.cu), and the attention cannot start streaming the
// cached keys into its ring until q exists. Here the cached K/V rows of
// earlier steps stream from the first instruction (they do not depend on
// this step at all), while the same CTAs compute q, k, v:
//
//   * grid (sequence, head), clusters of 8 sequences of one head; CTA rank r
//     owns the K-slice [r*Kc, (r+1)*Kc) of the hidden dimension (Kc = h/8);
//   * before griddepcontrol.wait: TMA of the CTA's QKV weight block (this
//     head's 3 x 64 rows x Kc columns, 48 KB at h1024), LN1 gamma/beta of the
//     slice, and the producer warp's cp.async.bulk K/V ring (no wait at all:
//     the rows are older than this step);
//   * after the wait: LayerNorm 1 of the cluster's 8 residual rows — each CTA
//     its slice's (mean, M2), all-gathered over DSMEM and combined in rank
//     order (Chan), identical in every CTA — then mma.sync m16n8k16 of the
//     normalised slice against the weight block: a split-K partial of the
//     192 q/k/v values of all 8 sequences, each sequence's part sent
//     (st.async) to the CTA that owns that sequence, which sums the 8
//     partials in rank order, rounds to the layer dtype (as the unfused path
//     stores q and the cache), writes this step's K/V slot and keeps q;
//   * the QKV block's shared memory is reused for the W_o block (TMA, lands
//     during the attention) and two more K/V ring slots (the ring is NBUF
//     deep while q/k/v are computed and NBUF + 2 deep for the attention);
//   * online-softmax attention over the ring (earlier keys) plus this step's
//     key from shared memory, then the attn_o.cu tail: context all-gather,
//     mma out-projection, 2^-32 fixed-point red.global.add.u64 into the
//     pending residual (order-independent, deterministic).
#include "mma_frag.cuh"

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

namespace eet {
namespace qao {
using namespace sm100;

constexpr int HD = 64, E = 16, LPK = 4, G = 32 / LPK, CW = 8, THREADS = (CW + 1) * 32, XP = 8, CB = 8;
constexpr int DCH = 64, NQ = 3 * HD, CST = HD + XP;
constexpr size_t CH = (size_t)DCH * HD;

// development trace (eet_debug_aotrace): per CTA globaltimer stamps [start,
// wait passed, LN staged, q/k/v reduced, attention done, contexts gathered]
// + end, (sequence << 16 | head) in [0]
__device__ int g_on = 0;
__device__ unsigned g_n = 0;
__device__ long long g_tr[4096][8];
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct Args {
  const float* x; long long x_sb;          // residual row b at x + b * x_sb
  const float* g; const float* bl;         // LayerNorm 1 gamma, beta
  const float* bqkv;                       // QKV bias [3 hq] or null
  void* kc; void* vc;                      // caches [b, heads, smax, HD]
  int heads, smax, h, hq, Kc, R;
  const int* pads;
  const int* kv_start; int kv_base;        // this step's slot = *kv_start + kv_base
  float scale;
  long long* acc; long long acc_sb;        // pending residual rows (2^-32 fixed point)
  const float* bo;                         // b_o (added by head 0) or null
  int l2pf;                                // prefetch the rows beyond the ring into L2
};

__host__ __device__ constexpr int al(int v, int a) { return (v + a - 1) / a * a; }

// shared-memory carve-up (host and device agree)
struct Lay {
  int ring, xs, recv, stats, cx, qkv, gb, total;
  __host__ __device__ Lay(int Kc, int R, int nbuf) {
    ring = al(NQ * Kc * 2 > R * HD * 2 ? NQ * Kc * 2 : R * HD * 2, 1024);
    xs = ring + nbuf * 2 * (int)CH * 2;
    recv = xs + al(8 * (Kc + XP) * 2, 16);
    stats = recv + CB * NQ * 4;
    cx = stats + CB * 8 * 8;
    qkv = cx + 8 * CST * 2;
    gb = qkv + NQ * 4;
    total = gb + 2 * Kc * 4 + 1024;        // + alignment slack of the 1024-aligned base
  }
};

// packed f32x2 math (FFMA2 / FMUL2)
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// two packed 16-bit values -> f32x2
template <typename T>
__device__ __forceinline__ uint64_t cvt2(uint32_t w) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    return f2pack(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
  } else {
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w));
    return f2pack(f.x, f.y);
  }
}

// q.k over two packed 16-bit pairs with fp32 accumulation and no conversion
// (FHFMA: the f16/bf16 products are exact in fp32, as after a conversion)
template <typename T>
__device__ __forceinline__ void hdot2(uint32_t q, uint32_t k, float& d0, float& d1) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    asm("{\n .reg .b16 ql, qh, kl, kh;\n mov.b32 {ql, qh}, %2;\n mov.b32 {kl, kh}, %3;\n"
        " fma.rn.f32.bf16 %0, ql, kl, %0;\n fma.rn.f32.bf16 %1, qh, kh, %1;\n}"
        : "+f"(d0), "+f"(d1) : "r"(q), "r"(k));
  } else {
    asm("{\n .reg .b16 ql, qh, kl, kh;\n mov.b32 {ql, qh}, %2;\n mov.b32 {kl, kh}, %3;\n"
        " fma.rn.f32.f16 %0, ql, kl, %0;\n fma.rn.f32.f16 %1, qh, kh, %1;\n}"
        : "+f"(d0), "+f"(d1) : "r"(q), "r"(k));
  }
}
template <typename T>
__device__ __forceinline__ uint32_t pack16(float a, float b) {
  T v[2] = {from_f<T>(a), from_f<T>(b)};
  return *reinterpret_cast<const uint32_t*>(v);
}
// four chains over E = 16 dims (8 packed words). fp16 uses the mixed FMA;
// bf16 converts (the bf16 form measured worse against the fp32 oracle at
// GPT-2-medium depth: elementwise ratio 2.2 vs 1.7 for the format itself)
template <typename T>
__device__ __forceinline__ float hdot16(const uint32_t* q, const uint32_t* k) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    uint64_t d2 = f2pack(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < 8; ++i) d2 = ffma2(cvt2<T>(q[i]), cvt2<T>(k[i]), d2);
    float lo, hi;
    f2unpack(d2, lo, hi);
    return lo + hi;
  } else {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      hdot2<T>(q[i], k[i], a0, a1);
      hdot2<T>(q[i + 1], k[i + 1], a2, a3);
    }
    return (a0 + a1) + (a2 + a3);
  }
}


__device__ __forceinline__ void st_async_b32(uint32_t addr, float v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(addr),
               "r"(__float_as_uint(v)), "r"(mbar)
               : "memory");
}

template <typename T, int NBUF>
__global__ void __launch_bounds__(THREADS) qkv_attn_o_kernel(const __grid_constant__ CUtensorMap mapQKV,
                                                             const __grid_constant__ CUtensorMap mapO,
                                                             const Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int Kc = a.Kc, R = a.R, XST = Kc + XP;
  const Lay Ly(Kc, R, NBUF);
  uint8_t* wbuf = smem;                                        // QKV block [3][Kc/64][64][64], then W_o [R][64]
  T* ring = reinterpret_cast<T*>(smem + Ly.ring);             // [NBUF][K chunk | V chunk]
  T* xs = reinterpret_cast<T*>(smem + Ly.xs);                 // [8][XST] normalised x slices
  float* recv = reinterpret_cast<float*>(smem + Ly.recv);     // [CB src][NQ] q/k/v partials of my sequence
  float2* stats = reinterpret_cast<float2*>(smem + Ly.stats); // [CB src][8 rows] slice (mean, M2)
  T* cx = reinterpret_cast<T*>(smem + Ly.cx);                 // [8][CST] the cluster's contexts
  float* qkvf = reinterpret_cast<float*>(smem + Ly.qkv);      // [NQ] my q, k, v (rounded to T)
  float* sgb = reinterpret_cast<float*>(smem + Ly.gb);        // [2][Kc] gamma, beta of my slice
  // ring slots: NBUF in their own bytes, plus up to XS more in the QKV
  // block's bytes once the QKV phase is done (next to the W_o block)
  constexpr int XS = 2;
  __shared__ __align__(8) uint64_t full[NBUF + XS], empty[NBUF + XS], wbar, obar, sbar, pbar, gbar, wfree;
  __shared__ float sm_m[CW], sm_l[CW];
  __shared__ float sm_acc[CW][HD];
  __shared__ __align__(16) T stage[HD];

  const int b = blockIdx.x, head = blockIdx.y;
  const int rank = (int)cluster_ctarank();                    // == b % CB
  const int b0 = b - rank;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k0 = rank * Kc;
  const int pad = a.pads[b];
  const int slot = (a.kv_start ? *a.kv_start : 0) + a.kv_base;  // this step's cache slot
  const int nk = max(slot - pad, 0);                          // earlier keys [pad, slot)
  const int nch = (nk + DCH - 1) / DCH;
  const long long base = ((long long)b * a.heads + head) * a.smax * HD;
  const int xoff = al(R * HD * 2, 1024);                      // extra slots after the W_o block
  const int S = NBUF + min(XS, (NQ * Kc * 2 - xoff) / (int)(2 * CH * 2));
  auto ring_slot = [&](int i) -> T* {
    return i < NBUF ? ring + i * 2 * CH : reinterpret_cast<T*>(wbuf + xoff) + (i - NBUF) * 2 * CH;
  };
  const bool trace = g_on && threadIdx.x == 0;
  long long ts[7] = {0, 0, 0, 0, 0, 0, 0};
  if (trace) ts[0] = gtime();

  if (threadIdx.x == 0) {
    for (int i = 0; i < NBUF + XS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CW);
    }
    mbar_init(&wfree, CW);
    mbar_init(&wbar, 1);
    mbar_init(&obar, 1);
    mbar_init(&sbar, 1);
    mbar_init(&pbar, 1);
    mbar_init(&gbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapQKV) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapO) : "memory");
    // static weights: this head's q, k, v rows x my K-slice, before the wait
    mbar_expect_tx(&wbar, (uint32_t)(NQ * Kc * 2));
#pragma unroll
    for (int j = 0; j < 3; ++j)
      tma_load_3d(wbuf + j * HD * Kc * 2, &mapQKV, &wbar, 0, j * a.hq + head * HD, k0 / 64, 0x1000000000000000ull);
    mbar_expect_tx(&sbar, (uint32_t)(CB * 8 * 8));
    mbar_expect_tx(&pbar, (uint32_t)(CB * NQ * 4));
    mbar_expect_tx(&gbar, (uint32_t)(CB * HD * 2));
  }
  for (int i = threadIdx.x; i < Kc; i += THREADS) {
    sgb[i] = __ldg(a.g + k0 + i);
    sgb[Kc + i] = __ldg(a.bl + k0 + i);
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");   // barriers initialised

  if (warp == CW) {                         // ---- producer warp: earlier keys, no dependency on this step
    if (lane == 0) {
      const T* Kc_ = reinterpret_cast<const T*>(a.kc) + base + (long long)pad * HD;
      const T* Vc_ = reinterpret_cast<const T*>(a.vc) + base + (long long)pad * HD;
      bool wfreed = false;
      auto load_wo = [&]() {                // QKV block consumed: W_o block into its first bytes
        mbar_wait(&wfree, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&obar, (uint32_t)(R * HD * 2));
        tma_load_2d(wbuf, &mapO, &obar, head * HD, rank * R, 0x1000000000000000ull);
        wfreed = true;
      };
      for (int c = 0; c < nch; ++c) {
        const int buf = c % S;
        if (c >= S) mbar_wait(&empty[buf], ((c / S) - 1) & 1);
        else if (buf >= NBUF && !wfreed) load_wo();
        const uint32_t bytes = (uint32_t)(min(DCH, nk - c * DCH) * HD * sizeof(T));
        T* dst = ring_slot(buf);
        mbar_expect_tx(&full[buf], 2 * bytes);
        bulk_load(dst, Kc_ + (size_t)c * CH, bytes, &full[buf]);
        bulk_load(dst + CH, Vc_ + (size_t)c * CH, bytes, &full[buf]);
        if (c == NBUF - 1 && a.l2pf)
          // The ring is full until q exists (after the wait, LN1 and the QKV
          // phase): the remaining rows of this (sequence, head) go to L2 in
          // the meantime, while HBM is otherwise idle, and the ring refills
          // from L2
          for (int c2 = NBUF; c2 < nch; ++c2) {
            const uint32_t pb = (uint32_t)(min(DCH, nk - c2 * DCH) * HD * sizeof(T));
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Kc_ + (size_t)c2 * CH), "r"(pb) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Vc_ + (size_t)c2 * CH), "r"(pb) : "memory");
          }
      }
      if (!wfreed) load_wo();
    }
    __syncwarp();
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    return;
  }

  // ---- consumer warps
  griddep_wait();                           // the residual rows come from the previous layer
  griddep_launch_dependents();
  if (trace) ts[1] = gtime();

  // 1. LayerNorm 1 of the cluster's 8 rows over the whole hidden dimension:
  //    warp w = sequence b0 + w, my slice's (mean, M2) to every CTA
  const bool lv = lane * 4 < Kc;
  const float inv_kc = 1.0f / (float)Kc;
  float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f);
  if (lv) v4 = *reinterpret_cast<const float4*>(a.x + (long long)(b0 + warp) * a.x_sb + k0 + lane * 4);
  const float mu = warp_sum((v4.x + v4.y) + (v4.z + v4.w)) * inv_kc;
  float ssq = 0.f;
  if (lv) {
    const float d0_ = v4.x - mu, d1 = v4.y - mu, d2 = v4.z - mu, d3 = v4.w - mu;
    ssq = (d0_ * d0_ + d1 * d1) + (d2 * d2 + d3 * d3);
  }
  ssq = warp_sum(ssq);
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");   // peers' barriers initialised
  if (lane < CB) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(
                     dsmem_addr(smem_u32(stats + rank * 8 + warp), (uint32_t)lane)),
                 "f"(mu), "f"(ssq), "r"(dsmem_addr(smem_u32(&sbar), (uint32_t)lane))
                 : "memory");
  }
  mbar_wait(&sbar, 0);
  {
    float sm = 0.f;
    for (int p = 0; p < CB; ++p) sm += stats[p * 8 + warp].x;
    const float mean = sm * (1.0f / CB);
    float m2 = 0.f, dd = 0.f;
    for (int p = 0; p < CB; ++p) {
      const float2 st = stats[p * 8 + warp];
      const float d = st.x - mean;
      m2 += st.y;
      dd += d * d;
    }
    m2 += dd * (float)Kc;
    const float rstd = rsqrtf(m2 / (float)a.h + 1e-5f);
    if (lv) {
      const int c = lane * 4;
      T o[4];
      o[0] = from_f<T>((v4.x - mean) * rstd * sgb[c + 0] + sgb[Kc + c + 0]);
      o[1] = from_f<T>((v4.y - mean) * rstd * sgb[c + 1] + sgb[Kc + c + 1]);
      o[2] = from_f<T>((v4.z - mean) * rstd * sgb[c + 2] + sgb[Kc + c + 2]);
      o[3] = from_f<T>((v4.w - mean) * rstd * sgb[c + 3] + sgb[Kc + c + 3]);
      *reinterpret_cast<uint2*>(xs + warp * XST + c) = *reinterpret_cast<const uint2*>(o);
    }
  }
  asm volatile("bar.sync 1, %0;" ::"n"(CW * 32) : "memory");   // consumer warps only
  if (trace) ts[2] = gtime();

  // 2. split-K partial of q/k/v (12 row tiles x 8 sequences); sequence t's
  //    values go to cluster CTA t
  mbar_wait(&wbar, 0);
  const int g4 = lane >> 2, c4 = lane & 3;
  for (int u = warp; u < NQ / 16; u += CW) {
    float pq[1][4];
    gc::warp_mma<T, 1>(smem_u32(wbuf + (u / 4) * HD * Kc * 2), HD, (u % 4) * 16, 0, Kc / 16, xs, XST, lane, pq);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int n = u * 16 + g4 + 8 * (i >> 1), t = 2 * c4 + (i & 1);
      st_async_b32(dsmem_addr(smem_u32(recv + rank * NQ + n), (uint32_t)t), pq[0][i],
                   dsmem_addr(smem_u32(&pbar), (uint32_t)t));
    }
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(&wfree);       // this warp is done with the QKV block

  // 3. my sequence's q, k, v: the 8 partials in rank order (+ bias), rounded
  //    to the layer dtype; this step's K/V into the cache slot
  mbar_wait(&pbar, 0);
  for (int n = threadIdx.x; n < NQ; n += CW * 32) {
    float v = 0.f;
#pragma unroll
    for (int s2 = 0; s2 < CB; ++s2) v += recv[s2 * NQ + n];
    const int which = n / HD, d = n - which * HD;
    if (a.bqkv) v += a.bqkv[which * a.hq + head * HD + d];
    const T tv = from_f<T>(v);
    qkvf[n] = to_f(tv);
    if (which) reinterpret_cast<T*>(which == 1 ? a.kc : a.vc)[base + (long long)slot * HD + d] = tv;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(CW * 32) : "memory");
  if (trace) ts[3] = gtime();

  // 4. online softmax: earlier keys from the ring, then this step's key.
  //    q.k as mixed-precision FMAs on the 16-bit operands (no conversions),
  //    packed f32x2 arithmetic (FFMA2) for p.v, and the running
  //    maximum rescales the accumulators only when it grows (corr would be
  //    exactly 1 otherwise): the chain per key is ~2/3 of the scalar form.
  const int g = lane / LPK, sub = lane % LPK, d0 = sub * E;
  uint32_t qh[E / 2];                      // q in the layer dtype (it was rounded to it)
  uint64_t acc2[E / 2];
#pragma unroll
  for (int i = 0; i < E / 2; ++i) {
    qh[i] = pack16<T>(qkvf[d0 + 2 * i], qkvf[d0 + 2 * i + 1]);
    acc2[i] = f2pack(0.f, 0.f);
  }
  float m = -INFINITY, l = 0.f;
  auto update = [&](float s, const uint64_t* v2) {          // one key of this lane group
    if (s > m) {
      const float corr = expf(m - s);                       // 0 for the first key
      l *= corr;
      const uint64_t c2 = f2pack(corr, corr);
#pragma unroll
      for (int i = 0; i < E / 2; ++i) acc2[i] = fmul2(acc2[i], c2);
      m = s;
    }
    const float p = expf(s - m);
    l += p;
    const uint64_t p2 = f2pack(p, p);
#pragma unroll
    for (int i = 0; i < E / 2; ++i) acc2[i] = ffma2(p2, v2[i], acc2[i]);
  };
  for (int c = 0; c < nch; ++c) {
    const int buf = c % S;
    mbar_wait(&full[buf], (c / S) & 1);
    const T* sK = ring_slot(buf);
    const T* sV = sK + CH;
    const int kn = min(DCH, nk - c * DCH);
    for (int jb = warp * G; jb < kn; jb += CW * G) {          // warp-uniform
      const int j = jb + g;
      const bool ok = j < kn;
      uint4 kr[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)}, vr[2] = {kr[0], kr[1]};
      if (ok) {
        kr[0] = *reinterpret_cast<const uint4*>(sK + (size_t)j * HD + d0);
        kr[1] = *reinterpret_cast<const uint4*>(sK + (size_t)j * HD + d0 + 8);
        vr[0] = *reinterpret_cast<const uint4*>(sV + (size_t)j * HD + d0);
        vr[1] = *reinterpret_cast<const uint4*>(sV + (size_t)j * HD + d0 + 8);
      }
      const uint32_t* kw = reinterpret_cast<const uint32_t*>(kr);
      const uint32_t* vw = reinterpret_cast<const uint32_t*>(vr);
      float dot = hdot16<T>(qh, kw);
#pragma unroll
      for (int o = 1; o < LPK; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      if (ok) {
        uint64_t v2[E / 2];
#pragma unroll
        for (int i = 0; i < E / 2; ++i) v2[i] = cvt2<T>(vw[i]);
        update(dot * a.scale, v2);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[buf]);
  }
  if (warp == 0) {                          // this step's key: group 0 of warp 0
    uint32_t kh[E / 2];
#pragma unroll
    for (int i = 0; i < E / 2; ++i) kh[i] = pack16<T>(qkvf[HD + d0 + 2 * i], qkvf[HD + d0 + 2 * i + 1]);
    float dot = hdot16<T>(qh, kh);
#pragma unroll
    for (int o = 1; o < LPK; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (g == 0) {
      uint64_t v2[E / 2];
#pragma unroll
      for (int i = 0; i < E / 2; ++i) v2[i] = f2pack(qkvf[2 * HD + d0 + 2 * i], qkvf[2 * HD + d0 + 2 * i + 1]);
      update(dot * a.scale, v2);
    }
  }
  float acc[E];
#pragma unroll
  for (int i = 0; i < E / 2; ++i) f2unpack(acc2[i], acc[2 * i], acc[2 * i + 1]);
#pragma unroll
  for (int o = LPK; o < 32; o <<= 1) {
    const float mo = __shfl_xor_sync(0xffffffffu, m, o);
    const float lo = __shfl_xor_sync(0xffffffffu, l, o);
    const float mn = fmaxf(m, mo);
    const float c1 = (m == -INFINITY) ? 0.f : expf(m - mn);
    const float c2 = (mo == -INFINITY) ? 0.f : expf(mo - mn);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const float ao = __shfl_xor_sync(0xffffffffu, acc[e], o);
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
  asm volatile("bar.sync 1, %0;" ::"n"(CW * 32) : "memory");
  if (trace) ts[4] = gtime();

  // 5. context row (layer dtype) -> every CTA of the cluster
  if (warp == 0) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < CW; ++w) M = fmaxf(M, sm_m[w]);
    float Lsum = 0.f, cw[CW];
#pragma unroll
    for (int w = 0; w < CW; ++w) {
      cw[w] = (sm_m[w] == -INFINITY) ? 0.f : expf(sm_m[w] - M);
      Lsum += sm_l[w] * cw[w];
    }
    for (int d = lane; d < HD; d += 32) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < CW; ++w) v += sm_acc[w][d] * cw[w];
      stage[d] = from_f<T>(v / Lsum);
    }
    __syncwarp();
    constexpr int PC = HD / 8;                                  // 16-byte pieces per context row
    for (int i = lane; i < CB * PC; i += 32) {
      const int peer = i / PC, c = i - peer * PC;
      const uint4 v = reinterpret_cast<const uint4*>(stage)[c];
      asm volatile(
          "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
              dsmem_addr(smem_u32(cx + rank * CST + c * 8), (uint32_t)peer)),
          "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(dsmem_addr(smem_u32(&gbar), (uint32_t)peer))
          : "memory");
    }
  }

  // 6. this head's share of the out-projection -> pending residual
  mbar_wait(&obar, 0);
  mbar_wait(&gbar, 0);
  if (trace) ts[5] = gtime();
  const bool add_bias = a.bo && head == 0;
  for (int u = warp; u < R / 16; u += CW) {
    float o[1][4];
    gc::warp_mma<T, 1>(smem_u32(wbuf), R, u * 16, 0, HD / 16, cx, CST, lane, o);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int n = rank * R + u * 16 + g4 + 8 * (i >> 1), tok = 2 * c4 + (i & 1);
      const float v = o[0][i] + (add_bias ? a.bo[n] : 0.f);
      const long long fx = __float2ll_rn(v * kAccScale);
      asm volatile("red.global.add.u64 [%0], %1;" ::"l"(a.acc + (long long)(b0 + tok) * a.acc_sb + n), "l"(fx)
                   : "memory");
    }
  }
  if (trace) {
    ts[6] = gtime();
    const unsigned i = atomicAdd(&g_n, 1u) & 4095u;
    g_tr[i][0] = ((long long)b << 16) | head;
#pragma unroll
    for (int j = 0; j < 7; ++j) g_tr[i][1 + j] = ts[j];
  }
}

}  // namespace qao

// trace control for eet_debug_aotrace (attn_o.cu)
void qao_trace(int on, long long* out, int* n) {
  if (on) {
    const int one = 1;
    const unsigned zero = 0;
    EET_CHECK_CUDA(cudaMemcpyToSymbol(qao::g_on, &one, sizeof(int)));
    EET_CHECK_CUDA(cudaMemcpyToSymbol(qao::g_n, &zero, sizeof(unsigned)));
  } else {
    const int zero = 0;
    unsigned cnt = 0;
    EET_CHECK_CUDA(cudaDeviceSynchronize());
    EET_CHECK_CUDA(cudaMemcpyToSymbol(qao::g_on, &zero, sizeof(int)));
    EET_CHECK_CUDA(cudaMemcpyFromSymbol(&cnt, qao::g_n, sizeof(unsigned)));
    EET_CHECK_CUDA(cudaMemcpyFromSymbol(out, qao::g_tr, sizeof(long long) * 4096 * 8));
    *n = (int)std::min<unsigned>(cnt, 4096u);
  }
}

// Eligible: 16-bit, head_dim 64, all heads on this GPU, hidden 512 or 1024
// (K-slices of 64 / 128 columns), the batch a multiple of 8.
bool qkv_attn_o_ok(int dtype, int batch, int h, int heads, int hd, int hq, const float* x, long long x_sb,
                   const void* kc, const void* vc, const void* wqkv, const void* wo) {
  static const bool on = [] {
    const char* v = std::getenv("EET_QKV_ATTN_O");
    return !(v && v[0] == '0');
  }();
  return on && (dtype == EET_F16 || dtype == EET_BF16) && hd == 64 && hq == heads * hd && hq == h &&
         (h == 512 || h == 1024) && batch % qao::CB == 0 && (x_sb & 3) == 0 &&
         ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(kc) | reinterpret_cast<uintptr_t>(vc) |
           reinterpret_cast<uintptr_t>(wqkv) | reinterpret_cast<uintptr_t>(wo)) & 15) == 0;
}

bool launch_qkv_attn_o(int dtype, int batch, int h, int heads, int smax, const float* x, long long x_sb,
                       const float* g, const float* bl, const void* wqkv, const float* bqkv, void* kc, void* vc,
                       const int* pads, const int* kv_start, int kv_base, const void* wo, const float* bo,
                       long long* acc, long long acc_sb, int L_host, const int* h_pads, cudaStream_t st) {
  const int hd = 64, hq = heads * hd;
  if (!qkv_attn_o_ok(dtype, batch, h, heads, hd, hq, x, x_sb, kc, vc, wqkv, wo)) return false;
  qao::Args a;
  a.x = x; a.x_sb = x_sb;
  a.g = g; a.bl = bl;
  a.bqkv = bqkv;
  a.kc = kc; a.vc = vc;
  a.heads = heads; a.smax = smax; a.h = h; a.hq = hq;
  a.Kc = h / qao::CB;
  a.R = h / qao::CB;
  a.pads = pads;
  a.kv_start = kv_start; a.kv_base = kv_base;
  a.scale = 1.0f / std::sqrt((float)hd);
  a.acc = acc; a.acc_sb = acc_sb;
  a.bo = bo;
  static const int l2pf = [] {                     // A/B: EET_QAO_L2PF=1 enables (measured no gain)
    const char* v = std::getenv("EET_QAO_L2PF");
    return (v && v[0] == '1') ? 1 : 0;
  }();
  a.l2pf = l2pf;

  static const int nbuf = [] {                     // A/B: EET_QAO_NBUF (2 or 3; 2 measured best)
    const char* v = std::getenv("EET_QAO_NBUF");
    return (v && v[0] == '3') ? 3 : 2;
  }();
  const size_t smem = (size_t)qao::Lay(a.Kc, a.R, nbuf).total;
  const CUtensorMap mq = make_tma_map_kblk(wqkv, 3 * hq, h, h, qao::HD, a.Kc / 64, dtype);
  const CUtensorMap mo = make_tma_map_2d(wo, h, hq, hq, a.R, dtype);
  double keys = 0;
  if (L_host >= 0)
    for (int b = 0; b < batch; ++b) keys += L_host - (h_pads ? h_pads[b] : 0);
  const double per_key_b = (double)heads * hd * 4;
  ProfScope ps(K_ATTN_DECODE, st,
               keys * per_key_b + 3.0 * h * hq * 2 + (double)h * hq * 2 + 4.0 * batch * h,
               keys * heads * 4.0 * hd + 2.0 * batch * 4 * h * hq, L_host >= 0 ? 0.0 : per_key_b,
               L_host >= 0 ? 0.0 : heads * 4.0 * hd);
  auto go = [&](auto kern) {
    static std::mutex mu;
    static std::unordered_map<const void*, size_t> set;
    {
      std::lock_guard<std::mutex> lk(mu);
      size_t& cur = set[reinterpret_cast<const void*>(kern)];
      if (cur < smem) {
        EET_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cur = smem;
      }
    }
    launch_cluster(kern, dim3(batch, heads), dim3(qao::THREADS), smem, st, true, dim3(qao::CB, 1, 1), mq, mo, a);
    EET_LAUNCH_CHECK();
  };
  if (dtype == EET_BF16) {
    if (nbuf == 2) go(qao::qkv_attn_o_kernel<__nv_bfloat16, 2>);
    else go(qao::qkv_attn_o_kernel<__nv_bfloat16, 3>);
  } else {
    if (nbuf == 2) go(qao::qkv_attn_o_kernel<__half, 2>);
    else go(qao::qkv_attn_o_kernel<__half, 3>);
  }
  return true;
}

}  // namespace eet
