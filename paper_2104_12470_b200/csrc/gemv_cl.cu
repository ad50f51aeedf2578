// Decode-step projections (16-bit modes, <= 16 token rows): runtime.py:131-136
// (QKV), :188 (out-proj), :206-213 (FFN) for one token per sequence, and the
// LM head + greedy argmax (:341-344, :425).
//
// A decode projection reads N*K weights once and <= 16 token rows; at c2
// (h1024) it is 2-8 MB, i.e. ~1 us of HBM time, so what matters is (a) that
// every SM streams its share of the weights, (b) that the weights are
// already on chip when the previous kernel finishes, and (c) the latency of
// what remains after griddepcontrol.wait. Layout of the work:
//
//   * clusters of C CTAs split K (C <= 8, K/C = Kc columns each); the G
//     clusters split N into blocks of R = 16*NT rows; G*C ~ one CTA per SM;
//   * each CTA TMA-loads its whole [R x Kc] weight block straight from the
//     K-major weight (128B swizzle, Kc/64 boxes) into shared memory BEFORE
//     griddepcontrol.wait — weights are static, so under programmatic
//     dependent launch they stream in while the previous kernel runs, and
//     the TMA engine keeps them out of the LSU queue the activation loads
//     use;
//   * after the wait a CTA reads only its own K-slice of the token rows
//     (fused LayerNorm from the fp32 residual stream, runtime.py:83-94: each
//     CTA's (mean, M2) of its slice is all-gathered through DSMEM and the C
//     partials are combined in rank order — Chan's parallel update, one
//     cluster barrier, deterministic);
//   * mma.sync m16n8k16 (weights = A via ldmatrix from the swizzled tile,
//     token rows = B), fp32 accumulators;
//   * split-K reduction through DSMEM: every 32-float accumulator chunk goes
//     to the cluster CTA that owns it, which sums the C (x k-group) partials
//     in a fixed order and applies the fused epilogue (Q + K/V-cache
//     scatter, residual add, GELU) — no global round trip, no atomics.
//
// The LM head (lm_head_kernel) is one persistent wave: the final LayerNorm
// of the token rows is staged once per CTA, then 16-row vocab tiles stream
// through a 4-stage TMA ring; each CTA keeps a running (max, lowest id) per
// token and argmax_cand_kernel reduces the per-CTA candidates.
#include "mma_frag.cuh"

#include <algorithm>
#include <cstdlib>

namespace eet {
namespace gc {
using namespace sm100;

constexpr int THREADS = 256, WARPS = 8, XPAD = 8;

// development trace (eet_debug_cltrace): CTA 0 and the last CTA of every
// launch record absolute globaltimer stamps [start, wait passed, X staged,
// weights landed, partials sent, reduced + epilogue done] plus (N, K).
__device__ int g_tr_on = 0;
__device__ unsigned g_tr_n = 0;
__device__ long long g_tr[8192][24];
__device__ __forceinline__ long long cyc() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr int MAX_KC = 512;                 // columns per CTA
constexpr int MAX_W_BYTES = 96 * 1024;      // weight block per CTA (two CTAs per SM under PDL)

struct LnSrc {                              // fused-LayerNorm operand source
  const float* x;                           // residual stream: decode row m at x + m * x_sb
  long long x_sb;
  const float* g;
  const float* b;
  const long long* acc;                     // pending fixed-point residual rows (or null), ld acc_sb
  long long acc_sb;
};

struct Shape {
  int M, N, K;
  int C, Kc, NT, KG;                        // cluster size, columns / CTA, 16-row tiles / cluster, k-groups
  const void* X; int ldx;                   // 16-bit activation rows (!LN)
  int warm;                                 // run the instruction-cache warm-up pass
  int ln;                                   // fused LayerNorm of fp32 rows (else X)
  int early;                                // trigger the dependent launch at kernel start
};

__host__ __device__ constexpr int align_up(int v, int a) { return (v + a - 1) / a * a; }

// shared-memory carve-up (host and device agree)
struct Lay {
  int w, x, gb, stats, recv, bar, total;
  __host__ __device__ Lay(int NT, int Kc, int C, int KG, int NB) {
    const int R = 16 * NT;
    w = 0;
    x = align_up(R * Kc * 2, 128);
    gb = x + align_up(16 * (Kc + XPAD) * 2, 128);
    stats = gb + Kc * 2 * 4;
    recv = stats + align_up(C * 16 * 8, 128);
    const int q = NT * NB;                     // 512 B accumulator chunks (one 16x8 block) per CTA
    const int per_owner = (q + C - 1) / C;
    bar = recv + C * KG * per_owner * 512;
    total = bar + 64 + 1024;                   // + alignment slack for the 1024-aligned base
  }
};

// decode epilogue (one mode per kernel instance: compact code): token row
// m is sequence m at cache slot kvs (runtime.py:136 cache write, :188/:212
// residual, :206-209 GELU)
template <typename T, int MODE>
__device__ __forceinline__ void dec_epi(const Epi& e, int kvs, int m, int n, float v) {
  if (e.bias) v += e.bias[n];
  if constexpr (MODE == EPI_STORE_F32) {
    reinterpret_cast<float*>(e.out)[(long long)m * e.ldo + n] = v;
  } else if constexpr (MODE == EPI_STORE_T) {
    reinterpret_cast<T*>(e.out)[(long long)m * e.ldo + n] = from_f<T>(v);
  } else if constexpr (MODE == EPI_GELU_T) {
    reinterpret_cast<T*>(e.out)[(long long)m * e.ldo + n] = from_f<T>(gelu_tanh(v));
  } else if constexpr (MODE == EPI_RESID) {
    float* xp = e.x + m * e.x_sb + n;
    if (e.acc) {                                    // fold in the pending out-projection, re-zero it
      long long* ap = e.acc + m * e.acc_sb + n;
      *xp = (*xp + acc_to_f(*ap)) + v;
      *ap = 0;
    } else {
      *xp += v;
    }
  } else if constexpr (MODE == EPI_QKV) {
    if (n < e.hq) {
      reinterpret_cast<T*>(e.out)[(long long)m * e.hq + n] = from_f<T>(v);
    } else {
      const int which = n >= 2 * e.hq;
      const int w = n - e.hq * (1 + which);
      const int head = (e.hd & (e.hd - 1)) ? w / e.hd : w >> (31 - __clz(e.hd));   // head_dim 64 / 128: shift
      const int d = w - head * e.hd;
      const long long off = (((long long)m * e.heads + head) * e.smax + kvs) * e.hd + d;
      reinterpret_cast<T*>(which ? e.vc : e.kc)[off] = from_f<T>(v);
    }
  }
}

// ---------------------------------------------------------------- projection
// One instance per (dtype, token n-blocks, LayerNorm width, epilogue): the
// code after the wait stays short (a unified runtime-mode kernel measured
// slower: r02, 935 vs 771 us per decode step).
template <typename T, int NB, int NV, int MODE, bool TRACE>
__global__ void __launch_bounds__(THREADS) gemv_cl_kernel(const __grid_constant__ CUtensorMap mapW,
                                                          const LnSrc ln, const Shape sh, const Epi e) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned (128B-swizzled TMA boxes) while staying a shared-space pointer
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr bool LN = NV > 0;
  const Lay L(sh.NT, sh.Kc, sh.C, sh.KG, NB);
  const int R = 16 * sh.NT, Kc = sh.Kc, C = sh.C, KG = sh.KG;
  const int xst = Kc + XPAD;
  T* xs = reinterpret_cast<T*>(smem + L.x);
  float2* stats = reinterpret_cast<float2*>(smem + L.stats);    // [C][16] (mean, M2) per slice
  float4* recv = reinterpret_cast<float4*>(smem + L.recv);      // [C*KG][per_owner][32 lanes]
  uint64_t* wbar = reinterpret_cast<uint64_t*>(smem + L.bar);   // weights landed (TMA)
  uint64_t* sbar = wbar + 1;                                    // all slices' LN statistics landed
  uint64_t* rbar = wbar + 2;                                    // all partials of my chunks landed
  const uint32_t sw = smem_u32(smem + L.w);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool trace = TRACE && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1);
  long long ts[6], cy[12] = {0};
  if (trace) { ts[0] = gtime(); cy[0] = cyc(); }
  const int rank = (int)cluster_ctarank();
  const int r0 = (blockIdx.x / C) * R;                          // first weight row of this cluster
  const int k0 = rank * Kc;
  const int Q = sh.NT * NB, per_owner = (Q + C - 1) / C;
  const int n_own = rank < Q ? (Q - rank + C - 1) / C : 0;      // chunks q = j*C + rank I reduce
  const float inv_kc = 1.0f / (float)Kc, inv_c = 1.0f / (float)C, inv_k = 1.0f / (float)sh.K;
  const bool warm_pass = sh.warm;

  // 1. before the wait (static data / data of kernels two or more launches
  //    back): barriers, the whole weight block (TMA), gamma/beta, the cache
  //    slot of this step
  if (threadIdx.x == 0) {
    mbar_init(wbar, 1);
    mbar_init(sbar, 1);
    mbar_init(rbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapW) : "memory");
    mbar_expect_tx(wbar, (uint32_t)(R * Kc * 2));
    const uint64_t pol = 0x12F0000000000000ull;              // EVICT_FIRST: read once per step
    tma_load_3d(smem + L.w, &mapW, wbar, 0, r0, k0 / 64, pol);     // [Kc/64][R][64] in one box
    if (C > 1) {                                              // DSMEM arrivals (one-CTA clusters stay local)
      if (LN) mbar_expect_tx(sbar, (uint32_t)(C * 16 * 8));
      mbar_expect_tx(rbar, (uint32_t)(n_own * C * KG * 512));
    }
  }
  constexpr int LNV = NV > 0 ? NV : 1;
  const int lrow = threadIdx.x >> 4, lsub = threadIdx.x & 15;  // LN: 16 threads per token row
  const int nv = Kc / 64;
  float* sgb = reinterpret_cast<float*>(smem + L.gb);         // [2][Kc] gamma, beta of this slice
  if constexpr (LN) {
    for (int i = threadIdx.x; i < Kc / 4; i += THREADS) {
      reinterpret_cast<float4*>(sgb)[i] = __ldg(reinterpret_cast<const float4*>(ln.g + k0) + i);
      reinterpret_cast<float4*>(sgb + Kc)[i] = __ldg(reinterpret_cast<const float4*>(ln.b + k0) + i);
    }
  }
  // the cursor is advanced once per step, many launches before this one
  const int kvs = (MODE == EPI_QKV) ? (e.kv_start ? *e.kv_start : 0) + e.kv_base : 0;
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  if (sh.early) griddep_launch_dependents();

  // The code after griddepcontrol.wait is what the decode step waits on, and
  // a decode step cycles ~5 different kernels through each SM: their code
  // does not stay in the instruction cache, and a cold pass measured 2-3x
  // the warm one (clock64 trace, r02). So the body runs twice: a dry pass
  // while the previous kernel is still finishing (inputs redirected to
  // harmless addresses, no stores / DSMEM / barrier waits) that pulls the
  // instructions in, then the real pass after the wait.
  const int KS = Kc / 16;
  const int units = sh.NT * KG;
  const int nsrc = C * KG;
#pragma unroll 1
  for (int pass = warm_pass ? 0 : 1; pass < 2; ++pass) {
    const bool dry = pass == 0;
    if (!dry) {
      griddep_wait();
      if (!sh.early) griddep_launch_dependents();
      if (trace) { ts[1] = gtime(); cy[1] = cyc(); }
    }

    // 2. this CTA's K-slice of the token rows -> xs (16-bit), rows >= M zero
    if constexpr (LN) {
      float4 v[LNV];
      const bool live = lrow < sh.M;
      const float4* xr = reinterpret_cast<const float4*>(
          dry ? ln.g + k0 : ln.x + (live ? lrow : 0) * ln.x_sb + k0);
      // x + the pending out-projection (attn_o.cu), both loads in flight together
      const bool pend = ln.acc && live && !dry;
      const longlong2* ar = reinterpret_cast<const longlong2*>(ln.acc + (pend ? lrow * ln.acc_sb + k0 : 0));
      longlong2 pa[LNV][2];
#pragma unroll
      for (int j = 0; j < LNV; ++j) {
        v[j] = (live && j < nv) ? xr[j * 16 + lsub] : make_float4(0.f, 0.f, 0.f, 0.f);
        pa[j][0] = pa[j][1] = make_longlong2(0, 0);
        if (pend && j < nv) {
          pa[j][0] = ar[(j * 16 + lsub) * 2];
          pa[j][1] = ar[(j * 16 + lsub) * 2 + 1];
        }
      }
      if (pend) {
#pragma unroll
        for (int j = 0; j < LNV; ++j) {
          v[j].x += acc_to_f(pa[j][0].x); v[j].y += acc_to_f(pa[j][0].y);
          v[j].z += acc_to_f(pa[j][1].x); v[j].w += acc_to_f(pa[j][1].y);
        }
      }
      // slice mean and M2 (two passes over registers), 16 lanes per row
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < LNV; ++j) s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
      if (trace && !dry) cy[2] = (s == 1.2345e-30f) ? 0 : cyc();
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      const float mu = s * inv_kc;
      float q = 0.f;
#pragma unroll
      for (int j = 0; j < LNV; ++j)
        if (j < nv) {
          const float a0 = v[j].x - mu, a1 = v[j].y - mu, a2 = v[j].z - mu, a3 = v[j].w - mu;
          q += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
        }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
      if (!dry) {
        if (trace) cy[3] = (q == 1.2345e-30f) ? 0 : cyc();
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");   // peers' barriers initialised
        if (trace) cy[4] = cyc();
        if (C > 1) {
          if (lsub < C)                                                        // all-gather (mean, M2)
            st_async_v2(dsmem_addr(smem_u32(stats + rank * 16 + lrow), lsub), mu, q, dsmem_addr(smem_u32(sbar), lsub));
          mbar_wait(sbar, 0);
        } else {                                                               // one-CTA cluster: local
          if (lsub == 0) stats[lrow] = make_float2(mu, q);
          __syncthreads();
        }
        if (trace) cy[5] = cyc();
      }
      // combine the C equal-size slices in rank order: identical in every CTA
      float sm = 0.f;
      for (int p = 0; p < C; ++p) sm += stats[p * 16 + lrow].x;
      const float mean = sm * inv_c;
      float m2 = 0.f, dd = 0.f;
      for (int p = 0; p < C; ++p) {
        const float2 st = stats[p * 16 + lrow];
        const float d = st.x - mean;
        m2 += st.y;
        dd += d * d;
      }
      m2 += dd * (float)Kc;
      const float rstd = rsqrtf(m2 * inv_k + 1e-5f);
      T* dst = xs + lrow * xst;
#pragma unroll
      for (int j = 0; j < LNV; ++j)
        if (j < nv) {
          const int c = (j * 16 + lsub) * 4;
          T o[4];
          if (live) {
            const float4 gg = *reinterpret_cast<const float4*>(sgb + c);
            const float4 bb = *reinterpret_cast<const float4*>(sgb + Kc + c);
            o[0] = from_f<T>((v[j].x - mean) * rstd * gg.x + bb.x);
            o[1] = from_f<T>((v[j].y - mean) * rstd * gg.y + bb.y);
            o[2] = from_f<T>((v[j].z - mean) * rstd * gg.z + bb.z);
            o[3] = from_f<T>((v[j].w - mean) * rstd * gg.w + bb.w);
          } else {
            o[0] = o[1] = o[2] = o[3] = from_f<T>(0.f);
          }
          *reinterpret_cast<uint2*>(dst + c) = *reinterpret_cast<const uint2*>(o);
        }
    } else {
      const T* X = reinterpret_cast<const T*>(sh.X);
      const int cpr = Kc / 8;                                   // 16-byte chunks per row
      // all of this thread's chunks in flight before the first shared store
      // (Kc <= 512: at most 4 per thread; one L2 round trip, not four)
      constexpr int XV = 4;
      uint4 tmp[XV];
#pragma unroll
      for (int k = 0; k < XV; ++k) {
        const int i = threadIdx.x + k * THREADS, r = i / cpr, c = i - r * cpr;
        tmp[k] = make_uint4(0, 0, 0, 0);
        if (i < 16 * cpr && r < sh.M && !dry) tmp[k] = *reinterpret_cast<const uint4*>(X + (size_t)r * sh.ldx + k0 + c * 8);
      }
#pragma unroll
      for (int k = 0; k < XV; ++k) {
        const int i = threadIdx.x + k * THREADS, r = i / cpr, c = i - r * cpr;
        if (i < 16 * cpr) *reinterpret_cast<uint4*>(xs + r * xst + c * 8) = tmp[k];
      }
    }
    __syncwarp();
    __syncthreads();
    if (!LN && !dry) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");   // before any DSMEM store
    if (!dry) {
      if (trace) { ts[2] = gtime(); cy[6] = cyc(); }
      mbar_wait(wbar, 0);
      if (trace) { ts[3] = gtime(); cy[7] = cyc(); }
    }

    // 3. MMA: unit (tile, k-group) per warp; 4. each 16x8 accumulator block
    //    to the cluster CTA that owns it (st.async, complete_tx on its rbar)
    for (int u = warp; u < units; u += WARPS) {
      const int t = u % sh.NT, kg = u / sh.NT;
      const int s0 = kg * (KS / KG), s1 = s0 + KS / KG;
      float acc[NB][4];
      warp_mma<T, NB>(sw, R, t * 16, s0, s1, xs, xst, lane, acc);
      if (trace && !dry && u == 0) cy[8] = (acc[0][0] == 1.2345e-30f) ? 0 : cyc();
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const int q = t * NB + nb;
        const int owner = q % C, j = q / C;
        float4* dst = recv + ((size_t)(rank * KG + kg) * per_owner + j) * 32 + lane;
        if (dry) continue;
        if (C > 1) st_async_v4(dsmem_addr(smem_u32(dst), owner), acc[nb], dsmem_addr(smem_u32(rbar), owner));
        else *dst = make_float4(acc[nb][0], acc[nb][1], acc[nb][2], acc[nb][3]);
      }
    }
    if (!dry) {
      if (trace) { ts[4] = gtime(); cy[9] = cyc(); }
      if (C == 1) __syncthreads();                     // local partials
      else if (n_own > 0) mbar_wait(rbar, 0);
      if (trace) cy[10] = cyc();
    }

    // 5. owner: fixed-order sum over (source rank, k-group), fused epilogue
    for (int idx = threadIdx.x; idx < n_own * 32; idx += THREADS) {
      const int j = idx >> 5, ln_ = idx & 31;
      const int q = j * C + rank;
      float4 v = recv[(size_t)j * 32 + ln_];
#pragma unroll 2
      for (int s2 = 1; s2 < nsrc; ++s2) {
        const float4 a = recv[((size_t)s2 * per_owner + j) * 32 + ln_];
        v.x += a.x; v.y += a.y; v.z += a.z; v.w += a.w;
      }
      const int t = q / NB, nb = q - t * NB;
      const int row = t * 16 + (ln_ >> 2), tok = nb * 8 + 2 * (ln_ & 3);
      const float vv[4] = {v.x, v.y, v.z, v.w};
      if constexpr (MODE == EPI_RESID) {
        // residual read-modify-write: the four elements' loads (x, and the
        // pending out-projection) all in flight before any store — one L2
        // round trip instead of four (the elements are distinct)
        float xv[4];
        long long av[4];
        bool ok[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int n = r0 + row + 8 * (i >> 1), m = tok + (i & 1);
          ok[i] = n < sh.N && m < sh.M && !dry;
          xv[i] = ok[i] ? e.x[m * e.x_sb + n] : 0.f;
          av[i] = (ok[i] && e.acc) ? e.acc[m * e.acc_sb + n] : 0;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (!ok[i]) continue;
          const int n = r0 + row + 8 * (i >> 1), m = tok + (i & 1);
          const float val = e.bias ? vv[i] + e.bias[n] : vv[i];
          if (e.acc) {
            e.x[m * e.x_sb + n] = (xv[i] + acc_to_f(av[i])) + val;
            e.acc[m * e.acc_sb + n] = 0;
          } else {
            e.x[m * e.x_sb + n] = xv[i] + val;
          }
        }
      } else {
#pragma unroll 1
        for (int i = 0; i < 4; ++i) {                  // rolled: one copy of the epilogue code
          const int n = r0 + row + 8 * (i >> 1), m = tok + (i & 1);
          if (n < sh.N && m < sh.M && !dry) dec_epi<T, MODE>(e, kvs, m, n, vv[i]);
        }
      }
    }
  }
  if (trace) {
    ts[5] = gtime();
    cy[11] = cyc();
    const unsigned i = atomicAdd(&g_tr_n, 1u) & 8191u;
    g_tr[i][0] = ((long long)sh.N << 32) | ((long long)sh.K << 1) | (LN ? 1 : 0);
    g_tr[i][1] = blockIdx.x;
#pragma unroll
    for (int k = 0; k < 6; ++k) g_tr[i][2 + k] = ts[k];
#pragma unroll
    for (int k = 1; k < 12; ++k) g_tr[i][8 + k - 1] = cy[k] ? cy[k] - cy[0] : -1;
  }
}

// ---------------------------------------------------------------- LM head
// Warp-specialised persistent wave: HCW consumer warps each take whole
// 16-row vocab tiles (full K, no cross-warp reduction) from an HSTAGES TMA
// ring filled by one producer warp; every consumer keeps a running
// (max, lowest id) per token in registers.
constexpr int HSTAGES = 6, HCW = 4, HTHREADS = (HCW + 1) * 32;   // 6 x 32 KB stages + 33 KB token rows

__device__ __forceinline__ bool better(float v, int i, float bv, int bi) {
  return v > bv || (v == bv && i < bi);
}

template <typename T, int NB>
__global__ void __launch_bounds__(HTHREADS) lm_head_kernel(const __grid_constant__ CUtensorMap mapW,
                                                           const LnSrc ln, int M, int N, int K, Epi e) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned (128B-swizzled TMA boxes) while staying a shared-space pointer
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int stage_bytes = 16 * K * 2;
  const int xst = K + XPAD;
  T* xs = reinterpret_cast<T*>(smem + HSTAGES * stage_bytes);
  float* bestv = reinterpret_cast<float*>(smem + HSTAGES * stage_bytes + align_up(16 * xst * 2, 128));  // [HCW][16]
  int* besti = reinterpret_cast<int*>(bestv + HCW * 16);                                              // [HCW][16]
  uint64_t* full = reinterpret_cast<uint64_t*>(besti + HCW * 16);                                     // [HSTAGES]
  uint64_t* empty = full + HSTAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles = (N + 15) / 16;
  const int nmine = tiles > (int)blockIdx.x ? (tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const uint64_t pol = 0x12F0000000000000ull;
  const bool trace = g_tr_on && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1);
  long long ts[6] = {0, 0, 0, 0, 0, 0};
  if (trace) ts[0] = gtime();
  if (threadIdx.x == 0) {
    for (int i = 0; i < HSTAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == HCW) {                                     // ---- producer warp
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mapW) : "memory");
      for (int i = 0; i < nmine; ++i) {
        const int st = i % HSTAGES;
        if (i >= HSTAGES) mbar_wait(&empty[st], (uint32_t)(((i / HSTAGES) - 1) & 1));
        const int t = blockIdx.x + i * gridDim.x;
        mbar_expect_tx(&full[st], stage_bytes);
        tma_load_3d(smem + st * stage_bytes, &mapW, &full[st], 0, t * 16, 0, pol);   // 16 whole rows
        if (i + 1 == HSTAGES) {                          // static weights: the first ring fill precedes the wait
          griddep_wait();
          griddep_launch_dependents();
        }
      }
      if (nmine < HSTAGES) {
        griddep_wait();
        griddep_launch_dependents();
      }
    }
    return;
  }
  // ---- consumers: final LayerNorm of the token rows -> xs. gamma / beta
  // of this lane's columns are static: loaded before the wait. Each warp
  // then takes two rows per pass (w, w+4 / w+8, w+12) with both rows' loads
  // in flight together: two dependent L2 round trips per warp instead of
  // eight (every CTA reads the same 16 rows at the same moment).
  const int nv = K / 4;
  float4 gg[8], bb[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int i = j * 32 + lane;
    gg[j] = i < nv ? __ldg(reinterpret_cast<const float4*>(ln.g) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    bb[j] = i < nv ? __ldg(reinterpret_cast<const float4*>(ln.b) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  griddep_wait();
  if (trace) ts[1] = gtime();
#pragma unroll 1
  for (int r0 = warp; r0 < 16; r0 += 2 * HCW) {
    float4 v[2][8];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int r = r0 + p * HCW;
      const float4* xr = reinterpret_cast<const float4*>(ln.x + (r < M ? r : 0) * ln.x_sb);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        v[p][j] = (r < M && j * 32 + lane < nv) ? xr[j * 32 + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float sm[2], rs[2];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) s += (v[p][j].x + v[p][j].y) + (v[p][j].z + v[p][j].w);
      sm[p] = s;
    }
#pragma unroll
    for (int p = 0; p < 2; ++p) sm[p] = warp_sum(sm[p]) / (float)K;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const float mu = sm[p];
      float qq = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j * 32 + lane < nv) {
          const float a0 = v[p][j].x - mu, a1 = v[p][j].y - mu, a2 = v[p][j].z - mu, a3 = v[p][j].w - mu;
          qq += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
        }
      rs[p] = qq;
    }
#pragma unroll
    for (int p = 0; p < 2; ++p) rs[p] = 1.0f / sqrtf(warp_sum(rs[p]) / (float)K + 1e-5f);
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int r = r0 + p * HCW;
      T* dst = xs + r * xst;
      const float mu = sm[p];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = j * 32 + lane;
        if (i < nv) {
          T o[4];
          if (r < M) {
            o[0] = from_f<T>((v[p][j].x - mu) * rs[p] * gg[j].x + bb[j].x);
            o[1] = from_f<T>((v[p][j].y - mu) * rs[p] * gg[j].y + bb[j].y);
            o[2] = from_f<T>((v[p][j].z - mu) * rs[p] * gg[j].z + bb[j].z);
            o[3] = from_f<T>((v[p][j].w - mu) * rs[p] * gg[j].w + bb[j].w);
          } else {
            o[0] = o[1] = o[2] = o[3] = from_f<T>(0.f);
          }
          *reinterpret_cast<uint2*>(dst + i * 4) = *reinterpret_cast<const uint2*>(o);
        }
      }
    }
  }
  asm volatile("bar.sync 1, %0;" ::"n"(HCW * 32) : "memory");   // consumers only
  if (trace) ts[2] = ts[3] = ts[4] = gtime();

  const int step = e.d_step ? *e.d_step : 0;
  const int g = lane >> 2, c4 = lane & 3;
  // lane (g == 0, c4) tracks tokens nb*8 + 2*c4 + {0, 1}
  float bv[NB][2];
  int bi[NB][2];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) { bv[nb][0] = bv[nb][1] = -INFINITY; bi[nb][0] = bi[nb][1] = 0x7fffffff; }
  for (int i = warp; i < nmine; i += HCW) {
    const int st = i % HSTAGES;
    const int t = blockIdx.x + i * gridDim.x;
    // A stage's successive tiles go to different consumer warps (HSTAGES is
    // not a multiple of HCW), so this warp can be two phases ahead of the
    // stage: tile i - HSTAGES (another warp's) may not even have landed yet,
    // and a parity wait on `full` alone would then pass on the older phase
    // and read the wrong tile. Waiting first for that tile's release
    // (the producer's own condition) makes the full-barrier parity
    // unambiguous.
    if (i >= HSTAGES) mbar_wait(&empty[st], (uint32_t)(((i / HSTAGES) - 1) & 1));
    mbar_wait(&full[st], (uint32_t)((i / HSTAGES) & 1));
    float acc[NB][4];
    warp_mma<T, NB>(smem_u32(smem + st * stage_bytes), 16, 0, 0, K / 16, xs, xst, lane, acc);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);             // stage consumed
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        // rows g and g + 8 of token nb*8 + 2*c4 + p, then over g (lanes ^4, ^8, ^16)
        const int n_lo = t * 16 + g, n_hi = n_lo + 8, tok = nb * 8 + 2 * c4 + p;
        float v = acc[nb][p], w = acc[nb][2 + p];
        if (e.out && step < e.steps && tok < M) {
          float* lo = reinterpret_cast<float*>(e.out) + ((long long)step * e.batch + tok) * e.ldo;
          if (n_lo < N) lo[n_lo] = v;
          if (n_hi < N) lo[n_hi] = w;
        }
        float cv = n_lo < N ? v : -INFINITY;
        int ci = n_lo;
        if (n_hi < N && better(w, n_hi, cv, ci)) { cv = w; ci = n_hi; }
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, cv, o);
          const int oi = __shfl_xor_sync(0xffffffffu, ci, o);
          if (better(ov, oi, cv, ci)) { cv = ov; ci = oi; }
        }
        if (better(cv, ci, bv[nb][p], bi[nb][p])) { bv[nb][p] = cv; bi[nb][p] = ci; }
      }
  }
  if (g == 0) {
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        bestv[warp * 16 + nb * 8 + 2 * c4 + p] = bv[nb][p];
        besti[warp * 16 + nb * 8 + 2 * c4 + p] = bi[nb][p];
      }
  }
  asm volatile("bar.sync 1, %0;" ::"n"(HCW * 32) : "memory");
  if (threadIdx.x < 16) {
    float v = -INFINITY;
    int id = 0x7fffffff;
    for (int w = 0; w < HCW; ++w)
      if (threadIdx.x < NB * 8 && better(bestv[w * 16 + threadIdx.x], besti[w * 16 + threadIdx.x], v, id)) {
        v = bestv[w * 16 + threadIdx.x];
        id = besti[w * 16 + threadIdx.x];
      }
    e.cand[blockIdx.x * 16 + threadIdx.x] = make_int2(__float_as_int(v), id);
  }
  if (trace) {
    ts[5] = gtime();
    const unsigned i = atomicAdd(&g_tr_n, 1u) & 8191u;
    g_tr[i][0] = ((long long)N << 32) | ((long long)K << 1) | 1;
    g_tr[i][1] = blockIdx.x;
    for (int k = 0; k < 6; ++k) g_tr[i][2 + k] = ts[k];
    for (int k = 8; k < 19; ++k) g_tr[i][k] = -1;
  }
}

// second stage of the fused argmax: one CTA per token reduces the per-CTA
// candidates (value, id) — any order gives the same answer: `better` is a
// total order (larger value, then lower id; runtime.py:425 np.argmax)
__global__ void __launch_bounds__(256) argmax_cand_kernel(const int2* __restrict__ cand, int ncand,
                                                          int* __restrict__ cur, long long* __restrict__ toks,
                                                          int steps, const int* __restrict__ d_step) {
  __shared__ float sv[8];
  __shared__ int si[8];
  griddep_wait();
  griddep_launch_dependents();
  const int tok = blockIdx.x;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int r = threadIdx.x; r < ncand; r += blockDim.x) {
    const int2 c = cand[r * 16 + tok];
    if (better(__int_as_float(c.x), c.y, bv, bi)) { bv = __int_as_float(c.x); bi = c.y; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = bv; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w)
      if (better(sv[w], si[w], bv, bi)) { bv = sv[w]; bi = si[w]; }
    if (bi == 0x7fffffff) bi = 0;          // all-NaN row: numpy returns 0
    cur[tok] = bi;
    const int step = d_step ? *d_step : 0;
    if (toks && step < steps) toks[(long long)tok * steps + step] = bi;
  }
}

// ---------------------------------------------------------------- host side
static bool plan(int M, int N, int K, int NB, Shape& sh, size_t& smem) {
  if (M < 1 || M > 16 || N < 1 || K % 64) return false;
  const int sms = device_sm_count();
  static const int c_max = [] {                  // A/B switch: EET_CL_C = largest cluster size tried
    const char* v = std::getenv("EET_CL_C");
    return v ? std::max(1, std::min(16, atoi(v))) : 8;
  }();
  int C = 0;
  for (int c : {16, 8, 6, 4, 3, 2, 1})
    if (c <= c_max && K % (64 * c) == 0 && K / c <= MAX_KC) { C = c; break; }
  if (!C) return false;
  const int Kc = K / C, KS = Kc / 16;
  const int tiles = (N + 15) / 16;
  const int clusters = std::max(1, sms / C);
  static const int nt_max = [] {                // A/B switch: 16-row tiles per cluster
    const char* e = std::getenv("EET_CL_NTMAX");
    return e ? std::max(1, std::min(16, atoi(e))) : 8;
  }();
  int NT = (tiles + clusters - 1) / clusters;
  NT = std::max(1, std::min({NT, nt_max, MAX_W_BYTES / (16 * Kc * 2)}));
  int KG = 1;
  if (NT < WARPS)
    for (int g = WARPS / NT; g >= 1; --g)
      if (KS % g == 0) { KG = g; break; }
  sh.M = M; sh.N = N; sh.K = K; sh.C = C; sh.Kc = Kc; sh.NT = NT; sh.KG = KG;
  smem = (size_t)Lay(NT, Kc, C, KG, NB).total;
  return true;
}

static std::atomic<int> g_trace_host{0};   // mirrors g_tr_on (set by eet_debug_cltrace)

template <typename T, int NB, int NV, int MODE, bool TRACE>
static void launch(const CUtensorMap& mw, const LnSrc& ln, const Shape& sh, size_t smem, const Epi& e,
                   cudaStream_t st) {
  auto kern = gemv_cl_kernel<T, NB, NV, MODE, TRACE>;
  static std::atomic<size_t> set{0};
  if (set.load() < smem) {
    EET_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));   // C = 16 (A/B)
    EET_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    size_t cur = set.load();
    while (cur < smem && !set.compare_exchange_weak(cur, smem)) {}
  }
  const int G = (sh.N + 16 * sh.NT - 1) / (16 * sh.NT);
  launch_cluster(kern, dim3(G * sh.C), dim3(THREADS), smem, st, true, dim3(sh.C, 1, 1), mw, ln, sh, e);
  EET_LAUNCH_CHECK();
}

template <typename T, int NB, int NV, int MODE>
static void go_t(const CUtensorMap& mw, const LnSrc& ln, const Shape& sh, size_t smem, const Epi& e, cudaStream_t st) {
  if (g_trace_host.load()) launch<T, NB, NV, MODE, true>(mw, ln, sh, smem, e, st);
  else launch<T, NB, NV, MODE, false>(mw, ln, sh, smem, e, st);
}

// LN-fused instances feed QKV (K/V scatter) and W1 (GELU); the others the
// residual (single GPU), fp32 partial (tensor parallel) or plain 16-bit store
template <typename T, int NB>
static void go(const CUtensorMap& mw, const LnSrc& ln, const Shape& sh, size_t smem, const Epi& e, cudaStream_t st) {
  if (sh.ln) {
    const bool small = sh.Kc <= 128;                 // LayerNorm slice: 2 (else 8) float4 per thread
    if (e.mode == EPI_QKV) {
      small ? go_t<T, NB, 2, EPI_QKV>(mw, ln, sh, smem, e, st) : go_t<T, NB, 8, EPI_QKV>(mw, ln, sh, smem, e, st);
    } else if (e.mode == EPI_STORE_F32) {             // test entry (eet_gemv_decode)
      small ? go_t<T, NB, 2, EPI_STORE_F32>(mw, ln, sh, smem, e, st) : go_t<T, NB, 8, EPI_STORE_F32>(mw, ln, sh, smem, e, st);
    } else {
      small ? go_t<T, NB, 2, EPI_GELU_T>(mw, ln, sh, smem, e, st) : go_t<T, NB, 8, EPI_GELU_T>(mw, ln, sh, smem, e, st);
    }
    return;
  }
  switch (e.mode) {
    case EPI_RESID: go_t<T, NB, 0, EPI_RESID>(mw, ln, sh, smem, e, st); break;
    case EPI_STORE_F32: go_t<T, NB, 0, EPI_STORE_F32>(mw, ln, sh, smem, e, st); break;
    case EPI_STORE_T: go_t<T, NB, 0, EPI_STORE_T>(mw, ln, sh, smem, e, st); break;
    default: go_t<T, NB, 0, EPI_GELU_T>(mw, ln, sh, smem, e, st); break;
  }
}

}  // namespace gc

// Decode projection Y[M, N] = X[M, K] W[N, K]^T (W K-major, ld = K) with the
// fused epilogue `e`. X: 16-bit rows (x == nullptr) or LayerNorm(x rows; g,
// b). Decode rows only: token m is sequence m at slot 0, i.e. x row m at
// x + m * x_sb (rinfo[m] == (m, 0) in the incremental plan) and the epilogue
// row is m. False when the shape is not eligible (caller falls back).
static bool cl_check(int dtype, const void* W, int M, int N, int K, const void* X, int ldx, const float* x,
                     long long x_sb, const float* g, const float* b, int mode, gc::Shape& sh, size_t& smem) {
  if (dtype != EET_F16 && dtype != EET_BF16) return false;
  const bool ln = x != nullptr;
  if (ln ? (mode != EPI_QKV && mode != EPI_GELU_T && mode != EPI_STORE_F32)
         : (mode != EPI_RESID && mode != EPI_STORE_F32 && mode != EPI_STORE_T && mode != EPI_GELU_T))
    return false;
  if (ln && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(b)) & 15 ||
             (x_sb & 3)))
    return false;
  if (!ln && ((reinterpret_cast<uintptr_t>(X) & 15) || (ldx % 8))) return false;
  if (reinterpret_cast<uintptr_t>(W) & 15) return false;
  return gc::plan(M, N, K, M <= 8 ? 1 : 2, sh, smem) && smem <= 227 * 1024;
}

bool gemv_cl_ok(int dtype, const void* W, int M, int N, int K, const void* X, int ldx, const float* x,
                long long x_sb, const float* g, const float* b, int mode) {
  gc::Shape sh{};
  size_t smem = 0;
  return cl_check(dtype, W, M, N, K, X, ldx, x, x_sb, g, b, mode, sh, smem);
}

bool gemv_cl(int dtype, const void* W, int M, int N, int K, const void* X, int ldx, const float* x,
             long long x_sb, long long x_ss, const int2* rinfo, const float* g, const float* b, const Epi& e,
             cudaStream_t st, const long long* acc, long long acc_sb) {
  const bool ln = x != nullptr;
  if (ln && (x_ss & 3)) return false;
  const int NB = M <= 8 ? 1 : 2;
  gc::Shape sh{};
  size_t smem = 0;
  if (!cl_check(dtype, W, M, N, K, X, ldx, x, x_sb, g, b, e.mode, sh, smem)) return false;
  sh.ln = ln ? 1 : 0;
  sh.X = X;
  sh.ldx = ldx;
  static const int warm = [] {                     // A/B switch: EET_CL_WARM=1 enables the dry pass
    const char* v = std::getenv("EET_CL_WARM");
    return (v && v[0] == '1') ? 1 : 0;
  }();
  sh.warm = warm;
  static const int early = [] {                    // A/B switch: EET_PDL_EARLY=1 (all) / 2 (QKV)
    const char* v = std::getenv("EET_PDL_EARLY");
    return v ? atoi(v) : 0;
  }();
  sh.early = early == 1 || (early == 2 && e.mode == EPI_QKV);   // 2: only QKV (its attention streams K/V early)
  (void)x_ss; (void)rinfo;
  const gc::LnSrc src{x, x_sb, g, b, acc, acc_sb};
  const CUtensorMap mw = make_tma_map_kblk(W, N, K, K, 16 * sh.NT, sh.Kc / 64, dtype);
  ProfScope ps(K_GEMV, st, (double)N * K * 2 + (double)M * K * (ln ? 4 : 2) + gemm_bytes(M, N, 0, 2, e),
               2.0 * M * N * K);
  if (dtype == EET_BF16) {
    NB == 1 ? gc::go<__nv_bfloat16, 1>(mw, src, sh, smem, e, st) : gc::go<__nv_bfloat16, 2>(mw, src, sh, smem, e, st);
  } else {
    NB == 1 ? gc::go<__half, 1>(mw, src, sh, smem, e, st) : gc::go<__half, 2>(mw, src, sh, smem, e, st);
  }
  return true;
}

// LM head + fused greedy argmax (runtime.py:341-344, :425) for <= 16 token
// rows: logits = LN(x rows) W_head^T, tokens -> e.cur / e.toks; optional fp32
// logits into e.out at step *e.d_step. W: [vocab, K] K-major.
bool lm_head_argmax(int dtype, const void* W, int M, int N, int K, const float* x, long long x_sb, long long x_ss,
                    const int2* rinfo, const float* g, const float* b, const Epi& e, cudaStream_t st) {
  if ((dtype != EET_F16 && dtype != EET_BF16) || M < 1 || M > 16 || K % 128 || K > 1024 || K < 128) return false;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(b) |
       reinterpret_cast<uintptr_t>(W)) & 15 || (x_sb & 3) || (x_ss & 3))
    return false;
  const int NB = M <= 8 ? 1 : 2;
  const int tiles = (N + 15) / 16;
  const int grid = std::min(tiles, device_sm_count());
  const size_t smem = (size_t)gc::HSTAGES * 16 * K * 2 + gc::align_up(16 * (K + gc::XPAD) * 2, 128) +
                      (size_t)gc::HCW * 16 * 8 + gc::HSTAGES * 16 + 1024 + 64;
  const CUtensorMap mw = make_tma_map_kblk(W, N, K, K, 16, K / 64, dtype);
  (void)x_ss; (void)rinfo;                       // rows: x + m * x_sb (decode plan)
  const gc::LnSrc src{x, x_sb, g, b, nullptr, 0};
  {
    ProfScope ps(K_GEMV, st, (double)N * K * 2 + (double)M * K * 4, 2.0 * M * N * K);
    auto run = [&](auto kern) {
      EET_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      launch_ex(kern, dim3(grid), dim3(gc::HTHREADS), smem, st, true, dim3(1, 1, 1), mw, src, M, N, K, e);
      EET_LAUNCH_CHECK();
    };
    if (dtype == EET_BF16) {
      if (NB == 1) run(gc::lm_head_kernel<__nv_bfloat16, 1>); else run(gc::lm_head_kernel<__nv_bfloat16, 2>);
    } else {
      if (NB == 1) run(gc::lm_head_kernel<__half, 1>); else run(gc::lm_head_kernel<__half, 2>);
    }
  }
  {
    ProfScope ps2(K_ARGMAX, st, 8.0 * grid * 16, 1.0 * grid * M);
    launch_ex(gc::argmax_cand_kernel, dim3(M), dim3(256), 0, st, true, dim3(1, 1, 1), (const int2*)e.cand, grid,
              e.cur, e.toks, e.steps, e.d_step);
    EET_LAUNCH_CHECK();
  }
  return true;
}

}  // namespace eet

namespace eet {
extern "C" int eet_gemv_decode(int dtype, const void* w, int N, int K, const void* X, const float* x, const float* g,
                               const float* b, int M, int mode, void* out, void* stream) {
  try {
    EET_REQUIRE(dtype == EET_F16 || dtype == EET_BF16, EET_ERR_ARG, "gemv_decode: 16-bit dtypes only");
    EET_REQUIRE(mode == EPI_STORE_F32 || mode == EPI_GELU_T || mode == EPI_RESID, EET_ERR_ARG, "gemv_decode: mode");
    EET_REQUIRE(!(x && mode == EPI_RESID), EET_ERR_ARG, "gemv_decode: LayerNorm input with residual mode");
    Epi e;
    e.mode = mode;
    if (mode == EPI_RESID) {
      e.x = reinterpret_cast<float*>(out);
      e.x_sb = N;
    } else {
      e.out = out;
      e.ldo = N;
    }
    const bool ok = gemv_cl(dtype, w, M, N, K, X, K, x, K, 0, nullptr, g, b, e, reinterpret_cast<cudaStream_t>(stream));
    EET_REQUIRE(ok, EET_ERR_UNSUPPORTED, "gemv_decode: unsupported shape");
    return EET_OK;
  } catch (const Fail& f) {
    return f.code;
  }
}

extern "C" int eet_debug_cltrace(int on, long long* out, int* n) {
  // on = 1: reset + enable; on = 0: disable and copy out (8192 x 8)
  try {
    if (on) {
      const int one = 1;
      const unsigned zero = 0;
      EET_CHECK_CUDA(cudaMemcpyToSymbol(gc::g_tr_on, &one, sizeof(int)));
      EET_CHECK_CUDA(cudaMemcpyToSymbol(gc::g_tr_n, &zero, sizeof(unsigned)));
      gc::g_trace_host.store(1);
    } else {
      gc::g_trace_host.store(0);
      const int zero = 0;
      unsigned cnt = 0;
      EET_CHECK_CUDA(cudaDeviceSynchronize());
      EET_CHECK_CUDA(cudaMemcpyToSymbol(gc::g_tr_on, &zero, sizeof(int)));
      EET_CHECK_CUDA(cudaMemcpyFromSymbol(&cnt, gc::g_tr_n, sizeof(unsigned)));
      EET_CHECK_CUDA(cudaMemcpyFromSymbol(out, gc::g_tr, sizeof(long long) * 8192 * 24));
      *n = (int)std::min<unsigned>(cnt, 8192u);
    }
    return EET_OK;
  } catch (const Fail& f) {
    return f.code;
  }
}
}  // namespace eet
