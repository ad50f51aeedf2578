// Decode-step projections from pre-permuted weights (16-bit modes, <= 16
// token rows): runtime.py:131-136 (QKV), :188 (out-proj), :206-213 (FFN) and
// :341-344 (LM head) for one token per sequence.
//
// Weights are packed once per generate call into 512 B mma.sync A-fragments
// (decode_mk.cu: mk_pack), fragment-major per 16-row tile. One CTA (8 warps)
// owns one 16-row output tile over the full K; warp w loads its K/8 slice
// of fragments straight into registers with 128-bit no-allocate loads —
// issued BEFORE griddepcontrol.wait, so under programmatic dependent launch
// the weight stream overlaps the previous kernel's tail. Then the <= 16
// activation rows are staged in shared memory (fused LayerNorm from the
// fp32 residual stream, runtime.py:83-94, or a 16-bit activation), each
// warp runs mma.sync m16n8k16 over its slice, and the 8 partial tiles are
// summed in warp order (deterministic) into the fused epilogue (QKV +
// K/V-cache scatter, residual add, GELU, fp32 logits).
#include "sm100.cuh"

#include <cstdlib>
#include <mutex>
#include <unordered_map>

namespace eet {
namespace gm {

constexpr int WARPS = 8, THREADS = WARPS * 32, XPAD = 8;

// development trace (EET_KTRACE=1): CTA 0 of every launch records
// globaltimer stamps [start, weights issued, wait passed, X staged, MMA done,
// reduced, end] plus (N, K) into a ring
__device__ int g_ktrace_on = 0;
__device__ unsigned g_ktrace_n = 0;
__device__ long long g_ktrace[4096][8];
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <typename T>
struct Args {
  const uint4* w;                 // packed [rtiles][ks][32] uint4
  int ks, N, M;                   // K / 16, output features, token rows
  const T* X; int ldx;            // 16-bit activation rows (!LN)
  const float* x; long long x_sb, x_ss; const int2* rinfo;   // LN: fp32 rows via row map
  const float* g; const float* b;
  Epi e;
  int persist;                    // LM head: one wave of CTAs loops over the tiles
};

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

template <typename T>
__device__ __forceinline__ void mma16816(float* d, const uint4& a, uint32_t b0, uint32_t b1) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
  }
}

// LM-head epilogue: greedy token per row (np.argmax, lowest id on ties,
// runtime.py:425). Each CTA reduces its 16 vocab rows per token into a
// candidate; the CTA that finishes last (acq_rel ticket) reduces all
// candidates — 16 threads per token, candidate ranges in id order — and
// records the token (argmax_kernel's job, without a logits round trip).
__device__ __forceinline__ bool better(float v, int i, float bv, int bi) {
  return v > bv || (v == bv && i < bi);
}
template <typename T>
__device__ __noinline__ void argmax_tail(const Args<T>& a, const float* red, int NB, int rt) {
  __shared__ float tile[16][17];
  __shared__ float bvs[16][16];
  __shared__ int bis[16][16];
  __shared__ int s_last;
  const Epi& e = a.e;
  const int step = *e.d_step;
  for (int t = threadIdx.x; t < 256; t += blockDim.x) tile[t >> 4][t & 15] = -INFINITY;
  __syncthreads();
  if (threadIdx.x < NB * 128) {
    const int el = threadIdx.x;
    float v = 0.f;
    for (int w = 0; w < WARPS; ++w) v += red[(w * NB * 4) * 32 + el];
    const int i = el >> 5, ln = el & 31;
    const int row = (ln >> 2) + 8 * ((i & 3) >> 1);
    const int tok = (i >> 2) * 8 + 2 * (ln & 3) + (i & 1);
    const int n = rt * 16 + row;
    if (n < a.N && tok < a.M) {
      tile[tok][row] = v;
      if (e.out && step < e.steps)
        reinterpret_cast<float*>(e.out)[((long long)step * e.batch + tok) * e.ldo + n] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < a.M && rt * 16 < a.N) {
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int r = 0; r < 16; ++r)
      if (rt * 16 + r < a.N && better(tile[threadIdx.x][r], rt * 16 + r, bv, bi)) {
        bv = tile[threadIdx.x][r];
        bi = rt * 16 + r;
      }
    e.cand[rt * 16 + threadIdx.x] = make_int2(__float_as_int(bv), bi);
  }
  __syncthreads();                                 // tile / red reusable by the next tile
}

// second stage: one CTA per token reduces the per-tile candidates in id order
__global__ void __launch_bounds__(256) argmax_cand_kernel(const int2* __restrict__ cand, int rtiles,
                                                          int* __restrict__ cur, long long* __restrict__ toks,
                                                          int steps, const int* __restrict__ d_step) {
  __shared__ float sv[8];
  __shared__ int si[8];
  sm100::griddep_wait();
  sm100::griddep_launch_dependents();
  const int tok = blockIdx.x;
  const int per = (rtiles + 255) / 256;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int r = threadIdx.x * per; r < min(rtiles, (threadIdx.x + 1) * per); ++r) {
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
    const int step = *d_step;
    if (toks && step < steps) toks[(long long)tok * steps + step] = bi;
  }
}

// NB n-blocks of 8 token rows; KW fragments per warp (K = 16 * 8 * KW);
// NV float4 per lane per LayerNorm row (h <= 128 * NV)
template <typename T, int NB, int KW, bool LN, int NV>
__global__ void __launch_bounds__(THREADS) gemv_mma_kernel(const __grid_constant__ Args<T> a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int K = a.ks * 16, xst = K + XPAD;
  T* xs = reinterpret_cast<T*>(smem);                                   // [16][K + XPAD]
  float* red = reinterpret_cast<float*>(smem + (size_t)16 * xst * sizeof(T));   // [WARPS][NB*4][32]
  const int rt = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rtiles = (a.N + 15) / 16;
  const bool trace = g_ktrace_on && blockIdx.x == 0 && threadIdx.x == 0;
  long long ts[7];
  if (trace) ts[0] = gtime();
  // 1. this warp's weight slice -> registers (static data: before the wait)
  uint4 wv[KW];
  {
    const uint4* wp = a.w + ((size_t)rt * a.ks + (size_t)warp * KW) * 32 + lane;
#pragma unroll
    for (int i = 0; i < KW; ++i) wv[i] = ldg_stream(wp + i * 32);
  }
  // LayerNorm gamma/beta are static too: stage them in shared memory now
  float* sgb = red + WARPS * NB * 4 * 32;                                // [2][K] (LN only)
  if constexpr (LN) {
    for (int i = threadIdx.x; i < K / 4; i += THREADS) {
      reinterpret_cast<float4*>(sgb)[i] = __ldg(reinterpret_cast<const float4*>(a.g) + i);
      reinterpret_cast<float4*>(sgb + K)[i] = __ldg(reinterpret_cast<const float4*>(a.b) + i);
    }
  }
  if (trace) ts[1] = gtime();
  sm100::griddep_wait();
  sm100::griddep_launch_dependents();
  if constexpr (LN) __syncthreads();             // gamma/beta staged by other threads (racecheck)
  if (trace) ts[2] = gtime();

  // 2. activation rows -> xs (rows >= M are zero)
  if constexpr (LN) {
    // warp w: rows w and w + 8, loaded together; two-pass statistics
    const int nv = K / 4;
    float4 v[2][NV];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = warp + q * WARPS;
      const float* xr = a.x;
      if (r < a.M) {
        const int2 ri = a.rinfo[r];
        xr = a.x + ri.x * a.x_sb + ri.y * a.x_ss;
      }
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const int i = j * 32 + lane;
        v[q][j] = (r < a.M && i < nv) ? reinterpret_cast<const float4*>(xr)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    if (trace) {                                   // x landed (values consumed)
      float z = v[0][0].x + v[1][NV - 1].w;
      ts[4] = (z == 1.2345e-38f) ? 0 : gtime();
    }
    // both rows' statistics interleaved: the shuffle chains run in parallel
    float mu[2], rs[2];
    {
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        s0 += (v[0][j].x + v[0][j].y) + (v[0][j].z + v[0][j].w);
        s1 += (v[1][j].x + v[1][j].y) + (v[1][j].z + v[1][j].w);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      }
      mu[0] = s0 / (float)K;
      mu[1] = s1 / (float)K;
      float q0 = 0.f, q1 = 0.f;
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        if (j * 32 + lane < nv) {
          const float a0 = v[0][j].x - mu[0], a1 = v[0][j].y - mu[0], a2 = v[0][j].z - mu[0], a3 = v[0][j].w - mu[0];
          const float b0 = v[1][j].x - mu[1], b1 = v[1][j].y - mu[1], b2 = v[1][j].z - mu[1], b3 = v[1][j].w - mu[1];
          q0 += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
          q1 += (b0 * b0 + b1 * b1) + (b2 * b2 + b3 * b3);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        q0 += __shfl_xor_sync(0xffffffffu, q0, o);
        q1 += __shfl_xor_sync(0xffffffffu, q1, o);
      }
      rs[0] = 1.0f / sqrtf(q0 / (float)K + 1e-5f);
      rs[1] = 1.0f / sqrtf(q1 / (float)K + 1e-5f);
    }
    if (trace) ts[5] = gtime();
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = warp + q * WARPS;
      T* dst = xs + r * xst;
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const int i = j * 32 + lane;
        if (i < nv) {
          uint2 o2 = make_uint2(0, 0);
          if (r < a.M) {
            const float4 gg = reinterpret_cast<const float4*>(sgb)[i];
            const float4 bb = reinterpret_cast<const float4*>(sgb + K)[i];
            T o[4] = {from_f<T>((v[q][j].x - mu[q]) * rs[q] * gg.x + bb.x), from_f<T>((v[q][j].y - mu[q]) * rs[q] * gg.y + bb.y),
                      from_f<T>((v[q][j].z - mu[q]) * rs[q] * gg.z + bb.z), from_f<T>((v[q][j].w - mu[q]) * rs[q] * gg.w + bb.w)};
            o2 = *reinterpret_cast<const uint2*>(o);
          }
          *reinterpret_cast<uint2*>(dst + i * 4) = o2;
        }
      }
    }
  } else {
    const int w8 = K / 8;                        // 16 B chunks per row
    for (int base = 0; base < 16 * w8; base += 8 * THREADS) {   // K <= 1024: one round trip
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * THREADS + threadIdx.x;
        const int r = i / w8, c = i - r * w8;
        v[u] = (i < 16 * w8 && r < a.M) ? reinterpret_cast<const uint4*>(a.X + (size_t)r * a.ldx)[c]
                                        : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * THREADS + threadIdx.x;
        const int r = i / w8, c = i - r * w8;
        if (i < 16 * w8) *reinterpret_cast<uint4*>(xs + r * xst + c * 8) = v[u];
      }
    }
  }
  __syncthreads();
  if (trace) ts[3] = gtime();

  // 3. this warp's K slice on the tensor cores
  float acc[NB][4];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[nb][i] = 0.f;
  {
    const int g = lane >> 2, c4 = lane & 3;
#pragma unroll
    for (int i = 0; i < KW; ++i) {
      const int k0 = (warp * KW + i) * 16;
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const T* xr = xs + (nb * 8 + g) * xst + k0 + 2 * c4;
        mma16816<T>(acc[nb], wv[i], *reinterpret_cast<const uint32_t*>(xr),
                    *reinterpret_cast<const uint32_t*>(xr + 8));
      }
    }
  }
  if (trace && !LN) {
    float z = acc[0][0];                        // MMA results materialised
    if (z == 1.2345e-38f) ts[4] = 0; else ts[4] = gtime();
  }
  // 4. warp-ordered reduction + epilogue
#pragma unroll
  for (int nb = 0; nb < NB; ++nb)
#pragma unroll
    for (int i = 0; i < 4; ++i) red[(warp * NB * 4 + nb * 4 + i) * 32 + lane] = acc[nb][i];
  __syncthreads();
  {
    if (a.persist) {
      // LM head: X staged once; this CTA's tiles rt, rt + G, ... with the
      // next tile's weights in flight while the current one is reduced
      for (int r = rt; r < rtiles; r += gridDim.x) {
        const int rn = r + (int)gridDim.x;
        if (rn < rtiles) {                         // next tile's weights in flight ...
          const uint4* wp = a.w + ((size_t)rn * a.ks + (size_t)warp * KW) * 32 + lane;
#pragma unroll
          for (int i = 0; i < KW; ++i) wv[i] = ldg_stream(wp + i * 32);
        }
        argmax_tail(a, red, NB, r);                // ... while this one is reduced
        if (rn >= rtiles) break;
        float acc2[NB][4];
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int i = 0; i < 4; ++i) acc2[nb][i] = 0.f;
        const int g = lane >> 2, c4 = lane & 3;
#pragma unroll
        for (int i = 0; i < KW; ++i) {
          const int k0 = (warp * KW + i) * 16;
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
            const T* xr = xs + (nb * 8 + g) * xst + k0 + 2 * c4;
            mma16816<T>(acc2[nb], wv[i], *reinterpret_cast<const uint32_t*>(xr),
                        *reinterpret_cast<const uint32_t*>(xr + 8));
          }
        }
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int i = 0; i < 4; ++i) red[(warp * NB * 4 + nb * 4 + i) * 32 + lane] = acc2[nb][i];
        __syncthreads();
      }
      return;
    }
    if (a.e.mode == EPI_ARGMAX) {
      argmax_tail(a, red, NB, rt);
      if (trace) {
        ts[4] = ts[5] = ts[6] = gtime();
        const unsigned i = atomicAdd(&g_ktrace_n, 1u) & 4095u;
        for (int k = 0; k < 6; ++k) g_ktrace[i][k] = ts[k + 1] - ts[0];
        g_ktrace[i][6] = a.N;
        g_ktrace[i][7] = a.ks * 16 + (LN ? 100000 : 0);
      }
      return;
    }
  }
  float v = 0.f;
  if (threadIdx.x < NB * 128) {
#pragma unroll
    for (int w = 0; w < WARPS; ++w) v += red[(w * NB * 4) * 32 + threadIdx.x];
  }
  if (trace && !LN) ts[5] = gtime();
  if (threadIdx.x < NB * 128) {
    const int e = threadIdx.x;
    const int i = e >> 5, ln = e & 31;
    const int row = (ln >> 2) + 8 * ((i & 3) >> 1);
    const int tok = (i >> 2) * 8 + 2 * (ln & 3) + (i & 1);
    const int n = rt * 16 + row;
    if (n < a.N && tok < a.M) epi_apply<T>(a.e, tok, n, v);
  }
  if (trace) {
    ts[6] = gtime();
    const unsigned i = atomicAdd(&g_ktrace_n, 1u) & 4095u;
    for (int k = 0; k < 6; ++k) g_ktrace[i][k] = ts[k + 1] - ts[0];
    g_ktrace[i][6] = a.N;
    g_ktrace[i][7] = a.ks * 16 + (LN ? 100000 : 0);
  }
}

template <typename T, int NB, int KW, bool LN, int NV>
static void go(const Args<T>& a, int rtiles, cudaStream_t st) {
  auto kern = gemv_mma_kernel<T, NB, KW, LN, NV>;
  const size_t smem = (size_t)16 * (a.ks * 16 + XPAD) * sizeof(T) + (size_t)WARPS * NB * 4 * 32 * 4 +
                      (LN ? (size_t)2 * a.ks * 16 * 4 : 0);
  static size_t set = 0;
  if (set < smem) {
    EET_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    set = smem;
  }
  int ctas = rtiles;
  if (a.persist) {                               // one wave
    int per_sm = 1;
    EET_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem));
    ctas = std::min(ctas, std::max(1, per_sm) * device_sm_count());
  }
  launch_ex(kern, dim3(ctas), dim3(THREADS), smem, st, true, dim3(1, 1, 1), a);
  EET_LAUNCH_CHECK();
}

template <typename T, int NB>
static bool dispatch(const Args<T>& a, int rtiles, bool ln, cudaStream_t st) {
  const int K = a.ks * 16;
  if (ln) {
    if (K == 1024) { go<T, NB, 8, true, 8>(a, rtiles, st); return true; }
    if (K == 768) { go<T, NB, 6, true, 6>(a, rtiles, st); return true; }
    if (K == 512) { go<T, NB, 4, true, 4>(a, rtiles, st); return true; }
    if (K == 256) { go<T, NB, 2, true, 2>(a, rtiles, st); return true; }
    return false;
  }
  switch (K) {
    case 256: go<T, NB, 2, false, 1>(a, rtiles, st); return true;
    case 512: go<T, NB, 4, false, 1>(a, rtiles, st); return true;
    case 768: go<T, NB, 6, false, 1>(a, rtiles, st); return true;
    case 1024: go<T, NB, 8, false, 1>(a, rtiles, st); return true;
    case 2048: go<T, NB, 16, false, 1>(a, rtiles, st); return true;
    case 3072: go<T, NB, 24, false, 1>(a, rtiles, st); return true;
    case 4096: go<T, NB, 32, false, 1>(a, rtiles, st); return true;
    default: return false;
  }
}

}  // namespace gm

// ---------------------------------------------------------------- registry
// source weight pointer -> packed copy, valid for the duration of one
// generate call (eet_generate registers and clears it)
static std::mutex g_pack_mu;
static std::unordered_map<const void*, const uint4*> g_packed;

void packed_register(const void* src, const void* packed) {
  std::lock_guard<std::mutex> lk(g_pack_mu);
  g_packed[src] = reinterpret_cast<const uint4*>(packed);
}
void packed_clear() {
  std::lock_guard<std::mutex> lk(g_pack_mu);
  g_packed.clear();
}
static const uint4* packed_lookup(const void* src) {
  std::lock_guard<std::mutex> lk(g_pack_mu);
  auto it = g_packed.find(src);
  return it == g_packed.end() ? nullptr : it->second;
}

// Decode projection through the packed weights of `wsrc` when registered
// and the shape is supported. X: 16-bit rows (ln == nullptr) or, with ln =
// {x, x_sb, x_ss, rinfo, g, b}, LayerNorm of the fp32 rows. Returns false to
// let the caller take the generic path.
bool gemv_packed(int dtype, const void* wsrc, int M, int N, int K, const void* X, int ldx,
                 const float* x, long long x_sb, long long x_ss, const int2* rinfo, const float* g,
                 const float* b, const Epi& e, cudaStream_t st) {
  static const bool off = [] {                  // A/B switch for measurements
    const char* e = std::getenv("EET_NO_PACKED");
    return e && e[0] == '1';
  }();
  if (off || (dtype != EET_F16 && dtype != EET_BF16) || M < 1 || M > 16 || K % 16) return false;
  const uint4* w = packed_lookup(wsrc);
  if (!w) return false;
  const bool ln = x != nullptr;
  if (ln && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(g) |
              reinterpret_cast<uintptr_t>(b)) & 15 || (x_sb & 3) || (x_ss & 3)))
    return false;
  if (!ln && ((reinterpret_cast<uintptr_t>(X) & 15) || (ldx % 8))) return false;
  // K > 1024 (W2) stays on the tcgen05 split-K kernel: in the decode graph
  // it costs 6.7 us per layer vs ~7.2 us for one CTA per tile or a 2-CTA
  // cluster K split of this kernel (r01 A/B)
  const int kl[] = {256, 512, 768, 1024}, kp[] = {256, 512, 768, 1024};
  bool ok = false;
  if (ln) { for (int k : kl) ok |= K == k; } else { for (int k : kp) ok |= K == k; }
  if (!ok) return false;
  const int rtiles = (N + 15) / 16;
  ProfScope ps(K_GEMV, st, (double)rtiles * 16 * K * 2 + (double)M * K * (ln ? 4 : 2) + (double)M * N * 4,
               2.0 * M * N * K);
  bool ok2;
  if (dtype == EET_BF16) {
    gm::Args<__nv_bfloat16> a{w, K / 16, N, M, reinterpret_cast<const __nv_bfloat16*>(X), ldx,
                              x, x_sb, x_ss, rinfo, g, b, e, e.mode == EPI_ARGMAX ? 1 : 0};
    ok2 = M <= 8 ? gm::dispatch<__nv_bfloat16, 1>(a, rtiles, ln, st) : gm::dispatch<__nv_bfloat16, 2>(a, rtiles, ln, st);
  } else {
    gm::Args<__half> a{w, K / 16, N, M, reinterpret_cast<const __half*>(X), ldx, x, x_sb, x_ss, rinfo, g, b, e,
                       e.mode == EPI_ARGMAX ? 1 : 0};
    ok2 = M <= 8 ? gm::dispatch<__half, 1>(a, rtiles, ln, st) : gm::dispatch<__half, 2>(a, rtiles, ln, st);
  }
  if (ok2 && e.mode == EPI_ARGMAX) {        // second stage of the fused argmax
    ProfScope ps2(K_ARGMAX, st, 8.0 * rtiles * 16, 1.0 * rtiles * M);
    launch_ex(gm::argmax_cand_kernel, dim3(M), dim3(256), 0, st, true, dim3(1, 1, 1), e.cand, rtiles, e.cur,
              e.toks, e.steps, e.d_step);
    EET_LAUNCH_CHECK();
  }
  return ok2;
}

}  // namespace eet

// ------------------------------------------------------------ C ABI (test)
namespace eet {
extern "C" int eet_gemv_packed(int dtype, const void* w, int N, int K, const void* X, int M,
                               float* out, int repack, void* stream) {
  try {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    static std::unordered_map<const void*, void*> own;    // packed copies made here
    static std::mutex mu;
    void* pk = nullptr;
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = own.find(w);
      if (it == own.end()) {
        EET_CHECK_CUDA(cudaMalloc(&pk, mk_packed_bytes(N, K)));
        own[w] = pk;
      } else {
        pk = it->second;
      }
    }
    if (repack) mk_pack(w, N, K, pk, st);
    packed_register(w, pk);
    Epi e;
    e.mode = EPI_STORE_F32;
    e.out = out;
    e.ldo = N;
    const bool ok = gemv_packed(dtype, w, M, N, K, X, K, nullptr, 0, 0, nullptr, nullptr, nullptr, e, st);
    EET_REQUIRE(ok, EET_ERR_UNSUPPORTED, "gemv_packed: unsupported shape");
    return EET_OK;
  } catch (const Fail& f) {
    return f.code;
  }
}
}  // namespace eet

namespace eet {
extern "C" int eet_debug_ktrace(int on, long long* out, int* n) {
  // on = 1: reset + enable; on = 0: disable and copy out (4096 x 8)
  try {
    if (on) {
      const int one = 1;
      const unsigned zero = 0;
      EET_CHECK_CUDA(cudaMemcpyToSymbol(gm::g_ktrace_on, &one, sizeof(int)));
      EET_CHECK_CUDA(cudaMemcpyToSymbol(gm::g_ktrace_n, &zero, sizeof(unsigned)));
    } else {
      const int zero = 0;
      unsigned cnt = 0;
      EET_CHECK_CUDA(cudaDeviceSynchronize());
      EET_CHECK_CUDA(cudaMemcpyToSymbol(gm::g_ktrace_on, &zero, sizeof(int)));
      EET_CHECK_CUDA(cudaMemcpyFromSymbol(&cnt, gm::g_ktrace_n, sizeof(unsigned)));
      EET_CHECK_CUDA(cudaMemcpyFromSymbol(out, gm::g_ktrace, sizeof(long long) * 4096 * 8));
      *n = (int)std::min<unsigned>(cnt, 4096u);
    }
    return EET_OK;
  } catch (const Fail& f) {
    return f.code;
  }
}
}  // namespace eet
