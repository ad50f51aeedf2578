// Decode attention fused with the attention output projection, one new token
// per sequence (runtime.py:160-178 attention over the cached keys, :186-188
// context @ W_o + b_o added to the residual stream; incremental phase).
//
// The out-projection of a decode step is a 2 MB (c2) GEMV whose hop costs a
// whole dependent launch (~5 us) for ~0.3 us of weight bytes.
// Here it rides on the attention kernel instead:
//
//   * grid (sequence, head), clusters of CB sequences of one head;
//   * each CTA streams the K/V rows of its (sequence, head) exactly like the
//     stand-alone decode kernel (producer warp, cp.async.bulk ring, 8
//     consumer warps, rows of earlier steps before griddepcontrol.wait);
//   * before the wait it also TMA-loads its W_o block: the R = hidden / CB
//     output rows it owns x this head's hd input columns (16 KB at c2);
//   * the CTA's context row (rounded to the layer dtype, as the unfused path
//     stores it) is all-gathered through DSMEM (st.async + complete_tx), so
//     every CTA holds the CB contexts of its head;
//   * mma.sync m16n8k16 (W_o block = A via ldmatrix, contexts = B) gives the
//     head's contribution to R output columns of CB sequences, added with
//     red.global.add.u64 to a pending-residual buffer in 2^-32 fixed point:
//     the heads' contributions arrive in any order, and integer addition
//     makes the sum independent of that order (deterministic). The next
//     projection's LayerNorm reads x + pending and the W2 epilogue folds it
//     into x (gemv_cl.cu). EET_ATTN_O=0 restores the two-kernel path.
#include "mma_frag.cuh"

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

namespace eet {
namespace ao {
using namespace sm100;

constexpr int DCH = 64, CW = 8, THREADS = (CW + 1) * 32, XP = 8;

// development trace (eet_debug_aotrace): per CTA globaltimer stamps [start,
// wait passed, attention done, contexts gathered, end] + (sequence, head)
__device__ int g_ao_on = 0;
__device__ unsigned g_ao_n = 0;
__device__ long long g_ao[4096][8];
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct Args {
  const void* q; int ldq;                  // query row b at q + b * ldq
  const void* kc; const void* vc;          // [b, heads, smax, hd]
  int heads, smax;
  const int* pads;
  const int* kv_start; int kv_base;        // keys [pad_b, *kv_start + kv_base + 1)
  float scale;
  long long* acc; long long acc_sb;        // pending residual row b at acc + b * acc_sb (2^-32 fixed point)
  const float* bias;                       // b_o (added by head 0) or null
  int R, CB;                               // out rows per CTA, sequences per cluster
  int pf;                                  // L2 prefetch distance in ring depths (0: off)
};

template <typename T, int LPK, int NB, int NBUF>
__global__ void __launch_bounds__(THREADS) attn_o_kernel(const __grid_constant__ CUtensorMap mapW, const Args a) {
  constexpr int E = 16, G = 32 / LPK, HD = LPK * E, XST = HD + XP;
  constexpr size_t CH = (size_t)DCH * HD;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[NBUF], empty[NBUF], wbar, gbar;
  __shared__ float sm_m[CW], sm_l[CW];
  __shared__ float sm_acc[CW][HD];
  __shared__ __align__(16) T stage[HD];
  const int R = a.R;
  T* ring = reinterpret_cast<T*>(smem + R * HD * 2);          // [NBUF][K chunk | V chunk]
  T* xs = ring + NBUF * 2 * CH;                               // [8 * NB][XST] contexts of the cluster
  const int b = blockIdx.x, head = blockIdx.y;
  const int rank = (int)cluster_ctarank();                    // == b % CB
  const int b0 = b - rank;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / LPK, sub = lane % LPK;
  const bool trace = g_ao_on && threadIdx.x == 0;
  long long ts[5] = {0, 0, 0, 0, 0};
  if (trace) ts[0] = gtime();

  if (threadIdx.x == 0) {
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CW);
    }
    mbar_init(&wbar, 1);
    mbar_init(&gbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapW) : "memory");
    // static weights: the W_o block lands while the previous kernel runs
    mbar_expect_tx(&wbar, (uint32_t)(R * HD * 2));
#pragma unroll
    for (int kb = 0; kb < HD / 64; ++kb)
      tma_load_2d(smem + kb * R * 128, &mapW, &wbar, head * HD + kb * 64, rank * R, 0x1000000000000000ull);
    mbar_expect_tx(&gbar, (uint32_t)(a.CB * HD * 2));
  }
  for (int i = a.CB * XST + threadIdx.x; i < 8 * NB * XST; i += THREADS) xs[i] = from_f<T>(0.f);
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");   // barriers initialised

  const int pad = a.pads[b];
  const int L = (a.kv_start ? *a.kv_start : 0) + a.kv_base + 1;
  const int nk = max(L - pad, 0);
  const int nch = (nk + DCH - 1) / DCH;
  const long long base = ((long long)b * a.heads + head) * a.smax * HD + (long long)pad * HD;

  if (warp == CW) {                         // ---- producer warp
    if (lane == 0) {
      const T* Kc = reinterpret_cast<const T*>(a.kc) + base;
      const T* Vc = reinterpret_cast<const T*>(a.vc) + base;
      bool waited = false;
      for (int c = 0; c < nch; ++c) {
        const int buf = c % NBUF;
        if (c >= NBUF) mbar_wait(&empty[buf], ((c / NBUF) - 1) & 1);
        const int kn = min(DCH, nk - c * DCH);
        if (!waited && pad + c * DCH + kn == L) {   // chunk holds this step's slot (written by the QKV GEMV)
          griddep_wait();
          waited = true;
        }
        const uint32_t bytes = (uint32_t)(kn * HD * sizeof(T));
        T* dst = ring + buf * 2 * CH;
        mbar_expect_tx(&full[buf], 2 * bytes);
        bulk_load(dst, Kc + (size_t)c * CH, bytes, &full[buf]);
        bulk_load(dst + CH, Vc + (size_t)c * CH, bytes, &full[buf]);
        // rolling L2 prefetch a ring's depth ahead: twice the bytes in
        // flight per (sequence, head) without more shared memory
        const int cp = c + a.pf * NBUF;
        if (a.pf && cp < nch) {
          const uint32_t pb = (uint32_t)(min(DCH, nk - cp * DCH) * HD * sizeof(T));
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Kc + (size_t)cp * CH), "r"(pb) : "memory");
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Vc + (size_t)cp * CH), "r"(pb) : "memory");
        }
      }
    }
    __syncwarp();
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    return;
  }

  // ---- consumer warps: online softmax over the key chunks
  griddep_wait();                           // q of this step comes from the QKV GEMV
  griddep_launch_dependents();
  if (trace) ts[1] = gtime();
  const T* Q = reinterpret_cast<const T*>(a.q) + (long long)b * a.ldq + head * HD;
  const int d0 = sub * E;
  float q[E];
#pragma unroll
  for (int c = 0; c < E; c += 16 / (int)sizeof(T)) load16<T>(Q + d0 + c, q + c);
  float m = -INFINITY, l = 0.f, acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;
  for (int c = 0; c < nch; ++c) {
    const int buf = c % NBUF;
    mbar_wait(&full[buf], (c / NBUF) & 1);
    const T* sK = ring + buf * 2 * CH;
    const T* sV = sK + CH;
    const int kn = min(DCH, nk - c * DCH);
    for (int jb = warp * G; jb < kn; jb += CW * G) {          // warp-uniform
      const int j = jb + g;
      const bool ok = j < kn;
      float kv[E], vv[E];
      if (ok) {
#pragma unroll
        for (int cc = 0; cc < E; cc += 16 / (int)sizeof(T)) {
          load16<T>(sK + (size_t)j * HD + d0 + cc, kv + cc);
          load16<T>(sV + (size_t)j * HD + d0 + cc, vv + cc);
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
    if (lane == 0) mbar_arrive(&empty[buf]);
  }
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
  asm volatile("bar.sync 1, %0;" ::"n"(CW * 32) : "memory");   // consumer warps only
  if (trace) ts[2] = gtime();

  // ---- context row (layer dtype) -> every CTA of the cluster
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
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");   // peers' barriers initialised
    constexpr int PC = HD / 8;                                            // 16-byte pieces per context row
    for (int i = lane; i < a.CB * PC; i += 32) {
      const int peer = i / PC, c = i - peer * PC;
      const uint4 v = reinterpret_cast<const uint4*>(stage)[c];
      asm volatile(
          "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
              dsmem_addr(smem_u32(xs + rank * XST + c * 8), (uint32_t)peer)),
          "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(dsmem_addr(smem_u32(&gbar), (uint32_t)peer))
          : "memory");
    }
  } else {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }

  // ---- this head's share of the out-projection: R rows x CB sequences
  mbar_wait(&wbar, 0);
  mbar_wait(&gbar, 0);
  if (trace) ts[3] = gtime();
  const int g4 = lane >> 2, c4 = lane & 3;
  const bool add_bias = a.bias && head == 0;
  for (int u = warp; u < R / 16; u += CW) {
    float o[NB][4];
    gc::warp_mma<T, NB>(smem_u32(smem), R, u * 16, 0, HD / 16, xs, XST, lane, o);
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int n = rank * R + u * 16 + g4 + 8 * (i >> 1), tok = nb * 8 + 2 * c4 + (i & 1);
        if (tok < a.CB) {
          const float v = o[nb][i] + (add_bias ? a.bias[n] : 0.f);
          const long long fx = __float2ll_rn(v * kAccScale);
          asm volatile("red.global.add.u64 [%0], %1;" ::"l"(a.acc + (long long)(b0 + tok) * a.acc_sb + n), "l"(fx)
                       : "memory");
        }
      }
  }
  if (trace) {
    ts[4] = gtime();
    const unsigned i = atomicAdd(&g_ao_n, 1u) & 4095u;
    g_ao[i][0] = b;
    g_ao[i][1] = head;
#pragma unroll
    for (int j = 0; j < 5; ++j) g_ao[i][2 + j] = ts[j];
  }
}

}  // namespace ao

// Fused decode attention + out-projection into the residual rows (see the
// file comment). False when the shape is not eligible: the caller runs the
// stand-alone attention kernel and the out-projection GEMV instead.
bool launch_attn_o(const DecodeArgs& d, const void* wo, int h, long long* acc, long long acc_sb,
                   const float* bias, cudaStream_t st) {
  static const bool on = [] {
    const char* v = std::getenv("EET_ATTN_O");
    return !(v && v[0] == '0');
  }();
  if (!on || (d.dtype != EET_F16 && d.dtype != EET_BF16) || d.splits != 1 || (d.hd != 64 && d.hd != 128))
    return false;
  const int hq = d.heads * d.hd;
  if (((reinterpret_cast<uintptr_t>(d.kc) | reinterpret_cast<uintptr_t>(d.vc) | reinterpret_cast<uintptr_t>(d.q) |
        reinterpret_cast<uintptr_t>(wo)) & 15) || d.ldq % 8 || hq % 8)
    return false;
  int CB = 0;
  for (int c : {8, 4})
    if (d.batch % c == 0 && h % c == 0 && (h / c) % 16 == 0 && h / c <= 256) { CB = c; break; }
  if (!CB) return false;
  const int R = h / CB;
  // K/V ring depth: small enough that two CTAs and the next projection's
  // 96 KB weight block share an SM (its weights stream in under PDL)
  static const int nbuf = [] {
    const char* v = std::getenv("EET_AO_NBUF");
    return v ? std::max(2, std::min(4, atoi(v))) : 3;
  }();
  const size_t smem = 1024 + (size_t)R * d.hd * 2 + (size_t)nbuf * 2 * ao::DCH * d.hd * 2 +
                      (size_t)16 * (d.hd + ao::XP) * 2;
  if (smem > 160 * 1024) return false;
  ao::Args a;
  a.q = d.q; a.ldq = d.ldq;
  a.kc = d.kc; a.vc = d.vc;
  a.heads = d.heads; a.smax = d.smax;
  a.pads = d.pads;
  a.kv_start = d.kv_start; a.kv_base = d.kv_base;
  a.scale = d.scale;
  a.acc = acc; a.acc_sb = acc_sb;
  a.bias = bias;
  a.R = R; a.CB = CB;
  static const int pf = [] {                       // A/B: EET_AO_PF = L2 prefetch distance (ring depths)
    const char* v = std::getenv("EET_AO_PF");
    return v ? std::max(0, std::min(4, atoi(v))) : 0;
  }();
  a.pf = pf;
  const CUtensorMap mw = make_tma_map_2d(wo, h, hq, hq, R, d.dtype);
  double keys = 0;
  if (d.L_host >= 0)
    for (int b = 0; b < d.batch; ++b) keys += d.L_host - (d.h_pads ? d.h_pads[b] : 0);
  const double per_key_b = (double)d.heads * d.hd * 4;   // K + V rows, 16-bit
  ProfScope ps(K_ATTN_DECODE, st, keys * per_key_b + (double)h * hq * 2 + 8.0 * d.batch * h,
               keys * d.heads * 4.0 * d.hd + 2.0 * d.batch * h * hq, d.L_host >= 0 ? 0.0 : per_key_b,
               d.L_host >= 0 ? 0.0 : d.heads * 4.0 * d.hd);
  auto go = [&](auto kern) {
    // every instance has the same signature: the attribute is tracked per
    // kernel address
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
    launch_cluster(kern, dim3(d.batch, d.heads), dim3(ao::THREADS), smem, st, true, dim3(CB, 1, 1), mw, a);
    EET_LAUNCH_CHECK();
  };
  auto by_depth = [&](auto t, auto lpk) {
    using T = decltype(t);
    constexpr int LPK = decltype(lpk)::value;
    if (nbuf == 2) go(ao::attn_o_kernel<T, LPK, 1, 2>);
    else if (nbuf == 3) go(ao::attn_o_kernel<T, LPK, 1, 3>);
    else go(ao::attn_o_kernel<T, LPK, 1, 4>);
  };
  using L4 = std::integral_constant<int, 4>;
  using L8 = std::integral_constant<int, 8>;
  if (d.dtype == EET_BF16) {
    if (d.hd == 64) by_depth(__nv_bfloat16{}, L4{});
    else by_depth(__nv_bfloat16{}, L8{});
  } else {
    if (d.hd == 64) by_depth(__half{}, L4{});
    else by_depth(__half{}, L8{});
  }
  return true;
}

void qao_trace(int on, long long* out, int* n);

extern "C" int eet_debug_aotrace(int on, long long* out, int* n) {
  // on = 1: reset + enable; on = 0: disable and copy out: attn_o records
  // [0, 4096) x 8, qkv_attn_o records [4096, 8192) x 8; n[0], n[1] counts
  try {
    qao_trace(on, on ? nullptr : out + 4096 * 8, on ? nullptr : n + 1);
    if (on) {
      const int one = 1;
      const unsigned zero = 0;
      EET_CHECK_CUDA(cudaMemcpyToSymbol(ao::g_ao_on, &one, sizeof(int)));
      EET_CHECK_CUDA(cudaMemcpyToSymbol(ao::g_ao_n, &zero, sizeof(unsigned)));
    } else {
      const int zero = 0;
      unsigned cnt = 0;
      EET_CHECK_CUDA(cudaDeviceSynchronize());
      EET_CHECK_CUDA(cudaMemcpyToSymbol(ao::g_ao_on, &zero, sizeof(int)));
      EET_CHECK_CUDA(cudaMemcpyFromSymbol(&cnt, ao::g_ao_n, sizeof(unsigned)));
      EET_CHECK_CUDA(cudaMemcpyFromSymbol(out, ao::g_ao, sizeof(long long) * 4096 * 8));
      *n = (int)std::min<unsigned>(cnt, 4096u);
    }
    return EET_OK;
  } catch (const Fail& f) {
    return f.code;
  }
}

}  // namespace eet
