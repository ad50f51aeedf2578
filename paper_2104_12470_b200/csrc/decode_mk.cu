// Persistent decode megakernel: one launch per incremental step of
// `generate` (runtime.py:372-437, decode half) in the 16-bit modes.
//
// A decode step at small batch is a ~2 GB HBM stream (every weight once,
// every cached K/V row once) chopped into ~125 dependent phases; as separate
// kernels it is bound by per-launch ramp-up, not by bandwidth. Here one CTA
// per SM runs the whole step:
//
//   embed -> for each layer: [LN1+QKV] | [attention] | [out-proj + residual]
//            | [LN2+W1+GELU] | [W2 + residual] -> [LNf + LM head + argmax]
//
// with a grid barrier between phases ('|'). Static data (weights,
// pre-permuted into 512 B mma.sync A-fragments, fragment-major per 16-row
// tile, and the LayerNorm parameters) and the cached K/V rows of earlier
// steps reach the SM through a shared-memory ring filled by a producer warp
// with cp.async.bulk; the producer never waits on a grid barrier, so the
// next phase's bytes are already on chip when a barrier opens. Consumers
// (8 warps) do the math from the ring: mma.sync m16n8k16 (weights = A, the
// <= 16 staged token rows = B, fp32 accumulators) for the projections, SIMT
// online softmax for attention (keys [pad_b, L), runtime.py:155-178).
//
// Work split: a projection's 16-row output tiles are owned whole by one CTA
// (round-robin, rotated per phase), so its epilogue (K/V-cache scatter,
// residual add, GELU) runs without cross-CTA reduction. Attention splits the
// concatenated key ranges of all (sequence, head) pairs evenly over the
// CTAs; a pair cut by a range boundary is merged by whichever CTA arrives
// last (acq_rel ticket), in key order: deterministic, no atomics on data.
#include "sm100.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace eet {
namespace mk {
using namespace sm100;

constexpr int CW = 8;                   // consumer warps
constexpr int NCT = CW * 32;            // consumer threads
constexpr int THREADS = NCT + 32;       // + producer warp
constexpr int NSLOT = 8;
constexpr int SLOT = 16384;
constexpr int FRAG = 512;               // 16x16 16-bit A fragment, lane-major
constexpr int FPS = SLOT / FRAG;        // 32 fragments per slot
constexpr int KPS = 64;                 // keys per attention slot (hd 64: 8 KB K + 8 KB V)
constexpr int XMAX = 2048;              // staged X columns
constexpr int XPAD = 8;                 // halves of row padding (conflict-free B loads)
constexpr int HD = 64;
constexpr int HB = 4;                   // LM-head tiles reduced together

struct Layer {
  const uint4* wqkv; const uint4* wo; const uint4* w1; const uint4* w2;
  const float* ln1_g; const float* ln1_b; const float* ln2_g; const float* ln2_b;
  void* kc; void* vc;
};

struct Args {
  const Layer* layers;
  int nlayers, h, heads, ffn, vocab, batch, smax;
  const uint4* head; const float* lnf_g; const float* lnf_b;
  const void* tok_emb; const void* pos_emb;
  float* x; long long x_sb;             // residual rows b * x_sb (fp32)
  void* q; void* ctx; void* mid;        // [batch, h], [batch, h], [batch, ffn] layer dtype
  float* wpart;                         // [s2][16][h] W2 split-K partials (s2 > 1)
  int s2;                               // W2 K-split: ffn / XMAX pieces
  float* apart;                         // [grid][2][HD + 2] split attention partials
  int* tickets;                         // [n_tile_tickets + bmax*heads + 1]
  int n_tile_tickets;
  unsigned* bar;                        // [2] count, generation
  float* cand_v; int* cand_i;           // [grid][16]
  const int* pads; int* d_filled; int* d_step; int* cur;
  long long* toks; int steps; float* logits;
  float scale;
  long long* trace;                     // optional [3 CTAs][nphase][8] globaltimer stamps
};

enum Kind { P_QKV = 0, P_ATTN, P_O, P_W1, P_W2, P_HEAD };

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"n"(NCT) : "memory"); }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ticket: one thread per CTA, after a CTA barrier that orders the CTA's
// partial stores before it (release) and the finisher's loads after (acquire)
__device__ __forceinline__ int ticket_add(int* p) {
  int prev;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(prev) : "l"(p) : "memory");
  return prev;
}

// grid barrier over the consumer threads of all CTAs (sense by generation)
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void grid_sync(unsigned* bar, long long* ts = nullptr) {
  csync();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acquire(bar + 1);
    unsigned prev;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(bar) : "memory");
    if (ts) ts[0] = gtimer();
    if (prev == gridDim.x - 1) {
      bar[0] = 0;
      asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(bar + 1), "r"(gen + 1) : "memory");
    } else {
#ifdef EET_WATCHDOG
      const long long t0 = clock64();
      while (ld_acquire(bar + 1) == gen) {
        if (clock64() - t0 > 8000000000ll) {
          printf("[eet watchdog] grid_sync block %d gen %u count %u\n", blockIdx.x, gen, *(volatile unsigned*)bar);
          __trap();
        }
      }
#else
      while (ld_acquire(bar + 1) == gen) {
      }
#endif
    }
    if (ts) ts[1] = gtimer();
  }
  csync();
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

template <typename T>
__device__ __forceinline__ void cvt8(const uint4& r, float* o) {
  const T* v = reinterpret_cast<const T*>(&r);
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i] = to_f(v[i]);
}

// Balanced contiguous ranges: CTA c owns [lo(c), lo(c+1)) of `total` units.
__device__ __forceinline__ long long range_lo(long long total, int c, int G) {
  return total * c / G;
}
// CTA owning unit index u
__device__ __forceinline__ int range_owner(long long total, long long u, int G) {
  int c = (int)((u * G) / total);
  while (c + 1 < G && range_lo(total, c + 1, G) <= u) ++c;
  while (c > 0 && range_lo(total, c, G) > u) --c;
  return c;
}
__device__ __forceinline__ bool range_nonempty(long long total, int c, int G) {
  return range_lo(total, c + 1, G) > range_lo(total, c, G);
}

// ------------------------------------------------------------------ shapes
struct Gemv {
  const uint4* w;
  int N, K, ks, rtiles;
};

__device__ __forceinline__ Gemv gemv_of(const Args& a, const Layer& L, int kind) {
  Gemv g;
  switch (kind) {
    case P_QKV: g.w = L.wqkv; g.N = 3 * a.h; g.K = a.h; break;
    case P_O: g.w = L.wo; g.N = a.h; g.K = a.h; break;
    case P_W1: g.w = L.w1; g.N = a.ffn; g.K = a.h; break;
    case P_W2: g.w = L.w2; g.N = a.h; g.K = a.ffn; break;
    default: g.w = a.head; g.N = a.vocab; g.K = a.h; break;
  }
  g.ks = g.K / 16;
  g.rtiles = (g.N + 15) / 16;
  return g;
}
// whole 16-row tiles, round-robin from a per-phase rotation: first tile of
// CTA c, stride G
__device__ __forceinline__ int first_tile(int c, int ph, int G) {
  const int rot = (int)(((long long)ph * 37) % G);
  return (c - rot + G) % G;
}
__device__ __forceinline__ bool has_ln(int kind) {
  return kind == P_QKV || kind == P_W1 || kind == P_HEAD;
}

// attention key space: pair p = b*heads + head holds keys [off_p, off_p + n_b)
struct AttnPlan {
  int L;                         // keys 0..L-1 exist; slot L-1 is this step's
  int n[16], off_b[16];          // per sequence: key count, offset of its first pair
  long long total;
};

// ------------------------------------------------------------------ kernel
template <typename T, int NB>
__global__ void __launch_bounds__(THREADS, 1) decode_step_kernel(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;                                               // NSLOT x SLOT
  T* xs = reinterpret_cast<T*>(smem + NSLOT * SLOT);                  // [16][xcols + XPAD]
  float* red = reinterpret_cast<float*>(xs + 16 * (XMAX + XPAD));    // [CW][NB*4][32]
  float* ared = red;                                                  // attention reuse
  __shared__ __align__(8) uint64_t full[NSLOT], empty[NSLOT];
  __shared__ AttnPlan ap;
  __shared__ int s_flag;
  __shared__ float best_v[16];
  __shared__ int best_i[16];

  const int G = gridDim.x, cta = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = a.h;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int filled = *a.d_filled;
    ap.L = filled + 1;
    long long tot = 0;
    for (int b = 0; b < a.batch; ++b) {
      ap.n[b] = ap.L - a.pads[b];
      ap.off_b[b] = (int)tot;
      tot += (long long)a.heads * ap.n[b];
    }
    ap.total = tot;
  }
  if (threadIdx.x < 16) { best_v[threadIdx.x] = -INFINITY; best_i[threadIdx.x] = 0x7fffffff; }
  __syncthreads();

  const int nphase = a.nlayers * 5 + 1;
  auto phase_kind = [&](int ph) { return ph == nphase - 1 ? (int)P_HEAD : ph % 5; };
  auto phase_layer = [&](int ph) { return ph == nphase - 1 ? 0 : ph / 5; };

  // =========================================================== producer
  if (warp == CW) {
    if (lane != 0) return;
    int slot = 0;
    uint32_t par = 0;
    auto push = [&](const void* s0, uint32_t b0, const void* s1, uint32_t b1) {
      mbar_wait(&empty[slot], par ^ 1);
      mbar_expect_tx(&full[slot], b0 + b1);
      bulk_load(ring + slot * SLOT, s0, b0, &full[slot]);
      if (b1) bulk_load(ring + slot * SLOT + SLOT / 2, s1, b1, &full[slot]);
      if (++slot == NSLOT) { slot = 0; par ^= 1; }
    };
    for (int ph = 0; ph < nphase; ++ph) {
      const int kind = phase_kind(ph);
      const Layer& Ly = a.layers[phase_layer(ph)];
      if (kind == P_ATTN) {
        const long long lo = range_lo(ap.total, cta, G), hi = range_lo(ap.total, cta + 1, G);
        long long k = lo;
        while (k < hi) {
          int b = 0;
          while (b + 1 < a.batch && ap.off_b[b + 1] <= k) ++b;
          const long long rel = k - ap.off_b[b];
          const int head = (int)(rel / ap.n[b]);
          const int k0 = (int)(rel - (long long)head * ap.n[b]);
          const long long pend = ap.off_b[b] + (long long)(head + 1) * ap.n[b];
          const int k1 = (int)(std::min(hi, pend) - (pend - ap.n[b]));
          const int kr = min(k1, ap.n[b] - 1);                      // ring keys: not the new slot
          const size_t base = (((size_t)b * a.heads + head) * a.smax + a.pads[b]) * HD;
          for (int j = k0; j < kr; j += KPS) {
            const uint32_t by = min(KPS, kr - j) * HD * sizeof(T);
            push(reinterpret_cast<const T*>(Ly.kc) + base + (size_t)j * HD, by,
                 reinterpret_cast<const T*>(Ly.vc) + base + (size_t)j * HD, by);
          }
          k = std::min(hi, pend);
        }
      } else {
        const Gemv gv = gemv_of(a, Ly, kind);
        if (has_ln(kind)) {                        // LayerNorm gamma | beta first
          const float* gam = kind == P_QKV ? Ly.ln1_g : kind == P_W1 ? Ly.ln2_g : a.lnf_g;
          const float* bet = kind == P_QKV ? Ly.ln1_b : kind == P_W1 ? Ly.ln2_b : a.lnf_b;
          push(gam, h * 4, bet, h * 4);
        }
        const int S = kind == P_W2 ? a.s2 : 1, kspan = gv.ks / S;
        for (int u = first_tile(cta, ph, G); u < gv.rtiles * S; u += G) {
          const int rt = u / S, k0 = (u - rt * S) * kspan;
          for (int j = k0; j < k0 + kspan; j += FPS)
            push(gv.w + ((size_t)rt * gv.ks + j) * 32, (uint32_t)(min(FPS, k0 + kspan - j) * FRAG), nullptr, 0);
        }
      }
    }
    return;
  }

  // =========================================================== consumers
  const int ct = threadIdx.x;                     // 0 .. NCT-1
  int slot = 0;
  uint32_t par = 0;
  auto pop = [&]() -> const uint8_t* {
    mbar_wait(&full[slot], par);
    return ring + slot * SLOT;
  };
  auto release = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (++slot == NSLOT) { slot = 0; par ^= 1; }
  };
  const int filled = ap.L - 1;
  const int step0 = *a.d_step;
  const T* tok = reinterpret_cast<const T*>(a.tok_emb);
  const T* pos = reinterpret_cast<const T*>(a.pos_emb);

  // stamps: 0 phase start, 1 X staged, 2 work done, 3 barrier passed
  const int tsel = cta == 0 ? 0 : cta == G / 2 ? 1 : cta == G - 1 ? 2 : -1;
  int cur_ph = 0;
  auto stamp = [&](int i) {
    if (a.trace && tsel >= 0 && ct == 0) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[((size_t)tsel * nphase + cur_ph) * 8 + i] = t;
    }
  };

  // ---- X staging (row stride xst = staged columns + XPAD halves)
  // LN rows m < batch of x (or, layer 0, of the token + position embedding)
  // with gamma/beta from the ring slot `gb` ([gamma h][beta h] fp32)
  auto stage_ln = [&](const float* gb, bool embed, bool fold, int xst) {
    const float* gam = gb;
    const float* bet = reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(gb) + SLOT / 2);
    auto run = [&](auto nr_c) {
      constexpr int NR = decltype(nr_c)::value;   // rows per warp pass (loaded together)
      constexpr int NV = 16 / NR;                  // float4 per lane per row
      for (int r0 = warp; r0 < 16; r0 += CW * NR) {
        float4 v[NR][NV];
        float mu[NR], rs[NR];
        const int nv = h / 4;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const int r = r0 + q * CW;
          const bool live = r < a.batch;
          const float* xr = a.x + (live ? r : 0) * a.x_sb;
          const T* tr = tok + (live ? (long long)a.cur[r] * h : 0);
          const T* pr = pos + (live ? (long long)(filled - a.pads[r]) * h : 0);
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            const int i = j * 32 + lane;
            v[q][j] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (live && i < nv) {
              if (embed) {
                const uint2 t2 = __ldg(reinterpret_cast<const uint2*>(tr) + i);
                const uint2 p2 = __ldg(reinterpret_cast<const uint2*>(pr) + i);
                const T* tv = reinterpret_cast<const T*>(&t2);
                const T* pv = reinterpret_cast<const T*>(&p2);
                v[q][j] = make_float4(to_f(tv[0]) + to_f(pv[0]), to_f(tv[1]) + to_f(pv[1]),
                                      to_f(tv[2]) + to_f(pv[2]), to_f(tv[3]) + to_f(pv[3]));
                if (cta == 0) reinterpret_cast<float4*>(a.x + r * a.x_sb)[i] = v[q][j];
              } else {
                v[q][j] = __ldcg(reinterpret_cast<const float4*>(xr) + i);
                if (fold) {                       // x += W2 split-K pieces, in piece order
                  for (int sp = 0; sp < a.s2; ++sp) {
                    const float4 p4 = __ldcg(reinterpret_cast<const float4*>(a.wpart + ((size_t)sp * 16 + r) * h) + i);
                    v[q][j].x += p4.x; v[q][j].y += p4.y; v[q][j].z += p4.z; v[q][j].w += p4.w;
                  }
                }
              }
            }
          }
        }
        if (r0 == 0) {                              // trace: x loads landed
          float t = v[0][0].x;
          if (t == 12345.f) t = 0.f;
          if (lane == 0 && t != 1e30f) stamp(4);
        }
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          float s = 0.f;
#pragma unroll
          for (int j = 0; j < NV; ++j) s += (v[q][j].x + v[q][j].y) + (v[q][j].z + v[q][j].w);
          mu[q] = warp_sum(s) / (float)h;
          float q2 = 0.f;
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            if (j * 32 + lane < nv) {
              const float d0 = v[q][j].x - mu[q], d1 = v[q][j].y - mu[q], d2 = v[q][j].z - mu[q],
                          d3 = v[q][j].w - mu[q];
              q2 += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
            }
          }
          rs[q] = 1.0f / sqrtf(warp_sum(q2) / (float)h + 1e-5f);
        }
        if (r0 == 0) stamp(5);
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const int r = r0 + q * CW;
          if (r >= 16) continue;
          T* dst = xs + r * xst;
          const bool live = r < a.batch;
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            const int i = j * 32 + lane;
            if (i < nv) {
              uint2 o2 = make_uint2(0, 0);
              if (live) {
                const float4 gg = reinterpret_cast<const float4*>(gam)[i];
                const float4 bb = reinterpret_cast<const float4*>(bet)[i];
                T o[4] = {from_f<T>((v[q][j].x - mu[q]) * rs[q] * gg.x + bb.x),
                          from_f<T>((v[q][j].y - mu[q]) * rs[q] * gg.y + bb.y),
                          from_f<T>((v[q][j].z - mu[q]) * rs[q] * gg.z + bb.z),
                          from_f<T>((v[q][j].w - mu[q]) * rs[q] * gg.w + bb.w)};
                o2 = *reinterpret_cast<const uint2*>(o);
              }
              *reinterpret_cast<uint2*>(dst + i * 4) = o2;
            }
          }
        }
      }
    };
    if (h <= 1024) run(std::integral_constant<int, 2>{});
    else run(std::integral_constant<int, 1>{});
  };
  // 16-bit activation rows, columns [klo, khi)
  auto stage_copy = [&](const T* src, int ld, int klo, int khi, int xst) {
    const int w8 = (khi - klo) / 8;
    const int n = 16 * w8;
    for (int base = 0; base < n; base += 8 * NCT) {  // 8 loads in flight per thread
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * NCT + ct;
        const int r = i / w8, cidx = i - r * w8;
        v[u] = (i < n && r < a.batch)
                   ? __ldcg(reinterpret_cast<const uint4*>(src + (long long)r * ld + klo) + cidx)
                   : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * NCT + ct;
        const int r = i / w8, cidx = i - r * w8;
        if (i < n) *reinterpret_cast<uint4*>(xs + r * xst + cidx * 8) = v[u];
      }
    }
  };

  // attention output for the out-projection: pairs finished whole by one
  // CTA are in ctx; pairs cut by CTA-range boundaries are merged here from
  // their pieces (apart[c][1] of the first owner, apart[c][0] of the
  // following ones), in key order
  auto stage_ctx = [&](int xst) {
    const int npair = a.batch * a.heads;
    for (int p = ct; p < 16 * a.heads; p += NCT) {
      const int b = p / a.heads, head = p - b * a.heads;
      T* dst = xs + b * xst + head * HD;
      if (p >= npair) {
#pragma unroll
        for (int c = 0; c < HD / 8; ++c) reinterpret_cast<uint4*>(dst)[c] = make_uint4(0, 0, 0, 0);
        continue;
      }
      const long long pstart = ap.off_b[b] + (long long)head * ap.n[b], pend = pstart + ap.n[b];
      const int c0 = range_owner(ap.total, pstart, G), c1 = range_owner(ap.total, pend - 1, G);
      if (c0 == c1) {
        const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(a.ctx) + (size_t)b * h + head * HD);
        uint4 v[HD / 8];
#pragma unroll
        for (int c = 0; c < HD / 8; ++c) v[c] = __ldcg(src + c);
#pragma unroll
        for (int c = 0; c < HD / 8; ++c) reinterpret_cast<uint4*>(dst)[c] = v[c];
        continue;
      }
      float M = -INFINITY;
      for (int cc = c0; cc <= c1; ++cc)
        if (range_nonempty(ap.total, cc, G))
          M = fmaxf(M, __ldcg(a.apart + ((size_t)cc * 2 + (cc == c0 ? 1 : 0)) * (HD + 2) + HD));
      float Ls = 0.f, acc[HD];
#pragma unroll
      for (int d = 0; d < HD; ++d) acc[d] = 0.f;
      for (int cc = c0; cc <= c1; ++cc) {
        if (!range_nonempty(ap.total, cc, G)) continue;
        const float* src = a.apart + ((size_t)cc * 2 + (cc == c0 ? 1 : 0)) * (HD + 2);
        const float ms = __ldcg(src + HD);
        const float cw = (ms == -INFINITY) ? 0.f : __expf(ms - M);
        Ls += __ldcg(src + HD + 1) * cw;
#pragma unroll
        for (int d = 0; d < HD; d += 2) {
          const float2 t2 = __ldcg(reinterpret_cast<const float2*>(src + d));
          acc[d] += t2.x * cw;
          acc[d + 1] += t2.y * cw;
        }
      }
      const float inv = 1.0f / Ls;
#pragma unroll
      for (int c = 0; c < HD / 8; ++c) {
        T o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = from_f<T>(acc[c * 8 + e] * inv);
        reinterpret_cast<uint4*>(dst)[c] = *reinterpret_cast<const uint4*>(o);
      }
    }
  };

  // ---- epilogue of one finished output element (out feature n, token m)
  auto epilogue = [&](int kind, const Layer& Ly, int n, int m, float v, int kpiece) {
    if (m >= a.batch) return;
    switch (kind) {
      case P_QKV: {
        if (n < h) {
          reinterpret_cast<T*>(a.q)[m * h + n] = from_f<T>(v);
        } else {
          const int which = n >= 2 * h;
          const int w = n - h * (1 + which);
          const int head = w / HD, d = w - head * HD;
          T* dst = reinterpret_cast<T*>(which ? Ly.vc : Ly.kc);
          dst[(((size_t)m * a.heads + head) * a.smax + filled) * HD + d] = from_f<T>(v);
        }
        break;
      }
      case P_O: {
        // x += attention output; also folds the previous layer's W2 pieces
        // into x (read by this layer's LN1 stage, two barriers ago)
        float* px = a.x + m * a.x_sb + n;          // L2-coherent: other CTAs update x too
        float xv = __ldcg(px);
        if (a.s2 > 1 && kpiece > 0)
          for (int sp = 0; sp < a.s2; ++sp) xv += __ldcg(a.wpart + ((size_t)sp * 16 + m) * h + n);
        __stcg(px, xv + v);
        break;
      }
      case P_W2: {                                 // piece s of the K split (folded by the next LN)
        if (a.s2 > 1) {
          __stcg(a.wpart + ((size_t)kpiece * 16 + m) * h + n, v);
        } else {
          float* px = a.x + m * a.x_sb + n;
          __stcg(px, __ldcg(px) + v);
        }
        break;
      }
      case P_W1:
        reinterpret_cast<T*>(a.mid)[(size_t)m * a.ffn + n] = from_f<T>(gelu_tanh(v));
        break;
      default:
        break;
    }
  };

  // element e of a reduced 16 x (8*NB) tile -> (row, token)
  auto elem = [&](int e, int& row, int& tokn) {
    const int i = e >> 5, ln = e & 31;
    const int nb = i >> 2, j = i & 3;
    row = (ln >> 2) + 8 * (j >> 1);
    tokn = nb * 8 + 2 * (ln & 3) + (j & 1);
  };

  // ---- k-steps [kq0, kq1) of projection tile rt from the ring into acc
  //      (X holds columns [xlo, xhi); W2 pieces restage mid when needed)
  auto gemv_range = [&](const Gemv& gv, int rt, int kq0, int kq1, float (*acc)[4], int xst, int xlo) {
    const int g = lane >> 2, c4 = lane & 3;
    for (int j = kq0; j < kq1; j += FPS) {
      const int nf = min(FPS, kq1 - j);
      const uint8_t* sl = pop();
      for (int i = warp; i < nf; i += CW) {
        const uint4 av = *reinterpret_cast<const uint4*>(sl + i * FRAG + lane * 16);
        const int kc = (j + i) * 16 - xlo;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          const T* xr = xs + (nb * 8 + g) * xst + kc + 2 * c4;
          mma16816<T>(acc[nb], av, *reinterpret_cast<const uint32_t*>(xr),
                      *reinterpret_cast<const uint32_t*>(xr + 8));
        }
      }
      release();
    }
    (void)gv;
  };

  for (int ph = 0; ph < nphase; ++ph) {
    const int kind = phase_kind(ph);
    const Layer& Ly = a.layers[phase_layer(ph)];
    cur_ph = ph;
    stamp(0);

    if (kind == P_ATTN) {
      // --------------------------------------------------- attention
      // 8 keys per warp step: lane group grp (4 lanes) owns one key, lane sub
      // 16 of its 64 dims
      const long long lo = range_lo(ap.total, cta, G), hi = range_lo(ap.total, cta + 1, G);
      const int grp = lane >> 2, sub = lane & 3;
      long long k = lo;
      while (k < hi) {
        int b = 0;
        while (b + 1 < a.batch && ap.off_b[b + 1] <= k) ++b;
        const int nb_ = ap.n[b];
        const long long rel = k - ap.off_b[b];
        const int head = (int)(rel / nb_);
        const int k0 = (int)(rel - (long long)head * nb_);
        const long long pstart = ap.off_b[b] + (long long)head * nb_, pend = pstart + nb_;
        const int k1 = (int)(std::min(hi, pend) - pstart);
        const int kr = min(k1, nb_ - 1);
        const int pair = b * a.heads + head;
        float q[16];
        {
          const T* qp = reinterpret_cast<const T*>(a.q) + (size_t)b * h + head * HD + sub * 16;
          cvt8<T>(__ldcg(reinterpret_cast<const uint4*>(qp)), q);
          cvt8<T>(__ldcg(reinterpret_cast<const uint4*>(qp) + 1), q + 8);
        }
        float m = -INFINITY, l = 0.f, acc[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[e] = 0.f;
        auto consume = [&](uint4 k0v, uint4 k1v, uint4 v0v, uint4 v1v, bool ok) {
          float kv[16];
          cvt8<T>(k0v, kv);
          cvt8<T>(k1v, kv + 8);
          float dot = 0.f;
#pragma unroll
          for (int e = 0; e < 16; ++e) dot = fmaf(q[e], kv[e], dot);
          dot += __shfl_xor_sync(0xffffffffu, dot, 1);
          dot += __shfl_xor_sync(0xffffffffu, dot, 2);
          if (ok) {
            float vv[16];
            cvt8<T>(v0v, vv);
            cvt8<T>(v1v, vv + 8);
            const float s = dot * a.scale;
            const float mn = fmaxf(m, s);
            const float corr = __expf(m - mn);             // m = -inf -> 0
            const float p = __expf(s - mn);
            l = l * corr + p;
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[e] = fmaf(p, vv[e], acc[e] * corr);
            m = mn;
          }
        };
        for (int j = k0; j < kr; j += KPS) {
          const int kn = min(KPS, kr - j);
          const uint8_t* sl = pop();
          const int jj = warp * 8 + grp;
          const bool ok = jj < kn;
          const uint4* kp = reinterpret_cast<const uint4*>(sl + jj * (HD * 2) + sub * 32);
          const uint4* vp = reinterpret_cast<const uint4*>(sl + SLOT / 2 + jj * (HD * 2) + sub * 32);
          uint4 k0v = make_uint4(0, 0, 0, 0), k1v = k0v, v0v = k0v, v1v = k0v;
          if (ok) {                                // no reads past the copied keys
            k0v = kp[0]; k1v = kp[1]; v0v = vp[0]; v1v = vp[1];
          }
          consume(k0v, k1v, v0v, v1v, ok);
          release();
        }
        if (k1 == nb_ && warp == 0) {            // this step's slot, written by LN1+QKV
          const size_t off = (((size_t)b * a.heads + head) * a.smax + filled) * HD + sub * 16;
          const uint4* kp = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(Ly.kc) + off);
          const uint4* vp = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(Ly.vc) + off);
          consume(__ldcg(kp), __ldcg(kp + 1), __ldcg(vp), __ldcg(vp + 1), grp == 0);
        }
        // merge the 8 key groups of the warp, then the warps
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          const float mo = __shfl_xor_sync(0xffffffffu, m, o);
          const float lo2 = __shfl_xor_sync(0xffffffffu, l, o);
          const float mn = fmaxf(m, mo);
          const float c1 = (m == -INFINITY) ? 0.f : __expf(m - mn);
          const float c2 = (mo == -INFINITY) ? 0.f : __expf(mo - mn);
#pragma unroll
          for (int e = 0; e < 16; ++e) acc[e] = acc[e] * c1 + __shfl_xor_sync(0xffffffffu, acc[e], o) * c2;
          l = l * c1 + lo2 * c2;
          m = mn;
        }
        if (grp == 0) {
#pragma unroll
          for (int e = 0; e < 16; ++e) ared[warp * (HD + 2) + sub * 16 + e] = acc[e];
          if (sub == 0) { ared[warp * (HD + 2) + HD] = m; ared[warp * (HD + 2) + HD + 1] = l; }
        }
        csync();
        const bool whole = (k0 == 0 && k1 == nb_);
        if (ct < HD) {
          float um = -INFINITY, ul = 0.f, ua = 0.f;
#pragma unroll
          for (int w = 0; w < CW; ++w) um = fmaxf(um, ared[w * (HD + 2) + HD]);
#pragma unroll
          for (int w = 0; w < CW; ++w) {
            const float mw = ared[w * (HD + 2) + HD];
            const float cw = (mw == -INFINITY) ? 0.f : __expf(mw - um);
            ul += ared[w * (HD + 2) + HD + 1] * cw;
            ua += ared[w * (HD + 2) + ct] * cw;
          }
          if (whole) {
            reinterpret_cast<T*>(a.ctx)[(size_t)b * h + head * HD + ct] = from_f<T>(ua / ul);
          } else {
            // piece continuing a pair from an earlier CTA -> slot 0; the
            // piece that starts a pair continued by later CTAs -> slot 1
            float* dst = a.apart + ((size_t)cta * 2 + (k0 > 0 ? 0 : 1)) * (HD + 2);
            dst[ct] = ua;
            if (ct == 0) { dst[HD] = um; dst[HD + 1] = ul; }
          }
        }
        csync();
        k = std::min(hi, pend);
      }
    } else {
      // --------------------------------------------------- projections
      const Gemv gv = gemv_of(a, Ly, kind);
      const int t0 = first_tile(cta, ph, G);
      const int S = kind == P_W2 ? a.s2 : 1, kspan = gv.ks / S;
      const int nunits = gv.rtiles * S;
      const int xst = min(gv.K, XMAX) + XPAD;
      int xlo = 0, xhi = 0;
      if (has_ln(kind)) {
        const uint8_t* gb = pop();                      // gamma | beta
        if (t0 < nunits || (ph == 0 && cta == 0))       // CTA 0 also writes the embedded x
          stage_ln(reinterpret_cast<const float*>(gb), kind == P_QKV && ph == 0,
                   a.s2 > 1 && (kind == P_HEAD || (kind == P_QKV && ph > 0)), xst);
        release();
        xhi = gv.K;
        csync();
      } else if (kind == P_O && t0 < nunits) {
        stage_ctx(xst);
        xhi = gv.K;
        csync();
      }
      stamp(1);
      if (kind != P_HEAD) {
        for (int u = t0; u < nunits; u += G) {
          const int rt = u / S, sp = u - rt * S;
          const int kq0 = sp * kspan, kq1 = kq0 + kspan;
          if (kq0 * 16 < xlo || kq1 * 16 > xhi) {       // W2: stage this piece of mid
            csync();
            xlo = kq0 * 16;
            xhi = kq1 * 16;
            stage_copy(reinterpret_cast<const T*>(a.mid), a.ffn, xlo, xhi, xst);
            csync();
          }
          float acc[NB][4];
#pragma unroll
          for (int nb = 0; nb < NB; ++nb)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[nb][i] = 0.f;
          gemv_range(gv, rt, kq0, kq1, acc, xst, xlo);
#pragma unroll
          for (int nb = 0; nb < NB; ++nb)
#pragma unroll
            for (int i = 0; i < 4; ++i) red[(warp * NB * 4 + nb * 4 + i) * 32 + lane] = acc[nb][i];
          csync();
          if (ct < NB * 128) {
            float v = 0.f;
#pragma unroll
            for (int w = 0; w < CW; ++w) v += red[(w * NB * 4) * 32 + ct];
            int row, tokn;
            elem(ct, row, tokn);
            const int n = rt * 16 + row;
            if (n < gv.N) epilogue(kind, Ly, n, tokn, v, kind == P_O ? (ph >= 5) : sp);
          }
          csync();
        }
      } else {
        // LM head: HB tiles per reduction; per-CTA running argmax (lowest id on ties)
        float* hred = reinterpret_cast<float*>(xs + 16 * xst);           // [HB][CW][NB*4][32]
        float* hres = hred + HB * CW * NB * 4 * 32;                       // [HB][16][16]
        for (int rt0 = t0; rt0 < gv.rtiles; rt0 += HB * G) {
          float acc[HB][NB][4];
#pragma unroll
          for (int u = 0; u < HB; ++u)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb)
#pragma unroll
              for (int i = 0; i < 4; ++i) acc[u][nb][i] = 0.f;
#pragma unroll
          for (int u = 0; u < HB; ++u)
            if (rt0 + u * G < gv.rtiles) gemv_range(gv, rt0 + u * G, 0, gv.ks, acc[u], xst, 0);
#pragma unroll
          for (int u = 0; u < HB; ++u)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb)
#pragma unroll
              for (int i = 0; i < 4; ++i)
                hred[((u * CW + warp) * NB * 4 + nb * 4 + i) * 32 + lane] = acc[u][nb][i];
          csync();
          for (int e = ct; e < HB * NB * 128; e += NCT) {
            const int u = e / (NB * 128), el = e - u * NB * 128;
            float v = 0.f;
#pragma unroll
            for (int w = 0; w < CW; ++w) v += hred[(u * CW + w) * NB * 4 * 32 + el];
            int row, tokn;
            elem(el, row, tokn);
            const int n = (rt0 + u * G) * 16 + row;
            const bool ok = rt0 + u * G < gv.rtiles && n < gv.N;
            if (ok && tokn < a.batch && a.logits && step0 + 1 < a.steps)
              a.logits[((size_t)(step0 + 1) * a.batch + tokn) * a.vocab + n] = v;
            hres[(u * 16 + tokn) * 16 + row] = ok ? v : -INFINITY;
          }
          csync();
          if (ct < a.batch) {
            float bv = best_v[ct];
            int bi = best_i[ct];
            for (int u = 0; u < HB; ++u)
              for (int r = 0; r < 16; ++r) {
                const float tv = hres[(u * 16 + ct) * 16 + r];
                const int id = (rt0 + u * G) * 16 + r;
                if (tv > bv || (tv == bv && id < bi)) { bv = tv; bi = id; }
              }
            best_v[ct] = bv;
            best_i[ct] = bi;
          }
          csync();
        }
      }
    }
    stamp(2);
    if (ph + 1 < nphase)
      grid_sync(a.bar, (a.trace && tsel >= 0) ? a.trace + ((size_t)tsel * nphase + cur_ph) * 8 + 6 : nullptr);
    stamp(3);
  }

  // ---- final argmax over the CTAs' candidates (last CTA), cursor advance
  if (ct < 16) {
    a.cand_v[cta * 16 + ct] = best_v[ct];
    a.cand_i[cta * 16 + ct] = best_i[ct];
  }
  csync();
  if (ct == 0) {
    const int tk = a.n_tile_tickets + 16 * a.heads;
    const int prev = ticket_add(&a.tickets[tk]);
    s_flag = prev == G - 1;
    if (s_flag) a.tickets[tk] = 0;
  }
  csync();
  if (s_flag) {
    const int step1 = step0 + 1;
    if (ct < a.batch) {
      float bv = -INFINITY;
      int bi = 0x7fffffff;
      for (int cc = 0; cc < G; ++cc) {
        const float v = __ldcg(a.cand_v + cc * 16 + ct);
        const int i = __ldcg(a.cand_i + cc * 16 + ct);
        if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
      }
      if (bi == 0x7fffffff) bi = 0;
      a.cur[ct] = bi;
      if (a.toks && step1 < a.steps) a.toks[(long long)ct * a.steps + step1] = bi;
    }
    if (ct == 0) {
      *a.d_filled = filled + 1;
      *a.d_step = step1;
    }
  }
}

}  // namespace mk

// ------------------------------------------------------------------ packing
// W [N, K] (K-major, row pitch K) -> fragment-major tiles: out[(rt*ks + kq)*32
// + lane] = the 8 halves lane holds of the m16n8k16 A operand
// (a0..a7 = (g,2c) (g,2c+1) (g+8,2c) (g+8,2c+1) (g,2c+8) (g,2c+9) (g+8,2c+8)
// (g+8,2c+9)); rows >= N are zero.
__global__ void mk_pack_kernel(const uint16_t* __restrict__ w, int N, int K, uint4* __restrict__ out) {
  const int ks = K / 16;
  const long long total = (long long)((N + 15) / 16) * ks * 32;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int lane = (int)(i & 31);
    const long long fr = i >> 5;
    const int rt = (int)(fr / ks), kq = (int)(fr - (long long)rt * ks);
    const int g = lane >> 2, c = lane & 3;
    const int r0 = rt * 16 + g, r1 = r0 + 8, k0 = kq * 16 + 2 * c;
    auto at = [&](int r, int k) -> uint32_t { return r < N ? w[(long long)r * K + k] : 0u; };
    uint4 v;
    v.x = at(r0, k0) | (at(r0, k0 + 1) << 16);
    v.y = at(r1, k0) | (at(r1, k0 + 1) << 16);
    v.z = at(r0, k0 + 8) | (at(r0, k0 + 9) << 16);
    v.w = at(r1, k0 + 8) | (at(r1, k0 + 9) << 16);
    out[i] = v;
  }
}

size_t mk_packed_bytes(int N, int K) { return (size_t)((N + 15) / 16) * (K / 16) * 512; }

void mk_pack(const void* w, int N, int K, void* out, cudaStream_t st) {
  const long long total = (long long)((N + 15) / 16) * (K / 16) * 32;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 4 * 148);
  mk_pack_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const uint16_t*>(w), N, K,
                                         reinterpret_cast<uint4*>(out));
  EET_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ host
bool mk_eligible(int dtype, int h, int heads, int batch, int ffn) {
  return (dtype == EET_F16 || dtype == EET_BF16) && heads >= 1 && h % heads == 0 &&
         h / heads == mk::HD && h % 128 == 0 && h <= 1024 && batch >= 1 && batch <= 16 &&
         ffn % 16 == 0 && ffn == 4 * h;
}

size_t mk_smem_bytes(int nb) {
  return (size_t)mk::NSLOT * mk::SLOT + 16 * (mk::XMAX + mk::XPAD) * 2 +
         (size_t)mk::CW * nb * 4 * 32 * 4;
}

struct MkState {
  int G = 0, dtype = -1, h = 0, heads = 0, bmax = 0, vocab = 0, layers = 0;
  void* wbuf = nullptr;
  size_t wcap = 0;
  mk::Layer* d_layers = nullptr;
  mk::Layer* h_layers = nullptr;       // pinned staging of the layer table
  int lcap = 0;
  void *q = nullptr, *ctx = nullptr, *mid = nullptr;
  float *gpart = nullptr, *apart = nullptr, *cand_v = nullptr;
  int *cand_i = nullptr, *tickets = nullptr;
  unsigned* bar = nullptr;
  int n_tile_tickets = 0;
  const uint4* head = nullptr;
  ~MkState() {
    for (void* p : {wbuf, (void*)d_layers, q, ctx, mid, (void*)gpart, (void*)apart, (void*)cand_v,
                    (void*)cand_i, (void*)tickets, (void*)bar})
      if (p) cudaFree(p);
    if (h_layers) cudaFreeHost(h_layers);
  }
};

void mk_state_free(MkState* s) { delete s; }

static void* dmalloc(size_t bytes) {
  void* p = nullptr;
  EET_CHECK_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
  return p;
}

static void mk_launch(int dtype, int batch, const mk::Args& args, int grid, cudaStream_t st) {
  const int nb = batch <= 8 ? 1 : 2;
  const size_t smem = mk_smem_bytes(nb);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(mk::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto go = [&](auto kern) {
    EET_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    EET_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, args));
  };
  if (dtype == EET_BF16) {
    nb == 1 ? go(mk::decode_step_kernel<__nv_bfloat16, 1>) : go(mk::decode_step_kernel<__nv_bfloat16, 2>);
  } else {
    nb == 1 ? go(mk::decode_step_kernel<__half, 1>) : go(mk::decode_step_kernel<__half, 2>);
  }
  EET_LAUNCH_CHECK();
}

void mk_pack_model(MkState*& st, int dtype, const eet_model* m, int h, cudaStream_t stream) {
  (void)dtype;
  if (!st) st = new MkState();
  MkState& Z = *st;
  const int V = m->vocab, L = m->layers, ffn = 4 * h;
  const size_t per_layer = mk_packed_bytes(3 * h, h) + mk_packed_bytes(h, h) +
                           mk_packed_bytes(ffn, h) + mk_packed_bytes(h, ffn);
  const size_t need = per_layer * L + mk_packed_bytes(V, h);
  if (Z.wcap < need) {
    if (Z.wbuf) cudaFree(Z.wbuf);
    Z.wbuf = dmalloc(need);
    Z.wcap = need;
  }
  if (Z.lcap < L) {
    if (Z.d_layers) cudaFree(Z.d_layers);
    if (Z.h_layers) cudaFreeHost(Z.h_layers);
    Z.d_layers = (mk::Layer*)dmalloc(sizeof(mk::Layer) * L);
    EET_CHECK_CUDA(cudaMallocHost(&Z.h_layers, sizeof(mk::Layer) * L));
    Z.lcap = L;
  }
  EET_CHECK_CUDA(cudaStreamSynchronize(stream));     // pinned table reuse
  uint8_t* wp = reinterpret_cast<uint8_t*>(Z.wbuf);
  auto pack = [&](const void* w, int N, int K) {
    mk_pack(w, N, K, wp, stream);
    packed_register(w, wp);
    const uint4* r = reinterpret_cast<const uint4*>(wp);
    wp += mk_packed_bytes(N, K);
    return r;
  };
  for (int l = 0; l < L; ++l) {
    const eet_layer_weights& w = m->layer[l];
    mk::Layer& D = Z.h_layers[l];
    D.wqkv = pack(w.wqkv, 3 * h, h);
    D.wo = pack(w.wo, h, h);
    D.w1 = pack(w.w1, ffn, h);
    D.w2 = pack(w.w2, h, ffn);
  }
  Z.head = pack(m->head, V, h);
}

// `steps` incremental steps of generate through the megakernel. The cursor
// (d_filled, d_step) and the current tokens (d_cur) are device state that
// each launch reads and advances, exactly as decode_iteration does.
void mk_generate(MkState*& st, int dtype, int h, int heads, int bmax, int smax,
                 const eet_model* m, int batch, const int* d_pads, const int* h_pads, int t,
                 int* d_filled, int* d_step, int* d_cur, long long* d_tokens, int steps,
                 float* d_logits, cudaStream_t stream) {
  const int G = device_sm_count();
  const int V = m->vocab, L = m->layers, ffn = 4 * h;
  if (!st) st = new MkState();
  MkState& S = *st;
  // ---- scratch (re)allocation
  if (S.G != G || S.dtype != dtype || S.h != h || S.heads != heads || S.bmax < bmax || S.vocab < V) {
    MkState* fresh = new MkState();
    std::swap(fresh->wbuf, S.wbuf);
    std::swap(fresh->wcap, S.wcap);
    delete st;
    st = fresh;
    MkState& N = *st;
    N.G = G; N.dtype = dtype; N.h = h; N.heads = heads; N.bmax = bmax; N.vocab = V;
    N.q = dmalloc((size_t)16 * h * 2);
    N.ctx = dmalloc((size_t)16 * h * 2);
    N.mid = dmalloc((size_t)16 * ffn * 2);
    N.gpart = (float*)dmalloc(sizeof(float) * 16 * h * std::max(1, ffn / mk::XMAX));
    N.apart = (float*)dmalloc(sizeof(float) * G * 2 * (mk::HD + 2));
    N.cand_v = (float*)dmalloc(sizeof(float) * G * 16);
    N.cand_i = (int*)dmalloc(sizeof(int) * G * 16);
    N.n_tile_tickets = (std::max(std::max(3 * h, ffn), V) + 15) / 16;
    const size_t nt = (size_t)N.n_tile_tickets + 16 * heads + 1;
    N.tickets = (int*)dmalloc(sizeof(int) * nt);
    N.bar = (unsigned*)dmalloc(sizeof(unsigned) * 2);
    EET_CHECK_CUDA(cudaMemsetAsync(N.tickets, 0, sizeof(int) * nt, stream));
    EET_CHECK_CUDA(cudaMemsetAsync(N.bar, 0, sizeof(unsigned) * 2, stream));
  }
  MkState& Z = *st;
  // ---- weights: re-packed every call (cheap next to the decode loop; the
  //      caller's buffers may change between calls)
  mk_pack_model(st, dtype, m, h, stream);
  MkState& Z2 = *st;
  for (int l = 0; l < L; ++l) {
    const eet_layer_weights& w = m->layer[l];
    mk::Layer& D = Z2.h_layers[l];
    D.ln1_g = w.ln1_g; D.ln1_b = w.ln1_b; D.ln2_g = w.ln2_g; D.ln2_b = w.ln2_b;
    D.kc = m->kcache[l];
    D.vc = m->vcache[l];
  }
  const uint4* head = Z2.head;
  EET_CHECK_CUDA(cudaMemcpyAsync(Z2.d_layers, Z2.h_layers, sizeof(mk::Layer) * L,
                                 cudaMemcpyHostToDevice, stream));
  mk::Args a{};
  a.layers = Z.d_layers;
  a.nlayers = L; a.h = h; a.heads = heads; a.ffn = ffn; a.vocab = V; a.batch = batch; a.smax = smax;
  a.head = head; a.lnf_g = m->lnf_g; a.lnf_b = m->lnf_b;
  a.tok_emb = m->tok_emb; a.pos_emb = m->pos_emb;
  a.x = m->hidden; a.x_sb = (long long)m->max_prompt * h;
  a.q = Z.q; a.ctx = Z.ctx; a.mid = Z.mid;
  a.wpart = Z.gpart; a.s2 = std::max(1, ffn / mk::XMAX); a.apart = Z.apart; a.tickets = Z.tickets; a.n_tile_tickets = Z.n_tile_tickets;
  a.bar = Z.bar; a.cand_v = Z.cand_v; a.cand_i = Z.cand_i;
  a.pads = d_pads; a.d_filled = d_filled; a.d_step = d_step; a.cur = d_cur;
  a.toks = d_tokens; a.steps = steps; a.logits = d_logits;
  a.scale = 1.0f / std::sqrt((float)mk::HD);
  const double es = 2.0;
  const double wbytes = (double)L * 12.0 * h * h * es + (double)V * h * es;
  static const bool tracing = [] {
    const char* e = std::getenv("EET_MK_TRACE");
    return e && e[0] == '1';
  }();
  const int nphase = L * 5 + 1;
  long long* d_trace = nullptr;
  const size_t tstride = (size_t)3 * nphase * 8;
  if (tracing) {
    d_trace = (long long*)dmalloc(sizeof(long long) * (size_t)steps * tstride);
    EET_CHECK_CUDA(cudaMemsetAsync(d_trace, 0, sizeof(long long) * (size_t)steps * tstride, stream));
  }
  for (int s = 0; s < steps; ++s) {
    a.trace = d_trace ? d_trace + (size_t)s * tstride : nullptr;
    double keys = 0;                                   // attended keys of this step
    for (int b = 0; b < batch; ++b) keys += t + s + 1 - h_pads[b];
    const double kvb = keys * 2.0 * h * es * L;
    ProfScope ps(K_DECODE_STEP, stream, wbytes + kvb, 2.0 * batch * wbytes / es + 4.0 * keys * h * L);
    mk_launch(dtype, batch, a, G, stream);
  }
  if (d_trace) {
    std::vector<long long> tr((size_t)steps * tstride);
    EET_CHECK_CUDA(cudaMemcpyAsync(tr.data(), d_trace, sizeof(long long) * tr.size(), cudaMemcpyDeviceToHost, stream));
    EET_CHECK_CUDA(cudaStreamSynchronize(stream));
    const char* nm[6] = {"qkv", "attn", "oproj", "w1", "w2", "head"};
    for (int w = 0; w < 3; ++w) {
      double acc[6][3] = {{0}}, ex[6][4] = {{0}};
      for (int s = 0; s < steps; ++s)
        for (int ph = 0; ph < nphase; ++ph) {
          const long long* t4 = &tr[(size_t)s * tstride + ((size_t)w * nphase + ph) * 8];
          const int k = ph == nphase - 1 ? 5 : ph % 5;
          const long long t1 = t4[1] ? t4[1] : t4[0];
          acc[k][0] += (double)(t1 - t4[0]);
          acc[k][1] += (double)(t4[2] - t1);
          acc[k][2] += (double)(t4[3] - t4[2]);
          if (t4[4]) ex[k][0] += (double)(t4[4] - t4[0]);
          if (t4[5]) ex[k][1] += (double)(t4[5] - t4[0]);
          if (t4[6]) ex[k][2] += (double)(t4[6] - t4[2]);
          if (t4[7]) ex[k][3] += (double)(t4[7] - t4[2]);
        }
      std::fprintf(stderr, "[eet mk trace] cta-sel %d, us per step (stage/work/barrier):", w);
      for (int k = 0; k < 6; ++k)
        std::fprintf(stderr, " %s %.1f/%.1f/%.1f", nm[k], acc[k][0] / steps / 1e3, acc[k][1] / steps / 1e3,
                     acc[k][2] / steps / 1e3);
      std::fprintf(stderr, "\n   x loads/LN stats since phase start; barrier: arrive-return/release since work done:");
      for (int k = 0; k < 6; ++k)
        std::fprintf(stderr, " %s %.1f/%.1f/%.1f/%.1f", nm[k], ex[k][0] / steps / 1e3, ex[k][1] / steps / 1e3,
                     ex[k][2] / steps / 1e3, ex[k][3] / steps / 1e3);
      std::fprintf(stderr, "\n");
    }
    cudaFree(d_trace);
  }
}

}  // namespace eet
