// Context-phase (prompt) mask-fused attention on tcgen05 for 16-bit modes,
// head_dim 64 / 128 (§2.1 Algorithm 1; attention.py:73-104 +
// runtime.py:164-178 in the reference).
//
// One CTA = one (sequence b, head, pair of 128-query tiles A/B). Causal and
// padding bounds come from slot indices: key tiles start at the sequence's
// pad offset and stop at each query tile's last query, so pad keys are never
// loaded and query tiles that lie wholly in the padding exit immediately.
//
//   warps 0-3   softmax for tile A, warps 4-7 for tile B (thread = query row)
//   warp 8      TMA producer: Q_A, Q_B once, then K/V tiles (64 keys) into a
//               two-stage ring straight from the [b, heads, s_max, hd] cache
//   warp 9      TMEM allocator + MMA issuer: S_X = Q_X K_j^T (M128 N64) and
//               O_X += P_X V_j (M128 N=hd; P read from TMEM, V MN-major)
//
// P goes through TMEM (default; EET_ATTN_PTMEM=0 keeps the smem path): the
// softmax writes P (16-bit pairs) over the S buffer it has just read and the
// PV MMA takes its A operand from TMEM. The 64 KB of smem P buffers this
// frees become K/V ring stages (5 at head_dim 128, 7 at 64): r02, c4
// attention 1.78 -> 1.49 ms, c5 215 -> 187 us, c3 119 -> 109 us.
//
// O accumulates in TMEM across key tiles; a softmax thread rescales its O
// row (tcgen05.ld/st) only when its running max grows by more than 2^8
// (lazy rescaling), so the common tile costs one TMEM read of S and one
// TMEM write of P per row. With two query tiles the tensor core works on
// one tile while the softmax warps of the other run.
#include "sm100.cuh"

#include <mutex>
#include <unordered_map>

#include <cstdlib>
#include <algorithm>
#include <atomic>
#include <vector>

namespace eet {
namespace fa {
using namespace sm100;

constexpr int BQ = 128, BKV = 64, NSM = 8, THREADS = (NSM + 2) * 32;
constexpr int NST = 3;                     // K/V ring stages
constexpr float RESCALE_LOG2 = 8.0f;       // lazy rescale threshold (log2 units)

template <int HD> struct Cfg {
  static constexpr int KSUB = HD / 64;                  // 64-wide (128 B) K-atoms per row
  static constexpr int QSUB = BQ * 128;                 // 128 rows x 128 B
  static constexpr int KVSUB = BKV * 128;               //  64 rows x 128 B
  static constexpr int Q_BYTES = KSUB * QSUB;           // one query tile
  static constexpr int KV_BYTES = KSUB * KVSUB;         // one K (or V) tile
  static constexpr int P_BYTES = BQ * BKV * 2;          // 128 queries x 64 keys, one atom wide
  // P double-buffered per tile: softmax(j+1) writes while PV(j) reads
  static constexpr int SMEM = 2 * Q_BYTES + 2 * NST * KV_BYTES + 4 * P_BYTES + 1024 + 256;
  // P through TMEM: no P buffers in smem, the space goes to K/V stages
  static constexpr int NST_PT = (2 * NST * KV_BYTES + 4 * P_BYTES) / (2 * KV_BYTES);
  static constexpr int SMEM_PT = 2 * Q_BYTES + 2 * NST_PT * KV_BYTES + 1024 + 256;
  // TMEM columns: S_A | S_B | O_A | O_B
  // TMEM columns: S_A[2] | S_B[2] (double-buffered scores) | O_A | O_B
  static constexpr uint32_t S_COL = 0, O_COL = 4 * BKV;
};

// tcgen05.mma with the A operand (P, 128 lanes x 16 keys as 8 packed
// 32-bit columns) read from TMEM: the softmax writes P over the S buffer it
// has just consumed, so P never round-trips through shared memory
__device__ __forceinline__ void mma_f16_ta(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accum));
}

// V is read MN-major: 8-key row groups 1024 B apart (SBO), 64-wide hd blocks
// one sub-tile apart (LBO).
__device__ __forceinline__ uint64_t smem_desc_mn(uint32_t saddr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// tcgen05.ld 32 lanes x 32 columns without the trailing wait (caller waits)
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// exp2 on the MUFU pipe (16 / clk / SM)
__device__ __forceinline__ float ex2_mufu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// exp2 on the FMA/ALU pipes: 2^round(x) by exponent add, 2^f (|f| <= 0.5) by
// a cubic (max rel. error 7.7e-5, below half an fp16 ulp of P). Used for half
// of the keys of full tiles so MUFU and FMA share the softmax (the MUFU alone
// caps the tensor pipe near 50% at head_dim 128).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;                     // 1.5 * 2^23: round to integer
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.0550886838f, f, 0.242604051f), f, 0.693276242f), f, 0.99992894f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}

// packed f32x2 math (FFMA2 / FADD2) for the softmax of full tiles
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
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// 2^x for a pair on the FMA pipe (cubic on |f| <= 0.5, exponent by IMAD)
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t x2) {
  float a, b;
  f2unpack(x2, a, b);
  x2 = f2pack(fmaxf(a, -126.f), fmaxf(b, -126.f));
  const uint64_t magic = f2pack(12582912.f, 12582912.f), nmagic = f2pack(-12582912.f, -12582912.f);
  const uint64_t t = fadd2(x2, magic);                       // round to integer (low mantissa bits)
  const uint64_t r = fadd2(t, nmagic);
  const uint64_t f = ffma2(r, f2pack(-1.f, -1.f), x2);       // x - round(x)
  uint64_t p = ffma2(f2pack(0.0550886838f, 0.0550886838f), f, f2pack(0.242604051f, 0.242604051f));
  p = ffma2(p, f, f2pack(0.693276242f, 0.693276242f));
  p = ffma2(p, f, f2pack(0.99992894f, 0.99992894f));
  float t0, t1, p0, p1;
  f2unpack(t, t0, t1);
  f2unpack(p, p0, p1);
  // (bits(t) - bits(1.5 * 2^23)) << 23 == bits(t) << 23 (mod 2^32)
  return f2pack(__int_as_float(__float_as_int(t0) * (1 << 23) + __float_as_int(p0)),
                __int_as_float(__float_as_int(t1) * (1 << 23) + __float_as_int(p1)));
}

__device__ __forceinline__ uint32_t pack2(float a, float b, bool bf) {
  if (bf) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
  }
  __half2 v = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
      "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// tcgen05.st 32 lanes x 4 columns, no wait (the caller waits once)
__device__ __forceinline__ void tmem_st4_nowait(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(r[0]), "r"(r[1]),
               "r"(r[2]), "r"(r[3])
               : "memory");
}

struct FaArgs {
  const int* pads;          // [b]
  const int* q_rowbase;     // packed row of slot s = q_rowbase[b] + s
  void* o; int ldo;
  int batch, seq, heads, smax, causal;
  float scale_log2;         // (1/sqrt(hd)) * log2(e)
  int poly;                 // polynomial exp2 for half of the keys of full tiles
  int p_tmem;               // P through TMEM (over the spent S buffer) instead of smem
  int nitems;               // > 0: persistent CTAs walk the work list
  int* ctr;                 // [2] next list entry, CTAs done (zero between launches)
  const int* ends;          // [b] valid end per sequence (windows), nullptr: seq
};

// Work list: one entry per non-empty (sequence, head, query-tile pair),
// (sequence, head) groups longest sequence first, the pairs of a group
// heaviest first and adjacent so they share the group's K/V through L2.
// Padding-only pairs are never visited. Passed by value: no host->device
// copy to order against the stream, and the launch stays graph-capturable.
constexpr int MAX_ITEMS = 7680;                 // kernel parameter space is 32 KB
struct FaItems {
  uint32_t v[MAX_ITEMS];                        // b << 16 | head << 8 | pair
};

template <typename T, int HD, bool PT>
__global__ void __launch_bounds__(THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                   const __grid_constant__ CUtensorMap mapV, FaArgs a,
                   const __grid_constant__ FaItems items) {
  using C = Cfg<HD>;
  constexpr bool BF = std::is_same<T, __nv_bfloat16>::value;
  // Items: with a work list the CTAs are persistent and take list entries
  // from a global counter (greedy, in list order); without one, the CTA runs
  // the single (pair, head, b) of its block index.
  const int n_work = a.nitems;
  struct Item { int b, head, q0, pad, end, ntA, ntB; };
  auto decode = [&](int lin, Item& w) -> bool {
    int pair;
    if (n_work > 0) {
      if (lin >= n_work) return false;
      const uint32_t it = items.v[lin];
      w.b = (int)(it >> 16);
      w.head = (int)((it >> 8) & 255u);
      pair = (int)(it & 255u);
    } else {
      if (lin != 0) return false;
      w.b = blockIdx.z;
      w.head = blockIdx.y;
      pair = gridDim.x - 1 - blockIdx.x;                  // heaviest (latest) queries first
    }
    w.q0 = pair * 2 * BQ;
    w.pad = a.pads[w.b];
    w.end = a.ends ? a.ends[w.b] : a.seq;                 // valid slots [pad, end)
    const int qhiA = min(w.q0 + BQ, w.end), qhiB = min(w.q0 + 2 * BQ, w.end);
    if (qhiB <= w.pad || w.q0 >= w.end) return false;     // both tiles in the padding
    const bool liveA = qhiA > w.pad && w.q0 < w.end;
    const int kendA = a.causal ? qhiA : w.end, kendB = a.causal ? qhiB : w.end;
    w.ntA = liveA ? (kendA - w.pad + BKV - 1) / BKV : 0;
    w.ntB = (kendB - w.pad + BKV - 1) / BKV;              // B's range covers A's
    return true;
  };
  if (n_work == 0) {
    Item w0;
    if (!decode(0, w0)) return;
  }

  constexpr int NST = PT ? C::NST_PT : fa::NST;           // K/V ring stages
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* sQ = sm;                                       // [2] query tiles
  uint8_t* sK = sQ + 2 * C::Q_BYTES;                      // [NST] stages
  uint8_t* sV = sK + NST * C::KV_BYTES;                   // [NST] stages
  uint8_t* sP = sV + NST * C::KV_BYTES;                   // [2] tiles (smem-P instance only)
  uint64_t* bars = reinterpret_cast<uint64_t*>(PT ? sP : sP + 4 * C::P_BYTES);     // sP: [2 tiles][2 buffers]
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;              // [NST]
  uint64_t* kv_empty = bars + 1 + NST;       // [NST]
  uint64_t* s_full = bars + 1 + 2 * NST;     // [2 tiles][2 buffers]
  uint64_t* p_full = s_full + 4;             // [2 tiles][2 P buffers]: P(j) in buffer j & 1
  uint64_t* o_done = p_full + 4;             // [2 tiles][2 P buffers]: PV(j) on buffer j & 1
  uint64_t* q_empty = o_done + 4;
  uint64_t* it_full = o_done + 5;            // [2] item ring: producer -> MMA / softmax
  uint64_t* it_empty = o_done + 7;           // [2]
  int* item_buf = reinterpret_cast<int*>(o_done + 9);     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 10);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&it_full[i], 1);
      mbar_init(&it_empty[i], 1 + 2 * 4);                 // MMA thread + 8 softmax warps
    }
    for (int i = 0; i < NST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&s_full[i], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&p_full[2 * i], 128);
      mbar_init(&p_full[2 * i + 1], 128);
      mbar_init(&o_done[2 * i], 1);
      mbar_init(&o_done[2 * i + 1], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapQ) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapK) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapV) : "memory");
  }
  if (warp == NSM + 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Barrier phases run on across items: K/V stages on the global tile
  // counter g, S/P/O buffers on per-query-tile counters, Q on the round r
  // (q_empty: the previous item's S MMAs have finished reading sQ).
  if (warp == NSM) {
    if (lane == 0) {
      const uint64_t pol = 0x14F0000000000000ull;         // EVICT_LAST: K/V reused by query tiles
      int g = 0;
      for (int r = 0;; ++r) {
        if (r > 0) mbar_wait(q_empty, (r - 1) & 1);       // sQ free; fetch the next item late
        const int lin = n_work > 0 ? atomicAdd(a.ctr, 1) : (r == 0 ? 0 : 1);
        if (r >= 2) mbar_wait(&it_empty[r & 1], ((r - 2) >> 1) & 1);
        atomicExch(&item_buf[r & 1], lin);              // (mbarrier-ordered; atomic for racecheck)
        mbar_arrive(&it_full[r & 1]);
        Item w;
        if (!decode(lin, w)) break;
        mbar_expect_tx(q_full, 2 * C::Q_BYTES);
        for (int t = 0; t < 2; ++t)
          for (int s = 0; s < C::KSUB; ++s)
            tma_load_2d(sQ + t * C::Q_BYTES + s * C::QSUB, &mapQ, q_full, w.head * HD + 64 * s,
                        a.q_rowbase[w.b] + w.q0 + t * BQ, pol);
        // K/V maps are 3-D [b * heads][seq][hd]: the last tile's slots at or
        // past seq (never written by this pass) arrive as zeros, so masked
        // keys carry P = 0 against finite V (no 0 * NaN from stale cache)
        const int plane = w.b * a.heads + w.head;
        for (int j = 0; j < w.ntB; ++j, ++g) {
          const int st = g % NST;
          mbar_wait(&kv_empty[st], ((g / NST) & 1) ^ 1);
          mbar_expect_tx(&kv_full[st], 2 * C::KV_BYTES);
          const int slot = w.pad + j * BKV;
          for (int s = 0; s < C::KSUB; ++s) {
            tma_load_3d(sK + st * C::KV_BYTES + s * C::KVSUB, &mapK, &kv_full[st], 64 * s, slot, plane, pol);
            tma_load_3d(sV + st * C::KV_BYTES + s * C::KVSUB, &mapV, &kv_full[st], 64 * s, slot, plane, pol);
          }
        }
      }
    }
  } else if (warp == NSM + 1) {
    if (lane == 0) {
      constexpr uint32_t fmt = BF ? 1 : 0;
      constexpr uint32_t id_s = instr_desc(fmt, BQ, BKV);
      constexpr uint32_t id_o = instr_desc(fmt, BQ, HD) | (1u << 16);   // B (V) MN-major
      int g0 = 0, cA = 0, cB = 0;                         // item-start counters
      for (int r = 0;; ++r) {
        mbar_wait(&it_full[r & 1], (r >> 1) & 1);
        const int lin = atomicAdd(&item_buf[r & 1], 0);
        mbar_arrive(&it_empty[r & 1]);
        Item w;
        if (!decode(lin, w)) break;
        mbar_wait(q_full, r & 1);
        tc_fence_after();
        const int ntA = w.ntA, nt = w.ntB;
        // Ping-pong: while the softmax warps of one query tile work on S(j),
        // the tensor core runs the other tile's PV(j) and S(j+1); S_t(j+1) is
        // issued as soon as tile t's softmax has released S_t(j).
        auto issue_s = [&](int t, int j) {
          const int c = (t ? cB : cA) + j;
          const uint32_t k_base = smem_u32(sK + ((g0 + j) % NST) * C::KV_BYTES);
          const uint32_t q_base = smem_u32(sQ + t * C::Q_BYTES);
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            const uint32_t qoff = (k >> 2) * C::QSUB + (k & 3) * 32;
            const uint32_t koff = (k >> 2) * C::KVSUB + (k & 3) * 32;
            mma_f16(tmem + C::S_COL + (t * 2 + (c & 1)) * BKV, smem_desc(q_base + qoff),
                    smem_desc(k_base + koff), id_s, k > 0);
          }
          mma_commit(&s_full[t * 2 + (c & 1)]);
        };
        auto issue_o = [&](int t, int j) {
          const int c = (t ? cB : cA) + j;
          mbar_wait(&p_full[t * 2 + (c & 1)], (c >> 1) & 1);
          tc_fence_after();
          const uint32_t v_base = smem_u32(sV + ((g0 + j) % NST) * C::KV_BYTES);
          if (PT) {
            // P(j) sits in the first BKV/2 columns of S_t buffer (c & 1)
            const uint32_t p_tm = tmem + C::S_COL + (t * 2 + (c & 1)) * BKV;
#pragma unroll
            for (int k = 0; k < BKV / 16; ++k)
              mma_f16_ta(tmem + C::O_COL + t * HD, p_tm + k * 8, smem_desc_mn(v_base + k * 2048, C::KVSUB), id_o,
                         (j > 0) | k);
          } else {
            const uint32_t p_base = smem_u32(sP + (t * 2 + (c & 1)) * C::P_BYTES);
#pragma unroll
            for (int k = 0; k < BKV / 16; ++k)
              mma_f16(tmem + C::O_COL + t * HD, smem_desc(p_base + k * 32),
                      smem_desc_mn(v_base + k * 2048, C::KVSUB), id_o, (j > 0) | k);
          }
          mma_commit(&o_done[t * 2 + (c & 1)]);
        };
        int kv_seen = -1;
        auto wait_kv = [&](int j) {
          if (kv_seen >= j) return;
          const int g = g0 + j;
          mbar_wait(&kv_full[g % NST], (g / NST) & 1);
          tc_fence_after();
          kv_seen = j;
        };
        // S is double-buffered per tile: S_t(j+2) goes out as soon as the
        // softmax of tile t has released S_t(j) (its P(j) is in smem)
        for (int j = 0; j < 2 && j < nt; ++j) {
          wait_kv(j);
          if (j < ntA) issue_s(0, j);
          issue_s(1, j);
        }
        if (nt <= 2) mma_commit(q_empty);                 // last S of the item issued
        for (int j = 0; j < nt; ++j) {
          if (j < ntA) {
            issue_o(0, j);
            if (j + 2 < ntA) {
              wait_kv(j + 2);
              issue_s(0, j + 2);
            }
          }
          issue_o(1, j);
          if (j + 2 < nt) {
            wait_kv(j + 2);
            issue_s(1, j + 2);
            if (j + 3 == nt) mma_commit(q_empty);
          }
          mma_commit(&kv_empty[(g0 + j) % NST]);
        }
        g0 += nt;
        cA += ntA;
        cB += nt;
      }
    }
  } else {
    // ---- softmax warps: thread <-> query row of tile t
    const int t = warp >> 2;
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    const uint32_t s_base = tmem + lane_addr + C::S_COL + t * 2 * BKV;
    const uint32_t o_addr = tmem + lane_addr + C::O_COL + t * HD;
    uint8_t* prow0 = sP + (t * 2) * C::P_BYTES + row * 128;
    int cb = 0;                                           // this tile's counter at item start
    for (int r = 0;; ++r) {
    mbar_wait(&it_full[r & 1], (r >> 1) & 1);
    const int lin = atomicAdd(&item_buf[r & 1], 0);
    __syncwarp();
    if (lane == 0) mbar_arrive(&it_empty[r & 1]);
    Item w;
    if (!decode(lin, w)) break;
    const int pad = w.pad;
    const int qs = w.q0 + t * BQ + row;
    const int ntile = t == 0 ? w.ntA : w.ntB;
    const bool live = qs >= pad && qs < w.end;
    const int row_kend = live ? (a.causal ? qs + 1 : w.end) : pad;   // keys [pad, row_kend)
    float m = -INFINITY, l = 0.f;                         // m in log2 units (scaled)
    for (int j = 0; j < ntile; ++j) {
      const int c = cb + j;
      const int kt = pad + j * BKV;
      const int nvalid = min(max(row_kend - kt, 0), BKV);
      mbar_wait(&s_full[t * 2 + (c & 1)], (c >> 1) & 1);
      const uint32_t s_addr = s_base + (c & 1) * BKV;
      tc_fence_after();
      float sv[BKV];
      {
        uint32_t r[BKV];                                  // both halves in flight, one wait
        tmem_ld32_nowait(s_addr, r);
        tmem_ld32_nowait(s_addr + 32, r + 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // tie every loaded register to the wait so no use is hoisted above it
#pragma unroll
        for (int i = 0; i < BKV; ++i) asm volatile("" : "+r"(r[i]));
#pragma unroll
        for (int i = 0; i < BKV; ++i) sv[i] = __uint_as_float(r[i]);
      }
      // raw scores; masking only on tiles that cut a causal / pad bound
      const bool full = __all_sync(0xffffffffu, nvalid == BKV);
      float tmax = -INFINITY;
      if (full) {
        // four independent 3-input max chains (ILP), then combined
        float t4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < BKV; i += 8)
#pragma unroll
          for (int q = 0; q < 4; ++q) t4[q] = fmax3(t4[q], sv[i + 2 * q], sv[i + 2 * q + 1]);
        tmax = fmax3(fmaxf(t4[0], t4[1]), t4[2], t4[3]);
      } else {
#pragma unroll
        for (int i = 0; i < BKV; ++i) {
          sv[i] = (i < nvalid) ? sv[i] : -INFINITY;
          tmax = fmaxf(tmax, sv[i]);
        }
      }
      tmax *= a.scale_log2;                               // scale > 0: max commutes
      // P buffer j & 1 was last read by PV(j-2)
      uint8_t* prow = prow0 + (c & 1) * C::P_BYTES;
      // smem P: buffer c & 1 was last read by PV(c - 2). TMEM P overwrites
      // the S buffer just read; S(c + 2) into it is issued after PV(c)
      // (tcgen05 MMAs of one thread execute in order)
      if (!PT && c >= 2) mbar_wait(&o_done[t * 2 + (c & 1)], ((c - 2) >> 1) & 1);
      tc_fence_after();
      // tcgen05.ld/st are .sync.aligned: the O rescale is decided per warp
      // (any row whose max grew past the threshold rescales the whole warp;
      // rescaling a row that did not need it is exact up to rounding)
      const bool need = tmax > m + RESCALE_LOG2 || (m == -INFINITY && tmax != -INFINITY);
      if (__any_sync(0xffffffffu, need && m != -INFINITY)) {
        // the O rows must be final up to PV(j-1) before they are rescaled
        if (j >= 1) mbar_wait(&o_done[t * 2 + ((c - 1) & 1)], ((c - 1) >> 1) & 1);
        tc_fence_after();
        const float m_new = fmaxf(m, tmax);
        const float f = (m == -INFINITY) ? 1.f : exp2f(m - m_new);   // -inf row: O is still zero
        l *= f;
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(o_addr + c * 32, r);
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
          tmem_st32(o_addr + c * 32, r);
        }
        m = m_new;
      } else if (need) {
        m = tmax;                                         // first live tile of this row
      }
      const float msub = (m == -INFINITY) ? 0.f : m;
      const float sc = a.scale_log2;
      float rs = 0.f;
      if (full) {
        // p = 2^(s * scale_log2 - m) in f32x2 pairs; chunks 1, 4, 6 (3/8 of
        // the keys) take the FMA-pipe polynomial, the rest the MUFU: balances
        // the 16/clk MUFU against the issue slots (the MUFU alone caps the
        // tensor pipe near 50% at head_dim 128)
        const uint64_t sc2 = f2pack(sc, sc), nm2 = f2pack(-msub, -msub);
        uint64_t rs2v[4] = {f2pack(0.f, 0.f), f2pack(0.f, 0.f), f2pack(0.f, 0.f), f2pack(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < BKV / 8; ++c) {
          uint32_t pk[4];
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            const uint64_t x2 = ffma2(f2pack(sv[c * 8 + i], sv[c * 8 + i + 1]), sc2, nm2);
            uint64_t p2;
            if (a.poly && (c == 1 || c == 4 || c == 6)) {
              p2 = ex2_poly2(x2);
            } else {
              float x0, x1;
              f2unpack(x2, x0, x1);
              p2 = f2pack(ex2_mufu(x0), ex2_mufu(x1));
            }
            rs2v[i >> 1] = fadd2(rs2v[i >> 1], p2);
            float p0, p1;
            f2unpack(p2, p0, p1);
            pk[i >> 1] = pack2(p0, p1, BF);
          }
          if (PT) tmem_st4_nowait(s_addr + c * 4, pk);    // 8 keys = 4 packed columns
          else *reinterpret_cast<uint4*>(prow + ((c ^ (row & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
        const uint64_t rs2 = fadd2(fadd2(rs2v[0], rs2v[1]), fadd2(rs2v[2], rs2v[3]));
        float r0, r1;
        f2unpack(rs2, r0, r1);
        rs = r0 + r1;
      } else {
#pragma unroll
        for (int c = 0; c < BKV / 8; ++c) {                 // 8 keys -> one 16 B swizzled chunk
          uint32_t pk[4];
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            const float p0 = ex2_mufu(fmaf(sv[c * 8 + i], sc, -msub));
            const float p1 = ex2_mufu(fmaf(sv[c * 8 + i + 1], sc, -msub));
            rs += p0 + p1;
            pk[i >> 1] = pack2(p0, p1, BF);
          }
          if (PT) tmem_st4_nowait(s_addr + c * 4, pk);
          else *reinterpret_cast<uint4*>(prow + ((c ^ (row & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      }
      l += rs;
      if (PT) {
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");   // P over the spent S buffer
      } else {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // P -> tensor core
      }
      tc_fence_before();
      mbar_arrive(&p_full[t * 2 + (c & 1)]);
    }
    const int cl = cb + ntile - 1;
    if (ntile > 0) mbar_wait(&o_done[t * 2 + (cl & 1)], (cl >> 1) & 1);
    tc_fence_after();
    if (ntile > 0) {                                      // warp-uniform TMEM reads
      const float inv = l > 0.f ? 1.0f / l : 0.f;
      T* dst = reinterpret_cast<T*>(a.o) + ((long long)a.q_rowbase[w.b] + qs) * a.ldo + w.head * HD;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(o_addr + c * 32, r);
        if (live) {
#pragma unroll
          for (int d = 0; d < 32; d += 8) {
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[d + i]) * inv;
            store16<T>(dst + c * 32 + d, v);
          }
        }
      }
    }
    cb += ntile;
    }
  }
  __syncthreads();
  if (warp == NSM + 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if (n_work > 0 && threadIdx.x == 0) {
    // the last CTA out re-arms the counter for the next launch
    __threadfence();
    if (atomicAdd(a.ctr + 1, 1) == (int)gridDim.x - 1) {
      a.ctr[0] = 0;
      a.ctr[1] = 0;
      __threadfence();
    }
  }
}

template <typename T, int HD>
static void launch(const PrefillArgs& p, int T_rows, cudaStream_t st, double bytes, double flops) {
  using C = Cfg<HD>;
  const int h_ld = p.ldq;
  CUtensorMap mq = make_tma_map_2d(p.q, T_rows, h_ld, h_ld, BQ, p.dtype);
  // K/V window of plane (b, head): slots [0, seq) of its s_max rows
  CUtensorMap mk = make_tma_map_3d(p.k, p.batch * p.heads, p.seq, HD, p.k_sh, BKV, p.dtype);
  CUtensorMap mv = make_tma_map_3d(p.v, p.batch * p.heads, p.seq, HD, p.k_sh, BKV, p.dtype);
  FaArgs a;
  a.pads = p.pads;
  a.q_rowbase = p.q_rowbase;
  a.o = p.o;
  a.ldo = p.ldo;
  a.batch = p.batch;
  a.seq = p.seq;
  a.ends = p.ends;
  a.heads = p.heads;
  a.smax = (int)(p.k_sh / p.hd);
  a.causal = p.causal;
  a.scale_log2 = p.scale * 1.4426950408889634f;
  static const int poly = [] {            // A/B switch: EET_ATTN_POLY=0 -> MUFU only
    const char* e = std::getenv("EET_ATTN_POLY");
    return e ? atoi(e) : 1;
  }();
  a.poly = poly;
  static const int p_tmem = [] {          // A/B switch: EET_ATTN_PTMEM=0 -> P through smem
    const char* e = std::getenv("EET_ATTN_PTMEM");
    return e ? atoi(e) : 1;
  }();
  a.p_tmem = p_tmem;
  auto kern = a.p_tmem ? attn_tc_kernel<T, HD, true> : attn_tc_kernel<T, HD, false>;
  static const bool attr = [] {                      // thread-safe one-time init (both instances)
    EET_CHECK_CUDA(cudaFuncSetAttribute(attn_tc_kernel<T, HD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        C::SMEM_PT));
    EET_CHECK_CUDA(cudaFuncSetAttribute(attn_tc_kernel<T, HD, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        C::SMEM));
    return true;
  }();
  (void)attr;
  const int npair = (p.seq + 2 * BQ - 1) / (2 * BQ);
  thread_local FaItems items;         // copied into the launch parameters
  a.nitems = 0;
  a.ctr = nullptr;
  static const bool no_list = std::getenv("EET_ATTN_GRID") != nullptr;   // A/B switch
  if (p.h_pads && !no_list && npair <= 256 && p.heads <= 256 && p.batch <= 65536) {
    auto end_of = [&](int b) { return p.h_ends ? p.h_ends[b] : p.seq; };   // valid slots [pad, end)
    auto live_pair = [&](int b, int pr) {
      return pr * 2 * BQ < end_of(b) && std::min((pr + 1) * 2 * BQ, end_of(b)) > p.h_pads[b];
    };
    thread_local std::vector<int> order;
    order.resize(p.batch);
    for (int b = 0; b < p.batch; ++b) order[b] = b;
    std::stable_sort(order.begin(), order.end(),
                     [&](int x, int y) { return end_of(x) - p.h_pads[x] > end_of(y) - p.h_pads[y]; });
    long long n = 0;
    for (int b : order) {
      int pairs = 0;                                    // non-empty pairs
      for (int pr = npair - 1; pr >= 0; --pr)
        if (live_pair(b, pr)) ++pairs;
      n += (long long)pairs * p.heads;
    }
    if (n <= MAX_ITEMS) {
      // Greedy dynamic scheduling wants the light items last (short tail);
      // L2 wants the pairs of a (sequence, head) adjacent (shared K/V). So:
      // NB cost phases, heaviest first, locality order inside each phase.
      static const int nb_env = [] {
        const char* e = std::getenv("EET_ATTN_NB");
        return e ? atoi(e) : 4;
      }();
      int maxc = 1;
      auto cost = [&](int b, int pr) {
        const int pad = p.h_pads[b], q0 = pr * 2 * BQ, end = end_of(b);
        const int qhiA = std::min(q0 + BQ, end), qhiB = std::min(q0 + 2 * BQ, end);
        const bool liveA = qhiA > pad && q0 < end;
        const int kA = p.causal ? qhiA : end, kB = p.causal ? qhiB : end;
        return (liveA ? (kA - pad + BKV - 1) / BKV : 0) + (kB - pad + BKV - 1) / BKV;
      };
      for (int b = 0; b < p.batch; ++b)
        for (int pr = npair - 1; pr >= 0; --pr)
          if (live_pair(b, pr)) { maxc = std::max(maxc, cost(b, pr)); break; }
      thread_local std::vector<std::pair<int, uint32_t>> work;
      work.clear();
      for (int b : order)
        for (int h = 0; h < p.heads; ++h)
          for (int pr = npair - 1; pr >= 0; --pr)
            if (live_pair(b, pr)) {
              const int c = cost(b, pr);
              const int phase = nb_env > 0 ? (int)((long long)(maxc - c) * nb_env / (maxc + 1)) : maxc - c;
              work.emplace_back(phase, ((uint32_t)b << 16) | ((uint32_t)h << 8) | (uint32_t)pr);
            }
      std::stable_sort(work.begin(), work.end(),
                       [](const std::pair<int, uint32_t>& x, const std::pair<int, uint32_t>& y) {
                         return x.first < y.first;
                       });
      int k = 0;
      for (const auto& e : work) items.v[k++] = e.second;
      a.nitems = k;
      if (k == 0) return;
    }
  }
  if (a.nitems > 0) {
    // work counter: one pair per stream, zeroed on the launch stream before
    // every launch (stream order keeps launches on one stream apart; other
    // streams use their own pair)
    static std::mutex mu;
    static std::unordered_map<cudaStream_t, int*> per_stream;
    int* c = nullptr;
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = per_stream.find(st);
      if (it == per_stream.end()) {
        EET_CHECK_CUDA(cudaMalloc(&c, 2 * sizeof(int)));
        per_stream[st] = c;
      } else {
        c = it->second;
      }
    }
    EET_CHECK_CUDA(cudaMemsetAsync(c, 0, 2 * sizeof(int), st));
    a.ctr = c;
  }
  // list: persistent, one CTA per SM (the smem footprint allows one)
  dim3 grid = a.nitems > 0 ? dim3((unsigned)std::min(a.nitems, device_sm_count()), 1, 1)
                           : dim3(npair, p.heads, p.batch);
  ProfScope ps(K_ATTN_PREFILL, st, bytes, flops);
  kern<<<grid, THREADS, a.p_tmem ? C::SMEM_PT : C::SMEM, st>>>(mq, mk, mv, a, items);
  EET_LAUNCH_CHECK();
}

}  // namespace fa

// Tensor-core path applies to the packed-Q / cache-K/V layout of the layer
// (q_rowbase given, K/V in [b, heads, smax, hd]) with hd 64 or 128.
bool attn_prefill_tc(const PrefillArgs& p, int T_rows, cudaStream_t st, double bytes, double flops) {
  if (p.dtype == EET_F32 || !p.q_rowbase || p.zero_pad_rows) return false;
  if (!(p.hd == 64 || p.hd == 128)) return false;
  if (p.k_ss != p.hd || p.k_sh % p.hd != 0 || p.k_sb != p.heads * p.k_sh || p.ldq % 8 != 0) return false;
  if (p.dtype == EET_BF16) {
    p.hd == 64 ? fa::launch<__nv_bfloat16, 64>(p, T_rows, st, bytes, flops)
               : fa::launch<__nv_bfloat16, 128>(p, T_rows, st, bytes, flops);
  } else {
    p.hd == 64 ? fa::launch<__half, 64>(p, T_rows, st, bytes, flops)
               : fa::launch<__half, 128>(p, T_rows, st, bytes, flops);
  }
  return true;
}

}  // namespace eet
