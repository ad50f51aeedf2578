// Context-phase (prompt) mask-fused attention on tcgen05 for 16-bit modes,
// head_dim 64 / 128 (§2.1 Algorithm 1; attention.py:73-104 +
// runtime.py:164-178 in the reference).
//
// One CTA = one (sequence b, head, 128-query tile). Causal and padding
// bounds come from slot indices: key tiles start at the sequence's pad
// offset and stop at the tile's last query, so pad keys are never loaded and
// query tiles that lie wholly in the padding exit immediately.
//
//   warp 0      TMA producer: Q tile once, then K/V tiles (128 keys) into a
//               two-stage ring, straight from the [b, heads, s_max, hd] cache.
//   warp 1      TMEM allocator + MMA issuer: S_j = Q K_j^T (M=128, N=128,
//               K-major both) into one of two TMEM score buffers, then
//               O_j = P_j V_j (M=128, N=hd; P K-major from smem, V MN-major).
//   warps 2..5  softmax: thread = query row; reads its S row from TMEM,
//               applies the index-derived mask, online max/sum in fp32,
//               writes P (16-bit, 128B-swizzled) to smem, then folds O_j into
//               a register accumulator with the running correction.
// The score matrix never reaches HBM; S_{j+1} overlaps the softmax of S_j.
#include "sm100.cuh"

namespace eet {
namespace fa {
using namespace sm100;

constexpr int BQ = 128, BKV = 128, THREADS = 192;

template <int HD> struct Cfg {
  static constexpr int KSUB = HD / 64;                  // 64-wide (128 B) K-atoms per row
  static constexpr int SUB = 128 * 128;                 // one 128-row x 128 B sub-tile
  static constexpr int Q_BYTES = KSUB * SUB;
  static constexpr int KV_BYTES = KSUB * SUB;           // K tile (V tile same size)
  static constexpr int P_BYTES = 2 * SUB;               // 128 queries x 128 keys
  static constexpr int SMEM = Q_BYTES + 4 * KV_BYTES + P_BYTES + 1024 + 256;
  static constexpr uint32_t S_COL = 0, O_COL = 256;     // TMEM: S0 | S1 | O
};

// K-major SW128 descriptor is sm100::smem_desc; V is read MN-major:
// 8-key row groups 1024 B apart (SBO), 64-wide hd blocks one sub-tile apart (LBO).
__device__ __forceinline__ uint64_t smem_desc_mn(uint32_t saddr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint32_t pack2(float a, float b, bool bf) {
  if (bf) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
  }
  __half2 v = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

struct FaArgs {
  const int* pads;          // [b]
  const int* q_rowbase;     // packed row of slot s = q_rowbase[b] + s
  void* o; int ldo;
  int batch, seq, heads, smax, causal;
  float scale_log2;         // (1/sqrt(hd)) * log2(e)
  float scale;              // 1/sqrt(hd)
};

template <typename T, int HD>
__global__ void __launch_bounds__(THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                   const __grid_constant__ CUtensorMap mapV, FaArgs a) {
  using C = Cfg<HD>;
  constexpr bool BF = std::is_same<T, __nv_bfloat16>::value;
  const int b = blockIdx.z, head = blockIdx.y;
  const int n_qt = gridDim.x;
  const int qt = n_qt - 1 - blockIdx.x;                  // heaviest (latest) tiles first
  const int q0 = qt * BQ;
  const int pad = a.pads[b];
  const int qhi = min(q0 + BQ, a.seq);
  if (qhi <= pad) return;                                 // tile wholly in the padding
  const int kend = a.causal ? qhi : a.seq;                // keys [pad, kend)
  const int nt = (kend - pad + BKV - 1) / BKV;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* sQ = sm;
  uint8_t* sK = sQ + C::Q_BYTES;                          // [2] stages
  uint8_t* sV = sK + 2 * C::KV_BYTES;                     // [2] stages
  uint8_t* sP = sV + 2 * C::KV_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + C::P_BYTES);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;      // [2]
  uint64_t* kv_empty = bars + 3;     // [2]
  uint64_t* s_full = bars + 5;       // [2]
  uint64_t* p_full = bars + 7;
  uint64_t* o_full = bars + 8;
  uint64_t* o_empty = bars + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
    }
    mbar_init(p_full, 128);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapQ) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapK) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapV) : "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int kv_row0 = (b * a.heads + head) * a.smax;      // cache row of slot 0

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = 0x14F0000000000000ull;         // EVICT_LAST: K/V reused by q tiles
      mbar_expect_tx(q_full, C::Q_BYTES);
      for (int s = 0; s < C::KSUB; ++s)
        tma_load_2d(sQ + s * C::SUB, &mapQ, q_full, head * HD + 64 * s, a.q_rowbase[b] + q0, pol);
      for (int j = 0; j < nt; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], 2 * C::KV_BYTES);
        const int row = kv_row0 + pad + j * BKV;
        for (int s = 0; s < C::KSUB; ++s) {
          tma_load_2d(sK + st * C::KV_BYTES + s * C::SUB, &mapK, &kv_full[st], 64 * s, row, pol);
          tma_load_2d(sV + st * C::KV_BYTES + s * C::SUB, &mapV, &kv_full[st], 64 * s, row, pol);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t fmt = BF ? 1 : 0;
      constexpr uint32_t id_s = instr_desc(fmt, BQ, BKV);
      constexpr uint32_t id_o = instr_desc(fmt, BQ, HD) | (1u << 16);   // B (V) MN-major
      const uint32_t q_base = smem_u32(sQ), p_base = smem_u32(sP);
      auto issue_s = [&](int j) {
        const int st = j & 1;
        const uint32_t k_base = smem_u32(sK + st * C::KV_BYTES);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k >> 2) * C::SUB + (k & 3) * 32;
          mma_f16(tmem + C::S_COL + st * 128, smem_desc(q_base + off), smem_desc(k_base + off), id_s,
                  k > 0);
        }
        mma_commit(&s_full[st]);
      };
      mbar_wait(q_full, 0);
      mbar_wait(&kv_full[0], 0);
      tc_fence_after();
      issue_s(0);
      for (int j = 0; j < nt; ++j) {
        if (j + 1 < nt) {
          mbar_wait(&kv_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
          tc_fence_after();
          issue_s(j + 1);
        }
        mbar_wait(p_full, j & 1);
        mbar_wait(o_empty, (j & 1) ^ 1);
        tc_fence_after();
        const uint32_t v_base = smem_u32(sV + (j & 1) * C::KV_BYTES);
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k) {
          const uint32_t poff = (k >> 2) * C::SUB + (k & 3) * 32;
          mma_f16(tmem + C::O_COL, smem_desc(p_base + poff), smem_desc_mn(v_base + k * 2048, C::SUB),
                  id_o, k > 0);
        }
        mma_commit(o_full);
        mma_commit(&kv_empty[j & 1]);
      }
    }
  } else {
    // ---- softmax warps: thread <-> query row
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const int qs = q0 + row;
    const bool live = qs >= pad && qs < a.seq;
    const int row_kend = live ? (a.causal ? qs + 1 : a.seq) : pad;   // keys [pad, row_kend)
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    float m = -INFINITY, l = 0.f;
    float o[HD];
#pragma unroll
    for (int d = 0; d < HD; ++d) o[d] = 0.f;
    uint8_t* prow = sP + row * 128;
    for (int j = 0; j < nt; ++j) {
      const int kt = pad + j * BKV;
      const int nvalid = min(max(row_kend - kt, 0), BKV);      // keys [kt, kt+nvalid) count
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t s_addr = tmem + lane_addr + C::S_COL + (j & 1) * 128;
      float tmax = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32(s_addr + c * 32, r);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c * 32 + i < nvalid) tmax = fmaxf(tmax, __uint_as_float(r[i]) * a.scale);
      }
      const float m_new = fmaxf(m, tmax);
      const float corr = (m == -INFINITY) ? (m_new == -INFINITY ? 1.f : 0.f)
                                          : exp2f((m - m_new) * 1.4426950408889634f);
      const float msub = (m_new == -INFINITY) ? 0.f : m_new * 1.4426950408889634f;
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32(s_addr + c * 32, r);
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float p0 = (c * 32 + i < nvalid) ? exp2f(__uint_as_float(r[i]) * a.scale_log2 - msub) : 0.f;
          float p1 = (c * 32 + i + 1 < nvalid) ? exp2f(__uint_as_float(r[i + 1]) * a.scale_log2 - msub) : 0.f;
          rs += p0 + p1;
          pk[i >> 1] = pack2(p0, p1, BF);
        }
        // keys c*32 .. c*32+31 -> sub-tile c/2, 16B chunks (c%2)*4 .. +3, 128B-swizzled
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int chunk = (c & 1) * 4 + q;
          uint8_t* dst = prow + (c >> 1) * C::SUB + ((chunk ^ (row & 7)) << 4);
          *reinterpret_cast<uint4*>(dst) = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
      }
      l = l * corr + rs;
      m = m_new;
      fence_async_smem();                    // P writes -> visible to the tensor core
      tc_fence_before();
      mbar_arrive(p_full);
      mbar_wait(o_full, j & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_addr + C::O_COL + c * 32, r);
#pragma unroll
        for (int i = 0; i < 32; ++i) o[c * 32 + i] = o[c * 32 + i] * corr + __uint_as_float(r[i]);
      }
      tc_fence_before();
      mbar_arrive(o_empty);
    }
    if (live) {
      const float inv = l > 0.f ? 1.0f / l : 0.f;
      T* dst = reinterpret_cast<T*>(a.o) + ((long long)a.q_rowbase[b] + qs) * a.ldo + head * HD;
#pragma unroll
      for (int d = 0; d < HD; d += 8) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = o[d + i] * inv;
        store16<T>(dst + d, v);
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <typename T, int HD>
static void launch(const PrefillArgs& p, int T_rows, cudaStream_t st, double bytes, double flops) {
  using C = Cfg<HD>;
  const int h_ld = p.ldq;
  CUtensorMap mq = make_tma_map_2d(p.q, T_rows, h_ld, h_ld, BQ, p.dtype);
  const int kv_rows = p.batch * p.heads * (int)(p.k_sh / p.hd);        // b * heads * smax
  CUtensorMap mk = make_tma_map_2d(p.k, kv_rows, HD, HD, BKV, p.dtype);
  CUtensorMap mv = make_tma_map_2d(p.v, kv_rows, HD, HD, BKV, p.dtype);
  FaArgs a;
  a.pads = p.pads;
  a.q_rowbase = p.q_rowbase;
  a.o = p.o;
  a.ldo = p.ldo;
  a.batch = p.batch;
  a.seq = p.seq;
  a.heads = p.heads;
  a.smax = (int)(p.k_sh / p.hd);
  a.causal = p.causal;
  a.scale = p.scale;
  a.scale_log2 = p.scale * 1.4426950408889634f;
  auto kern = attn_tc_kernel<T, HD>;
  static bool attr = false;
  if (!attr) {
    EET_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  dim3 grid((p.seq + BQ - 1) / BQ, p.heads, p.batch);
  ProfScope ps(K_ATTN_PREFILL, st, bytes, flops);
  kern<<<grid, THREADS, C::SMEM, st>>>(mq, mk, mv, a);
  EET_LAUNCH_CHECK();
}

}  // namespace fa

// Tensor-core path applies to the packed-Q / cache-K/V layout of the layer
// (q_rowbase given, K/V in [b, heads, smax, hd]) with hd 64 or 128.
bool attn_prefill_tc(const PrefillArgs& p, int T_rows, cudaStream_t st, double bytes, double flops) {
  if (p.dtype == EET_F32 || !p.q_rowbase || p.zero_pad_rows) return false;
  if (!(p.hd == 64 || p.hd == 128)) return false;
  if (p.k_ss != p.hd || p.k_sh % p.hd != 0 || p.ldq % 8 != 0) return false;
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
