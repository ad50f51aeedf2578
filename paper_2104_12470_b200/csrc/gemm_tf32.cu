// fp32-mode projections on the tensor cores: 3xTF32 on tcgen05
// (runtime.py:131,136,188,210,212 — the reference's float32 sgemm).
//
//   C[M, N] = A[M, K] * B[N, K]^T, A, B fp32 (B = weights, K-major)
//
// Every operand element is split in shared memory into a TF32 head and an
// fp32 tail, x = hi + lo with hi = cvt.rna.tf32(x), lo = x - hi (exact);
// the accumulator gets A_lo*B_hi + A_hi*B_lo + A_hi*B_hi (tcgen05.mma
// kind::tf32, fp32 accumulate in TMEM). Per product the dropped lo*lo term
// and the TF32 truncation of lo cost ~2^-21 relative, so the dot products
// carry about the error of an fp32 FFMA chain (plain TF32
// flips greedy tokens; this does not — fp32 goldens at 1e-5 and GPT-2-medium
// fp32 token identity are the tests).
//
// Warp roles (320 threads, one CTA per SM, persistent over (tile, k-split)):
//   warp 0      TMA producer: 128x32 fp32 A and 128x32 B boxes (128B rows,
//               128B swizzle) into a 3-stage ring
//   warp 1      TMEM allocator + MMA issuer (one lane): 3 x 4 MMAs of
//               M128 N128 K8 per 32-wide k-block
//   warps 2-5   epilogue: TMEM -> registers -> fused epilogue; with split
//               K, a partial tile in [col][row] order (coalesced stores),
//               summed over the splits in order 0..S-1 by a wide second
//               pass that runs the epilogue (deterministic)
//   warps 6-9   splitters: hi / lo of the landed stage, in place (the
//               swizzled layout is position-preserving), fence.proxy.async
// The c1 shapes (M = 205 tokens) have 12-48 output tiles, so K is split
// over ~one wave of CTAs.
#include "sm100.cuh"

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

namespace eet {
namespace t3 {
using namespace sm100;

constexpr int BM = 128, BN = 128, BK = 32, THREADS = 320, STAGES = 3;
constexpr int TILE_BYTES = BM * BK * 4;                 // 16 KB (A or B, BM == BN)
constexpr int STAGE_BYTES = 4 * TILE_BYTES;             // A_hi, B_hi (TMA), A_lo, B_lo
constexpr int TMEM_COLS = 2 * BN;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void split4(float4& v, float4& lo) {
  uint32_t h[4];
  const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h[i]) : "f"(x[i]));
  lo = make_float4(x[0] - __uint_as_float(h[0]), x[1] - __uint_as_float(h[1]), x[2] - __uint_as_float(h[2]),
                   x[3] - __uint_as_float(h[3]));
  v = make_float4(__uint_as_float(h[0]), __uint_as_float(h[1]), __uint_as_float(h[2]), __uint_as_float(h[3]));
}

struct Work {
  int num_m, num_n, splits, kb_per_split, nkb;
  int dev_mode;   // development A/B (EET_TF32_DEV): 0 normal, 1 no split (1xTF32), 2 split but 1 MMA
};

// second stage: every output element sums its S partials in split order
__global__ void __launch_bounds__(256) splitk_tiles_reduce_kernel(const float* __restrict__ part, int splits, int num_m,
                                                                  int num_n, int M, int N, Epi e) {
  const long long per_split = (long long)num_m * num_n * BM * BN;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < per_split; i += (long long)gridDim.x * 256) {
    const int tile = (int)(i / (BM * BN)), idx = (int)(i % (BM * BN));
    const int mb = tile % num_m, nb = tile / num_m;
    const int m = mb * BM + idx % BM, n = nb * BN + idx / BM;
    if (m >= M || n >= N) continue;
    float p8[8];
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2) p8[s2] = s2 < splits ? __ldcs(part + s2 * per_split + i) : 0.f;   // all in flight
    float v = 0.f;
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2) v += p8[s2];                                           // split order
    for (int s2 = 8; s2 < splits; ++s2) v += part[s2 * per_split + i];
    epi_apply<float>(e, m, n, v);
  }
}

__global__ void __launch_bounds__(THREADS, 1)
    gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int M,
                       int N, int K, Epi e, Work w, float* part) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // stage s: [A_hi | B_hi | A_lo | B_lo]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* conv = full + STAGES;
  uint64_t* empty = conv + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int items = w.num_m * w.num_n * w.splits;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&conv[i], 128);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // item -> (m tile, n tile, k split); k blocks [kb0, kb1)
  auto decode = [&](int it, int& mb, int& nb, int& sp, int& kb0, int& kb1) {
    sp = it % w.splits;
    const int t = it / w.splits;
    mb = t % w.num_m;
    nb = t / w.num_m;
    kb0 = sp * w.kb_per_split;
    kb1 = min(w.nkb, kb0 + w.kb_per_split);
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        int mb, nb, sp, kb0, kb1;
        decode(it, mb, nb, sp, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], 2 * TILE_BYTES);
          uint8_t* st = smem + stage * STAGE_BYTES;
          tma_load_2d(st, &mapA, &full[stage], kb * BK, mb * BM, 0x1000000000000000ull);
          tma_load_2d(st + TILE_BYTES, &mapB, &full[stage], kb * BK, nb * BN, 0x1000000000000000ull);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = instr_desc(2, BM, BN);          // A, B = TF32, D = F32
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int it = blockIdx.x; it < items; it += gridDim.x, ++local) {
        int mb, nb, sp, kb0, kb1;
        decode(it, mb, nb, sp, kb0, kb1);
        const int as = local & 1;
        mbar_wait(&tempty[as], ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&conv[stage], phase);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t ahi = st, bhi = st + TILE_BYTES, alo = st + 2 * TILE_BYTES, blo = st + 3 * TILE_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) {
            const uint32_t off = k * 32;                            // 8 tf32 = 32 bytes along K
            if (w.dev_mode == 0) {
              mma_tf32(d_tmem, smem_desc(alo + off), smem_desc(bhi + off), idesc, (kb > kb0) | k);
              mma_tf32(d_tmem, smem_desc(ahi + off), smem_desc(blo + off), idesc, 1);
            }
            mma_tf32(d_tmem, smem_desc(ahi + off), smem_desc(bhi + off), idesc, w.dev_mode ? ((kb > kb0) | k) : 1);
          }
          mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[as]);
      }
    }
  } else if (warp >= 6) {
    // splitters: 128 threads, 2 x 4096 floats per stage
    const int t = threadIdx.x - 192;
    int stage = 0;
    uint32_t phase = 0;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      int mb, nb, sp, kb0, kb1;
      decode(it, mb, nb, sp, kb0, kb1);
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        float4* hi = reinterpret_cast<float4*>(smem + stage * STAGE_BYTES);   // A_hi, B_hi
        float4* lo = reinterpret_cast<float4*>(smem + stage * STAGE_BYTES + 2 * TILE_BYTES);
#pragma unroll 4
        for (int i = t; i < (w.dev_mode == 1 ? 0 : 2 * TILE_BYTES / 16); i += 128) {
          float4 v = hi[i], l;
          split4(v, l);
          hi[i] = v;
          lo[i] = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> MMA
        mbar_arrive(&conv[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // epilogue warps 2-5: TMEM lane quadrant = warp % 4
    const int q = warp & 3;
    const int row = q * 32 + lane;
    int local = 0;
    for (int it = blockIdx.x; it < items; it += gridDim.x, ++local) {
      int mb, nb, sp, kb0, kb1;
      decode(it, mb, nb, sp, kb0, kb1);
      const int as = local & 1;
      mbar_wait(&tfull[as], (local >> 1) & 1);
      tc_fence_after();
      const int m = mb * BM + row;
      const int tile = it / w.splits;
      // split-K partial tile layout [col][row] (a warp's store = 32 consecutive rows: coalesced)
      float* ptile = part ? part + ((size_t)sp * w.num_m * w.num_n + tile) * (BM * BN) : nullptr;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + as * BN + c * 32, r);
        if (part) {
#pragma unroll
          for (int i = 0; i < 32; ++i) ptile[(c * 32 + i) * BM + row] = __uint_as_float(r[i]);
        } else if (m < M) {
          const int n0 = nb * BN + c * 32;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const int n = n0 + g * 8;
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[g * 8 + i]);
            if (n + 8 <= N) {
              epi_apply8<float>(e, m, n, v);
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (n + i < N) epi_apply<float>(e, m, n + i, v[i]);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[as]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

}  // namespace t3

bool gemm_tf32x3(const float* A, int lda, const float* B, int ldb, int M, int N, int K, const Epi& e,
                 cudaStream_t st) {
  using namespace t3;
  if (M <= 0 || N <= 0 || K <= 0) return true;
  if ((lda & 3) || (ldb & 3) || ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15))
    return false;
  const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN, nkb = (K + BK - 1) / BK;
  const int sms = device_sm_count();
  // split K so that (tiles x splits) fills about one wave, >= 4 k-blocks each
  int splits = std::max(1, std::min(sms / std::max(1, num_m * num_n), nkb / 4));
  const int kbps = (nkb + splits - 1) / splits;
  splits = (nkb + kbps - 1) / kbps;
  float* part = nullptr;
  if (splits > 1) {
    // per-stream workspace, grown outside graph capture (unsplit under capture if too small)
    static std::mutex mu;
    static std::unordered_map<cudaStream_t, std::pair<float*, size_t>> ws;
    const size_t need = sizeof(float) * (size_t)splits * num_m * num_n * BM * BN;
    std::lock_guard<std::mutex> lk(mu);
    auto& slot = ws[st];
    if (slot.second < need) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(st, &cs);
      if (cs != cudaStreamCaptureStatusNone) {
        splits = 1;
      } else {
        EET_CHECK_CUDA(cudaStreamSynchronize(st));
        if (slot.first) cudaFree(slot.first);
        EET_CHECK_CUDA(cudaMalloc(&slot.first, need));
        slot.second = need;
      }
    }
    if (splits > 1) part = slot.first;
  }
  static const int dev_mode = [] {               // development A/B: EET_TF32_DEV=1 (1xTF32) / 2
    const char* v = std::getenv("EET_TF32_DEV");
    return v ? atoi(v) : 0;
  }();
  const Work w{num_m, num_n, splits, splits > 1 ? kbps : nkb, nkb, dev_mode};
  const CUtensorMap ma = make_tma_map_2d_f32(A, M, K, lda, BM);
  const CUtensorMap mb = make_tma_map_2d_f32(B, N, K, ldb, BN);
  static const bool attr = [] {
    EET_CHECK_CUDA(cudaFuncSetAttribute(gemm_tf32x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    return true;
  }();
  (void)attr;
  const int items = num_m * num_n * splits;
  {
    ProfScope ps(K_GEMM_F32, st, gemm_bytes(M, N, K, 4, e), 2.0 * M * N * K);
    gemm_tf32x3_kernel<<<std::min(items, sms), THREADS, SMEM, st>>>(ma, mb, M, N, K, e, w, part);
    EET_LAUNCH_CHECK();
    if (part) {                             // the reduce pass is part of the GEMM's measured time
      const long long per_split = (long long)num_m * num_n * BM * BN;
      splitk_tiles_reduce_kernel<<<(int)std::min<long long>((per_split + 255) / 256, 4LL * sms), 256, 0, st>>>(
          part, splits, num_m, num_n, M, N, e);
      count_launch();
      EET_LAUNCH_CHECK();
    }
  }
  return true;
}

}  // namespace eet
