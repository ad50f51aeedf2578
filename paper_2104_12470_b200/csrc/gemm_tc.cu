// tcgen05 / TMEM / TMA tensor-core GEMM for sm_100a (bf16 / fp16 in, fp32
// accumulate) — the QKV, out-proj, FFN and LM-head projections of the
// 16-bit modes (runtime.py:131,136,188,210,212,344 in the reference).
//
//   C[M, N] = A[M, K] * B[N, K]^T      A: packed valid-token activations
//                                      B: weights, K-major ([out, in])
//
// Persistent, warp-specialised CTA (192 threads, one CTA per SM):
//   warp 0      TMA producer (one elected lane): 128x64 A and BNx64 B tiles,
//               128B-swizzled, into a STAGES-deep smem ring (full/empty
//               mbarriers).
//   warp 1      TMEM allocator + MMA issuer (one lane): tcgen05.mma
//               kind::f16 M=128 N=BN K=16, accumulating into one of two
//               TMEM accumulator stages; tcgen05.commit frees smem slots and
//               signals the epilogue.
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 -> registers -> fused
//               epilogue (bias, GELU, residual add, KV-cache scatter) ->
//               global. Double-buffered TMEM lets tile i's epilogue overlap
//               tile i+1's MMAs.
// Row tails and K tails are handled by TMA zero fill (OOB) + epilogue guards.
#include "sm100.cuh"

#include <cstdlib>

#include <cudaTypedefs.h>

#include <mutex>

namespace eet {

// ------------------------------------------------------------------ host
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  EET_REQUIRE(fn != nullptr, EET_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2-D K-major map: rows x K elements, row pitch ld elements, box 64 x box_rows.
CUtensorMap make_tma_map_2d(const void* ptr, int rows, int K, int ld, int box_rows, int dtype) {
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64u, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&map,
                           dtype == EET_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                           2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  EET_REQUIRE(r == CUDA_SUCCESS, EET_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return map;
}

// K-major 16-bit rows x K seen as [K/64 blocks][rows][64]: one box brings
// box_rows rows x box_kblocks swizzled 128-byte column blocks (the smem
// layout of that many box_rows x 64 2-D boxes stacked along K) in a single
// TMA instruction
CUtensorMap make_tma_map_kblk(const void* ptr, int rows, int K, int ld, int box_rows, int box_kblocks, int dtype) {
  CUtensorMap map;
  cuuint64_t dims[3] = {64u, (cuuint64_t)rows, (cuuint64_t)(K / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 2, 128u};
  cuuint32_t box[3] = {64u, (cuuint32_t)box_rows, (cuuint32_t)box_kblocks};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&map,
                           dtype == EET_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                           3, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  EET_REQUIRE(r == CUDA_SUCCESS, EET_ERR_CUDA, "cuTensorMapEncodeTiled (k-blocks) failed");
  return map;
}

// fp32 K-major map: box 32 x box_rows (128-byte rows, 128B swizzle)
CUtensorMap make_tma_map_2d_f32(const void* ptr, int rows, int K, int ld, int box_rows) {
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32u, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  EET_REQUIRE(r == CUDA_SUCCESS, EET_ERR_CUDA, "cuTensorMapEncodeTiled (fp32) failed");
  return map;
}

// 3-D map over [planes][rows][K] with a plane pitch of plane_ld elements: a
// box that runs past `rows` inside a plane is zero-filled instead of reading
// the plane's tail (or the next plane).
CUtensorMap make_tma_map_3d(const void* ptr, int planes, int rows, int K, long long plane_ld,
                            int box_rows, int dtype) {
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)K * 2, (cuuint64_t)plane_ld * 2};
  cuuint32_t box[3] = {64u, (cuuint32_t)box_rows, 1u};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&map,
                           dtype == EET_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                           3, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  EET_REQUIRE(r == CUDA_SUCCESS, EET_ERR_CUDA, "cuTensorMapEncodeTiled (3-D) failed");
  return map;
}

int device_sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    EET_CHECK_CUDA(cudaGetDevice(&dev));
    EET_CHECK_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

namespace tc {
using namespace sm100;

constexpr int BM = 128, BK = 64, THREADS = 192;
constexpr int A_BYTES = BM * BK * 2;

template <int BN> struct Cfg {
  static constexpr int STAGES = BN >= 256 ? 4 : 6;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;                 // two accumulator stages
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

// Grouped raster: tiles run in panels of GM M-tiles; inside a panel the
// N-tiles advance slowest, so the ~148 concurrently running CTAs share one
// A panel (GM*128 rows, kept in L2) and a few B column blocks. The plain
// M-fastest order re-streamed all of A from HBM for every N-tile (c4 QKV:
// 13.3 GB of DRAM reads per launch for 1.2 GB of operands).
// GM is chosen on the host so that the A panel fits well inside L2.
__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int GM, int& mb, int& nb) {
  const int panel = GM * num_n;
  const int p = tile / panel;
  const int m0 = p * GM;
  const int gm = min(GM, num_m - m0);
  const int r = tile - p * panel;
  nb = r / gm;
  mb = m0 + r % gm;
}

struct L2Plan {
  int gm;                  // M-tiles per raster group
  int resid_pipe;          // pipelined residual epilogue (A/B: EET_GEMM_RESID_PIPE=0)
  uint64_t pol_a, pol_b;   // L2 cache policies of the A / B TMA loads
};

template <typename T, int BN>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA,
                   const __grid_constant__ CUtensorMap mapB, int M, int N, int K, Epi e, L2Plan L) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
  const int tiles = num_m * num_n;
  const int nk = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
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
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // the A panel is re-read by every N-tile of its group (kept in L2);
      // a B block is re-read only by the group's M-tiles running next to it
      const uint64_t pol_first = L.pol_a;
      const uint64_t pol_last = L.pol_b;
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        int mb, nb;
        tile_coords(tile, num_m, num_n, L.gm, mb, nb);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          tma_load_2d(sA + stage * A_BYTES, &mapA, &full[stage], kb * BK, mb * BM, pol_first);
          tma_load_2d(sB + stage * C::B_BYTES, &mapB, &full[stage], kb * BK, nb * BN, pol_last);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = instr_desc(std::is_same<T, __nv_bfloat16>::value ? 1 : 0, BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
        const int as = local & 1;
        const uint32_t aphase = (local >> 1) & 1;
        mbar_wait(&tempty[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_f16(d_tmem, smem_desc(a0 + k * 32), smem_desc(b0 + k * 32), idesc,
                    (kb | k) != 0);
          mma_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[as]);
      }
    }
  } else {
    const int q = warp & 3;                 // TMEM lane quadrant of this warp
    const int row = q * 32 + lane;
    int local = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
      int mb, nb;
      tile_coords(tile, num_m, num_n, L.gm, mb, nb);
      const int as = local & 1;
      const uint32_t aphase = (local >> 1) & 1;
      const int m = mb * BM + row;
      // Residual epilogue (out-proj / W2): the fp32 row segment x[m, nb*BN ..
      // +BN) is read-modify-written. Its loads are issued two 32-column
      // chunks ahead (the first two before the accumulator is ready), so
      // the row's DRAM latency is paid ~once per tile instead of once per
      // 8 columns (c4 out-proj, K = 4096: the per-chunk load stalls made
      // the epilogue longer than the tile's MMA).
      float* xrow = nullptr;
      if (e.mode == EPI_RESID && m < M && nb * BN + BN <= N) {
        const int2 rr = e.rinfo[m];
        xrow = e.x + rr.x * e.x_sb + rr.y * e.x_ss + nb * BN;
        if ((reinterpret_cast<uintptr_t>(xrow) | reinterpret_cast<uintptr_t>(e.bias)) & 15) xrow = nullptr;
      }
      // tcgen05.ld is warp-collective: the whole warp takes one path
      if (__all_sync(0xffffffffu, xrow != nullptr) && L.resid_pipe) {
        constexpr int NCH = BN / 32;
        float4 xv[NCH][8];
#pragma unroll
        for (int c = 0; c < 2 && c < NCH; ++c)
#pragma unroll
          for (int j = 0; j < 8; ++j) xv[c][j] = *reinterpret_cast<const float4*>(xrow + c * 32 + j * 4);
        mbar_wait(&tfull[as], aphase);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          if (c + 2 < NCH) {
#pragma unroll
            for (int j = 0; j < 8; ++j) xv[c + 2][j] = *reinterpret_cast<const float4*>(xrow + (c + 2) * 32 + j * 4);
          }
          uint32_t r[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + as * BN + c * 32, r);
          const int n0 = nb * BN + c * 32;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 a = xv[c][j];
            float b0 = 0.f, b1 = 0.f, b2 = 0.f, b3 = 0.f;
            if (e.bias) {
              const float4 bb = *reinterpret_cast<const float4*>(e.bias + n0 + j * 4);
              b0 = bb.x; b1 = bb.y; b2 = bb.z; b3 = bb.w;
            }
            a.x += __uint_as_float(r[j * 4 + 0]) + b0;
            a.y += __uint_as_float(r[j * 4 + 1]) + b1;
            a.z += __uint_as_float(r[j * 4 + 2]) + b2;
            a.w += __uint_as_float(r[j * 4 + 3]) + b3;
            *reinterpret_cast<float4*>(xrow + c * 32 + j * 4) = a;
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[as]);
        continue;
      }
      mbar_wait(&tfull[as], aphase);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + as * BN + c * 32, r);
        if (m < M) {
          const int n0 = nb * BN + c * 32;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const int n = n0 + g * 8;
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[g * 8 + i]);
            if (n + 8 <= N) {
              epi_apply8<T>(e, m, n, v);
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (n + i < N) epi_apply<T>(e, m, n + i, v[i]);
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
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(C::TMEM_COLS));
  }
}

template <typename T, int BN>
static void launch(const void* A, int lda, const void* B, int ldb, int M, int N, int K,
                   const Epi& e, int dtype, cudaStream_t st) {
  using C = Cfg<BN>;
  CUtensorMap ma = make_tma_map_2d(A, M, K, lda, BM, dtype);
  CUtensorMap mb = make_tma_map_2d(B, N, K, ldb, BN, dtype);
  auto kern = gemm_tc_kernel<T, BN>;
  static const bool attr_set = [&] {                 // thread-safe one-time init
    EET_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    return true;
  }();
  (void)attr_set;
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = std::min(tiles, device_sm_count());
  // A panel of GM M-tiles <= ~40 MB (a third of L2), GM in [4, 32]
  // (panel budget sweep, tools/gpu_gemm_panel.sh: 20-96 MB within 1% on c3/c4)
  static const int mode = [] {
    const char* v = std::getenv("EET_GEMM_L2");
    return v ? atoi(v) : 1;
  }();
  constexpr uint64_t EVICT_NORMAL = 0x1000000000000000ull, EVICT_FIRST = 0x12F0000000000000ull,
                     EVICT_LAST = 0x14F0000000000000ull;
  L2Plan L;
  const long long panel_row_bytes = (long long)BM * K * 2;
  static const long long panel_mb_env = [] {
    const char* v = std::getenv("EET_GEMM_PANEL_MB");
    return v ? atoll(v) : 0LL;
  }();
  // K >= 8192 (c4 W2, K = 16384: a 4 MB A row-panel per M tile): a 40 MB
  // group is 10 M tiles and B (128 MB) streams once per group; 88 MB keeps
  // 22 M tiles resident (B streamed 12x instead of 26x; time within 1% over
  // 20-96 MB at K <= 4096)
  const long long panel_mb = panel_mb_env ? panel_mb_env : (K >= 8192 ? 88LL : 40LL);
  L.gm = (int)std::max(4LL, std::min(32LL, (panel_mb << 20) / std::max(1LL, panel_row_bytes)));
  // all of A within ~96 MB: one group, B streamed exactly once (c5: -4%)
  const int num_m = (M + BM - 1) / BM;
  if (num_m <= 32 && (long long)num_m * panel_row_bytes <= (96LL << 20)) L.gm = num_m;
  L.pol_a = EVICT_LAST;
  L.pol_b = EVICT_NORMAL;
  static const int resid_pipe = [] {
    const char* v = std::getenv("EET_GEMM_RESID_PIPE");
    return v ? atoi(v) : 1;
  }();
  L.resid_pipe = resid_pipe;
  if (mode == 0) {                       // previous plan: GM 32, A evict-first, B evict-last
    L.gm = 32;
    L.pol_a = EVICT_FIRST;
    L.pol_b = EVICT_LAST;
  } else if (mode == 2) {
    L.pol_a = EVICT_NORMAL;
  }
  ProfScope ps(K_GEMM_TC, st, gemm_bytes(M, N, K, 2, e), 2.0 * M * N * K);
  kern<<<grid, THREADS, C::SMEM, st>>>(ma, mb, M, N, K, e, L);
  EET_LAUNCH_CHECK();
}

}  // namespace tc

void gemm_tc_sm100(int dtype, const void* A, int lda, const void* B, int ldb, int M, int N,
                   int K, const Epi& e, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  EET_REQUIRE(dtype == EET_BF16 || dtype == EET_F16, EET_ERR_ARG, "tcgen05 GEMM needs bf16/fp16");
  const bool wide = N >= 256;
  if (dtype == EET_BF16) {
    wide ? tc::launch<__nv_bfloat16, 256>(A, lda, B, ldb, M, N, K, e, dtype, st)
         : tc::launch<__nv_bfloat16, 128>(A, lda, B, ldb, M, N, K, e, dtype, st);
  } else {
    wide ? tc::launch<__half, 256>(A, lda, B, ldb, M, N, K, e, dtype, st)
         : tc::launch<__half, 128>(A, lda, B, ldb, M, N, K, e, dtype, st);
  }
}

}  // namespace eet
