// Decode-step projections on tcgen05 ("swap-AB" split-K GEMV), 16-bit modes.
//
// In the incremental phase every projection has M = batch <= 32 token rows
// against a weight matrix of 1-50k output features, so it is bound by the
// weight read from HBM (runtime.py:155-188 / 204-213, one token per
// sequence). The weight tile takes the 128-row MMA operand and the token rows
// the narrow N = 16/32 operand:
//
//   D[n (128 weight rows), m (token)] += W[n, k:k+64] . X[m, k:k+64]^T
//
// Each CTA (128 threads) streams a K-range of one 128-row weight block
// through a TMA ring (16 KB W + 2-4 KB X per 64-wide k-block), one lane
// issues tcgen05.mma kind::f16 M=128 N=MN into TMEM, and all four warps read
// the accumulator back (TMEM lane = weight row). K is split across CTAs to
// put ~2 CTAs on every SM; partial sums go to a workspace and the last CTA of
// each row block adds them in split order (deterministic) and runs the fused
// epilogue (bias / GELU / residual / KV-cache scatter / logits).
#include "sm100.cuh"

namespace eet {
namespace gv {
using namespace sm100;

constexpr int ROWS = 128, BK = 64, THREADS = 128, STAGES = 4;
constexpr int W_BYTES = ROWS * BK * 2;

template <int MN> struct Cfg {
  static constexpr int X_BYTES = MN * BK * 2;               // 2 KB (16) / 4 KB (32)
  static constexpr int SMEM = STAGES * (W_BYTES + X_BYTES) + 1024 + 128;
};

template <typename T, int MN>
__global__ void __launch_bounds__(THREADS) gemv_tc_kernel(
    const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapX, int M,
    int N, int K, int kb_per_split, int splits, float* __restrict__ ws, int* __restrict__ counters,
    Epi e) {
  using C = Cfg<MN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sW = smem;                                   // STAGES x 16 KB (1024-aligned)
  uint8_t* sX = smem + STAGES * W_BYTES;                // STAGES x X_BYTES
  uint64_t* full = reinterpret_cast<uint64_t*>(sX + STAGES * C::X_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = blockIdx.x, split = blockIdx.y;
  const int nkb = (K + BK - 1) / BK;
  const int kb0 = split * kb_per_split;
  const int kb1 = min(nkb, kb0 + kb_per_split);

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapW) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapX) : "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // weights are read exactly once per step: stream them past L2
    const uint64_t pol_w = 0x12F0000000000000ull;   // EVICT_FIRST
    const uint64_t pol_x = 0x14F0000000000000ull;   // EVICT_LAST (re-read by every CTA)
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&empty[stage], phase ^ 1);
      mbar_expect_tx(&full[stage], W_BYTES + C::X_BYTES);
      tma_load_2d(sW + stage * W_BYTES, &mapW, &full[stage], kb * BK, rb * ROWS, pol_w);
      tma_load_2d(sX + stage * C::X_BYTES, &mapX, &full[stage], kb * BK, 0, pol_x);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = instr_desc(std::is_same<T, __nv_bfloat16>::value ? 1 : 0, ROWS, MN);
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      const uint32_t w0 = smem_u32(sW + stage * W_BYTES);
      const uint32_t x0 = smem_u32(sX + stage * C::X_BYTES);
#pragma unroll
      for (int k = 0; k < BK / 16; ++k)
        mma_f16(tmem, smem_desc(w0 + k * 32), smem_desc(x0 + k * 32), idesc, (kb > kb0) | k);
      mma_commit(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    mma_commit(done);
  }
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();

  // accumulator row = this thread's weight row; columns = token rows
  const int row = warp * 32 + lane;
  const int n = rb * ROWS + row;
  float acc[MN];
  {
    uint32_t r[MN];
    if constexpr (MN == 16) tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), r);
    else tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), r);
#pragma unroll
    for (int m = 0; m < MN; ++m) acc[m] = __uint_as_float(r[m]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 32);

  if (splits == 1) {
    if (n < N)
#pragma unroll
      for (int m = 0; m < MN; ++m)
        if (m < M) epi_apply<T>(e, m, n, acc[m]);
    return;
  }
  // publish this split's partial tile, then the last split reduces in order
  float* mine = ws + (((size_t)rb * splits + split) * ROWS + row) * MN;
#pragma unroll
  for (int m = 0; m < MN; m += 4)
    __stcg(reinterpret_cast<float4*>(mine + m), make_float4(acc[m], acc[m + 1], acc[m + 2], acc[m + 3]));
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(&counters[rb], 1) == splits - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
#pragma unroll
  for (int m = 0; m < MN; ++m) acc[m] = 0.f;
  for (int s = 0; s < splits; ++s) {
    const float* src = ws + (((size_t)rb * splits + s) * ROWS + row) * MN;
#pragma unroll
    for (int m = 0; m < MN; m += 4) {
      float4 v = __ldcg(reinterpret_cast<const float4*>(src + m));
      acc[m] += v.x; acc[m + 1] += v.y; acc[m + 2] += v.z; acc[m + 3] += v.w;
    }
  }
  if (n < N)
#pragma unroll
    for (int m = 0; m < MN; ++m)
      if (m < M) epi_apply<T>(e, m, n, acc[m]);
  if (threadIdx.x == 0) counters[rb] = 0;
}

// Grow-only split-K scratch (allocated outside graph capture: the eager
// warm-up step of every shape reaches here before any capture does).
static float* g_ws = nullptr;
static size_t g_ws_bytes = 0;
static int* g_cnt = nullptr;
static size_t g_cnt_n = 0;

static void ensure_scratch(size_t ws_bytes, size_t counters) {
  if (ws_bytes > g_ws_bytes) {
    if (g_ws) cudaFree(g_ws);
    EET_CHECK_CUDA(cudaMalloc(&g_ws, ws_bytes));
    g_ws_bytes = ws_bytes;
  }
  if (counters > g_cnt_n) {
    if (g_cnt) cudaFree(g_cnt);
    EET_CHECK_CUDA(cudaMalloc(&g_cnt, counters * sizeof(int)));
    EET_CHECK_CUDA(cudaMemset(g_cnt, 0, counters * sizeof(int)));
    g_cnt_n = counters;
  }
}

template <typename T, int MN>
static void launch(const void* A, int lda, const void* B, int ldb, int M, int N, int K,
                   const Epi& e, int dtype, cudaStream_t st) {
  using C = Cfg<MN>;
  const int rbs = (N + ROWS - 1) / ROWS;
  const int nkb = (K + BK - 1) / BK;
  const int target = 2 * device_sm_count();
  int splits = std::min(std::max(1, (target + rbs - 1) / rbs), std::min(nkb, 16));
  const int kbps = (nkb + splits - 1) / splits;
  splits = (nkb + kbps - 1) / kbps;
  if (splits > 1) ensure_scratch((size_t)rbs * splits * ROWS * MN * sizeof(float), (size_t)rbs);
  CUtensorMap mw = make_tma_map_2d(B, N, K, ldb, ROWS, dtype);
  CUtensorMap mx = make_tma_map_2d(A, M, K, lda, MN, dtype);
  auto kern = gemv_tc_kernel<T, MN>;
  static bool attr = false;
  if (!attr) {
    EET_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  ProfScope ps(K_GEMV, st, gemm_bytes(M, N, K, 2, e), 2.0 * M * N * K);
  kern<<<dim3(rbs, splits), THREADS, C::SMEM, st>>>(mw, mx, M, N, K, kbps, splits, g_ws, g_cnt, e);
  EET_LAUNCH_CHECK();
}

}  // namespace gv

void gemv_tc_sm100(int dtype, const void* A, int lda, const void* B, int ldb, int M, int N, int K,
                   const Epi& e, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  EET_REQUIRE(M <= 32, EET_ERR_ARG, "gemv_tc: more than 32 token rows");
  if (dtype == EET_BF16) {
    M <= 16 ? gv::launch<__nv_bfloat16, 16>(A, lda, B, ldb, M, N, K, e, dtype, st)
            : gv::launch<__nv_bfloat16, 32>(A, lda, B, ldb, M, N, K, e, dtype, st);
  } else {
    M <= 16 ? gv::launch<__half, 16>(A, lda, B, ldb, M, N, K, e, dtype, st)
            : gv::launch<__half, 32>(A, lda, B, ldb, M, N, K, e, dtype, st);
  }
}

}  // namespace eet
