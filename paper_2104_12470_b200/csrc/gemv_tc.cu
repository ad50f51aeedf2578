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
// the accumulator back (TMEM lane = weight row). K is split across the CTAs
// of a thread-block cluster (<= 8) so ~2 CTAs land on every SM; the partial
// tiles are summed through distributed shared memory in split order
// (deterministic, no global round trip), each CTA finishing a slice of the
// fused epilogue (bias / GELU / residual / KV-cache scatter / logits).
//
// Launched with programmatic dependent launch: weights are static, so the
// first ring stages of W are requested before griddepcontrol.wait and
// stream in while the previous kernel is still finishing.
#include "sm100.cuh"

namespace eet {
namespace gv {
using namespace sm100;

constexpr int ROWS = 128, BK = 64, THREADS = 128, STAGES = 4;
constexpr int W_BYTES = ROWS * BK * 2;

template <int MN> struct Lay {
  static constexpr int X_BYTES = MN * BK * 2;
  static constexpr int RED_OFF = STAGES * (W_BYTES + X_BYTES);
  static constexpr int SMEM = RED_OFF + ROWS * MN * 4 + 1024 + 128;
};

template <typename T, int MN>
__global__ void __launch_bounds__(THREADS) gemv_tc_kernel(
    const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapX, int M,
    int N, int K, int kb_per_split, int splits, Epi e) {
  using L = Lay<MN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sW = smem;                                   // STAGES x 16 KB (1024-aligned)
  uint8_t* sX = smem + STAGES * W_BYTES;                // STAGES x X_BYTES
  float* red = reinterpret_cast<float*>(smem + L::RED_OFF);        // [MN][128] partial tile
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::RED_OFF + ROWS * MN * 4);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

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
    const uint64_t pol_w = 0x12F0000000000000ull;   // EVICT_FIRST: weights read once per step
    const uint64_t pol_x = 0x14F0000000000000ull;   // EVICT_LAST: X re-read by every CTA
    // weights are static: fill the ring before waiting on the previous grid
    const int pre = min(STAGES, kb1 - kb0);
    for (int i = 0; i < pre; ++i) {
      mbar_expect_tx(&full[i], W_BYTES + L::X_BYTES);
      tma_load_2d(sW + i * W_BYTES, &mapW, &full[i], (kb0 + i) * BK, rb * ROWS, pol_w);
    }
    griddep_wait();
    griddep_launch_dependents();
    for (int i = 0; i < pre; ++i)
      tma_load_2d(sX + i * L::X_BYTES, &mapX, &full[i], (kb0 + i) * BK, 0, pol_x);
    int stage = pre % STAGES;
    uint32_t phase = pre == STAGES ? 1 : 0;
    for (int kb = kb0 + pre; kb < kb1; ++kb) {
      mbar_wait(&empty[stage], phase ^ 1);
      mbar_expect_tx(&full[stage], W_BYTES + L::X_BYTES);
      tma_load_2d(sW + stage * W_BYTES, &mapW, &full[stage], kb * BK, rb * ROWS, pol_w);
      tma_load_2d(sX + stage * L::X_BYTES, &mapX, &full[stage], kb * BK, 0, pol_x);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  } else {
    griddep_wait();
    griddep_launch_dependents();
    if (warp == 1 && lane == 0) {
      constexpr uint32_t idesc = instr_desc(std::is_same<T, __nv_bfloat16>::value ? 1 : 0, ROWS, MN);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t w0 = smem_u32(sW + stage * W_BYTES);
        const uint32_t x0 = smem_u32(sX + stage * L::X_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          mma_f16(tmem, smem_desc(w0 + k * 32), smem_desc(x0 + k * 32), idesc, (kb > kb0) | k);
        mma_commit(&empty[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      mma_commit(done);
    }
  }
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();

  // accumulator row = this thread's weight row; columns = token rows
  const int row = warp * 32 + lane;
  const int n0 = rb * ROWS;
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
    if (n0 + row < N)
#pragma unroll
      for (int m = 0; m < MN; ++m)
        if (m < M) epi_apply<T>(e, m, n0 + row, acc[m]);
    return;
  }
  // split-K reduction through distributed shared memory: publish the
  // partial tile transposed ([m][row]), then every CTA of the cluster sums
  // a contiguous slice over the splits in rank order and finishes it.
#pragma unroll
  for (int m = 0; m < MN; ++m) red[m * ROWS + row] = acc[m];
  cluster_sync();
  const int total = M * ROWS;
  const int chunk = (total + splits - 1) / splits;
  const int lo = (int)cluster_ctarank() * chunk, hi = min(total, lo + chunk);
  const float* peer[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) peer[p] = map_peer(red, p < splits ? p : 0);
  for (int idx = lo + threadIdx.x; idx < hi; idx += THREADS) {
    float part[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) part[p] = p < splits ? peer[p][idx] : 0.f;   // all in flight
    float v = 0.f;
#pragma unroll
    for (int p = 0; p < 8; ++p) v += part[p];                                 // rank order
    const int m = idx / ROWS, n = n0 + idx % ROWS;
    if (n < N) epi_apply<T>(e, m, n, v);
  }
  cluster_sync();                       // peers may still be reading our slice
}

template <typename T, int MN>
static void launch(const void* A, int lda, const void* B, int ldb, int M, int N, int K,
                   const Epi& e, int dtype, cudaStream_t st) {
  using L = Lay<MN>;
  const int rbs = (N + ROWS - 1) / ROWS;
  const int nkb = (K + BK - 1) / BK;
  const int target = 2 * device_sm_count();
  int splits = std::min(std::max(1, (target + rbs - 1) / rbs), std::min(nkb, 8));
  const int kbps = (nkb + splits - 1) / splits;
  splits = (nkb + kbps - 1) / kbps;
  CUtensorMap mw = make_tma_map_2d(B, N, K, ldb, ROWS, dtype);
  CUtensorMap mx = make_tma_map_2d(A, M, K, lda, MN, dtype);
  auto kern = gemv_tc_kernel<T, MN>;
  static bool attr = false;
  if (!attr) {
    EET_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM));
    attr = true;
  }
  ProfScope ps(K_GEMV, st, gemm_bytes(M, N, K, 2, e), 2.0 * M * N * K);
  launch_ex(kern, dim3(rbs, splits), dim3(THREADS), L::SMEM, st, true, dim3(1, splits, 1), mw, mx, M,
            N, K, kbps, splits, e);
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
