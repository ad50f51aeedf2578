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
// through a TMA ring (16 KB per 64-wide k-block), one lane issues
// tcgen05.mma kind::f16 M=128 N=MN into TMEM, and all four warps read the
// accumulator back (TMEM lane = weight row). K is split across the CTAs of a
// thread-block cluster (<= 8) so ~2 CTAs land on every SM; the partial tiles
// are summed through distributed shared memory in split order
// (deterministic, no global round trip), each CTA finishing a slice of the
// fused epilogue (bias / GELU / residual / KV-cache scatter / logits).
//
// X comes either from a 16-bit activation buffer (TMA) or — LNX — straight
// from the fp32 residual stream: the CTA normalises its token rows
// (runtime.py:83-94, single-pass statistics) for its own K-range and writes
// them into the 128B-swizzled operand layout, so the decode step needs no
// separate LayerNorm launch before QKV, W1 and the LM head.
//
// Launched with programmatic dependent launch: weights are static, so the
// first ring stages of W are requested before griddepcontrol.wait and
// stream in while the previous kernel is still finishing.
#include "sm100.cuh"

#include <map>
#include <mutex>

namespace eet {
namespace gv {
using namespace sm100;

constexpr int ROWS = 128, BK = 64, THREADS = 128, STAGES = 4, MAX_KBPS = 16;
// LNX: a CTA's K-slice (<= LNX_MAX_COLS columns) of the token rows stays in registers
constexpr int LNX_MAX_COLS = 256;
constexpr int W_BYTES = ROWS * BK * 2;

struct LnSrc {                      // LNX operand source
  const float* x;                   // residual stream, row m at rinfo[m]
  long long x_sb, x_ss;
  const int2* rinfo;
  const float* g;
  const float* b;
};

template <int MN, bool LNX> struct Lay {
  static constexpr int X_TILE = MN * BK * 2;                 // one [MN x 64] operand tile
  static constexpr int X_TILES = LNX ? LNX_MAX_COLS / BK : STAGES;   // whole K-slice vs TMA ring
  static constexpr int X_OFF = STAGES * W_BYTES;
  static constexpr int RED_OFF = X_OFF + X_TILES * X_TILE;
  static constexpr int STATS_OFF = RED_OFF + ROWS * MN * 4;   // LNX row stats [MN] float2
  static constexpr int BAR_OFF = STATS_OFF + MN * 8;
  static constexpr int SMEM = BAR_OFF + 128 + 1024;
};

template <typename T, int MN, bool LNX>
__global__ void __launch_bounds__(THREADS) gemv_tc_kernel(
    const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapX, LnSrc ln,
    int M, int N, int K, int kb_per_split, int splits, Epi e) {
  using L = Lay<MN, LNX>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sW = smem;                                   // STAGES x 16 KB (1024-aligned)
  uint8_t* sX = smem + L::X_OFF;                        // X tiles (2-4 KB each, 1024-aligned)
  float* red = reinterpret_cast<float*>(smem + L::RED_OFF);        // [MN][128] partial tile
  float2* stats = reinterpret_cast<float2*>(smem + L::STATS_OFF);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint64_t* x_ready = done + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(x_ready + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = blockIdx.x, split = blockIdx.y;
  const int nkb = (K + BK - 1) / BK;
  const int kb0 = split * kb_per_split;
  const int kb1 = min(nkb, kb0 + kb_per_split);
  constexpr uint32_t STAGE_TX = LNX ? W_BYTES : W_BYTES + L::X_TILE;

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    mbar_init(x_ready, THREADS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapW) : "memory");
    if (!LNX) asm volatile("prefetch.tensormap [%0];" ::"l"(&mapX) : "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const uint64_t pol_w = 0x12F0000000000000ull;   // EVICT_FIRST: weights read once per step
  const uint64_t pol_x = 0x14F0000000000000ull;   // EVICT_LAST: X re-read by every CTA
  const int pre = min(STAGES, kb1 - kb0);
  if (warp == 0 && lane == 0) {
    // weights are static: fill the ring before waiting on the previous grid
    for (int i = 0; i < pre; ++i) {
      mbar_expect_tx(&full[i], STAGE_TX);
      tma_load_2d(sW + i * W_BYTES, &mapW, &full[i], (kb0 + i) * BK, rb * ROWS, pol_w);
    }
  }
  griddep_wait();
  griddep_launch_dependents();

  if constexpr (LNX) {
    // ---- fused LayerNorm of the token rows into the swizzled X tiles.
    // Every CTA of the split-K cluster loads only its own K-slice of the M
    // rows (the columns it normalises), keeps it in registers, and the row
    // statistics (sum, sum of squares) are combined across the cluster
    // through DSMEM in rank order: one L2 round trip per CTA.
    constexpr int TPR = THREADS / MN;                   // threads per row: 8 (MN 16) / 4 (MN 32)
    constexpr int GPT = LNX_MAX_COLS / 8 / TPR;         // 8-column groups per thread
    const int h = K;
    const int m = threadIdx.x / TPR, sub = threadIdx.x % TPR;
    const int c0 = kb0 * BK, ngrp = (kb1 - kb0) * BK / 8;
    const float* xr = ln.x;
    if (m < M) {
      const int2 ri = ln.rinfo[m];
      xr = ln.x + ri.x * ln.x_sb + ri.y * ln.x_ss;
    }
    float v[GPT][8];
    float s = 0.f, ss = 0.f;
#pragma unroll
    for (int i = 0; i < GPT; ++i) {                     // all loads in flight together
      const int grp = sub + i * TPR;
      if (m < M && grp < ngrp) {
        const float4 a = *reinterpret_cast<const float4*>(xr + c0 + grp * 8);
        const float4 b = *reinterpret_cast<const float4*>(xr + c0 + grp * 8 + 4);
        v[i][0] = a.x; v[i][1] = a.y; v[i][2] = a.z; v[i][3] = a.w;
        v[i][4] = b.x; v[i][5] = b.y; v[i][6] = b.z; v[i][7] = b.w;
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[i][j] = 0.f;
      }
    }
#pragma unroll
    for (int i = 0; i < GPT; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) { s += v[i][j]; ss += v[i][j] * v[i][j]; }
#pragma unroll
    for (int o = 1; o < TPR; o <<= 1) {           // all lanes take part
      s += __shfl_xor_sync(0xffffffffu, s, o);
      ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    if (sub == 0) stats[m] = make_float2(s, ss);
    cluster_sync();
    float ts = 0.f, tss = 0.f;
    for (int p = 0; p < splits; ++p) {            // rank order: deterministic
      const float2 q = map_peer(stats, p)[m];
      ts += q.x;
      tss += q.y;
    }
    const float mean = ts / (float)h;
    const float rstd = 1.0f / sqrtf(fmaxf(tss / (float)h - mean * mean, 0.f) + 1e-5f);
#pragma unroll
    for (int i = 0; i < GPT; ++i) {
      const int grp = sub + i * TPR;
      if (grp >= ngrp) continue;
      const int col = c0 + grp * 8;
      float y[8];
      if (m < M) {
        const float4 g0 = *reinterpret_cast<const float4*>(ln.g + col);
        const float4 g1 = *reinterpret_cast<const float4*>(ln.g + col + 4);
        const float4 b0 = *reinterpret_cast<const float4*>(ln.b + col);
        const float4 b1 = *reinterpret_cast<const float4*>(ln.b + col + 4);
        const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) y[j] = (v[i][j] - mean) * rstd * gv[j] + bv[j];
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) y[j] = 0.f;
      }
      const int tile = grp >> 3, chunk = grp & 7;
      uint8_t* dst = sX + tile * L::X_TILE + (m >> 3) * 1024 + (m & 7) * 128 + ((chunk ^ (m & 7)) << 4);
      store16<T>(reinterpret_cast<T*>(dst), y);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> MMA
    mbar_arrive(x_ready);
  }

  if (warp == 0 && lane == 0) {
    if constexpr (!LNX) {
      for (int i = 0; i < pre; ++i)
        tma_load_2d(sX + i * L::X_TILE, &mapX, &full[i], (kb0 + i) * BK, 0, pol_x);
    }
    int stage = pre % STAGES;
    uint32_t phase = pre == STAGES ? 1 : 0;
    for (int kb = kb0 + pre; kb < kb1; ++kb) {
      mbar_wait(&empty[stage], phase ^ 1);
      mbar_expect_tx(&full[stage], STAGE_TX);
      tma_load_2d(sW + stage * W_BYTES, &mapW, &full[stage], kb * BK, rb * ROWS, pol_w);
      if constexpr (!LNX)
        tma_load_2d(sX + stage * L::X_TILE, &mapX, &full[stage], kb * BK, 0, pol_x);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = instr_desc(std::is_same<T, __nv_bfloat16>::value ? 1 : 0, ROWS, MN);
    if constexpr (LNX) mbar_wait(x_ready, 0);
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      const uint32_t w0 = smem_u32(sW + stage * W_BYTES);
      const uint32_t x0 = smem_u32(sX + (LNX ? (kb - kb0) : stage) * L::X_TILE);
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

// splits: ~2 CTAs per SM, <= 8 per cluster, every split non-empty, and all
// clusters co-resident (one wave): ncu r01 showed 8-CTA clusters capped at 15
// active clusters, i.e. 3 waves for the QKV / W1 shapes. `max_clusters(s)`
// is the occupancy query for cluster size s. LNX keeps the whole K-range of
// a CTA in shared memory (<= MAX_KBPS k-blocks).
template <typename F>
static void plan_splits(int rbs, int nkb, bool lnx, int* splits, int* kbps, F max_clusters) {
  const int target = 2 * device_sm_count();
  int s = std::min(std::max(1, (target + rbs - 1) / rbs), std::min(nkb, 8));
  while (s > 1 && rbs > max_clusters(s)) --s;
  if (lnx) s = std::max(s, (nkb * BK + LNX_MAX_COLS - 1) / LNX_MAX_COLS);
  const int k = (nkb + s - 1) / s;
  *kbps = k;
  *splits = (nkb + k - 1) / k;
}

template <typename Kern>
static int active_clusters(Kern kern, int smem, int s) {
  static std::map<std::pair<const void*, int>, int> cache;   // (kernel, s)
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_pair(reinterpret_cast<const void*>(kern), s);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1, s, 1);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = s;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = 2 * device_sm_count() / s;
  }
  cache[key] = n;
  return n;
}

template <typename T, int MN, bool LNX>
static void launch(const void* A, int lda, const LnSrc& ln, const void* B, int ldb, int M, int N,
                   int K, const Epi& e, int dtype, cudaStream_t st) {
  using L = Lay<MN, LNX>;
  const int rbs = (N + ROWS - 1) / ROWS;
  const int nkb = (K + BK - 1) / BK;
  auto kern = gemv_tc_kernel<T, MN, LNX>;
  static const bool attr = [&] {                     // thread-safe one-time init
    EET_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM));
    EET_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    return true;
  }();
  (void)attr;
  int splits, kbps;
  plan_splits(rbs, nkb, LNX, &splits, &kbps, [&](int s) { return active_clusters(kern, L::SMEM, s); });
  EET_REQUIRE(splits <= 8, EET_ERR_UNSUPPORTED, "gemv_tc: K too long for one cluster");
  CUtensorMap mw = make_tma_map_2d(B, N, K, ldb, ROWS, dtype);
  CUtensorMap mx = LNX ? mw : make_tma_map_2d(A, M, K, lda, MN, dtype);
  const double xbytes = LNX ? (double)M * K * 4 : (double)M * K * 2;
  ProfScope ps(K_GEMV, st, gemm_bytes(M, N, K, 2, e) - (double)M * K * 2 + xbytes, 2.0 * M * N * K);
  launch_ex(kern, dim3(rbs, splits), dim3(THREADS), L::SMEM, st, true, dim3(1, splits, 1), mw, mx,
            ln, M, N, K, kbps, splits, e);
  EET_LAUNCH_CHECK();
}

}  // namespace gv

void gemv_tc_sm100(int dtype, const void* A, int lda, const void* B, int ldb, int M, int N, int K,
                   const Epi& e, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  EET_REQUIRE(M <= 32, EET_ERR_ARG, "gemv_tc: more than 32 token rows");
  const gv::LnSrc none{};
  if (dtype == EET_BF16) {
    M <= 16 ? gv::launch<__nv_bfloat16, 16, false>(A, lda, none, B, ldb, M, N, K, e, dtype, st)
            : gv::launch<__nv_bfloat16, 32, false>(A, lda, none, B, ldb, M, N, K, e, dtype, st);
  } else {
    M <= 16 ? gv::launch<__half, 16, false>(A, lda, none, B, ldb, M, N, K, e, dtype, st)
            : gv::launch<__half, 32, false>(A, lda, none, B, ldb, M, N, K, e, dtype, st);
  }
}

// LayerNorm-fused variant: X = LN(x[rows]) * g + b computed in the prologue.
// Returns false (caller runs LN + GEMV separately) when the shape does not fit.
bool gemv_tc_ln_sm100(int dtype, const float* x, long long x_sb, long long x_ss,
                      const int2* rinfo, const float* g, const float* b, const void* B, int ldb,
                      int M, int N, int K, const Epi& e, cudaStream_t st) {
  if (dtype == EET_F32 || M <= 0 || M > 32 || K % 64 != 0 || ldb % 8 != 0 ||
      (reinterpret_cast<uintptr_t>(x) & 15) || (x_sb & 3) || (x_ss & 3) ||
      (reinterpret_cast<uintptr_t>(B) & 15) || (K + gv::LNX_MAX_COLS - 1) / gv::LNX_MAX_COLS > 8 ||
      (reinterpret_cast<uintptr_t>(g) & 15) || (reinterpret_cast<uintptr_t>(b) & 15))
    return false;
  {
    int sp, kb;
    auto kern = dtype == EET_BF16 ? (M <= 16 ? gv::gemv_tc_kernel<__nv_bfloat16, 16, true> : gv::gemv_tc_kernel<__nv_bfloat16, 32, true>)
                                  : (M <= 16 ? gv::gemv_tc_kernel<__half, 16, true> : gv::gemv_tc_kernel<__half, 32, true>);
    const int smem = M <= 16 ? gv::Lay<16, true>::SMEM : gv::Lay<32, true>::SMEM;
    EET_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    gv::plan_splits((N + gv::ROWS - 1) / gv::ROWS, K / 64, false, &sp, &kb,
                    [&](int s) { return gv::active_clusters(kern, smem, s); });
    if (kb * 64 > gv::LNX_MAX_COLS) return false;       // e.g. LM head: 1 split of 1024 columns
  }
  const gv::LnSrc ln{x, x_sb, x_ss, rinfo, g, b};
  if (dtype == EET_BF16) {
    M <= 16 ? gv::launch<__nv_bfloat16, 16, true>(nullptr, 0, ln, B, ldb, M, N, K, e, dtype, st)
            : gv::launch<__nv_bfloat16, 32, true>(nullptr, 0, ln, B, ldb, M, N, K, e, dtype, st);
  } else {
    M <= 16 ? gv::launch<__half, 16, true>(nullptr, 0, ln, B, ldb, M, N, K, e, dtype, st)
            : gv::launch<__half, 32, true>(nullptr, 0, ln, B, ldb, M, N, K, e, dtype, st);
  }
  return true;
}

}  // namespace eet
