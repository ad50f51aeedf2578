// CUDA-core GEMMs:
//  * gemm_f32_simt — true-fp32 FFMA GEMM for the reference's "fp32 mode"
//    (no TF32: identical greedy tokens need ~1e-6 logit accuracy, SURVEY
//    Appendix B.4). Replaces the OpenBLAS sgemm calls at runtime.py:131,136,
//    188,210,212,344.
//  * gemv_small_m — M <= 16 rows (decode steps, LM head): HBM-bound on the
//    weight read, so it streams W with 128-bit loads and keeps the few
//    activation rows in shared memory. Works for every dtype.
// Both compute C = A[M,K] * B[N,K]^T with the fused epilogue of common.cuh.
#include "sm100.cuh"

#include <algorithm>
#include <mutex>
#include <string>
#include <unordered_map>

namespace eet {

// ------------------------------------------------------------- fp32 GEMM
namespace {
constexpr int BM = 128, BN = 128, BK = 16;
}

// 128x128x16 tile, 256 threads, 8x8 outputs per thread as 2x2 blocks of 4x4
// (rows ty*4 and 64+ty*4, columns tx*4 and 64+tx*4: conflict-free float4
// shared reads, 16 FFMA per 128-bit shared load). A and B k-slices are
// staged transposed ([k][m], [k][n]) in a double-buffered ring; global
// loads are 128-bit along k when rows are 16-byte aligned (VEC).
// split-K: blockIdx.z = split, K range [z * kspan, (z+1) * kspan); with
// part != nullptr the tile is stored raw to part[z][M][N] (the reduction
// kernel applies the epilogue), else the epilogue runs here.
template <bool VEC>
__global__ void __launch_bounds__(256, 2) gemm_f32_kernel(const float* __restrict__ A, int lda,
                                                          const float* __restrict__ B, int ldb,
                                                          int M, int N, int K, Epi e, int kspan,
                                                          float* __restrict__ part) {
  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kbeg = blockIdx.z * kspan;
  A += kbeg;
  B += kbeg;
  K = min(kspan, K - kbeg);
  // loader: 128 rows x 16 k per operand; thread -> rows lr and lr + 64,
  // k lk..lk+3 (two float4 per operand per slice)
  const int lr = tid >> 2, lk = (tid & 3) * 4;
  bool a_ok[2], b_ok[2];
  const float* Ap[2];
  const float* Bp[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    a_ok[h] = m0 + lr + 64 * h < M;
    b_ok[h] = n0 + lr + 64 * h < N;
    Ap[h] = A + (long long)(a_ok[h] ? m0 + lr + 64 * h : 0) * lda;
    Bp[h] = B + (long long)(b_ok[h] ? n0 + lr + 64 * h : 0) * ldb;
  }
  float acc[8][8] = {};
  float4 ra[2], rb[2];
  auto gload = [&](int k0) {
    const int k = k0 + lk;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (VEC && k + 3 < K) {
        ra[h] = a_ok[h] ? __ldg(reinterpret_cast<const float4*>(Ap[h] + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
        rb[h] = b_ok[h] ? __ldg(reinterpret_cast<const float4*>(Bp[h] + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        float va[4], vb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          va[j] = (a_ok[h] && k + j < K) ? Ap[h][k + j] : 0.f;
          vb[j] = (b_ok[h] && k + j < K) ? Bp[h][k + j] : 0.f;
        }
        ra[h] = make_float4(va[0], va[1], va[2], va[3]);
        rb[h] = make_float4(vb[0], vb[1], vb[2], vb[3]);
      }
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = lr + 64 * h;
      As[buf][lk + 0][r] = ra[h].x; As[buf][lk + 1][r] = ra[h].y;
      As[buf][lk + 2][r] = ra[h].z; As[buf][lk + 3][r] = ra[h].w;
      Bs[buf][lk + 0][r] = rb[h].x; Bs[buf][lk + 1][r] = rb[h].y;
      Bs[buf][lk + 2][r] = rb[h].z; Bs[buf][lk + 3][r] = rb[h].w;
    }
  };
  const int nk = (K + BK - 1) / BK;
  gload(0);
  sstore(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) gload((kt + 1) * BK);
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][k][64 + tx * 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < nk) {
      sstore(buf ^ 1);
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (n >= N) continue;
      if (part) part[((size_t)blockIdx.z * M + m) * N + n] = acc[i][j];
      else epi_apply<float>(e, m, n, acc[i][j]);
    }
  }
}

// second stage of split-K: partial sums in split order (deterministic), epilogue
__global__ void gemm_f32_reduce_kernel(const float* __restrict__ part, int splits, int M, int N, Epi e) {
  const long long total = (long long)M * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    float v = 0.f;
    for (int s = 0; s < splits; ++s) v += part[s * total + i];
    epi_apply<float>(e, (int)(i / N), (int)(i % N), v);
  }
}

void launch_splitk_reduce(const float* part, int splits, int M, int N, const Epi& e, cudaStream_t st) {
  const long long total = (long long)M * N;
  gemm_f32_reduce_kernel<<<(int)std::min<long long>((total + 255) / 256, 8 * device_sm_count()), 256, 0, st>>>(
      part, splits, M, N, e);
  count_launch();
  EET_LAUNCH_CHECK();
}

// Split-K plan: ~2 CTAs of 256 threads per SM, >= 128 k per split. The
// partial workspace is device memory grown outside graph capture; under
// capture (or if it would have to grow) the GEMM runs unsplit.
void gemm_f32_simt(const float* A, int lda, const float* B, int ldb, int M, int N, int K,
                   const Epi& e, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  const int tiles = ((N + BN - 1) / BN) * ((M + BM - 1) / BM);
  int splits = std::max(1, std::min(2 * device_sm_count() / std::max(1, tiles), K / 128));
  float* ws = nullptr;
  if (splits > 1) {
    // per-stream split-K workspace (concurrent layers on several streams),
    // grown outside graph capture (unsplit under capture if too small)
    static std::mutex mu;
    static std::unordered_map<cudaStream_t, std::pair<float*, size_t>> wss;
    const size_t need = sizeof(float) * (size_t)splits * M * N;
    std::lock_guard<std::mutex> lk(mu);
    auto& slot = wss[st];
    if (need > slot.second) {
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
    if (splits > 1) ws = slot.first;
  }
  const int kspan = ((K + splits - 1) / splits + BK - 1) / BK * BK;
  splits = (K + kspan - 1) / kspan;
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, splits);
  ProfScope ps(K_GEMM_F32, st, gemm_bytes(M, N, K, 4, e), 2.0 * M * N * K);
  const bool vec = lda % 4 == 0 && ldb % 4 == 0 && kspan % 4 == 0 &&
                   (reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0;
  if (vec)
    gemm_f32_kernel<true><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, e, kspan, ws);
  else
    gemm_f32_kernel<false><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, e, kspan, ws);
  EET_LAUNCH_CHECK();
  if (splits > 1) {
    const long long total = (long long)M * N;
    gemm_f32_reduce_kernel<<<(int)std::min<long long>((total + 255) / 256, 8 * device_sm_count()), 256, 0, st>>>(
        ws, splits, M, N, e);
    count_launch();
    EET_LAUNCH_CHECK();
  }
}

// --------------------------------------------------------- small-M GEMV
// Block = 8 warps; warp w owns COLS consecutive output columns. Each lane
// streams 16-byte slices of the COLS weight rows and multiplies them with
// the MT activation rows staged (chunk by chunk along K) in shared memory.
template <typename T, int MT, int COLS, bool VEC>
__global__ void __launch_bounds__(256) gemv_kernel(const T* __restrict__ A, int lda,
                                                   const T* __restrict__ B, int ldb, int M,
                                                   int N, int K, int KC, Epi e) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* xs = reinterpret_cast<T*>(smem_raw);          // [MT][KC]
  constexpr int E = VEC ? 16 / sizeof(T) : 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nbase = (blockIdx.x * 8 + warp) * COLS;
  float acc[COLS][MT];
#pragma unroll
  for (int c = 0; c < COLS; ++c)
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[c][m] = 0.f;

  for (int k0 = 0; k0 < K; k0 += KC) {
    const int kc = min(KC, K - k0);
    __syncthreads();
    // stage activation rows [0, M) x [k0, k0+kc)
    if constexpr (VEC) {
      const int nv = kc / E;
      for (int idx = threadIdx.x; idx < M * nv; idx += blockDim.x) {
        int m = idx / nv, v = idx - m * nv;
        *reinterpret_cast<uint4*>(xs + m * KC + v * E) =
            *reinterpret_cast<const uint4*>(A + (long long)m * lda + k0 + v * E);
      }
    } else {
      for (int idx = threadIdx.x; idx < M * kc; idx += blockDim.x) {
        int m = idx / kc, k = idx - m * kc;
        xs[m * KC + k] = A[(long long)m * lda + k0 + k];
      }
    }
    __syncthreads();
    for (int kk = lane * E; kk < kc; kk += 32 * E) {
      float w[COLS][E];
#pragma unroll
      for (int c = 0; c < COLS; ++c) {
        int n = nbase + c;
        if (n < N) {
          const T* src = B + (long long)n * ldb + k0 + kk;
          if constexpr (VEC) {
            load16<T>(src, w[c]);
          } else {
            w[c][0] = to_f(src[0]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < E; ++j) w[c][j] = 0.f;
        }
      }
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        if (m < M) {
          float xv[E];
          if constexpr (VEC) {
            load16<T>(xs + m * KC + kk, xv);
          } else {
            xv[0] = to_f(xs[m * KC + kk]);
          }
#pragma unroll
          for (int c = 0; c < COLS; ++c)
#pragma unroll
            for (int j = 0; j < E; ++j) acc[c][m] = fmaf(w[c][j], xv[j], acc[c][m]);
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < COLS; ++c)
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[c][m] = warp_sum(acc[c][m]);
#pragma unroll
  for (int c = 0; c < COLS; ++c)
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      int p = c * MT + m;
      if ((p & 31) == lane && m < M && nbase + c < N) epi_apply<T>(e, m, nbase + c, acc[c][m]);
    }
}

template <typename T, int MT>
static void gemv_launch(const T* A, int lda, const T* B, int ldb, int M, int N, int K,
                        const Epi& e, cudaStream_t st) {
  constexpr int COLS = 4;
  constexpr int E = 16 / sizeof(T);
  const bool vec = (K % E == 0) && (lda % E == 0) && (ldb % E == 0) &&
                   ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
  int KC = (int)(65536 / (MT * sizeof(T)));          // 64 KB of staged activations
  KC = std::min(KC, (K + E - 1) / E * E);
  KC = std::max(E, KC / E * E);
  size_t smem = (size_t)MT * KC * sizeof(T);
  dim3 grid((N + 8 * COLS - 1) / (8 * COLS));
  ProfScope ps(K_GEMV, st, gemm_bytes(M, N, K, sizeof(T), e), 2.0 * M * N * K);
  if (vec) {
    auto k = gemv_kernel<T, MT, COLS, true>;
    EET_CHECK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, 256, smem, st>>>(A, lda, B, ldb, M, N, K, KC, e);
  } else {
    auto k = gemv_kernel<T, MT, COLS, false>;
    EET_CHECK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, 256, smem, st>>>(A, lda, B, ldb, M, N, K, KC, e);
  }
  EET_LAUNCH_CHECK();
}

template <typename T>
static void gemv_dispatch(const T* A, int lda, const T* B, int ldb, int M, int N, int K,
                          const Epi& e, cudaStream_t st) {
  if (M <= 1) gemv_launch<T, 1>(A, lda, B, ldb, M, N, K, e, st);
  else if (M <= 2) gemv_launch<T, 2>(A, lda, B, ldb, M, N, K, e, st);
  else if (M <= 4) gemv_launch<T, 4>(A, lda, B, ldb, M, N, K, e, st);
  else if (M <= 8) gemv_launch<T, 8>(A, lda, B, ldb, M, N, K, e, st);
  else gemv_launch<T, 16>(A, lda, B, ldb, M, N, K, e, st);
}

void gemv_small_m(int dtype, const void* A, int lda, const void* B, int ldb, int M, int N, int K,
                  const Epi& e, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  EET_REQUIRE(M <= 16, EET_ERR_ARG, "gemv_small_m: M > 16");
  switch (dtype) {
    case EET_F32: gemv_dispatch<float>((const float*)A, lda, (const float*)B, ldb, M, N, K, e, st); break;
    case EET_BF16: gemv_dispatch<__nv_bfloat16>((const __nv_bfloat16*)A, lda, (const __nv_bfloat16*)B, ldb, M, N, K, e, st); break;
    default: gemv_dispatch<__half>((const __half*)A, lda, (const __half*)B, ldb, M, N, K, e, st);
  }
}

// The GEMM entry the runtime uses: fp32 mode -> FFMA kernels (GEMV for the
// decode rows); 16-bit modes -> tcgen05 tensor cores fed by TMA: the tiled
// persistent GEMM for prompt passes, the swap-AB split-K GEMV for decode.
static bool tc_eligible(const void* A, int lda, const void* B, int ldb, int K) {
  return (K % 8 == 0) && (lda % 8 == 0) && (ldb % 8 == 0) &&
         ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
}

void gemm(int dtype, const void* A, int lda, const void* B, int ldb, int M, int N, int K,
          const Epi& e, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  if (dtype == EET_F32) {
    // fp32 mode: 3xTF32 on tcgen05 (gemm_tf32.cu) for the prompt-pass
    // projections, FFMA for decode rows and unaligned operands
    static const bool ffma = [] {                  // A/B switch: EET_F32_GEMM=ffma
      const char* v = std::getenv("EET_F32_GEMM");
      return v && std::string(v) == "ffma";
    }();
    if (M <= 16) gemv_small_m(dtype, A, lda, B, ldb, M, N, K, e, st);
    else if (ffma || !gemm_tf32x3(static_cast<const float*>(A), lda, static_cast<const float*>(B), ldb, M, N, K, e, st))
      gemm_f32_simt((const float*)A, lda, (const float*)B, ldb, M, N, K, e, st);
    return;
  }
  if (tc_eligible(A, lda, B, ldb, K)) {
    M <= 32 ? gemv_tc_sm100(dtype, A, lda, B, ldb, M, N, K, e, st)     // decode: swap-AB split-K
            : gemm_tc_sm100(dtype, A, lda, B, ldb, M, N, K, e, st);
    return;
  }
  // 16-bit operands whose rows are not 16-byte aligned (tiny hidden sizes in
  // tests): stream them through the GEMV 16 rows at a time.
  const size_t es = dtype_size(dtype);
  for (int m0 = 0; m0 < M; m0 += 16) {
    Epi em = e;
    // shift row-indexed epilogue state to the chunk
    if (e.mode == EPI_RESID || e.mode == EPI_QKV) em.rinfo = e.rinfo + m0;
    if (e.mode == EPI_QKV) em.out = (char*)e.out + (size_t)m0 * e.hq * es;
    else if (e.mode == EPI_STORE_F32) em.out = (char*)e.out + (size_t)m0 * e.ldo * 4;
    else if (e.mode != EPI_RESID) em.out = (char*)e.out + (size_t)m0 * e.ldo * es;
    gemv_small_m(dtype, (const char*)A + (size_t)m0 * lda * es, lda, B, ldb, std::min(16, M - m0),
                 N, K, em, st);
  }
}

}  // namespace eet
