// Calibration for a persistent decode step: cost of a grid-wide barrier
// among one-CTA-per-SM persistent CTAs (flat vs cluster-hierarchical).
#include "gridsync.cuh"

#include <algorithm>

namespace eet {

__global__ void __launch_bounds__(256) barrier_bench_kernel(unsigned* ctr, int n, int mode, unsigned nclusters) {
  for (int i = 1; i <= n; ++i) {
    if (mode == 0) gs::grid_sync_flat(ctr, (unsigned)i);
    else gs::grid_sync_cluster(ctr, (unsigned)i, nclusters);
  }
}

extern "C" int eet_debug_grid_barrier(int n, int ctas, int mode, float* us_per_barrier) {
  try {
    unsigned* ctr = nullptr;
    EET_CHECK_CUDA(cudaMalloc(&ctr, 64));
    cudaEvent_t a, b;
    EET_CHECK_CUDA(cudaEventCreate(&a));
    EET_CHECK_CUDA(cudaEventCreate(&b));
    const int cl = mode == 0 ? 1 : 8;
    ctas = ctas / cl * cl;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      EET_CHECK_CUDA(cudaMemset(ctr, 0, 64));
      EET_CHECK_CUDA(cudaEventRecord(a));
      launch_cluster(barrier_bench_kernel, dim3(ctas), dim3(256), 0, nullptr, false, dim3(cl, 1, 1), ctr, n, mode,
                     (unsigned)(ctas / cl));
      EET_CHECK_CUDA(cudaEventRecord(b));
      EET_CHECK_CUDA(cudaEventSynchronize(b));
      float ms = 0;
      EET_CHECK_CUDA(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms * 1e3f / n);
    }
    *us_per_barrier = best;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(ctr);
    return EET_OK;
  } catch (const Fail& f) {
    return f.code;
  }
}

}  // namespace eet
