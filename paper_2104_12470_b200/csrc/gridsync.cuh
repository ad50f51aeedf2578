// Grid-wide barriers for persistent kernels (all CTAs co-resident).
// Monotonic counters: barrier number g (1, 2, ...) completes when the
// counter reaches g * arrivals, so nothing is reset between barriers; the
// counter is zeroed (memset on the launch stream) before each launch.
#pragma once

#include "sm100.cuh"

namespace eet {
namespace gs {

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// flat: every CTA arrives on one counter; thread 0 spins
__device__ __forceinline__ void grid_sync_flat(unsigned* ctr, unsigned gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_release_gpu(ctr, 1u);
    const unsigned target = gen * gridDim.x;
    while (ld_acquire_gpu(ctr) < target) {
    }
  }
  __syncthreads();
}

// hierarchical: cluster barrier, one arrival per cluster (rank 0), rank 0
// spins, cluster barrier releases the other CTAs of the cluster
__device__ __forceinline__ void grid_sync_cluster(unsigned* ctr, unsigned gen, unsigned nclusters) {
  sm100::cluster_sync();
  if (threadIdx.x == 0 && sm100::cluster_ctarank() == 0) {
    red_release_gpu(ctr, 1u);
    const unsigned target = gen * nclusters;
    while (ld_acquire_gpu(ctr) < target) {
    }
  }
  sm100::cluster_sync();
}

}  // namespace gs
}  // namespace eet
