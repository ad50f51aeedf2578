// mma.sync fragment helpers shared by the decode projections (gemv_cl.cu)
// and the fused decode attention + out-projection (attn_o.cu): 16x16 weight
// sub-tiles read with ldmatrix from a 128B-swizzled [K/64][rows][64] TMA
// block, token rows as the B operand, m16n8k16 with fp32 accumulators, and
// the st.async DSMEM stores that complete_tx on the receiver's mbarrier.
#pragma once

#include "sm100.cuh"

namespace eet {
namespace gc {

__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                            uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// remote (DSMEM) stores that complete_tx on the receiver's mbarrier
__device__ __forceinline__ void st_async_v4(uint32_t addr, const float* v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
               ::"r"(addr), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t addr, float a, float b, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];"
               ::"r"(addr), "f"(a), "f"(b), "r"(mbar)
               : "memory");
}

template <typename T>
__device__ __forceinline__ void mma16816(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
}

// A fragment of the 16x16 weight sub-tile (rows row0.., k-step ks) from a
// weight block laid out as [Kc/64 boxes][rows][64] with 128B swizzle
__device__ __forceinline__ void load_a(uint32_t sw, int rows, int row0, int ks, int lane, uint32_t* a) {
  const int r = row0 + (lane & 15);
  const int chunk = ((ks & 3) << 1) | (lane >> 4);              // 16-byte chunk within the 128 B row
  const uint32_t addr = sw + (uint32_t)((ks >> 2) * rows * 128 + r * 128 + ((chunk ^ (r & 7)) << 4));
  ldmatrix_x4(addr, a[0], a[1], a[2], a[3]);
}

// one warp: tile rows [row0, row0+16) x k-steps [s0, s1) x NB n-blocks of
// token rows; four independent accumulator chains, summed in a fixed order
template <typename T, int NB>
__device__ __forceinline__ void warp_mma(uint32_t sw, int rows, int row0, int s0, int s1, const T* xs,
                                         int xst, int lane, float (&acc)[NB][4]) {
  float part[4][NB][4];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int i = 0; i < 4; ++i) part[c][nb][i] = 0.f;
  const int g = lane >> 2, c4 = lane & 3;
  int s = s0;
#pragma unroll 1
  for (; s + 3 < s1; s += 4) {
    uint32_t a[4][4];
#pragma unroll
    for (int c = 0; c < 4; ++c) load_a(sw, rows, row0, s + c, lane, a[c]);
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const T* xr = xs + (nb * 8 + g) * xst + (s + c) * 16 + 2 * c4;
        mma16816<T>(part[c][nb], a[c][0], a[c][1], a[c][2], a[c][3], *reinterpret_cast<const uint32_t*>(xr),
                    *reinterpret_cast<const uint32_t*>(xr + 8));
      }
  }
#pragma unroll 1
  for (; s < s1; ++s) {
    uint32_t a[4];
    load_a(sw, rows, row0, s, lane, a);
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      const T* xr = xs + (nb * 8 + g) * xst + s * 16 + 2 * c4;
      mma16816<T>(part[0][nb], a[0], a[1], a[2], a[3], *reinterpret_cast<const uint32_t*>(xr),
                  *reinterpret_cast<const uint32_t*>(xr + 8));
    }
  }
#pragma unroll
  for (int nb = 0; nb < NB; ++nb)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[nb][i] = (part[0][nb][i] + part[1][nb][i]) + (part[2][nb][i] + part[3][nb][i]);
}

}  // namespace gc
}  // namespace eet
