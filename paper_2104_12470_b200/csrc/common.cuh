// Device-side helpers shared by the kernels: dtype conversion, vector access,
// warp/block reductions and the epilogue applicator.
#pragma once

#include "eet_internal.h"

namespace eet {

template <typename T> struct DT;
template <> struct DT<float> {
  static __device__ __forceinline__ float to_f(float v) { return v; }
  static __device__ __forceinline__ float from_f(float v) { return v; }
};
template <> struct DT<__nv_bfloat16> {
  static __device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  static __device__ __forceinline__ __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};
template <> struct DT<__half> {
  static __device__ __forceinline__ float to_f(__half v) { return __half2float(v); }
  static __device__ __forceinline__ __half from_f(float v) { return __float2half_rn(v); }
};

template <typename T> __device__ __forceinline__ float to_f(T v) { return DT<T>::to_f(v); }
template <typename T> __device__ __forceinline__ T from_f(float v) { return DT<T>::from_f(v); }

// Load / store 16 bytes as N values converted to/from float.
template <typename T> struct Vec16 {
  static constexpr int N = 16 / sizeof(T);
};

template <typename T>
__device__ __forceinline__ void load16(const T* p, float* out) {
  uint4 raw = *reinterpret_cast<const uint4*>(p);
  const T* v = reinterpret_cast<const T*>(&raw);
#pragma unroll
  for (int i = 0; i < Vec16<T>::N; ++i) out[i] = to_f(v[i]);
}

template <typename T>
__device__ __forceinline__ void store16(T* p, const float* in) {
  uint4 raw;
  T* v = reinterpret_cast<T*>(&raw);
#pragma unroll
  for (int i = 0; i < Vec16<T>::N; ++i) v[i] = from_f<T>(in[i]);
  *reinterpret_cast<uint4*>(p) = raw;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide reduction; `red` must hold >= 32 floats. All threads get the
// result. Deterministic for a fixed launch shape.
template <bool IS_MAX>
__device__ __forceinline__ float block_reduce(float v, float* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = IS_MAX ? warp_max(v) : warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  float r = (lane < nw) ? red[lane] : (IS_MAX ? -INFINITY : 0.f);
  r = IS_MAX ? warp_max(r) : warp_sum(r);
  return r;
}

// tanh-GELU exactly as runtime.py:97-103 (float32).
__device__ __forceinline__ float gelu_tanh(float u) {
  const float c = 0.7978845608028654f;   // sqrt(2/pi)
  const float a = 0.044715f;
  return u * (0.5f * (1.0f + tanhf(c * (u + a * u * u * u))));
}

// Algorithmic bytes of one GEMM launch: operands once + epilogue traffic.
inline double gemm_bytes(int M, int N, int K, size_t es, const Epi& e) {
  double out = e.mode == EPI_STORE_F32 ? 4.0 : e.mode == EPI_RESID ? 8.0 : (double)es;
  return ((double)M * K + (double)N * K) * es + (double)M * N * out;
}

// Scalar epilogue for one accumulator element. T = layer dtype.
template <typename T>
__device__ __forceinline__ void epi_store(const Epi& e, int m, int n, float acc) {
  switch (e.mode) {
    case EPI_STORE_F32:
      reinterpret_cast<float*>(e.out)[(long long)m * e.ldo + n] = acc;
      break;
    case EPI_STORE_T:
      reinterpret_cast<T*>(e.out)[(long long)m * e.ldo + n] = from_f<T>(acc);
      break;
    case EPI_GELU_T:
      reinterpret_cast<T*>(e.out)[(long long)m * e.ldo + n] = from_f<T>(gelu_tanh(acc));
      break;
    case EPI_RESID: {
      int2 r = e.rinfo[m];
      e.x[r.x * e.x_sb + r.y * e.x_ss + n] += acc;
      break;
    }
    case EPI_QKV: {
      if (n < e.hq) {
        reinterpret_cast<T*>(e.out)[(long long)m * e.hq + n] = from_f<T>(acc);
      } else {
        int which = n >= 2 * e.hq;        // 0 = K, 1 = V
        int w = n - e.hq * (1 + which);
        int head = w / e.hd, d = w - head * e.hd;
        int2 r = e.rinfo[m];
        int slot = (e.kv_start ? *e.kv_start : 0) + e.kv_base + r.y;
        long long off = (((long long)r.x * e.heads + head) * e.smax + slot) * e.hd + d;
        T* dst = reinterpret_cast<T*>(which ? e.vc : e.kc);
        dst[off] = from_f<T>(acc);
      }
      break;
    }
  }
}

template <typename T>
__device__ __forceinline__ void epi_apply(const Epi& e, int m, int n, float acc) {
  if (e.bias) acc += e.bias[n];
  epi_store<T>(e, m, n, acc);
}

// Vector epilogue for 8 consecutive columns n0..n0+7 of row m (n0 % 8 == 0,
// all < N). Falls back to scalar where a vector store would straddle.
template <typename T>
__device__ __forceinline__ void epi_apply8(const Epi& e, int m, int n0, float* v) {
  if (e.bias) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += e.bias[n0 + i];
  }
  switch (e.mode) {
    case EPI_STORE_F32: {
      float* p = reinterpret_cast<float*>(e.out) + (long long)m * e.ldo + n0;
      if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
        reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) p[i] = v[i];
      }
      break;
    }
    case EPI_STORE_T:
    case EPI_GELU_T: {
      if (e.mode == EPI_GELU_T) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = gelu_tanh(v[i]);
      }
      T* p = reinterpret_cast<T*>(e.out) + (long long)m * e.ldo + n0;
      if (sizeof(T) == 2 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
        store16<T>(p, v);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) p[i] = from_f<T>(v[i]);
      }
      break;
    }
    case EPI_RESID: {
      int2 r = e.rinfo[m];
      float* p = e.x + r.x * e.x_sb + r.y * e.x_ss + n0;
      if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
        float4 a = reinterpret_cast<float4*>(p)[0], b = reinterpret_cast<float4*>(p)[1];
        a.x += v[0]; a.y += v[1]; a.z += v[2]; a.w += v[3];
        b.x += v[4]; b.y += v[5]; b.z += v[6]; b.w += v[7];
        reinterpret_cast<float4*>(p)[0] = a;
        reinterpret_cast<float4*>(p)[1] = b;
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) p[i] += v[i];
      }
      break;
    }
    case EPI_QKV: {
      if (sizeof(T) == 2 && (e.hd & 7) == 0 && (e.hq & 7) == 0) {
        if (n0 < e.hq) {
          store16<T>(reinterpret_cast<T*>(e.out) + (long long)m * e.hq + n0, v);
        } else {
          int which = n0 >= 2 * e.hq;
          int w = n0 - e.hq * (1 + which);
          int head = w / e.hd, d = w - head * e.hd;
          int2 r = e.rinfo[m];
          int slot = (e.kv_start ? *e.kv_start : 0) + e.kv_base + r.y;
          long long off = (((long long)r.x * e.heads + head) * e.smax + slot) * e.hd + d;
          store16<T>(reinterpret_cast<T*>(which ? e.vc : e.kc) + off, v);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) epi_store<T>(e, m, n0 + i, v[i]);
      }
      break;
    }
  }
}

}  // namespace eet
