// Thread-block-folded row kernels: LayerNorm (+ pad-skipping pack), the
// operator-level mask-fused softmaxes, embeddings, argmax.
//
// Folding (folding.py:30-54, §2.2): a row of `n` work items is cut
// into t = 2^k sub-blocks of `threads` lanes; lane `tid` of the CTA owns items
// sb*threads + tid for sb < t (folding.py:57-70 map_index). One launch shape
// therefore covers h up to 16384 and seq up to 4096 with <= 1024 threads.
#include "sm100.cuh"

namespace eet {

FoldPlan plan_folding(int logical, int cap) {
  if (cap < 1) cap = 1024;
  int k = 0;
  while (((logical + (1 << k) - 1) >> k) > cap) ++k;
  int t = 1 << k;
  return FoldPlan{k, t, (logical + t - 1) / t};
}

static inline int round32(int n) { return (n + 31) & ~31; }

// ------------------------------------------------------------------ LayerNorm
// y[r] = (x[r] - mean) / sqrt(var_pop + 1e-5) * g + b   (runtime.py:83-94)
// Row r reads x at (rinfo[r].x, rinfo[r].y) when rinfo != null (pad-skipping
// pack: only valid tokens are normalised), else at r * x_sb. VEC float4 lanes
// when h % 4 == 0. Two-pass (mean, then centred second moment) like numpy.
template <typename TO, int VEC, int MAXT>
__global__ void __launch_bounds__(1024) ln_kernel(
    const float* __restrict__ x, long long x_sb, long long x_ss,
    const int2* __restrict__ rinfo, const float* __restrict__ g,
    const float* __restrict__ b, TO* __restrict__ y, int ldy, int h,
    int sub_blocks, int lanes) {
  __shared__ float red[32];
  sm100::griddep_wait();
  sm100::griddep_launch_dependents();
  const int r = blockIdx.x;
  const float* xr;
  if (rinfo) {
    int2 ri = rinfo[r];
    xr = x + ri.x * x_sb + ri.y * x_ss;
  } else {
    xr = x + (long long)r * x_sb;     // no row map: row r at batch stride
  }
  const int nvec = h / VEC;
  float v[MAXT][VEC];
  float s = 0.f;
#pragma unroll
  for (int sb = 0; sb < MAXT; ++sb) {
    int i = sb * lanes + threadIdx.x;
    bool ok = sb < sub_blocks && threadIdx.x < lanes && i < nvec;
    if constexpr (VEC == 4) {
      float4 q = ok ? reinterpret_cast<const float4*>(xr)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      v[sb][0] = q.x; v[sb][1] = q.y; v[sb][2] = q.z; v[sb][3] = q.w;
    } else {
      v[sb][0] = ok ? xr[i] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < VEC; ++j) s += v[sb][j];
  }
  const float mean = block_reduce<false>(s, red) / (float)h;
  float q2 = 0.f;
#pragma unroll
  for (int sb = 0; sb < MAXT; ++sb) {
    int i = sb * lanes + threadIdx.x;
    bool ok = sb < sub_blocks && threadIdx.x < lanes && i < nvec;
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      float d = v[sb][j] - mean;
      q2 += ok ? d * d : 0.f;
    }
  }
  const float var = block_reduce<false>(q2, red) / (float)h;
  const float rstd = 1.0f / sqrtf(var + 1e-5f);
  TO* yr = y + (long long)r * ldy;
#pragma unroll
  for (int sb = 0; sb < MAXT; ++sb) {
    int i = sb * lanes + threadIdx.x;
    if (!(sb < sub_blocks && threadIdx.x < lanes && i < nvec)) continue;
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      int c = i * VEC + j;
      yr[c] = from_f<TO>((v[sb][j] - mean) * rstd * g[c] + b[c]);
    }
  }
}

// Row-group LayerNorm for the layer path: W warps own one row (folded into
// NV float4 sub-blocks per lane, the same folding as above with a fixed
// 32*W-lane unit), 8/W rows per 256-thread CTA, warp-shuffle reductions,
// float4 loads of x / gamma / beta and 8-16 B packed stores. Two-pass
// statistics (mean, then centred second moment) as numpy.
template <int W>
__device__ __forceinline__ float row_sum(float v, float (*red)[2], int slot, int warp, int lane) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if constexpr (W == 1) {
    return v;
  } else {
    if (lane == 0) red[warp][slot] = v;
    __syncthreads();
    const int base = (warp / W) * W;
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) t += red[base + w][slot];
    return t;
  }
}

template <typename TO, int W, int NV>
__global__ void __launch_bounds__(256) ln_rows_kernel(
    const float* __restrict__ x, long long x_sb, long long x_ss, const int2* __restrict__ rinfo,
    const float* __restrict__ g, const float* __restrict__ b, TO* __restrict__ y, int ldy, int h,
    int rows) {
  __shared__ float red[8][2];
  sm100::griddep_wait();
  sm100::griddep_launch_dependents();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * (8 / W) + warp / W;
  const int tid = (warp % W) * 32 + lane;
  const bool active = r < rows;
  const float* xr = x;
  if (active) {
    if (rinfo) {
      const int2 ri = rinfo[r];
      xr = x + ri.x * x_sb + ri.y * x_ss;
    } else {
      xr = x + (long long)r * x_sb;
    }
  }
  const int nvec = h >> 2;
  float4 v[NV];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int idx = i * 32 * W + tid;
    v[i] = (active && idx < nvec) ? __ldg(reinterpret_cast<const float4*>(xr) + idx)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
    s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
  const float mean = row_sum<W>(s, red, 0, warp, lane) / (float)h;
  float q2 = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int idx = i * 32 * W + tid;
    if (active && idx < nvec) {
      const float a = v[i].x - mean, c = v[i].y - mean, d = v[i].z - mean, e = v[i].w - mean;
      q2 += (a * a + c * c) + (d * d + e * e);
    }
  }
  const float rstd = 1.0f / sqrtf(row_sum<W>(q2, red, 1, warp, lane) / (float)h + 1e-5f);
  if (!active) return;
  TO* yr = y + (long long)r * ldy;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int idx = i * 32 * W + tid;
    if (idx >= nvec) continue;
    const float4 gg = __ldg(reinterpret_cast<const float4*>(g) + idx);
    const float4 bb = __ldg(reinterpret_cast<const float4*>(b) + idx);
    const float o0 = (v[i].x - mean) * rstd * gg.x + bb.x;
    const float o1 = (v[i].y - mean) * rstd * gg.y + bb.y;
    const float o2 = (v[i].z - mean) * rstd * gg.z + bb.z;
    const float o3 = (v[i].w - mean) * rstd * gg.w + bb.w;
    if constexpr (sizeof(TO) == 4) {
      reinterpret_cast<float4*>(yr)[idx] = make_float4(o0, o1, o2, o3);
    } else {
      TO t[4] = {from_f<TO>(o0), from_f<TO>(o1), from_f<TO>(o2), from_f<TO>(o3)};
      reinterpret_cast<uint2*>(yr)[idx] = *reinterpret_cast<const uint2*>(t);
    }
  }
}

// rows kernel when the shape allows (h % 4, 16-byte aligned rows, output
// rows 8/16-byte aligned); returns false otherwise
template <typename TO>
static bool ln_rows_dispatch(const float* x, long long x_sb, long long x_ss, const int2* rinfo,
                             int rows, const float* g, const float* b, TO* y, int ldy, int h,
                             cudaStream_t st) {
  const uintptr_t al = reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(g) |
                       reinterpret_cast<uintptr_t>(b);
  if (h % 4 || (al & 15) || (x_ss & 3) || (x_sb & 3) || (!rinfo && x_sb == 0) ||
      (ldy % 4) || (reinterpret_cast<uintptr_t>(y) & (sizeof(TO) * 4 - 1)))
    return false;
  const int nvec = h / 4;
  int W = 1;
  while (W < 8 && (nvec + 32 * W - 1) / (32 * W) > 8) W *= 2;
  const int nv = (nvec + 32 * W - 1) / (32 * W);
  ProfScope ps(K_LAYERNORM, st, (double)rows * h * (4 + sizeof(TO)) + 8.0 * h, 8.0 * rows * h);
#define LNR(W_, NV_)                                                                          \
  if (W == W_ && nv <= NV_) {                                                                 \
    launch_ex(ln_rows_kernel<TO, W_, NV_>, dim3((rows + 8 / W_ - 1) / (8 / W_)), dim3(256), 0, st, \
              true, dim3(1, 1, 1), x, x_sb, x_ss, rinfo, g, b, y, ldy, h, rows);             \
    EET_LAUNCH_CHECK();                                                                       \
    return true;                                                                              \
  }
  LNR(1, 2) LNR(1, 4) LNR(1, 8) LNR(2, 8) LNR(4, 8) LNR(8, 8) LNR(8, 12) LNR(8, 16)
#undef LNR
  return false;
}

template <typename TO, int VEC>
static void ln_dispatch(const float* x, long long x_sb, long long x_ss, const int2* rinfo, int rows,
                        const float* g, const float* b, TO* y, int ldy, int h, int cap,
                        cudaStream_t st) {
  FoldPlan p = plan_folding(h / VEC, cap);
  int threads = round32(p.threads);
  EET_REQUIRE(threads <= 1024, EET_ERR_ARG, "layer norm: fold cap too large");
#define LN_CASE(T_)                                                                      \
  if (p.sub_blocks <= T_) {                                                              \
    ProfScope ps(K_LAYERNORM, st, (double)rows * h * (4 + sizeof(TO)) + 8.0 * h, 8.0 * rows * h); \
    launch_ex(ln_kernel<TO, VEC, T_>, dim3(rows), dim3(threads), 0, st, true, dim3(1, 1, 1), x,   \
              x_sb, x_ss, rinfo, g, b, y, ldy, h, p.sub_blocks, p.threads);              \
    EET_LAUNCH_CHECK();                                                                  \
    return;                                                                              \
  }
  LN_CASE(1) LN_CASE(2) LN_CASE(4) LN_CASE(8) LN_CASE(16)
#undef LN_CASE
  EET_REQUIRE(false, EET_ERR_UNSUPPORTED, "layer norm: hidden too large for the fold cap");
}

void launch_layer_norm(const float* x, long long x_sb, long long x_ss, const int2* rinfo,
                       int rows, const float* g, const float* b, void* y, int y_dtype, int ldy,
                       int h, int cap, cudaStream_t st) {
  if (rows <= 0) return;
  EET_REQUIRE(h >= 1 && h <= 16384, EET_ERR_ARG, "layer norm: hidden outside [1, 16384]");
  if (cap == 0) {          // layer path: row-group kernel; explicit fold caps keep the folded CTA shape
    const bool done =
        y_dtype == EET_F32    ? ln_rows_dispatch(x, x_sb, x_ss, rinfo, rows, g, b, (float*)y, ldy, h, st)
        : y_dtype == EET_BF16 ? ln_rows_dispatch(x, x_sb, x_ss, rinfo, rows, g, b, (__nv_bfloat16*)y, ldy, h, st)
                              : ln_rows_dispatch(x, x_sb, x_ss, rinfo, rows, g, b, (__half*)y, ldy, h, st);
    if (done) return;
  }
  bool v4 = (h % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0) &&
            (x_ss % 4 == 0) && (x_sb % 4 == 0) && (rinfo || x_sb != 0);
  switch (y_dtype) {
    case EET_F32:
      v4 ? ln_dispatch<float, 4>(x, x_sb, x_ss, rinfo, rows, g, b, (float*)y, ldy, h, cap, st)
         : ln_dispatch<float, 1>(x, x_sb, x_ss, rinfo, rows, g, b, (float*)y, ldy, h, cap, st);
      break;
    case EET_BF16:
      v4 ? ln_dispatch<__nv_bfloat16, 4>(x, x_sb, x_ss, rinfo, rows, g, b, (__nv_bfloat16*)y, ldy, h, cap, st)
         : ln_dispatch<__nv_bfloat16, 1>(x, x_sb, x_ss, rinfo, rows, g, b, (__nv_bfloat16*)y, ldy, h, cap, st);
      break;
    default:
      v4 ? ln_dispatch<__half, 4>(x, x_sb, x_ss, rinfo, rows, g, b, (__half*)y, ldy, h, cap, st)
         : ln_dispatch<__half, 1>(x, x_sb, x_ss, rinfo, rows, g, b, (__half*)y, ldy, h, cap, st);
  }
}

// ------------------------------------------------------- mask-fused softmax
// One CTA per query row of one (batch, head) plane; window bounds come from
// the row index and the sequence's pad offset — no mask tensor exists.
// Window: causal [pad, i], bidirectional [pad, s); pad-query rows (i < pad)
// and everything outside the window are written as exact zeros
// (attention.py:73-135). Reductions run sub-block by sub-block in fixed
// order, so results are deterministic for a fixed plan (attention.py:55-66).
__global__ void __launch_bounds__(1024) masked_softmax_kernel(
    float* __restrict__ s, const int* __restrict__ pads, int heads, int seq, int causal,
    int sub_blocks, int lanes) {
  __shared__ float red[32];
  const int i = blockIdx.x;             // query row
  const int plane = blockIdx.y;         // b * heads + head
  const int pad = pads[plane / heads];
  float* row = s + ((long long)plane * seq + i) * seq;
  const int lo = pad, hi = causal ? i + 1 : seq;
  const bool live = i >= pad;
  float m = -INFINITY;
  if (live) {
    for (int sb = 0; sb < sub_blocks; ++sb) {
      int j = sb * lanes + threadIdx.x;
      if (threadIdx.x < lanes && j >= lo && j < hi) m = fmaxf(m, row[j]);
    }
  }
  m = block_reduce<true>(m, red);
  float sum = 0.f;
  if (live) {
    for (int sb = 0; sb < sub_blocks; ++sb) {
      int j = sb * lanes + threadIdx.x;
      if (threadIdx.x < lanes && j >= lo && j < hi) sum += expf(row[j] - m);
    }
  }
  sum = block_reduce<false>(sum, red);
  for (int sb = 0; sb < sub_blocks; ++sb) {
    int j = sb * lanes + threadIdx.x;
    if (threadIdx.x < lanes && j < seq) {
      float o = 0.f;
      if (live && j >= lo && j < hi) o = expf(row[j] - m) / sum;
      row[j] = o;
    }
  }
}

void launch_masked_softmax(float* s, const int* pads, int batch, int heads, int seq, int causal,
                           int cap, cudaStream_t st) {
  if (batch * heads == 0 || seq == 0) return;
  FoldPlan p = plan_folding(seq, cap);
  int threads = round32(p.threads);
  EET_REQUIRE(threads <= 1024, EET_ERR_ARG, "softmax: fold cap too large");
  dim3 grid(seq, batch * heads);
  ProfScope ps(K_SOFTMAX, st, 8.0 * batch * heads * seq * seq, 3.0 * batch * heads * seq * seq);
  masked_softmax_kernel<<<grid, threads, 0, st>>>(s, pads, heads, seq, causal, p.sub_blocks,
                                                  p.threads);
  EET_LAUNCH_CHECK();
}

// Decode-step softmax over [b, heads, L]: window [pad_b, L) (attention.py:138-163).
__global__ void __launch_bounds__(1024) step_softmax_kernel(
    float* __restrict__ s, const int* __restrict__ pads, int heads, int len, int sub_blocks,
    int lanes) {
  __shared__ float red[32];
  const int plane = blockIdx.x;
  const int pad = pads[plane / heads];
  float* row = s + (long long)plane * len;
  float m = -INFINITY;
  for (int sb = 0; sb < sub_blocks; ++sb) {
    int j = sb * lanes + threadIdx.x;
    if (threadIdx.x < lanes && j >= pad && j < len) m = fmaxf(m, row[j]);
  }
  m = block_reduce<true>(m, red);
  float sum = 0.f;
  for (int sb = 0; sb < sub_blocks; ++sb) {
    int j = sb * lanes + threadIdx.x;
    if (threadIdx.x < lanes && j >= pad && j < len) sum += expf(row[j] - m);
  }
  sum = block_reduce<false>(sum, red);

  for (int sb = 0; sb < sub_blocks; ++sb) {
    int j = sb * lanes + threadIdx.x;
    if (threadIdx.x < lanes && j < len) row[j] = (j >= pad) ? expf(row[j] - m) / sum : 0.f;
  }
}

void launch_step_softmax(float* s, const int* pads, int batch, int heads, int len, int cap,
                         cudaStream_t st) {
  if (batch * heads == 0 || len == 0) return;
  FoldPlan p = plan_folding(len, cap);
  int threads = round32(p.threads);
  EET_REQUIRE(threads <= 1024, EET_ERR_ARG, "softmax: fold cap too large");
  ProfScope ps(K_SOFTMAX, st, 8.0 * batch * heads * len, 3.0 * batch * heads * len);
  step_softmax_kernel<<<batch * heads, threads, 0, st>>>(s, pads, heads, len, p.sub_blocks,
                                                         p.threads);
  EET_LAUNCH_CHECK();
}

// --------------------------------------------------------------- embeddings
// Prompt: slot < pad -> zero row; else tok_emb[id] + pos_emb[slot - pad]
// (runtime.py:304-323; logical positions).
template <typename T>
__global__ void embed_prompt_kernel(const T* __restrict__ tok, const T* __restrict__ pos,
                                    const int* __restrict__ prompts, int max_len,
                                    const int* __restrict__ pads, float* __restrict__ x,
                                    long long x_sb, int t, int h) {
  const int slot = blockIdx.x, b = blockIdx.y;
  const int pad = pads[b];
  float* xr = x + b * x_sb + (long long)slot * h;
  if (slot < pad) {
    for (int c = threadIdx.x; c < h; c += blockDim.x) xr[c] = 0.f;
    return;
  }
  const int p = slot - pad;
  const int id = prompts[b * max_len + p];
  const T* tr = tok + (long long)id * h;
  const T* pr = pos + (long long)p * h;
  for (int c = threadIdx.x; c < h; c += blockDim.x) xr[c] = to_f(tr[c]) + to_f(pr[c]);
}

// Step: one token per sequence at absolute slot *d_filled (runtime.py:326-338).
template <typename T>
__global__ void embed_step_kernel(const T* __restrict__ tok, const T* __restrict__ pos,
                                  const int* __restrict__ cur, const int* __restrict__ pads,
                                  const int* __restrict__ d_filled, float* __restrict__ x,
                                  long long x_sb, int h) {
  sm100::griddep_wait();
  sm100::griddep_launch_dependents();
  const int b = blockIdx.x;
  const int p = *d_filled - pads[b];
  const T* tr = tok + (long long)cur[b] * h;
  const T* pr = pos + (long long)p * h;
  float* xr = x + b * x_sb;
  for (int c = threadIdx.x; c < h; c += blockDim.x) xr[c] = to_f(tr[c]) + to_f(pr[c]);
}

void launch_embed_prompt(int dtype, const void* tok, const void* pos, const int* prompts,
                         int max_len, const int* pads, float* x, long long x_sb, int batch, int t,
                         int h, cudaStream_t st) {
  dim3 grid(t, batch);
  int threads = std::min(256, round32(h));
  ProfScope ps(K_EMBED, st, (double)batch * t * h * (4 + 2 * dtype_size(dtype)), 1.0 * batch * t * h);
  if (dtype == EET_F32)
    embed_prompt_kernel<float><<<grid, threads, 0, st>>>((const float*)tok, (const float*)pos, prompts, max_len, pads, x, x_sb, t, h);
  else if (dtype == EET_BF16)
    embed_prompt_kernel<__nv_bfloat16><<<grid, threads, 0, st>>>((const __nv_bfloat16*)tok, (const __nv_bfloat16*)pos, prompts, max_len, pads, x, x_sb, t, h);
  else
    embed_prompt_kernel<__half><<<grid, threads, 0, st>>>((const __half*)tok, (const __half*)pos, prompts, max_len, pads, x, x_sb, t, h);
  EET_LAUNCH_CHECK();
}

void launch_embed_step(int dtype, const void* tok, const void* pos, const int* cur,
                       const int* pads, const int* d_filled, float* x, long long x_sb, int batch,
                       int h, cudaStream_t st) {
  int threads = std::min(256, round32(h));
  ProfScope ps(K_EMBED, st, (double)batch * h * (4 + 2 * dtype_size(dtype)), 1.0 * batch * h);
  const dim3 one(1, 1, 1);
  if (dtype == EET_F32)
    launch_ex(embed_step_kernel<float>, dim3(batch), dim3(threads), 0, st, true, one, (const float*)tok, (const float*)pos, cur, pads, d_filled, x, x_sb, h);
  else if (dtype == EET_BF16)
    launch_ex(embed_step_kernel<__nv_bfloat16>, dim3(batch), dim3(threads), 0, st, true, one, (const __nv_bfloat16*)tok, (const __nv_bfloat16*)pos, cur, pads, d_filled, x, x_sb, h);
  else
    launch_ex(embed_step_kernel<__half>, dim3(batch), dim3(threads), 0, st, true, one, (const __half*)tok, (const __half*)pos, cur, pads, d_filled, x, x_sb, h);
  EET_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ argmax
// Greedy next token, lowest id on ties (runtime.py:425, np.argmax). Also
// records the token at step *d_step and optionally copies the logits row.
__global__ void __launch_bounds__(1024) argmax_kernel(
    const float* __restrict__ logits, int vocab, int* __restrict__ cur,
    long long* __restrict__ toks, int steps, const int* __restrict__ d_step,
    float* __restrict__ logits_all, int batch) {
  __shared__ float sv[32];
  __shared__ int si[32];
  sm100::griddep_wait();
  sm100::griddep_launch_dependents();
  const int b = blockIdx.x;
  const float* row = logits + (long long)b * vocab;
  const int step = d_step ? *d_step : 0;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int j = threadIdx.x; j < vocab; j += blockDim.x) {
    float v = row[j];
    if (v > best || (v == best && j < bi)) { best = v; bi = j; }
    if (logits_all && step < steps) logits_all[((long long)step * batch + b) * vocab + j] = v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { sv[wid] = best; si[wid] = bi; }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    best = lane < nw ? sv[lane] : -INFINITY;
    bi = lane < nw ? si[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float ov = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) {
      if (bi == 0x7fffffff) bi = 0;      // all-NaN row: numpy returns 0
      cur[b] = bi;
      if (toks && step < steps) toks[(long long)b * steps + step] = bi;
    }
  }
}

void launch_argmax(const float* logits, int batch, int vocab, int* cur, long long* toks,
                   int steps, const int* d_step, float* logits_all, cudaStream_t st) {
  ProfScope ps(K_ARGMAX, st, 4.0 * batch * vocab * (logits_all ? 2 : 1), 1.0 * batch * vocab);
  launch_ex(argmax_kernel, dim3(batch), dim3(1024), 0, st, true, dim3(1, 1, 1), logits, vocab, cur,
            toks, steps, d_step, logits_all, batch);
  EET_LAUNCH_CHECK();
}

// x[valid row m] += reduced[m] : the residual add after a tensor-parallel
// all-reduce (runtime.py:259 / :212 across shards). The reduced partial is
// fp32 (fp32 mode) or the layer dtype (16-bit modes: half the NVLink bytes).
template <typename R>
__global__ void residual_add_kernel(float* __restrict__ x, long long x_sb, long long x_ss,
                                    const int2* __restrict__ rinfo, const R* __restrict__ r,
                                    int h) {
  sm100::griddep_wait();
  sm100::griddep_launch_dependents();
  const int m = blockIdx.x;
  const int2 ri = rinfo[m];
  float* xr = x + ri.x * x_sb + ri.y * x_ss;
  const R* rr = r + (long long)m * h;
  for (int c = threadIdx.x; c < h; c += blockDim.x) xr[c] += to_f(rr[c]);
}

void launch_residual_add(float* x, long long x_sb, long long x_ss, const int2* rinfo,
                         const void* reduced, int dtype, int rows, int h, cudaStream_t st) {
  if (rows <= 0) return;
  ProfScope ps(K_LAYERNORM, st, (8.0 + dtype_size(dtype)) * rows * h, 1.0 * rows * h);
  if (dtype == EET_F32)
    launch_ex(residual_add_kernel<float>, dim3(rows), dim3(256), 0, st, true, dim3(1, 1, 1), x, x_sb, x_ss,
              rinfo, reinterpret_cast<const float*>(reduced), h);
  else if (dtype == EET_BF16)
    launch_ex(residual_add_kernel<__nv_bfloat16>, dim3(rows), dim3(256), 0, st, true, dim3(1, 1, 1), x, x_sb,
              x_ss, rinfo, reinterpret_cast<const __nv_bfloat16*>(reduced), h);
  else
    launch_ex(residual_add_kernel<__half>, dim3(rows), dim3(256), 0, st, true, dim3(1, 1, 1), x, x_sb, x_ss,
              rinfo, reinterpret_cast<const __half*>(reduced), h);
  EET_LAUNCH_CHECK();
}

__global__ void advance_kernel(int* d_filled, int* d_step) {
  sm100::griddep_wait();
  sm100::griddep_launch_dependents();
  *d_filled += 1;
  *d_step += 1;
}

void launch_advance(int* d_filled, int* d_step, cudaStream_t st) {
  ProfScope ps(K_ADVANCE, st, 16.0, 2.0);
  launch_ex(advance_kernel, dim3(1), dim3(1), 0, st, true, dim3(1, 1, 1), d_filled, d_step);
  EET_LAUNCH_CHECK();
}

// ------------------------------------------------- launch-chain calibration
// n back-to-back dependent launches of a (nearly) empty kernel, with or
// without programmatic dependent launch: the per-link floor of a decode graph
__global__ void empty_link_kernel(int* p) {
  sm100::griddep_wait();
  sm100::griddep_launch_dependents();
  if (p && threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(p, 1);
}

// ------------------------------------------------------- weight packing
// dst[c][r] = cast(src[r][c]): the reference's [in, out] float32 matrices
// (weights.py:31-51, MFW1 payload order) become the kernels' K-major
// [out, in] layout in the compute dtype, on the device, in one pass
// through a 32x33 shared tile (coalesced reads and writes).
template <typename T>
__global__ void transpose_cast_kernel(const float* __restrict__ src, int rows, int cols,
                                      T* __restrict__ dst) {
  __shared__ float tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = src[(size_t)r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (c < cols && r < rows) dst[(size_t)c * rows + r] = from_f<T>(tile[threadIdx.x][i]);
  }
}

extern "C" int eet_transpose_cast(int dtype, const float* src, int rows, int cols, void* dst,
                                  void* stream) {
  try {
    EET_REQUIRE(src && dst, EET_ERR_ARG, "transpose_cast: null pointer");
    EET_REQUIRE(rows >= 0 && cols >= 0, EET_ERR_SHAPE, "transpose_cast: negative extent");
    if (rows == 0 || cols == 0) return EET_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const dim3 grid((cols + 31) / 32, (rows + 31) / 32), block(32, 8);
    EET_REQUIRE(grid.y <= 65535u, EET_ERR_SHAPE, "transpose_cast: too many rows");
    if (dtype == EET_F32)
      transpose_cast_kernel<float><<<grid, block, 0, st>>>(src, rows, cols, static_cast<float*>(dst));
    else if (dtype == EET_BF16)
      transpose_cast_kernel<__nv_bfloat16><<<grid, block, 0, st>>>(src, rows, cols, static_cast<__nv_bfloat16*>(dst));
    else if (dtype == EET_F16)
      transpose_cast_kernel<__half><<<grid, block, 0, st>>>(src, rows, cols, static_cast<__half*>(dst));
    else
      EET_REQUIRE(false, EET_ERR_ARG, "transpose_cast: unknown dtype");
    count_launch();
    EET_LAUNCH_CHECK();
    return EET_OK;
  } catch (const Fail& f) {
    return f.code;
  }
}

}  // namespace eet

extern "C" int eet_debug_launch_chain(int n, int ctas, int pdl, int* counter, void* stream) {
  try {
    for (int i = 0; i < n; ++i) {
      eet::launch_ex(eet::empty_link_kernel, dim3(ctas), dim3(128), 0, reinterpret_cast<cudaStream_t>(stream),
                     pdl != 0, dim3(1, 1, 1), counter);
      EET_CHECK_CUDA(cudaGetLastError());
    }
    return EET_OK;
  } catch (const eet::Fail& f) {
    return f.code;
  }
}
