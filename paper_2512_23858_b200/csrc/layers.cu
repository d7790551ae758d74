// Forward-pass ops other than the GEMM: embedding gather, RMSNorm, tree/prefix attention
// (SIMT variant for both dtypes; the tcgen05 variant lives in attn_tc.cu), per-row logit
// statistics for greedy / sampled acceptance, and the K8 on-device stage timer.
#include <cmath>

#include "common.cuh"
#include "host_util.h"

namespace ygg {

template <typename T>
__global__ void embed_kernel(const T* __restrict__ table, int V, int d, const int32_t* __restrict__ tokens,
                             float* __restrict__ out) {
  // One CTA per row, 8 features per thread with every load in flight at once (a strided loop would
  // serialise one round trip per iteration).
  pdl_wait();
  pdl_launch_dependents();
  const int m = blockIdx.x;
  int tok = tokens[m];
  tok = tok < 0 ? 0 : (tok >= V ? V - 1 : tok);
  const T* row = table + static_cast<size_t>(tok) * d;
  const int n = threadIdx.x * 8;
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = n + i < d ? to_f32(row[n + i]) : 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (n + i < d) out[static_cast<size_t>(m) * d + n + i] = v[i];
}

// Embedding + the first RMSNorm in one pass (verify / AR / prefill entry): one CTA per row, 8
// features per thread; writes the f32 residual and the normalised activations.  Same arithmetic as
// embed_kernel followed by rmsnorm_kernel.
template <typename T>
__global__ void __launch_bounds__(1024) embed_rmsnorm_kernel(const T* __restrict__ table, int V, int d,
                                                             const int32_t* __restrict__ tokens,
                                                             const T* __restrict__ w, float eps,
                                                             float* __restrict__ resid, T* __restrict__ xn) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ float red[32];
  const int m = blockIdx.x;
  int tok = tokens[m];
  tok = tok < 0 ? 0 : (tok >= V ? V - 1 : tok);
  const T* row = table + static_cast<size_t>(tok) * d;
  const int n = threadIdx.x * 8;
  float v[8], g[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = n + i < d ? to_f32(row[n + i]) : 0.f;
    g[i] = n + i < d ? to_f32(w[n + i]) : 0.f;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (n + i < d) resid[static_cast<size_t>(m) * d + n + i] = v[i];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) ss += v[i] * v[i];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float t = 0.f;
  for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) t += red[k];
  const float r = rsqrtf(t / static_cast<float>(d) + eps);
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (n + i < d) xn[static_cast<size_t>(m) * d + n + i] = from_f32<T>(v[i] * r * g[i]);
}

// Embedding for the fused path: one CTA per token row, d/8 threads with 8 features (one 16-byte
// load) each, so the whole row is a single round trip.  Writes the f32 residual, its bf16 copy
// (next GEMM operand) and each 128-feature tile's sum of squares (16 threads per tile, fixed xor
// order: deterministic).
__global__ void __launch_bounds__(1024) embed_fused_kernel(const __nv_bfloat16* __restrict__ table, int V, int d,
                                                           const int32_t* __restrict__ tokens, float* __restrict__ resid,
                                                           __nv_bfloat16* __restrict__ hb, float* __restrict__ ss_out,
                                                           int M, unsigned long long* trace) {
  if (threadIdx.x == 0) trace_min(trace, 0);
  pdl_wait();
  if (threadIdx.x == 0) trace_min(trace, 1);
  pdl_launch_dependents();
  const int m = blockIdx.x;
  int tok = tokens[m];
  tok = tok < 0 ? 0 : (tok >= V ? V - 1 : tok);
  const int n = threadIdx.x * 8;
  float s = 0.f;
  if (n < d) {
    const uint4 raw = __ldg(reinterpret_cast<const uint4*>(table + static_cast<size_t>(tok) * d + n));
    const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
    float h[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
      h[2 * i] = __bfloat162float(b.x);
      h[2 * i + 1] = __bfloat162float(b.y);
    }
    float4* rp = reinterpret_cast<float4*>(resid + static_cast<size_t>(m) * d + n);
    rp[0] = make_float4(h[0], h[1], h[2], h[3]);
    rp[1] = make_float4(h[4], h[5], h[6], h[7]);
    *reinterpret_cast<uint4*>(hb + static_cast<size_t>(m) * d + n) = raw;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += h[i] * h[i];
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (n < d && (threadIdx.x & 15) == 0) ss_out[static_cast<size_t>(n / 128) * M + m] = s;
  if (threadIdx.x == 0) trace_max(trace, 2);
}

template <typename T>
__global__ void __launch_bounds__(1024) rmsnorm_kernel(const float* __restrict__ x, const T* __restrict__ w, int d,
                                                       float eps, T* __restrict__ out) {
  // One CTA per row, 8 features per thread, all loads in flight at once; one block reduction
  // (warp sums, then the warps' sums in fixed order: deterministic).
  pdl_wait();
  pdl_launch_dependents();
  __shared__ float red[32];
  const int m = blockIdx.x;
  const float* row = x + static_cast<size_t>(m) * d;
  const int n = threadIdx.x * 8;
  float v[8], g[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = n + i < d ? row[n + i] : 0.f;
    g[i] = n + i < d ? to_f32(w[n + i]) : 0.f;
  }
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) ss += v[i] * v[i];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float t = 0.f;
  for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) t += red[k];
  const float r = rsqrtf(t / static_cast<float>(d) + eps);
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (n + i < d) out[static_cast<size_t>(m) * d + n + i] = from_f32<T>(v[i] * r * g[i]);
}

// ---------------------------------------------------------------------------
// SIMT attention.  CTA = (query chunk, kv head, request); rows = chunk tokens x G q-heads.
// 4 consecutive lanes own one row for both the score and the P.V stage.
// ---------------------------------------------------------------------------
constexpr int kAttnRows = 64;
constexpr int kAttnKeys = 32;
constexpr int kAttnThreads = 256;

template <typename T, int HD>
__global__ void __launch_bounds__(kAttnThreads) attn_simt_kernel(
    const T* __restrict__ q, const T* __restrict__ cache, int T_per_req, int Hq, int Hkv, int S,
    const int32_t* __restrict__ blk_start, const int32_t* __restrict__ blk_len, const uint32_t* __restrict__ qmask,
    int mask_words, float scale_log2, T* __restrict__ out) {
  pdl_wait();
  pdl_launch_dependents();
  const int G = Hq / Hkv;
  const int qc = kAttnRows / G;  // query tokens per CTA
  const int r = blockIdx.z, kvh = blockIdx.y;
  const int t0 = blockIdx.x * qc;
  extern __shared__ float attn_smem[];
  float (*sq)[HD + 1] = reinterpret_cast<float (*)[HD + 1]>(attn_smem);
  float (*sk)[HD + 1] = reinterpret_cast<float (*)[HD + 1]>(attn_smem + kAttnRows * (HD + 1));
  float (*sv)[HD + 1] = reinterpret_cast<float (*)[HD + 1]>(attn_smem + (kAttnRows + kAttnKeys) * (HD + 1));
  const int tid = threadIdx.x;
  const int row = tid >> 2, sub = tid & 3;
  const int tq = t0 + row / G;            // query token within request
  const int head = kvh * G + row % G;      // q head
  const bool row_valid = (row < qc * G) && (tq < T_per_req);
  const int m = r * T_per_req + tq;        // global query row
  for (int i = tid; i < kAttnRows * HD; i += kAttnThreads) {
    const int rr = i / HD, dd = i % HD;
    const int tt = t0 + rr / G, hh = kvh * G + rr % G;
    float v = 0.f;
    if (rr < qc * G && tt < T_per_req) v = to_f32(q[(static_cast<size_t>(r * T_per_req + tt) * Hq + hh) * HD + dd]);
    sq[rr][dd] = v;
  }
  const int bs = blk_start[r], bl = blk_len[r];
  const int nkeys = bs + bl;
  const T* kbase = cache + ((static_cast<size_t>(r) * 2 + 0) * Hkv + kvh) * static_cast<size_t>(S) * HD;
  const T* vbase = cache + ((static_cast<size_t>(r) * 2 + 1) * Hkv + kvh) * static_cast<size_t>(S) * HD;
  const uint32_t* mrow = (qmask && row_valid) ? qmask + static_cast<size_t>(m) * mask_words : nullptr;
  constexpr int DPT = HD / 4;  // output dims per thread
  float o[DPT];
#pragma unroll
  for (int i = 0; i < DPT; ++i) o[i] = 0.f;
  float mx = -INFINITY, l = 0.f;
  for (int k0 = 0; k0 < nkeys; k0 += kAttnKeys) {
    __syncthreads();
    for (int i = tid; i < kAttnKeys * HD; i += kAttnThreads) {
      const int kk = i / HD, dd = i % HD;
      const int key = k0 + kk;
      float kv = 0.f, vv = 0.f;
      if (key < nkeys) {
        kv = to_f32(kbase[static_cast<size_t>(key) * HD + dd]);
        vv = to_f32(vbase[static_cast<size_t>(dd) * S + key]);  // V^T [hd][S]
      }
      sk[kk][dd] = kv;
      sv[kk][dd] = vv;
    }
    __syncthreads();
    float sc[8];
    float tmax = -INFINITY;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int kk = sub * 8 + j;
      const int key = k0 + kk;
      bool vis = row_valid && key < nkeys;
      if (vis && key >= bs) {
        const int jb = key - bs;
        if (mrow) vis = (mrow[jb >> 5] >> (jb & 31)) & 1u;
        else vis = jb <= tq;  // causal block
      }
      float s = -INFINITY;
      if (vis) {
        float acc = 0.f;
#pragma unroll 16
        for (int d = 0; d < HD; ++d) acc = fmaf(sq[row][d], sk[kk][d], acc);
        s = acc * scale_log2;
      }
      sc[j] = s;
      tmax = fmaxf(tmax, s);
    }
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
    const float new_mx = fmaxf(mx, tmax);
    const float corr = (new_mx == -INFINITY) ? 1.f : exp2f(mx - new_mx);
    float psum = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sc[j] = (sc[j] == -INFINITY) ? 0.f : exp2f(sc[j] - new_mx);
      psum += sc[j];
    }
    psum += __shfl_xor_sync(0xffffffffu, psum, 1);
    psum += __shfl_xor_sync(0xffffffffu, psum, 2);
    l = l * corr + psum;
    mx = new_mx;
#pragma unroll
    for (int i = 0; i < DPT; ++i) o[i] *= corr;
    // P.V: gather the row's 32 probabilities from the 4 lanes of the row.
#pragma unroll
    for (int src = 0; src < 4; ++src) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float p = __shfl_sync(0xffffffffu, sc[j], (threadIdx.x & ~3) | src);
        const int kk = src * 8 + j;
#pragma unroll
        for (int i = 0; i < DPT; ++i) o[i] = fmaf(p, sv[kk][sub * DPT + i], o[i]);
      }
    }
  }
  if (row_valid) {
    const float inv = l > 0.f ? 1.f / l : 0.f;
    T* dst = out + (static_cast<size_t>(m) * Hq + head) * HD + sub * DPT;
#pragma unroll
    for (int i = 0; i < DPT; ++i) dst[i] = from_f32<T>(o[i] * inv);
  }
}

// Per-row max, argmax (first max) and log-sum-exp(x / T); f64 accumulation, fixed order.
// One 1024-thread CTA per row, float4 loads when the row is 16-byte aligned; the log-sum-exp
// pass runs only when `stats` is requested (sampling), greedy acceptance needs the argmax alone.
constexpr int kRowStatsThreads = 1024;
template <typename T>
__global__ void __launch_bounds__(kRowStatsThreads) row_stats_kernel(const T* __restrict__ logits, int V, int ld,
                                                                     float inv_temp, int32_t* __restrict__ argmax,
                                                                     float* __restrict__ stats) {
  pdl_wait();
  pdl_launch_dependents();
  constexpr int NW = kRowStatsThreads / 32;
  const int row = blockIdx.x;
  const T* x = logits + static_cast<size_t>(row) * ld;
  __shared__ float smax[NW];
  __shared__ int sarg[NW];
  __shared__ double ssum[NW];
  float bm = -INFINITY;
  int ba = 0x7fffffff;
  auto take = [&](float f, int v) {
    if (f > bm || (f == bm && v < ba)) { bm = f; ba = v; }
  };
  if constexpr (sizeof(T) == 4) {
    if ((reinterpret_cast<uintptr_t>(x) & 15) == 0) {
      const int nv = V >> 2;
      const float4* x4 = reinterpret_cast<const float4*>(x);
      // 8 loads in flight per thread (through L2: the logits were just written by the LM head).
      int i = threadIdx.x;
      for (; i + 7 * kRowStatsThreads < nv; i += 8 * kRowStatsThreads) {
        float4 q[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) q[u] = __ldcg(x4 + i + u * kRowStatsThreads);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int b = 4 * (i + u * kRowStatsThreads);
          take(q[u].x, b); take(q[u].y, b + 1); take(q[u].z, b + 2); take(q[u].w, b + 3);
        }
      }
      for (; i < nv; i += kRowStatsThreads) {
        const float4 q = __ldcg(x4 + i);
        take(q.x, 4 * i); take(q.y, 4 * i + 1); take(q.z, 4 * i + 2); take(q.w, 4 * i + 3);
      }
      for (int v = (nv << 2) + threadIdx.x; v < V; v += kRowStatsThreads) take(to_f32(x[v]), v);
    } else {
      for (int v = threadIdx.x; v < V; v += kRowStatsThreads) take(to_f32(x[v]), v);
    }
  } else {
    for (int v = threadIdx.x; v < V; v += kRowStatsThreads) take(to_f32(x[v]), v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, bm, o);
    const int oa = __shfl_xor_sync(0xffffffffu, ba, o);
    if (om > bm || (om == bm && oa < ba)) { bm = om; ba = oa; }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { smax[warp] = bm; sarg[warp] = ba; }
  __syncthreads();
  float gm = smax[0];
  int ga = sarg[0];
  for (int w = 1; w < NW; ++w)
    if (smax[w] > gm || (smax[w] == gm && sarg[w] < ga)) { gm = smax[w]; ga = sarg[w]; }
  if (stats == nullptr) {
    if (threadIdx.x == 0 && argmax) argmax[row] = ga;
    return;
  }
  const double ms = static_cast<double>(gm) * inv_temp;
  double s = 0.0;
  for (int v = threadIdx.x; v < V; v += kRowStatsThreads) s += exp(static_cast<double>(to_f32(x[v]) * inv_temp) - ms);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) ssum[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < NW; ++w) tot += ssum[w];
    if (argmax) argmax[row] = ga;
    stats[2 * row] = static_cast<float>(ms);
    stats[2 * row + 1] = static_cast<float>(ms + log(tot));
  }
}

__global__ void stamp_kernel(unsigned long long* slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *slot = t;
}

}  // namespace ygg

using namespace ygg;

extern "C" {

int ygg_prepare_layers(void) {
  cudaFuncSetAttribute(attn_simt_kernel<float, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(attn_simt_kernel<float, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(attn_simt_kernel<__nv_bfloat16, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaError_t e =
      cudaFuncSetAttribute(attn_simt_kernel<__nv_bfloat16, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "attention attribute: %s", cudaGetErrorString(e));
  return YGG_OK;
}

int ygg_embed(const void* table, int dtype, int V, int d, const int32_t* tokens, int M, float* resid_out,
              ygg_stream_t stream) {
  YGG_CHECK_ARG(table && tokens && resid_out && V >= 1 && d >= 1 && d <= 8192, "invalid arguments");
  if (M <= 0) return YGG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int threads = ((d + 7) / 8 + 31) / 32 * 32;  // 8 features per thread
  if (dtype == YGG_F32)
    YGG_LAUNCH_PDL(embed_kernel<float>, dim3(M), dim3(threads), 0, s, static_cast<const float*>(table), V, d, tokens,
                   resid_out);
  else
    YGG_LAUNCH_PDL(embed_kernel<__nv_bfloat16>, dim3(M), dim3(threads), 0, s, static_cast<const __nv_bfloat16*>(table),
                   V, d, tokens, resid_out);
  return YGG_OK;
}

int ygg_embed_fused(const void* table, int V, int d, const int32_t* tokens, int M, float* resid, void* hb,
                    float* ss_out, ygg_stream_t stream) {
  YGG_CHECK_ARG(table && tokens && resid && hb && ss_out && V >= 1, "invalid arguments");
  YGG_CHECK_ARG(d % 128 == 0 && d <= 8192, "model width must be a multiple of 128 and <= 8192");
  if (M <= 0) return YGG_OK;
  YGG_LAUNCH_PDL(embed_fused_kernel, dim3(M), dim3(((d / 8 + 31) / 32) * 32), 0, reinterpret_cast<cudaStream_t>(stream),
                 static_cast<const __nv_bfloat16*>(table), V, d, tokens, resid, static_cast<__nv_bfloat16*>(hb),
                 ss_out, M, trace_next(14));
  return YGG_OK;
}

int ygg_embed_rmsnorm(const void* table, const void* norm_w, int dtype, int V, int d, const int32_t* tokens, int M,
                      float eps, float* resid_out, void* xn_out, ygg_stream_t stream) {
  YGG_CHECK_ARG(table && norm_w && tokens && resid_out && xn_out && V >= 1 && d >= 1 && d <= 8192,
                "invalid arguments");
  if (M <= 0) return YGG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int threads = ((d + 7) / 8 + 31) / 32 * 32;
  if (dtype == YGG_F32)
    YGG_LAUNCH_PDL(embed_rmsnorm_kernel<float>, dim3(M), dim3(threads), 0, s, static_cast<const float*>(table), V, d,
                   tokens, static_cast<const float*>(norm_w), eps, resid_out, static_cast<float*>(xn_out));
  else
    YGG_LAUNCH_PDL(embed_rmsnorm_kernel<__nv_bfloat16>, dim3(M), dim3(threads), 0, s,
                   static_cast<const __nv_bfloat16*>(table), V, d, tokens, static_cast<const __nv_bfloat16*>(norm_w),
                   eps, resid_out, static_cast<__nv_bfloat16*>(xn_out));
  return YGG_OK;
}

int ygg_rmsnorm(const float* x, const void* w, int dtype, int M, int d, float eps, void* out, ygg_stream_t stream) {
  YGG_CHECK_ARG(x && w && out && d >= 1 && d <= 8192, "invalid arguments");
  if (M <= 0) return YGG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int threads = ((d + 7) / 8 + 31) / 32 * 32;  // 8 features per thread
  if (dtype == YGG_F32)
    YGG_LAUNCH_PDL(rmsnorm_kernel<float>, dim3(M), dim3(threads), 0, s, x, static_cast<const float*>(w), d, eps,
                   static_cast<float*>(out));
  else
    YGG_LAUNCH_PDL(rmsnorm_kernel<__nv_bfloat16>, dim3(M), dim3(threads), 0, s, x, static_cast<const __nv_bfloat16*>(w),
                   d, eps, static_cast<__nv_bfloat16*>(out));
  return YGG_OK;
}

int ygg_attention(const void* q, const void* cache, int dtype, int M, int B, int Hq, int Hkv, int hd, int S,
                  const int32_t* blk_start, const int32_t* blk_len, const uint32_t* qmask, int mask_words, float scale,
                  void* out, ygg_stream_t stream) {
  YGG_CHECK_ARG(q && cache && blk_start && blk_len && out, "invalid arguments");
  YGG_CHECK_ARG(B >= 1 && M % B == 0, "query rows must split evenly over requests");
  YGG_CHECK_ARG(Hkv >= 1 && Hq % Hkv == 0 && (Hq / Hkv) <= kAttnRows, "bad head grouping");
  YGG_CHECK_ARG(mask_words >= 0 && mask_words <= 64, "bad mask words");
  if (M == 0) return YGG_OK;
  const int T = M / B;
  const int G = Hq / Hkv;
  const int qc = kAttnRows / G;
  dim3 grid((T + qc - 1) / qc, Hkv, B);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const float sl2 = scale * 1.4426950408889634f;
  const size_t smem = static_cast<size_t>(kAttnRows + 2 * kAttnKeys) * (hd + 1) * sizeof(float);
  if (dtype == YGG_F32) {
    if (hd == 64)
      YGG_LAUNCH_PDL((attn_simt_kernel<float, 64>), grid, dim3(kAttnThreads), smem, s, static_cast<const float*>(q),
                     static_cast<const float*>(cache), T, Hq, Hkv, S, blk_start, blk_len, qmask, mask_words, sl2,
                     static_cast<float*>(out));
    else if (hd == 128)
      YGG_LAUNCH_PDL((attn_simt_kernel<float, 128>), grid, dim3(kAttnThreads), smem, s, static_cast<const float*>(q),
                     static_cast<const float*>(cache), T, Hq, Hkv, S, blk_start, blk_len, qmask, mask_words, sl2,
                     static_cast<float*>(out));
    else
      return ygg_fail(YGG_ERR_UNSUPPORTED, "head dim must be 64 or 128");
  } else {
    if (hd == 64)
      YGG_LAUNCH_PDL((attn_simt_kernel<__nv_bfloat16, 64>), grid, dim3(kAttnThreads), smem, s,
                     static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(cache), T, Hq, Hkv, S,
                     blk_start, blk_len, qmask, mask_words, sl2, static_cast<__nv_bfloat16*>(out));
    else if (hd == 128)
      YGG_LAUNCH_PDL((attn_simt_kernel<__nv_bfloat16, 128>), grid, dim3(kAttnThreads), smem, s,
                     static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(cache), T, Hq, Hkv, S,
                     blk_start, blk_len, qmask, mask_words, sl2, static_cast<__nv_bfloat16*>(out));
    else
      return ygg_fail(YGG_ERR_UNSUPPORTED, "head dim must be 64 or 128");
  }
  return YGG_OK;
}

int ygg_row_stats(const void* logits, int dtype, int rows, int V, int ld, float temperature, int32_t* argmax,
                  float* stats, ygg_stream_t stream) {
  YGG_CHECK_ARG(logits && V >= 1 && ld >= V && temperature > 0.f, "invalid arguments");
  if (rows <= 0) return YGG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const float inv_t = 1.0f / temperature;
  if (dtype == YGG_F32)
    YGG_LAUNCH_PDL(row_stats_kernel<float>, dim3(rows), dim3(kRowStatsThreads), 0, s, static_cast<const float*>(logits), V, ld,
                   inv_t, argmax, stats);
  else
    YGG_LAUNCH_PDL(row_stats_kernel<__nv_bfloat16>, dim3(rows), dim3(kRowStatsThreads), 0, s,
                   static_cast<const __nv_bfloat16*>(logits), V, ld, inv_t, argmax, stats);
  return YGG_OK;
}

int ygg_stamp(unsigned long long* slot, ygg_stream_t stream) {
  YGG_CHECK_ARG(slot != nullptr, "null slot");
  stamp_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(slot);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "stamp launch: %s", cudaGetErrorString(e));
  return YGG_OK;
}

}  // extern "C"
