// K2: tree / prefix attention on tcgen05 (bf16), split over the key sequence.
//
// CTA = (key chunk of KC=128 keys, query tile of 128 rows, kv head, request).  Query rows are
// (token, q-head-in-group) pairs of one kv head, so GQA shares every K/V tile across the G
// heads of the group.  Flow per CTA:
//   TMA  : Q tile [128 x hd], K chunk [KC x hd], V^T chunk [hd x KC] (V is cached transposed so
//          both MMAs read K-major, 128B-swizzled operands)
//   MMA1 : S[128 x KC] = Q . K^T            -> TMEM columns [0, KC)
//   soft : one thread per row: tcgen05.ld S, ancestor mask on the fly (prefix keys always
//          visible; block keys by the row's tree-mask bit), max / exp2 / sum, P (bf16) -> smem
//   MMA2 : O[128 x hd] = P . V              -> TMEM columns [KC, KC + hd)
//   out  : unnormalised O + (max, sum) partials per chunk; a combine kernel merges chunks in
//          fixed order (deterministic).
// Chunks past a request's key count exit immediately after recording an empty partial.
#include <cudaTypedefs.h>

#include <cmath>
#include <cstring>

#include "common.cuh"
#include "host_util.h"

namespace ygg {

constexpr int kKC = 128;           // keys per CTA
constexpr int kQRows = 128;        // query rows per CTA (UMMA M)
constexpr int kAttnTcThreads = 288; // warps 0-7 softmax/epilogue (2 per TMEM lane quarter), warp 8 TMA + MMA
constexpr int kSoftThreads = 256;

struct AttnPlan {
  uint32_t magic;
  int B, M, Hq, Hkv, hd, S, T;  // T = query rows (tokens) per request
  int G, tok_per_tile, q_tiles, chunks;
  alignas(64) CUtensorMap tm_q;
  alignas(64) CUtensorMap tm_k;
  alignas(64) CUtensorMap tm_vt;
};
constexpr uint32_t kAttnMagic = 0x59474741u;

struct AttnArgs {
  int M, Hq, Hkv, hd, S, T, G, tok_per_tile, chunks, mask_words;
  float scale_log2;
  const int32_t* blk_start;
  const int32_t* blk_len;
  const uint32_t* qmask;
  float* opart;  // [chunks][M*Hq][hd]
  float* ml;     // [chunks][M*Hq][2]
  unsigned long long* trace;  // kernel-timeline slot (profiling only) or nullptr
};

YGG_DEV void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
YGG_DEV void tma_load_2d_nohint(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
YGG_DEV void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
YGG_DEV uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int HD>
__global__ void __launch_bounds__(kAttnTcThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_vt, AttnArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int DCH = HD / 64;            // 64-wide d chunks
  constexpr int KCH = kKC / 64;           // 64-wide key chunks
  unsigned char* sq = base;                                   // DCH x [128 rows x 128 B]
  unsigned char* sk = sq + DCH * kQRows * 128;                // DCH x [KC rows x 128 B]
  unsigned char* svt = sk + DCH * kKC * 128;                  // KCH x [HD rows x 128 B]
  unsigned char* sp = svt + KCH * HD * 128;                   // KCH x [128 rows x 128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sp + KCH * kQRows * 128);  // load, s, p, o
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);
  float* red_max = reinterpret_cast<float*>(bars + 6);  // [2][128]
  float* red_sum = red_max + 2 * kQRows;                 // [2][128]

  const int chunk = blockIdx.x, qt = blockIdx.y, kvh = blockIdx.z % a.Hkv, r = blockIdx.z / a.Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) trace_min(a.trace, 0);
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 0) trace_min(a.trace, 1);
  const int bs = a.blk_start[r], bl = a.blk_len[r];
  const int nkeys = bs + bl;
  const int key0 = chunk * kKC;
  const int t0 = qt * a.tok_per_tile;
  // Row owned by this thread (softmax warps): TMEM lane = row; the two warps of a lane quarter
  // split the key columns (half 0: keys [0, 64), half 1: keys [64, 128) of the chunk).
  const int row = (warp & 3) * 32 + lane;
  const int half = (warp >> 2) & 1;
  const int tq = t0 + row / a.G;
  const int head = kvh * a.G + row % a.G;
  const bool row_valid = warp < 8 && tq < a.T;
  const int m = r * a.T + tq;
  const size_t orow = static_cast<size_t>(m) * a.Hq + head;
  const size_t slot_stride = static_cast<size_t>(a.M) * a.Hq;
  // Causal prefill tiles never need keys past their last query token.
  const int last_tok = min(a.T - 1, t0 + a.tok_per_tile - 1);
  const bool skip = key0 >= nkeys || (a.mask_words == 0 && key0 > bs + last_tok);
  if (skip) {
    if (row_valid && half == 0) {
      a.ml[(static_cast<size_t>(chunk) * slot_stride + orow) * 2] = -INFINITY;
      a.ml[(static_cast<size_t>(chunk) * slot_stride + orow) * 2 + 1] = 0.f;
    }
    return;
  }
  if (warp == 8) {
    if (lane == 0) {
      for (int i = 0; i < 4; ++i) mbar_init(&bars[i], i == 2 ? kSoftThreads : 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(tmem_slot, 256);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + kKC;

  if (warp == 8) {
    if (lane == 0) {
      const uint32_t bytes = DCH * kQRows * 128 + DCH * kKC * 128 + KCH * HD * 128;
      mbar_arrive_expect_tx(&bars[0], bytes);
      for (int c = 0; c < DCH; ++c) {
        tma_load_3d(sq + c * kQRows * 128, &tm_q, &bars[0], c * 64, kvh * a.G, r * a.T + t0);
        tma_load_2d_nohint(sk + c * kKC * 128, &tm_k, &bars[0], c * 64,
                           (r * 2 * a.Hkv + kvh) * a.S + key0);
      }
      for (int c = 0; c < KCH; ++c)
        tma_load_2d_nohint(svt + c * HD * 128, &tm_vt, &bars[0], key0 + c * 64, ((r * 2 + 1) * a.Hkv + kvh) * HD);
      mbar_wait(&bars[0], 0);
      tc_fence_after();
      // MMA1: S = Q . K^T  (M=128, N=KC, K=HD)
      const uint32_t id1 = umma_idesc_bf16(kQRows, kKC);
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const uint64_t ad = umma_desc_sw128(smem_u32(sq + (kk / 4) * kQRows * 128) + (kk % 4) * 32);
        const uint64_t bd = umma_desc_sw128(smem_u32(sk + (kk / 4) * kKC * 128) + (kk % 4) * 32);
        umma_bf16(tS, ad, bd, id1, kk > 0 ? 1u : 0u);
      }
      umma_commit(&bars[1]);
      // MMA2 after the softmax warps published P.
      mbar_wait(&bars[2], 0);
      tc_fence_after();
      const uint32_t id2 = umma_idesc_bf16(kQRows, HD);
#pragma unroll
      for (int kk = 0; kk < kKC / 16; ++kk) {
        const uint64_t ad = umma_desc_sw128(smem_u32(sp + (kk / 4) * kQRows * 128) + (kk % 4) * 32);
        const uint64_t bd = umma_desc_sw128(smem_u32(svt + (kk / 4) * HD * 128) + (kk % 4) * 32);
        umma_bf16(tO, ad, bd, id2, kk > 0 ? 1u : 0u);
      }
      umma_commit(&bars[3]);
    }
  } else {
    // ===== softmax: two threads per query row (64 key columns each) =====
    uint32_t mw[YGG_MAX_MASK_WORDS];
#pragma unroll
    for (int w = 0; w < YGG_MAX_MASK_WORDS; ++w)
      mw[w] = (row_valid && w < a.mask_words) ? a.qmask[static_cast<size_t>(m) * a.mask_words + w] : 0u;
    // Visibility bits of 32 keys starting at absolute key kw: prefix keys (< bs) always, block keys
    // by the row's tree-mask bit (causal when no mask is given), nothing at or past nkeys.
    auto vis_word = [&](int kw) -> uint32_t {
      if (!row_valid) return 0u;
      uint32_t pre = 0u;
      if (kw + 32 <= bs) pre = 0xffffffffu;
      else if (kw < bs) pre = (1u << (bs - kw)) - 1u;
      const int jb0 = kw - bs;  // block index of this word's bit 0
      uint32_t blk = 0u;
      if (jb0 + 32 > 0 && jb0 < bl) {
        if (a.mask_words == 0) {
          const int lo = jb0 < 0 ? -jb0 : 0;
          const int hi = min(31, tq - jb0);
          if (hi >= lo) blk = ((hi == 31) ? 0xffffffffu : ((1u << (hi + 1)) - 1u)) & ~((1u << lo) - 1u);
        } else if (jb0 < 0) {
          blk = mw[0] << (-jb0);
        } else {
          const int i = jb0 >> 5, s = jb0 & 31;
          uint32_t w0 = 0u, w1 = 0u;
#pragma unroll
          for (int w = 0; w < YGG_MAX_MASK_WORDS; ++w) {
            if (w == i) w0 = mw[w];
            if (w == i + 1) w1 = mw[w];
          }
          blk = s ? ((w0 >> s) | (w1 << (32 - s))) : w0;
        }
        const int keep = bl - jb0;  // bits j with jb0 + j < bl
        if (keep < 32) blk &= (1u << keep) - 1u;
      }
      return pre | blk;
    };
    const int cbase = half * 64;
    const uint32_t vis0 = vis_word(key0 + cbase), vis1 = vis_word(key0 + cbase + 32);
    mbar_wait(&bars[1], 0);
    tc_fence_after();
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    // Pass 1: partial row max over this thread's 64 columns, straight from TMEM.
    float mx = -INFINITY;
#pragma unroll
    for (int c = 0; c < 64; c += 16) {
      float v[16];
      tmem_ld16(tS + lane_base + cbase + c, v);
      const uint32_t bits = (c < 32 ? vis0 : vis1) >> (c & 31);
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if ((bits >> j) & 1u) mx = fmaxf(mx, v[j] * a.scale_log2);
    }
    red_max[half * kQRows + row] = mx;
    asm volatile("bar.sync 1, %0;" ::"n"(kSoftThreads) : "memory");
    mx = fmaxf(red_max[row], red_max[kQRows + row]);
    // Pass 2: P = 2^(s - max) -> bf16 -> smem (this half's 64-key block, 128B-swizzled rows).
    float l = 0.f;
    const uint32_t rbase = smem_u32(sp + half * kQRows * 128 + row * 128);
#pragma unroll
    for (int c = 0; c < 64; c += 16) {
      float v[16];
      tmem_ld16(tS + lane_base + cbase + c, v);
      const uint32_t bits = (c < 32 ? vis0 : vis1) >> (c & 31);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        v[j] = ((bits >> j) & 1u) ? exp2f(v[j] * a.scale_log2 - mx) : 0.f;
        l += v[j];
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = c / 8 + h;
        const float* p8 = v + 8 * h;
        st_shared_v4(rbase + ((u ^ (row & 7)) << 4), pack_bf16(p8[0], p8[1]), pack_bf16(p8[2], p8[3]),
                     pack_bf16(p8[4], p8[5]), pack_bf16(p8[6], p8[7]));
      }
    }
    red_sum[half * kQRows + row] = l;
    fence_proxy_async();
    tc_fence_before();
    mbar_arrive(&bars[2]);
    mbar_wait(&bars[3], 0);
    tc_fence_after();
    // O readback: each half stores HD/2 columns.  Every lane executes the (warp-collective,
    // .aligned) TMEM loads; only valid rows store.
    float* op = a.opart + (static_cast<size_t>(chunk) * slot_stride + (row_valid ? orow : 0)) * HD + half * (HD / 2);
#pragma unroll
    for (int c = 0; c < HD / 2; c += 16) {
      float o[16];
      tmem_ld16(tO + lane_base + half * (HD / 2) + c, o);
      if (row_valid) {
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(op + c + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
      }
    }
    if (row_valid && half == 0) {
      a.ml[(static_cast<size_t>(chunk) * slot_stride + orow) * 2] = mx;
      a.ml[(static_cast<size_t>(chunk) * slot_stride + orow) * 2 + 1] = red_sum[row] + red_sum[kQRows + row];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace_max(a.trace, 2);
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

// Merge chunk partials in fixed chunk order: out = sum_c 2^(m_c - M) O_c / sum_c 2^(m_c - M) l_c.
// One warp per (query row, head); only the chunks holding the request's keys are read.
template <int HD>
__global__ void __launch_bounds__(128) attn_combine_kernel(const float* __restrict__ opart,
                                                           const float* __restrict__ ml, int rows, int Hq, int T,
                                                           const int32_t* __restrict__ blk_start,
                                                           const int32_t* __restrict__ blk_len,
                                                           __nv_bfloat16* __restrict__ out,
                                                           unsigned long long* trace) {
  if (threadIdx.x == 0) trace_min(trace, 0);
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 0) trace_min(trace, 1);
  const int rr = blockIdx.x * 4 + (threadIdx.x >> 5);  // m*Hq + head
  const int lane = threadIdx.x & 31;
  if (rr >= rows) return;
  const int req = (rr / Hq) / T;
  const int nch = (blk_start[req] + blk_len[req] + kKC - 1) / kKC;
  constexpr int DPL = HD / 32;
  float M = -INFINITY;
  for (int c = 0; c < nch; ++c) M = fmaxf(M, __ldg(ml + (static_cast<size_t>(c) * rows + rr) * 2));
  float acc[DPL];
#pragma unroll
  for (int i = 0; i < DPL; ++i) acc[i] = 0.f;
  float L = 0.f;
  if (M != -INFINITY) {
    for (int c = 0; c < nch; ++c) {
      const float mc = __ldg(ml + (static_cast<size_t>(c) * rows + rr) * 2);
      if (mc == -INFINITY) continue;
      const float w = exp2f(mc - M);
      L += w * __ldg(ml + (static_cast<size_t>(c) * rows + rr) * 2 + 1);
      const float* o = opart + (static_cast<size_t>(c) * rows + rr) * HD + lane * DPL;
#pragma unroll
      for (int i = 0; i < DPL; ++i) acc[i] += w * __ldg(o + i);
    }
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  __nv_bfloat16* dst = out + static_cast<size_t>(rr) * HD + lane * DPL;
#pragma unroll
  for (int i = 0; i < DPL; ++i) dst[i] = __float2bfloat16_rn(acc[i] * inv);
  if (lane == 0) trace_max(trace, 2);
}

static int encode(CUtensorMap* map, int rank, const void* ptr, const cuuint64_t* dims, const cuuint64_t* strides,
                  const cuuint32_t* box) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return ygg_fail(YGG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  cuuint32_t es[3] = {1, 1, 1};
  CUresult rc = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) return ygg_fail(YGG_ERR_CUDA, "attention tensor map encode failed (%d)", static_cast<int>(rc));
  return YGG_OK;
}

template <int HD>
size_t attn_smem() {
  return 1024 + (HD / 64) * kQRows * 128 + (HD / 64) * kKC * 128 + (kKC / 64) * HD * 128 + (kKC / 64) * kQRows * 128 +
         64 + 4 * kQRows * sizeof(float);
}

static const AttnPlan* attn_plan_of(const void* p) {
  const AttnPlan* a = reinterpret_cast<const AttnPlan*>((reinterpret_cast<uintptr_t>(p) + 63) & ~uintptr_t(63));
  return (a && a->magic == kAttnMagic) ? a : nullptr;
}

}  // namespace ygg

using namespace ygg;

extern "C" {

int ygg_prepare_attn_tc(void) {
  cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(attn_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "attention attribute: %s", cudaGetErrorString(e));
  return YGG_OK;
}

size_t ygg_attn_plan_size(void) { return sizeof(AttnPlan) + 64; }

/* q [M, Hq, hd] bf16; cache_layer = this layer's [B, 2, Hkv, S, hd] block (K rows, V^T rows). */
int ygg_attn_plan_init(void* plan_mem, const void* q, const void* cache_layer, int B, int M, int Hq, int Hkv, int hd,
                       int S, size_t* partial_bytes) {
  YGG_CHECK_ARG(plan_mem && q && cache_layer, "null pointer");
  YGG_CHECK_ARG(hd == 64 || hd == 128, "head dim must be 64 or 128");
  YGG_CHECK_ARG(Hkv >= 1 && Hq % Hkv == 0, "bad head grouping");
  const int G = Hq / Hkv;
  YGG_CHECK_ARG(kQRows % G == 0, "group size must divide 128");
  YGG_CHECK_ARG(B >= 1 && M % B == 0, "rows must split evenly over requests");
  YGG_CHECK_ARG(S % 64 == 0, "cache capacity must be a multiple of 64");
  AttnPlan* p = reinterpret_cast<AttnPlan*>((reinterpret_cast<uintptr_t>(plan_mem) + 63) & ~uintptr_t(63));
  std::memset(p, 0, sizeof(AttnPlan));
  p->magic = kAttnMagic;
  p->B = B;
  p->M = M;
  p->Hq = Hq;
  p->Hkv = Hkv;
  p->hd = hd;
  p->S = S;
  p->T = M / B;
  p->G = G;
  p->tok_per_tile = kQRows / G;
  p->q_tiles = (p->T + p->tok_per_tile - 1) / p->tok_per_tile;
  p->chunks = (S + kKC - 1) / kKC;
  {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(hd), static_cast<cuuint64_t>(Hq), static_cast<cuuint64_t>(M)};
    cuuint64_t str[2] = {static_cast<cuuint64_t>(hd) * 2, static_cast<cuuint64_t>(Hq) * hd * 2};
    cuuint32_t box[3] = {64, static_cast<cuuint32_t>(G), static_cast<cuuint32_t>(p->tok_per_tile)};
    if (int rc = encode(&p->tm_q, 3, q, dims, str, box)) return rc;
  }
  {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(hd), static_cast<cuuint64_t>(B) * 2 * Hkv * S};
    cuuint64_t str[1] = {static_cast<cuuint64_t>(hd) * 2};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(kKC)};
    if (int rc = encode(&p->tm_k, 2, cache_layer, dims, str, box)) return rc;
  }
  {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(S), static_cast<cuuint64_t>(B) * 2 * Hkv * hd};
    cuuint64_t str[1] = {static_cast<cuuint64_t>(S) * 2};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(hd)};
    if (int rc = encode(&p->tm_vt, 2, cache_layer, dims, str, box)) return rc;
  }
  if (partial_bytes) *partial_bytes = static_cast<size_t>(p->chunks) * M * Hq * (hd + 2) * sizeof(float);
  return YGG_OK;
}

int ygg_attention_tc(const void* plan, const int32_t* blk_start, const int32_t* blk_len, const uint32_t* qmask,
                     int mask_words, float scale, float* partials, void* out, ygg_stream_t stream) {
  const AttnPlan* p = attn_plan_of(plan);
  YGG_CHECK_ARG(p != nullptr, "invalid attention plan");
  YGG_CHECK_ARG(blk_start && blk_len && partials && out, "null pointer");
  YGG_CHECK_ARG(mask_words >= 0 && mask_words <= YGG_MAX_MASK_WORDS, "mask too wide for the tcgen05 path");
  YGG_CHECK_ARG(mask_words == 0 || qmask != nullptr, "mask words without a mask");
  AttnArgs a;
  a.M = p->M;
  a.Hq = p->Hq;
  a.Hkv = p->Hkv;
  a.hd = p->hd;
  a.S = p->S;
  a.T = p->T;
  a.G = p->G;
  a.tok_per_tile = p->tok_per_tile;
  a.chunks = p->chunks;
  a.mask_words = mask_words;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.blk_start = blk_start;
  a.blk_len = blk_len;
  a.qmask = qmask;
  a.opart = partials;
  a.ml = partials + static_cast<size_t>(p->chunks) * p->M * p->Hq * p->hd;
  a.trace = trace_next(8);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  dim3 grid(p->chunks, p->q_tiles, p->Hkv * p->B);
  if (p->hd == 64)
    YGG_LAUNCH_PDL(attn_tc_kernel<64>, grid, dim3(kAttnTcThreads), attn_smem<64>(), s, p->tm_q, p->tm_k, p->tm_vt, a);
  else
    YGG_LAUNCH_PDL(attn_tc_kernel<128>, grid, dim3(kAttnTcThreads), attn_smem<128>(), s, p->tm_q, p->tm_k, p->tm_vt,
                   a);
  const int rows = p->M * p->Hq;
  unsigned long long* ctrace = trace_next(9);
  if (p->hd == 64)
    YGG_LAUNCH_PDL(attn_combine_kernel<64>, dim3((rows + 3) / 4), dim3(128), 0, s, static_cast<const float*>(a.opart),
                   static_cast<const float*>(a.ml), rows, p->Hq, p->T, blk_start, blk_len,
                   static_cast<__nv_bfloat16*>(out), ctrace);
  else
    YGG_LAUNCH_PDL(attn_combine_kernel<128>, dim3((rows + 3) / 4), dim3(128), 0, s, static_cast<const float*>(a.opart),
                   static_cast<const float*>(a.ml), rows, p->Hq, p->T, blk_start, blk_len,
                   static_cast<__nv_bfloat16*>(out), ctrace);
  return YGG_OK;
}

}  // extern "C"
