// Weight-streaming small-M GEMM for the draft and verify forwards (K3) and its fused
// epilogues.  Y[M,N] = X[M,K] . W[N,K]^T.
//
// bf16 path ("swap-AB"): the weight tile is the 128-row UMMA A operand, the M<=256 tokens are
// the UMMA N dimension, so a decode-sized batch still issues full 128-row tcgen05.mma
// instructions.  Work is split stream-K over the persistent grid: the (tile, k-block) unit
// space is cut into num_ctas equal contiguous ranges, so every SM streams the same number
// of weight bytes regardless of N.  Each CTA: warp 0 = TMA producer (weights prefetched
// before griddepcontrol.wait, activations after), warp 1 = single-thread MMA issuer with a
// double-buffered TMEM accumulator, warps 2-5 = TMEM->global partial epilogue.
// Partials ws[seg][BN][128] f32 are reduced by the epilogue kernels in fixed segment order
// (deterministic), which also apply RoPE/KV-append, residual+RMSNorm or SwiGLU.
//
// f32 path (parity mode): SIMT tiled GEMM writing the same partial layout, one segment per tile.
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "host_util.h"

namespace ygg {

constexpr int kBM = 128;          // weight rows per tile (UMMA M)
constexpr int kBK = 64;           // k per stage: 64 bf16 = one 128B swizzle row
constexpr int kGemmThreads = 192; // 6 warps
constexpr int kMaxRstdTokensHost = 1024;
// alignment slack + barriers (<= 2*12+4 u64) + tmem slot/pending + red_s[64] + rstd_s[1024]
constexpr int kSmemExtra = 1024 + 28 * 8 + 32 + 64 * 4 + kMaxRstdTokensHost * 4;

struct GemmPlan {
  uint32_t magic;
  int dtype;
  int M, N, K;
  int BN;        // tokens per tile (multiple of 16, <= 256)
  int m_tiles, n_tiles, tiles, kb;
  int num_ctas;
  int dp_per_cta;
  long long units;
  int segments;
  int stages;
  int tmem_cols;
  int cluster;   // > 0: cluster split-K (one cluster of `cluster` CTAs per tile, DSMEM reduction)
  const void* W;
  const void* X;
  int32_t* seg_table;  // device: seg_first[tiles+1], seg_base[num_ctas]
  const char* epi_pf;  // L2 prefetch region of this plan's separate epilogue kernel (or nullptr)
  size_t epi_pf_bytes;
  int interleaved;     // W rows in the fused layout (RoPE pairs / gate-up pairs adjacent): separate epilogues
  alignas(64) CUtensorMap tmap_w;
  alignas(64) CUtensorMap tmap_x;
};
constexpr uint32_t kPlanMagic = 0x59474750u;  // "YGGP"

struct GemmParams {
  int M, BN, m_tiles, kb, num_ctas, stages, tmem_cols;
  int dp_per_cta;   // whole tiles per CTA (tiles [0, dp_per_cta * num_ctas) are data-parallel)
  long long units;  // stream-K units (remainder tiles x kb)
  const int32_t* seg_first;
  const int32_t* seg_base;
  int prewait;      // weight stages issued before the grid-dependency wait (<= stages)
};

// ---------------------------------------------------------------------------
// Fused epilogues.  A tile owned by one CTA is finished straight from TMEM.  A tile split over
// several stream-K CTAs is finished cooperatively: every participant publishes its f32 partial
// and, at the end of its own range, waits for the tile's arrival counter and reduces a disjoint
// slice of token columns in fixed segment order (deterministic) before applying the op.  The
// grid is persistent (<= one CTA per SM), so all participants are co-resident and the wait is
// short; concurrently running fused GEMMs must therefore split the SMs between them.
// RMSNorm is folded: its gain lives in the next weight matrix and the per-token rstd (from the
// producer's per-tile sums of squares) scales the consumer's output rows.
// ---------------------------------------------------------------------------
enum EpiKind : int { kEpiNone = 0, kEpiStoreF32 = 1, kEpiQkvRope = 2, kEpiSwiglu = 3, kEpiResid = 4, kEpiArgmax = 5 };
constexpr int kArgmaxKeyOffset = 512;  // u64 key scratch inside rstd_s (argmax plans keep M <= 512)
constexpr int kMaxRstdTokens = 1024;

struct EpiArgs {
  const float* ss_in;   // [ss_tiles][M] sums of squares of the (un-normalised) input rows, or null
  int ss_tiles;
  int norm_dim;
  float eps;
  float* out;           // STORE_F32 [M][ld]
  int ld;
  __nv_bfloat16* q_out; // QKV_ROPE (rows permuted: pairs (i, i+hd/2) adjacent)
  __nv_bfloat16* cache;
  int S, Hq, Hkv, hd;
  float log2_theta;
  const int32_t* pos;
  const int32_t* slot;
  const int32_t* req;
  __nv_bfloat16* act_out; // SWIGLU [M][N/2] (rows interleaved gate/up)
  float* resid;           // RESID [M][N]
  __nv_bfloat16* hb;      // RESID bf16 copy of the residual = next GEMM's X
  float* ss_out;          // RESID [N/128][M]
  int n_total;
  int32_t* counters;      // [tiles] arrival counters, self-resetting
  unsigned long long* dbg; // optional per-CTA %globaltimer stamps [num_ctas][8] (profiling only)
  unsigned long long* trace;  // kernel-timeline slot (profiling only) or nullptr
  const float2* rope_cs;   // optional [positions][hd/2] (cos, sin) table; else sincosf
};


YGG_DEV void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
YGG_DEV uint32_t cluster_ctarank_u32() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
YGG_DEV int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Apply the fused op to 16 token columns of one 128-feature tile row (thread = feature row).
// Every global load of a chunk (token metadata, RoPE table, residual) is issued before any store:
// the EpiArgs pointers may alias as far as the compiler knows, so interleaving would serialise
// one L2 round trip per token.
template <int KIND>
YGG_DEV void epi_apply(const EpiArgs& e, int M, int n, int m0, int valid16, float* v, const float* rstd_s,
                       float* red_s, int quarter, int lane) {
  if (e.ss_in) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] *= (j < valid16) ? rstd_s[m0 + j] : 0.f;
  }
  if constexpr (KIND == kEpiStoreF32) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < valid16) e.out[static_cast<size_t>(m0 + j) * e.ld + n] = v[j];
  } else if constexpr (KIND == kEpiSwiglu) {
    const bool odd = n & 1;
    const int F = e.n_total / 2;
    float o[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float other = __shfl_xor_sync(0xffffffffu, v[j], 1);
      o[j] = v[j] / (1.f + __expf(-v[j])) * other;
    }
    if (!odd) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < valid16) e.act_out[static_cast<size_t>(m0 + j) * F + (n >> 1)] = __float2bfloat16_rn(o[j]);
    }
  } else if constexpr (KIND == kEpiQkvRope) {
    const int head = n / e.hd, p = n % e.hd, half = e.hd / 2;
    const int pair = p >> 1;
    const bool odd = p & 1;
    const int orig = pair + (odd ? half : 0);
    const bool rope = head < e.Hq + e.Hkv;
    const bool is_q = head < e.Hq;
    const bool is_v = head >= e.Hq + e.Hkv;
    // ---- load phase
    int pos[16], req[16], slot[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int m = min(m0 + j, M - 1);  // chunks past M (valid16 <= 0) still run: clamp their loads
      pos[j] = __ldg(e.pos + m);
      req[j] = __ldg(e.req + m);
      slot[j] = __ldg(e.slot + m);
    }
    float cs[16], sn[16];
    if (rope) {
      if (e.rope_cs) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 t = __ldg(e.rope_cs + static_cast<size_t>(pos[j]) * half + pair);
          cs[j] = t.x;
          sn[j] = t.y;
        }
      } else {
        const float inv_freq = 1.0f / exp2f(e.log2_theta * (static_cast<float>(2 * pair) / static_cast<float>(e.hd)));
#pragma unroll
        for (int j = 0; j < 16; ++j) sincosf(static_cast<float>(pos[j]) * inv_freq, &sn[j], &cs[j]);
      }
    }
    // ---- compute
    float y[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float other = __shfl_xor_sync(0xffffffffu, v[j], 1);
      y[j] = v[j];
      if (rope) {
        const float x1 = odd ? other : v[j], x2 = odd ? v[j] : other;
        y[j] = odd ? (x2 * cs[j] + x1 * sn[j]) : (x1 * cs[j] - x2 * sn[j]);
      }
    }
    // ---- store phase
    const int kvh = is_v ? head - e.Hq - e.Hkv : head - e.Hq;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j >= valid16) continue;
      const __nv_bfloat16 yb = __float2bfloat16_rn(y[j]);
      if (is_q) {
        e.q_out[(static_cast<size_t>(m0 + j) * e.Hq + head) * e.hd + orig] = yb;
      } else {
        const size_t base =
            ((static_cast<size_t>(req[j]) * 2 + (is_v ? 1 : 0)) * e.Hkv + kvh) * static_cast<size_t>(e.S) * e.hd;
        if (!is_v) e.cache[base + static_cast<size_t>(slot[j]) * e.hd + orig] = yb;
        else e.cache[base + static_cast<size_t>(orig) * e.S + slot[j]] = yb;  // V^T [hd][S]
      }
    }
  } else if constexpr (KIND == kEpiArgmax) {
    // Greedy LM head: the first maximum of each token column over this tile's 128 vocabulary rows as
    // a u64 key (ordered f32 bits << 32 | ~row), max-reduced over the warp, then over the 4 warps.
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(const_cast<float*>(rstd_s) + kArgmaxKeyOffset);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t u = __float_as_uint(v[j]);
      const uint32_t ord = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
      unsigned long long k = j < valid16 ? ((static_cast<unsigned long long>(ord) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(n))) : 0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long q = __shfl_xor_sync(0xffffffffu, k, o);
        k = q > k ? q : k;
      }
      if (lane == 0) keys[quarter * 16 + j] = k;
    }
    epi_bar();
    const int t = quarter * 32 + lane;
    if (t < 16 && t < valid16) {
      unsigned long long best = keys[t];
#pragma unroll
      for (int q = 1; q < 4; ++q) best = keys[q * 16 + t] > best ? keys[q * 16 + t] : best;
      reinterpret_cast<unsigned long long*>(e.out)[static_cast<size_t>(n / kBM) * M + m0 + t] = best;
    }
    epi_bar();
  } else if constexpr (KIND == kEpiResid) {
    float h[16], sq[16];
#pragma unroll
    for (int j = 0; j < 16; ++j)  // load phase
      h[j] = (j < valid16) ? e.resid[static_cast<size_t>(m0 + j) * e.n_total + n] : 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      h[j] += (j < valid16) ? v[j] : 0.f;
      sq[j] = h[j] * h[j];
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {  // store phase
      if (j < valid16) {
        const size_t idx = static_cast<size_t>(m0 + j) * e.n_total + n;
        e.resid[idx] = h[j];
        e.hb[idx] = __float2bfloat16_rn(h[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float s = sq[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red_s[quarter * 16 + j] = s;
    }
    epi_bar();
    const int t = quarter * 32 + lane;
    if (t < 16 && t < valid16)  // fixed order over the four 32-row quarters => deterministic
      e.ss_out[static_cast<size_t>(n / kBM) * M + m0 + t] =
          red_s[0 * 16 + t] + red_s[1 * 16 + t] + red_s[2 * 16 + t] + red_s[3 * 16 + t];
    epi_bar();
  }
}

// ---------------------------------------------------------------------------
// tcgen05 kernel
// ---------------------------------------------------------------------------
template <int KIND>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x,
                        GemmParams p, float* __restrict__ ws, EpiArgs e) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-align the dynamic smem base (SW128 atoms).
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int BN = p.BN, S = p.stages;
  const uint32_t a_bytes = kBM * kBK * 2;
  const uint32_t b_bytes = BN * kBK * 2;
  unsigned char* sa = base;
  unsigned char* sb = base + static_cast<size_t>(S) * a_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + static_cast<size_t>(S) * b_bytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;   // [2]
  uint64_t* tempty = tfull + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* pend_tile = reinterpret_cast<int*>(tmem_slot + 1);  // [2] split tiles awaiting their fixup
  int* pend_j = pend_tile + 2;                               // [2] participant index in the tile
  int* pend_tgt = pend_j + 2;                                // [2] epoch-counter target
  float* red_s = reinterpret_cast<float*>(tmem_slot + 8);    // [4][16]
  float* rstd_s = red_s + 64;                               // [kMaxRstdTokens]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  // Hybrid split: dp_per_cta whole tiles per CTA (tiles c, c+G, ...) plus an equal share of the
  // stream-K units of the remaining tiles, which start at tile t_dp.
  const long long sk_base = static_cast<long long>(p.dp_per_cta) * p.num_ctas * p.kb;
  const long long u0 = sk_base + p.units * c / p.num_ctas, u1 = sk_base + p.units * (c + 1) / p.num_ctas;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_w);
    tma_prefetch_desc(&tmap_x);
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 128); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (e.dbg && threadIdx.x == 0) e.dbg[c * 8 + 0] = gtimer();
  if (threadIdx.x == 0) trace_min(e.trace, 0);
  pdl_launch_dependents();

  // Processing order of this CTA's range: the (possibly split) first and last tiles first, then
  // the whole middle tiles, so the cooperative fixups of split tiles overlap the whole-tile stream.
  const int n_sk = (u1 > u0) ? static_cast<int>((u1 - 1) / p.kb - u0 / p.kb + 1) : 0;
  const int nsegs = n_sk + p.dp_per_cta;
  const long long tfirst = u0 / p.kb, tlast = (u1 > u0) ? (u1 - 1) / p.kb : tfirst;
  auto segment = [&](int k, long long& a, long long& b) {
    if (k >= n_sk) {  // whole data-parallel tile
      const long long t = c + static_cast<long long>(k - n_sk) * p.num_ctas;
      a = t * p.kb;
      b = a + p.kb;
      return;
    }
    const long long t = (k == 0) ? tfirst : (k == 1 ? tlast : tfirst + (k - 1));
    a = u0 > t * p.kb ? u0 : t * p.kb;
    b = u1 < (t + 1) * p.kb ? u1 : (t + 1) * p.kb;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      const long long n_units = u1 - u0;
      const int pre = static_cast<int>(n_units < p.prewait ? n_units : p.prewait);
      // Unit coordinates are stepped incrementally inside a segment (one tile): the single producer
      // thread must not pay 64-bit divisions per stage (that alone capped a CTA near 30 GB/s).
      int k = 0, left = 0, kblk = 0, wrow = 0, xrow = 0;
      auto seg_start = [&](int kk) {
        long long a, b;
        segment(kk, a, b);
        const int tile = static_cast<int>(a / p.kb);
        kblk = static_cast<int>(a - static_cast<long long>(tile) * p.kb);
        left = static_cast<int>(b - a);
        wrow = (tile / p.m_tiles) * kBM;
        xrow = (tile % p.m_tiles) * BN;
      };
      if (nsegs) seg_start(0);
      auto advance = [&]() {
        ++kblk;
        if (--left == 0 && ++k < nsegs) seg_start(k);
      };
      int pre_xrow[12], pre_kblk[12];
      // Weights never depend on the previous kernel: stream them before the grid dependency.
      for (int i = 0; i < pre; ++i) {
        pre_xrow[i] = xrow;
        pre_kblk[i] = kblk;
        mbar_arrive_expect_tx(&full[i], a_bytes + b_bytes);
        tma_load_2d(sa + static_cast<size_t>(i) * a_bytes, &tmap_w, &full[i], kblk * kBK, wrow, pol_w);
        advance();
      }
      pdl_wait();
      trace_min(e.trace, 1);
      for (int i = 0; i < pre; ++i)
        tma_load_2d(sb + static_cast<size_t>(i) * b_bytes, &tmap_x, &full[i], pre_kblk[i] * kBK, pre_xrow[i], pol_x);
      int stage = pre % S;
      uint32_t phase = (pre == S) ? 1u : 0u;
      while (k < nsegs) {
        mbar_wait(&empty[stage], phase ^ 1u);
        mbar_arrive_expect_tx(&full[stage], a_bytes + b_bytes);
        tma_load_2d(sa + static_cast<size_t>(stage) * a_bytes, &tmap_w, &full[stage], kblk * kBK, wrow, pol_w);
        tma_load_2d(sb + static_cast<size_t>(stage) * b_bytes, &tmap_x, &full[stage], kblk * kBK, xrow, pol_x);
        if (++stage == S) { stage = 0; phase ^= 1u; }
        advance();
      }
      if (e.dbg) e.dbg[c * 8 + 6] = gtimer();
      trace_max(e.trace, 3);  // producer: last load issued
    }
  } else if (warp == 1) {
    pdl_wait();
    // ===== MMA issuer =====
    const uint32_t idesc = umma_idesc_bf16(kBM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase[2] = {0u, 0u};
    for (int k = 0; k < nsegs; ++k) {
      long long a, b;
      segment(k, a, b);
      // Wait for the epilogue to drain this accumulator buffer.
      mbar_wait(&tempty[acc], acc_phase[acc] ^ 1u);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
      for (long long u = a; u < b; ++u) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_addr = smem_u32(sa + static_cast<size_t>(stage) * a_bytes);
          const uint32_t b_addr = smem_u32(sb + static_cast<size_t>(stage) * b_bytes);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t ad = umma_desc_sw128(a_addr + kk * 32);
            const uint64_t bd = umma_desc_sw128(b_addr + kk * 32);
            umma_bf16(d_tmem, ad, bd, idesc, (u == a && kk == 0) ? 0u : 1u);
          }
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == S) { stage = 0; phase ^= 1u; }
      }
      if (lane == 0) umma_commit(&tfull[acc]);
      __syncwarp();
      acc_phase[acc] ^= 1u;
      acc ^= 1;
    }
    if (e.dbg && lane == 0) e.dbg[c * 8 + 5] = gtimer();
    if (lane == 0) trace_max(e.trace, 4);  // mma: last commit
  } else {
    pdl_wait();
    // ===== Epilogue warps: TMEM -> (partials | fused op) =====
    const int quarter = warp & 3;  // TMEM lanes accessible by this warp
    const int row = quarter * 32 + lane;
    const int et = threadIdx.x - 64;  // 0..127
    if (KIND != kEpiNone && e.ss_in) {
      for (int m = et; m < p.M; m += 128) {
        float s = 0.f;
#pragma unroll 16
        for (int t = 0; t < e.ss_tiles; ++t) s += __ldg(e.ss_in + static_cast<size_t>(t) * p.M + m);
        rstd_s[m] = rsqrtf(s / static_cast<float>(e.norm_dim) + e.eps);
      }
      epi_bar();
    }
    int acc = 0;
    uint32_t acc_phase[2] = {0u, 0u};
    int npend = 0;
    for (int k = 0; k < nsegs; ++k) {
      long long a, b;
      segment(k, a, b);
      const int tile = static_cast<int>(a / p.kb);
      const int s_first = p.seg_first[tile], s_end = p.seg_first[tile + 1];
      const int nseg = s_end - s_first;
      const int seg = (k == 0 && n_sk > 0) ? p.seg_base[c] : s_first;
      const int m_tile = tile % p.m_tiles, n_tile = tile / p.m_tiles;
      const int valid = min(BN, p.M - m_tile * BN);
      const int n = n_tile * kBM + row;
      mbar_wait(&tfull[acc], acc_phase[acc]);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * BN);
      if (KIND != kEpiNone && nseg == 1) {
        // Whole tile accumulated here: finish it straight from TMEM.
        for (int c0 = 0; c0 < BN; c0 += 16) {
          float v[16];
          tmem_ld16(taddr + c0, v);
          epi_apply<KIND>(e, p.M, n, m_tile * BN + c0, valid - c0, v, rstd_s, red_s, quarter, lane);
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
      } else {
        float* dst = ws + static_cast<size_t>(seg) * BN * kBM + row;
        for (int c0 = 0; c0 < BN; c0 += 16) {
          float v[16];
          tmem_ld16(taddr + c0, v);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < valid) dst[static_cast<size_t>(c0 + j) * kBM] = v[j];
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        if (KIND != kEpiNone) {
          // Publish the partial: CTA barrier, then one release-ordered arrival on the tile's epoch
          // counter (monotonic: launch L of this plan moves it from L*nseg to (L+1)*nseg).
          epi_bar();
          if (et == 0) {
            int old;
            asm volatile("atom.add.release.gpu.global.s32 %0, [%1], 1;" : "=r"(old) : "l"(e.counters + tile) : "memory");
            pend_tile[npend] = tile;
            pend_j[npend] = seg - s_first;
            pend_tgt[npend] = (old / nseg + 1) * nseg;
          }
          ++npend;
        }
      }
      acc_phase[acc] ^= 1u;
      acc ^= 1;
      if (k == min(n_sk, 2) - 1 && npend > 0) {
        if (e.dbg && et == 0) e.dbg[c * 8 + 1] = gtimer();
        if (et == 0) trace_max(e.trace, 5);  // fixups start
        // Cooperative fixups (right after this CTA's split segments, overlapping the whole tiles
        // still streaming): participant j reduces 16-token column chunks j, j+nseg, ... in fixed
        // segment order and applies the op.
        for (int i = 0; i < npend; ++i) {
          epi_bar();
          const int ft = pend_tile[i], fj = pend_j[i], target = pend_tgt[i];
          const int fs = p.seg_first[ft];
          const int fn = p.seg_first[ft + 1] - fs;
          const int fm = ft % p.m_tiles;
          const int fvalid = min(BN, p.M - fm * BN);
          const int fcol = (ft / p.m_tiles) * kBM + row;
          if (et == 0) {
            const long long t0 = clock64();
            while (ld_acquire(e.counters + ft) < target) {
              __nanosleep(32);
              if (clock64() - t0 > (1ll << 34)) __trap();
            }
          }
          epi_bar();
          if (e.dbg && et == 0) e.dbg[c * 8 + 2 + i] = gtimer();
          if (et == 0) trace_max(e.trace, 6);  // a fixup's partials all arrived
          const float* src = ws + static_cast<size_t>(fs) * BN * kBM + row;
          for (int c0 = fj * 16; c0 < BN; c0 += fn * 16) {
            const int nv = min(16, fvalid - c0);
            float v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = 0.f;
            // Four segments' loads in flight at a time; summed in segment order (deterministic).
            for (int s = 0; s < fn; s += 4) {
              float t[4][16];
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const float* ps = src + static_cast<size_t>(s + kk) * BN * kBM;
#pragma unroll
                for (int q = 0; q < 16; ++q)
                  t[kk][q] = (s + kk < fn && q < nv) ? __ldcg(ps + static_cast<size_t>(c0 + q) * kBM) : 0.f;
              }
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                for (int q = 0; q < 16; ++q) v[q] += t[kk][q];
            }
            epi_apply<KIND>(e, p.M, fcol, fm * BN + c0, fvalid - c0, v, rstd_s, red_s, quarter, lane);
          }
        }
        npend = 0;
      }
    }
    if (e.dbg && et == 0) e.dbg[c * 8 + 4] = gtimer();
    if (et == 0) trace_max(e.trace, 7);  // epilogue warps done
  }
  __syncthreads();
  if (threadIdx.x == 0) trace_max(e.trace, 2);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// ---------------------------------------------------------------------------
// Cluster split-K kernel: one (cs, 1, 1) thread-block cluster per output tile, the tile's K range
// split evenly over the cs CTAs, the partials reduce-scattered through DSMEM: the tile's 16-token
// column chunks are owned round-robin by the cluster's CTAs (chunk q -> rank q % cs), every CTA
// stores the chunks it does not own into their owner's receive slots, and after one cluster barrier
// each owner sums its chunk's cs partials in rank order (deterministic) and applies the fused
// epilogue.  No global partials, no arrival counters, no fixups, and the epilogue's global round
// trips are spread over the cluster (one chunk per CTA at cs = 4).  A tile's CTAs are co-scheduled
// and stream the same number of weight bytes, so they reach the exchange together.  Used where the
// tile count times the cluster size fits one wave (the cfg2 verify's O / down: 32 tiles x 4 CTAs).
// ---------------------------------------------------------------------------
struct ClusterParams {
  int M, BN, m_tiles, kb, stages, tmem_cols, cs;
  int own_max;  // chunks owned per CTA (ceil(BN/16 / cs)); receive slots per CTA = (cs-1) * own_max
};

constexpr int kChunkBytes = 16 * kBM * 4;  // one 16-token x 128-feature f32 partial chunk

__host__ __device__ inline size_t cluster_recv_bytes(int cs, int BN) {
  const int nchunks = BN / 16;
  const int own_max = (nchunks + cs - 1) / cs;
  return static_cast<size_t>(cs - 1) * own_max * kChunkBytes;
}

template <int KIND>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_cluster_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x,
                        ClusterParams p, EpiArgs e) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int BN = p.BN, S = p.stages, cs = p.cs;
  const uint32_t a_bytes = kBM * kBK * 2;
  const uint32_t b_bytes = BN * kBK * 2;
  unsigned char* sa = base;
  unsigned char* sb = base + static_cast<size_t>(S) * a_bytes;
  // receive slots [cs-1][own_max][16/4][128][4] f32, outside the ring: peers may store into them
  // while this CTA is still streaming
  float* recv = reinterpret_cast<float*>(sb + static_cast<size_t>(S) * b_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(recv) +
                                               static_cast<size_t>(cs - 1) * p.own_max * kChunkBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 2);
  float* red_s = reinterpret_cast<float*>(tmem_slot + 8);  // [4][16]
  float* rstd_s = red_s + 64;                             // [kMaxRstdTokens]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = static_cast<int>(cluster_ctarank_u32());
  const int tile = blockIdx.x / cs;
  const int m_tile = tile % p.m_tiles, n_tile = tile / p.m_tiles;
  const int k0 = p.kb * rank / cs, k1 = p.kb * (rank + 1) / cs;
  const int nk = k1 - k0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_w);
    tma_prefetch_desc(&tmap_x);
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&tfull[0], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // first cluster-barrier phase: "this CTA has started"; waited on just before the DSMEM scatter
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) trace_min(e.trace, 0);
  pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer: weights before the grid-dependency wait, activations after =====
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      const int wrow = n_tile * kBM, xrow = m_tile * BN;
      const int pre = nk < S ? nk : S;
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], a_bytes + b_bytes);
        tma_load_2d(sa + static_cast<size_t>(i) * a_bytes, &tmap_w, &full[i], (k0 + i) * kBK, wrow, pol_w);
      }
      pdl_wait();
      trace_min(e.trace, 1);
      for (int i = 0; i < pre; ++i)
        tma_load_2d(sb + static_cast<size_t>(i) * b_bytes, &tmap_x, &full[i], (k0 + i) * kBK, xrow, pol_x);
      int stage = pre % S;
      uint32_t phase = (pre == S) ? 1u : 0u;
      for (int kb = k0 + pre; kb < k1; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1u);
        mbar_arrive_expect_tx(&full[stage], a_bytes + b_bytes);
        tma_load_2d(sa + static_cast<size_t>(stage) * a_bytes, &tmap_w, &full[stage], kb * kBK, wrow, pol_w);
        tma_load_2d(sb + static_cast<size_t>(stage) * b_bytes, &tmap_x, &full[stage], kb * kBK, xrow, pol_x);
        if (++stage == S) { stage = 0; phase ^= 1u; }
      }
      trace_max(e.trace, 3);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===== MMA issuer (one accumulator: one K range per CTA) =====
    const uint32_t idesc = umma_idesc_bf16(kBM, BN);
    int stage = 0;
    uint32_t phase = 0;
    for (int u = 0; u < nk; ++u) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a_addr = smem_u32(sa + static_cast<size_t>(stage) * a_bytes);
        const uint32_t b_addr = smem_u32(sb + static_cast<size_t>(stage) * b_bytes);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)
          umma_bf16(tmem_base, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32), idesc,
                    (u == 0 && kk == 0) ? 0u : 1u);
        umma_commit(&empty[stage]);
      }
      __syncwarp();
      if (++stage == S) { stage = 0; phase ^= 1u; }
    }
    if (lane == 0) {
      umma_commit(&tfull[0]);
      trace_max(e.trace, 4);
    }
    __syncwarp();
  } else {
    // ===== epilogue warps: the previous kernel's outputs become visible, then the folded-RMSNorm
    // rstd of every token is computed while the mainloop runs =====
    pdl_wait();
    if (KIND != kEpiNone && e.ss_in) {
      const int et = threadIdx.x - 64;
      for (int m = et; m < p.M; m += 128) {
        float s = 0.f;
#pragma unroll 16
        for (int t = 0; t < e.ss_tiles; ++t) s += __ldg(e.ss_in + static_cast<size_t>(t) * p.M + m);
        rstd_s[m] = rsqrtf(s / static_cast<float>(e.norm_dim) + e.eps);
      }
      epi_bar();
    }
  }
  const int quarter = warp & 3;
  const int row = quarter * 32 + lane;
  const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16);
  const int valid = min(BN, p.M - m_tile * BN);
  const int nchunks = (valid + 15) / 16;  // chunks holding at least one real token
  // every CTA of the cluster has started (arrived right after its set-up) before any DSMEM store
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  if (warp >= 2) {
    mbar_wait(&tfull[0], 0);
    tc_fence_after();
    // scatter: every chunk this CTA does not own goes to its owner's receive slot for this rank
    for (int q = 0; q < nchunks; ++q) {
      const int owner = q % cs;
      if (owner == rank) continue;
      float v[16];
      tmem_ld16(taddr + q * 16, v);
      const int slot = (rank - owner - 1 + cs) % cs;  // 0..cs-2, the source's position after the owner
      const int local = q / cs;
      const uint32_t dst = mapa_shared(smem_u32(recv), static_cast<uint32_t>(owner)) +
                           static_cast<uint32_t>((((slot * p.own_max + local) * 4) * kBM + row) * 16);
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4)
        st_cluster_v4(dst + static_cast<uint32_t>(c4 * kBM * 16), v[4 * c4], v[4 * c4 + 1], v[4 * c4 + 2],
                      v[4 * c4 + 3]);
    }
  }
  // every partial is in its owner's shared memory (release / acquire at cluster scope)
  cluster_sync();
  if (warp >= 2) {
    const int n = n_tile * kBM + row;
    for (int q = rank; q < nchunks; q += cs) {
      const int local = q / cs;
      float own[16], v[16];
      tmem_ld16(taddr + q * 16, own);
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = 0.f;
      for (int r = 0; r < cs; ++r) {  // rank order: deterministic
        if (r == rank) {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] += own[j];
        } else {
          const int slot = (r - rank - 1 + cs) % cs;
          const float4* src = reinterpret_cast<const float4*>(recv) + ((slot * p.own_max + local) * 4) * kBM + row;
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const float4 x = src[c4 * kBM];
            v[4 * c4] += x.x;
            v[4 * c4 + 1] += x.y;
            v[4 * c4 + 2] += x.z;
            v[4 * c4 + 3] += x.w;
          }
        }
      }
      if constexpr (KIND != kEpiNone)
        epi_apply<KIND>(e, p.M, n, m_tile * BN + q * 16, valid - q * 16, v, rstd_s, red_s, quarter, lane);
    }
    if (threadIdx.x == 64) trace_max(e.trace, 7);
  }
  __syncthreads();
  if (threadIdx.x == 0) trace_max(e.trace, 2);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// ---------------------------------------------------------------------------
// SIMT f32 kernel (parity mode): 128 (n) x 32 (m) tile per CTA, 256 threads, 4x4 per thread.
// ---------------------------------------------------------------------------
constexpr int kSimtBN = 32, kSimtBK = 32;
__global__ void __launch_bounds__(256) gemm_f32_simt_kernel(const float* __restrict__ W, const float* __restrict__ X,
                                                            int M, int N, int K, int BN, int m_tiles,
                                                            float* __restrict__ ws) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ float sw[kSimtBK][kBM + 4];
  __shared__ float sx[kSimtBK][kSimtBN + 4];
  const int n_tile = blockIdx.x, msub = blockIdx.y;  // msub: 32-token slice of the full M
  const int m0 = msub * kSimtBN;
  const int tid = threadIdx.x;
  const int tn = tid % 32, tm = tid / 32;  // thread owns n = tn + 32*i, m = tm + 8*j
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += kSimtBK) {
    for (int i = tid; i < kBM * kSimtBK; i += 256) {
      const int r = i / kSimtBK, kk = i % kSimtBK;
      sw[kk][r] = W[static_cast<size_t>(n_tile * kBM + r) * K + k0 + kk];
    }
    for (int i = tid; i < kSimtBN * kSimtBK; i += 256) {
      const int r = i / kSimtBK, kk = i % kSimtBK;
      const int m = m0 + r;
      sx[kk][r] = (m < M) ? X[static_cast<size_t>(m) * K + k0 + kk] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < kSimtBK; ++kk) {
      float a[4], bx[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sw[kk][tn + 32 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bx[j] = sx[kk][tm + 8 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bx[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int m = m0 + tm + 8 * j;
    if (m >= M) continue;
    const int m_tile = m / BN, mr = m % BN;
    const int seg = n_tile * m_tiles + m_tile;
#pragma unroll
    for (int i = 0; i < 4; ++i) ws[(static_cast<size_t>(seg) * BN + mr) * kBM + tn + 32 * i] = acc[i][j];
  }
}

// ---------------------------------------------------------------------------
// Epilogues.  value(m, n) = sum over segments of tile(n/128, m/BN) of ws[seg][m%BN][n%128].
// ---------------------------------------------------------------------------
struct EpiGeom {
  int M, N, BN, m_tiles;
  const int32_t* seg_first;
  unsigned long long* trace;  // kernel-timeline slot (profiling only) or nullptr
  const char* pf;             // L2 prefetch region (a later weight stream) or nullptr
  size_t pf_bytes;
  int il;                     // fused-layout rows (model.prepare_fused_): pairs are adjacent rows
};

// The epilogue kernels barely touch HBM (their partials are L2 hits): right after the dependency
// wait, thread 0 of every CTA pulls its share of a later weight stream into L2 (bulk prefetch,
// <= 64 KB per instruction, fire and forget), so the next GEMM starts that much of its stream from L2.
YGG_DEV void epi_l2_prefetch(const EpiGeom& g) {
  if (!g.pf || threadIdx.x != 0) return;
  const size_t ncta = static_cast<size_t>(gridDim.x) * gridDim.y;
  const size_t cta = static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x;
  const size_t per = ((g.pf_bytes / ncta) + 255) & ~static_cast<size_t>(255);
  const size_t b0 = cta * per, b1 = b0 + per < g.pf_bytes ? b0 + per : g.pf_bytes;
  for (size_t o = b0; o < b1; o += 65536) {
    const uint32_t n = static_cast<uint32_t>(b1 - o < 65536 ? ((b1 - o) & ~static_cast<size_t>(15)) : 65536);
    if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g.pf + o), "r"(n) : "memory");
  }
}

YGG_DEV float epi_value(const EpiGeom& g, const float* __restrict__ ws, int m, int n) {
  const int t = (n / kBM) * g.m_tiles + m / g.BN;
  const int s0 = g.seg_first[t], s1 = g.seg_first[t + 1];
  const size_t off = static_cast<size_t>(m % g.BN) * kBM + (n % kBM);
  float v = 0.f;
  for (int s = s0; s < s1; ++s) v += ws[static_cast<size_t>(s) * g.BN * kBM + off];
  return v;
}

// Segment range [s0, s1) of the tile holding (row m, feature n): plan constants, so the epilogue
// kernels load them before their grid-dependency wait.
YGG_DEV int2 epi_segs(const EpiGeom& g, int m, int n) {
  const int t = (n / kBM) * g.m_tiles + m / g.BN;
  return make_int2(__ldg(g.seg_first + t), __ldg(g.seg_first + t + 1));
}

template <int V>
YGG_DEV void epi_values(const EpiGeom& g, const float* __restrict__ ws, int m, int n, float* v, int2 sg);

template <int V>
YGG_DEV void epi_values(const EpiGeom& g, const float* __restrict__ ws, int m, int n, float* v) {
  epi_values<V>(g, ws, m, n, v, epi_segs(g, m, n));
}

// Sum of the partials of V consecutive features [n, n+V) of row m (n % V == 0, one tile).
template <int V>
YGG_DEV void epi_values(const EpiGeom& g, const float* __restrict__ ws, int m, int n, float* v, int2 sg) {
  const int s0 = sg.x, s1 = sg.y;
  const float* p = ws + static_cast<size_t>(m % g.BN) * kBM + (n % kBM);
  const size_t seg_stride = static_cast<size_t>(g.BN) * kBM;
#pragma unroll
  for (int i = 0; i < V; ++i) v[i] = 0.f;
#pragma unroll 4
  for (int s = s0; s < s1; ++s) {
    const float4* q = reinterpret_cast<const float4*>(p + s * seg_stride);
#pragma unroll
    for (int i = 0; i < V / 4; ++i) {
      const float4 x = __ldcg(q + i);
      v[4 * i] += x.x;
      v[4 * i + 1] += x.y;
      v[4 * i + 2] += x.z;
      v[4 * i + 3] += x.w;
    }
  }
}

// Partial sums of two V-wide feature runs [n1, n1+V) and [n2, n2+V) of row m (possibly different
// tiles), both runs' loads in flight together; each run summed in its own segment order.
template <int V>
YGG_DEV void epi_values2(const EpiGeom& g, const float* __restrict__ ws, int m, int n1, int n2, float* v1, float* v2,
                         int2 sa, int2 sb) {
  const int a0 = sa.x, a1 = sa.y, b0 = sb.x, b1 = sb.y;
  const size_t row = static_cast<size_t>(m % g.BN) * kBM;
  const float* p1 = ws + row + (n1 % kBM);
  const float* p2 = ws + row + (n2 % kBM);
  const size_t seg_stride = static_cast<size_t>(g.BN) * kBM;
#pragma unroll
  for (int i = 0; i < V; ++i) v1[i] = v2[i] = 0.f;
  const int na = a1 - a0, nb = b1 - b0, n = na > nb ? na : nb;
  for (int j = 0; j < n; j += 4) {
    float4 x[4][2][V / 4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4* q1 = reinterpret_cast<const float4*>(p1 + (a0 + j + k) * seg_stride);
      const float4* q2 = reinterpret_cast<const float4*>(p2 + (b0 + j + k) * seg_stride);
#pragma unroll
      for (int i = 0; i < V / 4; ++i) {
        x[k][0][i] = (j + k < na) ? __ldcg(q1 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        x[k][1][i] = (j + k < nb) ? __ldcg(q2 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int i = 0; i < V / 4; ++i) {
        v1[4 * i] += x[k][0][i].x; v1[4 * i + 1] += x[k][0][i].y; v1[4 * i + 2] += x[k][0][i].z; v1[4 * i + 3] += x[k][0][i].w;
        v2[4 * i] += x[k][1][i].x; v2[4 * i + 1] += x[k][1][i].y; v2[4 * i + 2] += x[k][1][i].z; v2[4 * i + 3] += x[k][1][i].w;
      }
  }
}

template <typename T>
YGG_DEV void store8(T* dst, const float* v);
template <>
YGG_DEV void store8<float>(float* dst, const float* v) {
  reinterpret_cast<float4*>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
}
template <>
YGG_DEV void store8<__nv_bfloat16>(__nv_bfloat16* dst, const float* v) {
  uint4 u;
  __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
  __nv_bfloat162 c = __floats2bfloat162_rn(v[4], v[5]), d = __floats2bfloat162_rn(v[6], v[7]);
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  u.z = *reinterpret_cast<uint32_t*>(&c);
  u.w = *reinterpret_cast<uint32_t*>(&d);
  *reinterpret_cast<uint4*>(dst) = u;
}
template <typename T>
YGG_DEV void load8(const T* src, float* v);
template <>
YGG_DEV void load8<float>(const float* src, float* v) {
  const float4 a = reinterpret_cast<const float4*>(src)[0], b = reinterpret_cast<const float4*>(src)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
template <>
YGG_DEV void load8<__nv_bfloat16>(const __nv_bfloat16* src, float* v) {
  const uint4 u = *reinterpret_cast<const uint4*>(src);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
    v[2 * i] = __bfloat162float(b.x);
    v[2 * i + 1] = __bfloat162float(b.y);
  }
}

constexpr int kEpiThreads = 128;  // x 8 features = 1024 features per CTA

template <typename OutT>
__global__ void __launch_bounds__(kEpiThreads) epi_store_kernel(EpiGeom g, const float* __restrict__ ws,
                                                                OutT* __restrict__ out, int ld) {
  if (threadIdx.x == 0) trace_min(g.trace, 0);
  const int m = blockIdx.y;
  const int n = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  const int2 sg = n < g.N ? epi_segs(g, m, n) : make_int2(0, 0);
  pdl_wait();
  pdl_launch_dependents();
  epi_l2_prefetch(g);
  if (threadIdx.x == 0) trace_min(g.trace, 1);
  if (n >= g.N) return;
  float v[8];
  epi_values<8>(g, ws, m, n, v, sg);
  store8<OutT>(out + static_cast<size_t>(m) * ld + n, v);
  if (threadIdx.x == 0) trace_max(g.trace, 2);
}

YGG_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
YGG_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
YGG_DEV float ld_dsmem_f32(const float* local, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(rank));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
  return v;
}

// Residual add + RMSNorm of one row per CTA (N/8 threads, 8 features each): every global load of the
// row (partials, residual, norm gains) is issued before any use, and the sum of squares is one
// block reduction in fixed warp order (deterministic).
template <typename ActT>
__global__ void __launch_bounds__(1024) epi_residual_norm_kernel(EpiGeom g, const float* __restrict__ ws,
                                                                 float* __restrict__ resid,
                                                                 const ActT* __restrict__ norm_w, float eps,
                                                                 ActT* __restrict__ xn) {
  if (threadIdx.x == 0) trace_min(g.trace, 0);
  __shared__ float red[32];
  const int m = blockIdx.x;
  const int n = threadIdx.x * 8;
  const bool live = n < g.N;
  float h[8], w[8], v[8];
  int2 sg = make_int2(0, 0);
  if (live) {  // plan constants and the norm gains before the dependency wait
    sg = epi_segs(g, m, n);
    load8<ActT>(norm_w + n, w);
  }
  pdl_wait();
  pdl_launch_dependents();
  epi_l2_prefetch(g);
  if (threadIdx.x == 0) trace_min(g.trace, 1);
  float ss = 0.f;
  if (live) {
    float* hp = resid + static_cast<size_t>(m) * g.N + n;
    load8<float>(hp, h);
    epi_values<8>(g, ws, m, n, v, sg);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      h[i] += v[i];
      ss += h[i] * h[i];
    }
    store8<float>(hp, h);
  }
  ss = warp_sum(ss);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  float total = 0.f;
  for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) total += red[k];
  const float rs = rsqrtf(total / static_cast<float>(g.N) + eps);
  if (live) {
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = h[i] * rs * w[i];
    store8<ActT>(xn + static_cast<size_t>(m) * g.N + n, h);
  }
  if (threadIdx.x == 0) trace_max(g.trace, 2);
}

// R tokens per thread (R > 1 for wide passes: fewer, fuller CTAs, R tokens' loads in flight together).
template <typename ActT, int R>
__global__ void __launch_bounds__(kEpiThreads) epi_swiglu_kernel(EpiGeom g, const float* __restrict__ ws,
                                                                 ActT* __restrict__ out) {
  if (threadIdx.x == 0) trace_min(g.trace, 0);
  const int m0 = blockIdx.y * R;
  const int F = g.N / 2;
  const int f = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  // fused layout: gate j / up j are rows 2j / 2j + 1, so this thread's 16 rows start at 2f (one tile)
  const int na = g.il ? 2 * f : f, nb = g.il ? 2 * f + 8 : F + f;
  int2 sa[R], sb[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const bool ok = f < F && m0 + r < g.M;
    sa[r] = ok ? epi_segs(g, m0 + r, na) : make_int2(0, 0);
    sb[r] = ok ? epi_segs(g, m0 + r, nb) : make_int2(0, 0);
  }
  pdl_wait();
  pdl_launch_dependents();
  epi_l2_prefetch(g);
  if (threadIdx.x == 0) trace_min(g.trace, 1);
  if (f >= F) return;
  float a[R][8], b[R][8];
  bool single = true;  // every run of this thread's tokens lies in a whole (one-segment) tile
#pragma unroll
  for (int r = 0; r < R; ++r) single = single && sa[r].y - sa[r].x <= 1 && sb[r].y - sb[r].x <= 1;
  if (single) {
    const size_t seg_stride = static_cast<size_t>(g.BN) * kBM;
    float4 xa[R][2], xb[R][2];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const size_t row = static_cast<size_t>((m0 + r) % g.BN) * kBM;
      const float4* qa = reinterpret_cast<const float4*>(ws + sa[r].x * seg_stride + row + (na % kBM));
      const float4* qb = reinterpret_cast<const float4*>(ws + sb[r].x * seg_stride + row + (nb % kBM));
      const bool ok = sa[r].y > sa[r].x;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        xa[r][i] = ok ? __ldcg(qa + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        xb[r][i] = ok ? __ldcg(qb + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        a[r][4 * i] = xa[r][i].x; a[r][4 * i + 1] = xa[r][i].y; a[r][4 * i + 2] = xa[r][i].z; a[r][4 * i + 3] = xa[r][i].w;
        b[r][4 * i] = xb[r][i].x; b[r][4 * i + 1] = xb[r][i].y; b[r][4 * i + 2] = xb[r][i].z; b[r][4 * i + 3] = xb[r][i].w;
      }
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (m0 + r < g.M) epi_values2<8>(g, ws, m0 + r, na, nb, a[r], b[r], sa[r], sb[r]);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (m0 + r >= g.M) break;
    float gate[8], up[8], o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (g.il) {
        gate[i] = i < 4 ? a[r][2 * i] : b[r][2 * (i - 4)];
        up[i] = i < 4 ? a[r][2 * i + 1] : b[r][2 * (i - 4) + 1];
      } else {
        gate[i] = a[r][i];
        up[i] = b[r][i];
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = gate[i] / (1.f + expf(-gate[i])) * up[i];
    store8<ActT>(out + static_cast<size_t>(m0 + r) * F + f, o);
  }
  if (threadIdx.x == 0) trace_max(g.trace, 2);
}

// Row argmax over the ARGMAX epilogue's per-tile keys: one CTA per token row, max over tiles.
__global__ void __launch_bounds__(256) argmax_reduce_kernel(const unsigned long long* __restrict__ keys, int ntiles,
                                                            int M, int32_t* __restrict__ out) {
  pdl_wait();
  pdl_launch_dependents();
  const int m = blockIdx.x;
  unsigned long long best = 0ull;
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
    const unsigned long long k = __ldcg(keys + static_cast<size_t>(t) * M + m);
    best = k > best ? k : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long q = __shfl_xor_sync(0xffffffffu, best, o);
    best = q > best ? q : best;
  }
  __shared__ unsigned long long wb[8];
  if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) best = wb[w] > best ? wb[w] : best;
    out[m] = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(best & 0xFFFFFFFFull));
  }
}

// QKV epilogue: RoPE (rotate-half convention) on q and k at pos[m]; q -> q_out, k/v -> KV cache.
// Work item = 4 rotation pairs (i..i+3, i+half..i+half+3) of one head; one item per thread.
// cos/sin come from the host table rope_cs [positions][hd/2] when given (else sincosf).
template <typename ActT>
__global__ void __launch_bounds__(256) epi_qkv_rope_kernel(EpiGeom g, const float* __restrict__ ws, int Hq, int Hkv,
                                                           int hd, float log2_theta, const int32_t* __restrict__ pos,
                                                           const int32_t* __restrict__ slot,
                                                           const int32_t* __restrict__ req, ActT* __restrict__ q_out,
                                                           ActT* __restrict__ cache, int S,
                                                           const float2* __restrict__ rope_cs) {
  if (threadIdx.x == 0) trace_min(g.trace, 0);
  const int m = blockIdx.x;
  const int half = hd / 2;
  const int per_head = half / 4;
  const int items = (Hq + 2 * Hkv) * per_head;
  const int it = blockIdx.y * blockDim.x + threadIdx.x;
  const int head = it / per_head;
  const int i0 = (it % per_head) * 4;
  const int n0 = head * hd;
  // fused layout: rotation pair (i, i + hd/2) of a head is rows (2i, 2i + 1): this thread's 8 rows from 2*i0
  const int2 sa = it < items ? epi_segs(g, m, g.il ? n0 + 2 * i0 : n0 + i0) : make_int2(0, 0);
  const int2 sb = it < items ? epi_segs(g, m, g.il ? n0 + 2 * i0 : n0 + i0 + half) : make_int2(0, 0);
  pdl_wait();
  pdl_launch_dependents();
  epi_l2_prefetch(g);
  if (threadIdx.x == 0) trace_min(g.trace, 1);
  if (it >= items) return;
  const int pm = pos[m];
  float x1[4], x2[4], cs[4], sn[4];
  const bool rot = head < Hq + Hkv;
  if (rot && rope_cs) {  // table loads first: they overlap the partial-sum loads below
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 t = __ldg(rope_cs + static_cast<size_t>(pm) * half + i0 + j);
      cs[j] = t.x;
      sn[j] = t.y;
    }
  }
  if (g.il) {
    float v[8];
    epi_values<8>(g, ws, m, n0 + 2 * i0, v, sa);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x1[j] = v[2 * j];
      x2[j] = v[2 * j + 1];
    }
  } else {
    epi_values2<4>(g, ws, m, n0 + i0, n0 + i0 + half, x1, x2, sa, sb);
  }
  if (rot) {
    if (rope_cs) {
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        // inv_freq = theta^(-2i/hd), as 1/(theta**(2i/hd)) in f32
        const float inv_freq = 1.0f / exp2f(log2_theta * (static_cast<float>(2 * (i0 + j)) / static_cast<float>(hd)));
        sincosf(static_cast<float>(pm) * inv_freq, &sn[j], &cs[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float y1 = x1[j] * cs[j] - x2[j] * sn[j];
      const float y2 = x2[j] * cs[j] + x1[j] * sn[j];
      x1[j] = y1;
      x2[j] = y2;
    }
  }
  if (head < Hq) {
    ActT* q = q_out + (static_cast<size_t>(m) * Hq + head) * hd;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      q[i0 + j] = from_f32<ActT>(x1[j]);
      q[i0 + j + half] = from_f32<ActT>(x2[j]);
    }
  } else {
    const bool is_v = head >= Hq + Hkv;
    const int kvh = is_v ? head - Hq - Hkv : head - Hq;
    const size_t base = ((static_cast<size_t>(req[m]) * 2 + (is_v ? 1 : 0)) * Hkv + kvh) * static_cast<size_t>(S) * hd;
    const int sl = slot[m];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (!is_v) {  // K rows: [S][hd]
        cache[base + static_cast<size_t>(sl) * hd + i0 + j] = from_f32<ActT>(x1[j]);
        cache[base + static_cast<size_t>(sl) * hd + i0 + j + half] = from_f32<ActT>(x2[j]);
      } else {      // V transposed: [hd][S], so attention reads K-major V^T tiles
        cache[base + static_cast<size_t>(i0 + j) * S + sl] = from_f32<ActT>(x1[j]);
        cache[base + static_cast<size_t>(i0 + j + half) * S + sl] = from_f32<ActT>(x2[j]);
      }
    }
  }
  if (threadIdx.x == 0) trace_max(g.trace, 2);
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

static int make_map_bf16(CUtensorMap* map, const void* ptr, int rows, int cols, int box_rows) {
  auto enc = get_encode();
  if (!enc) return ygg_fail(YGG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return ygg_fail(YGG_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return YGG_OK;
}

static const GemmPlan* as_plan(const void* p) {
  const GemmPlan* g = static_cast<const GemmPlan*>(p);
  return (g && g->magic == kPlanMagic) ? g : nullptr;
}

static EpiGeom geom_of(const GemmPlan* g, int kernel_id) {
  return EpiGeom{g->M, g->N, g->BN, g->m_tiles, g->seg_table, trace_next(kernel_id), g->epi_pf, g->epi_pf_bytes,
                 g->interleaved};
}

}  // namespace ygg

using namespace ygg;

// Ring stages of a cluster plan: the stream-K budget minus the receive slots.
static int cluster_stages(const GemmPlan* g, int cs) {
  const int stage_bytes = kBM * kBK * 2 + g->BN * kBK * 2;
  const long long avail = 190LL * 1024 - kSmemExtra - static_cast<long long>(cluster_recv_bytes(cs, g->BN));
  return static_cast<int>(std::min<long long>(12, avail / stage_bytes));
}

static size_t cluster_smem(const GemmPlan* g) {
  return kSmemExtra + static_cast<size_t>(cluster_stages(g, g->cluster)) * (kBM * kBK * 2 + g->BN * kBK * 2) +
         cluster_recv_bytes(g->cluster, g->BN);
}

template <int KIND>
static int launch_cluster_kind(const GemmPlan* g, const EpiArgs& e, cudaStream_t s) {
  const int nchunks = g->BN / 16;
  ClusterParams cp{g->M, g->BN, g->m_tiles, g->kb, cluster_stages(g, g->cluster), g->tmem_cols, g->cluster,
                   (nchunks + g->cluster - 1) / g->cluster};
  return launch_pdl_cluster_x(gemm_cluster_kernel<KIND>, dim3(g->tiles * g->cluster), dim3(kGemmThreads),
                              cluster_smem(g), g->cluster, s, g->tmap_w, g->tmap_x, cp, e);
}

extern "C" {

int ygg_prepare_gemm(void) {
  cudaError_t e = cudaSuccess;
  for (auto fn : {gemm_bf16_tc_kernel<kEpiNone>, gemm_bf16_tc_kernel<kEpiStoreF32>, gemm_bf16_tc_kernel<kEpiQkvRope>,
                  gemm_bf16_tc_kernel<kEpiSwiglu>, gemm_bf16_tc_kernel<kEpiResid>, gemm_bf16_tc_kernel<kEpiArgmax>}) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "gemm attribute: %s", cudaGetErrorString(e));
  }
  for (auto fn : {gemm_cluster_kernel<kEpiNone>, gemm_cluster_kernel<kEpiStoreF32>, gemm_cluster_kernel<kEpiQkvRope>,
                  gemm_cluster_kernel<kEpiSwiglu>, gemm_cluster_kernel<kEpiResid>}) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "gemm attribute: %s", cudaGetErrorString(e));
  }
  for (auto fn : {gemm_cluster_kernel<kEpiNone>, gemm_cluster_kernel<kEpiStoreF32>, gemm_cluster_kernel<kEpiQkvRope>,
                  gemm_cluster_kernel<kEpiSwiglu>, gemm_cluster_kernel<kEpiResid>}) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "gemm cluster attribute: %s", cudaGetErrorString(e));
  }
  return YGG_OK;
}

size_t ygg_gemm_plan_size(void) { return sizeof(GemmPlan) + 64; }

int ygg_gemm_plan_init(void* plan_mem, int dtype, const void* W, const void* X, int M, int N, int K, int num_ctas,
                       int32_t* seg_table_dev, int* num_segments, size_t* workspace_bytes) {
  YGG_CHECK_ARG(plan_mem && W && X && seg_table_dev, "null pointer");
  YGG_CHECK_ARG(M >= 1 && N >= kBM && K >= kBK, "bad GEMM shape");
  YGG_CHECK_ARG(N % kBM == 0, "N must be a multiple of 128");
  YGG_CHECK_ARG(K % kBK == 0, "K must be a multiple of 64");
  GemmPlan* g = reinterpret_cast<GemmPlan*>((reinterpret_cast<uintptr_t>(plan_mem) + 63) & ~uintptr_t(63));
  std::memset(g, 0, sizeof(GemmPlan));
  g->magic = kPlanMagic;
  g->dtype = dtype;
  g->M = M;
  g->N = N;
  g->K = K;
  const int mp = (M + 15) / 16 * 16;
  // Token tile (UMMA N): as few tiles of <= 256 as the rows need, split evenly (multiple of 16), so a
  // 520-row cfg5 verify runs 3 x 176 instead of 3 x 256 columns of MMA work (2 x 256 at 512 rows).
  {
    const int mt = (mp + 255) / 256;
    g->BN = ((mp + mt - 1) / mt + 15) / 16 * 16;
  }
  g->m_tiles = (M + g->BN - 1) / g->BN;
  g->n_tiles = N / kBM;
  g->tiles = g->n_tiles * g->m_tiles;
  g->kb = K / kBK;
  g->W = W;
  g->X = X;
  g->seg_table = seg_table_dev;
  std::vector<int32_t> table;
  if (dtype == YGG_BF16) {
    g->units = static_cast<long long>(g->tiles) * g->kb;
    // Default grid: every SM, but never fewer than 8 k-blocks (128 KB of weights) per CTA, which
    // bounds how many CTAs share (and must later reduce) one output tile for small layers.
    constexpr int min_units = 8;
    if (num_ctas <= 0)
      num_ctas = static_cast<int>(std::max(1LL, std::min<long long>(kNumSMs, g->units / min_units)));
    if (num_ctas > g->units) num_ctas = static_cast<int>(g->units);
    g->num_ctas = num_ctas;
    const int stage_bytes = kBM * kBK * 2 + g->BN * kBK * 2;
    // Shared-memory budget: 190 KB (one CTA per SM with a 7-stage ring at
    // BN = 64; the small epilogue CTAs still co-reside under programmatic dependent launch, the
    // decode attention of the verify (up to 190 KB itself) does not either way).  Same-box sweeps
    // of the cfg2 verify forward — with the split-KV tcgen05 attention: 113 KB 4.37 ms, 135 KB
    // 4.24, 150 KB 4.22, 165 KB 4.22, 190 KB 4.25, 227 KB 4.47; with the decode attention: 120 KB
    // 3.76, 150 KB 3.605, 190 KB 3.586, 216 KB 3.605.  Compute-bound 256-token tiles (prefill chunks):
    // 190 KB holds only 3 of their 48 KB stages; 4 stages (224 KB) run the cfg2 target prefill in 9.30
    // vs 9.91 ms (scripts/prefill_stages_ab.py), the 1B draft's unchanged.
    const int smem_kb = g->BN >= 256 ? 224 : 190;
    g->stages = std::min(12, (smem_kb * 1024 - kSmemExtra) / stage_bytes);
    YGG_CHECK_ARG(g->stages >= 2, "tile too large for shared memory");
    int cols = 32;
    while (cols < 2 * g->BN) cols *= 2;
    g->tmem_cols = cols;
    // Hybrid split: whole tiles first (one segment each), then the remainder tiles' units are
    // cut stream-K over all CTAs; their segments are enumerated in (cta, tile) == (tile, cta) order.
    g->dp_per_cta = g->tiles / num_ctas;
    const int t_dp = g->dp_per_cta * num_ctas;
    g->units = static_cast<long long>(g->tiles - t_dp) * g->kb;
    std::vector<int32_t> seg_first(g->tiles + 1, 0), seg_base(num_ctas, 0);
    std::vector<int> count(g->tiles, 0);
    for (int t = 0; t < t_dp; ++t) count[t] = 1;
    int seg = t_dp;
    for (int c = 0; c < num_ctas; ++c) {
      const long long u0 = static_cast<long long>(t_dp) * g->kb + g->units * c / num_ctas;
      const long long u1 = static_cast<long long>(t_dp) * g->kb + g->units * (c + 1) / num_ctas;
      seg_base[c] = seg;
      if (u1 > u0) {
        const int t0 = static_cast<int>(u0 / g->kb), t1 = static_cast<int>((u1 - 1) / g->kb);
        for (int t = t0; t <= t1; ++t) ++count[t];
        seg += t1 - t0 + 1;
      }
    }
    int acc = 0;
    for (int t = 0; t < g->tiles; ++t) { seg_first[t] = acc; acc += count[t]; }
    seg_first[g->tiles] = acc;
    g->segments = seg;
    table = seg_first;
    table.insert(table.end(), seg_base.begin(), seg_base.end());
    if (int rc = make_map_bf16(&g->tmap_w, W, N, K, kBM)) return rc;
    if (int rc = make_map_bf16(&g->tmap_x, X, M, K, g->BN)) return rc;
  } else if (dtype == YGG_F32) {
    g->num_ctas = 0;
    g->segments = g->tiles;
    table.resize(g->tiles + 1);
    for (int t = 0; t <= g->tiles; ++t) table[t] = t;
  } else {
    return ygg_fail(YGG_ERR_VALUE, "unknown dtype");
  }
  cudaError_t e = cudaMemcpy(seg_table_dev, table.data(), table.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "seg table upload: %s", cudaGetErrorString(e));
  if (num_segments) *num_segments = g->segments;
  if (workspace_bytes) *workspace_bytes = static_cast<size_t>(g->segments) * g->BN * kBM * sizeof(float);
  return YGG_OK;
}

int ygg_gemm_seg_table_len(const void* plan) {
  const GemmPlan* g = as_plan(reinterpret_cast<const void*>((reinterpret_cast<uintptr_t>(plan) + 63) & ~uintptr_t(63)));
  if (!g) return -1;
  return g->tiles + 1 + g->num_ctas;
}

static const GemmPlan* plan_of(const void* plan) {
  return as_plan(reinterpret_cast<const void*>((reinterpret_cast<uintptr_t>(plan) + 63) & ~uintptr_t(63)));
}

static int gemm_launch(const GemmPlan* g, float* workspace, const ygg_epilogue* epi, cudaStream_t s) {
  if (g->dtype == YGG_BF16) {
    GemmParams p;
    p.M = g->M;
    p.BN = g->BN;
    p.m_tiles = g->m_tiles;
    p.kb = g->kb;
    p.num_ctas = g->num_ctas;
    p.dp_per_cta = g->dp_per_cta;
    p.stages = g->stages;
    p.tmem_cols = g->tmem_cols;
    p.prewait = g->stages;  // every weight stage is streamed before the grid-dependency wait
    p.units = g->units;
    p.seg_first = g->seg_table;
    p.seg_base = g->seg_table + g->tiles + 1;
    const size_t smem = kSmemExtra + static_cast<size_t>(g->stages) * (kBM * kBK * 2 + g->BN * kBK * 2);
    EpiArgs e;
    std::memset(&e, 0, sizeof(e));
    e.trace = trace_next(3);
    int kind = kEpiNone;
    if (epi) {
      kind = epi->kind;
      e.ss_in = epi->ss_in;
      e.ss_tiles = epi->ss_tiles;
      e.norm_dim = epi->norm_dim;
      e.eps = epi->eps;
      e.out = epi->out;
      e.ld = epi->ld;
      e.q_out = static_cast<__nv_bfloat16*>(epi->q_out);
      e.cache = static_cast<__nv_bfloat16*>(epi->cache);
      e.S = epi->S;
      e.Hq = epi->Hq;
      e.Hkv = epi->Hkv;
      e.hd = epi->hd;
      e.log2_theta = epi->rope_theta > 0.f ? log2f(epi->rope_theta) : 0.f;
      e.pos = epi->pos;
      e.slot = epi->slot;
      e.req = epi->req;
      e.act_out = static_cast<__nv_bfloat16*>(epi->act_out);
      e.resid = epi->resid;
      e.hb = static_cast<__nv_bfloat16*>(epi->hb);
      e.ss_out = epi->ss_out;
      e.n_total = g->N;
      e.counters = epi->counters;
      e.dbg = reinterpret_cast<unsigned long long*>(epi->dbg);
      e.rope_cs = reinterpret_cast<const float2*>(epi->rope_cs);
      YGG_CHECK_ARG(kind == kEpiNone || g->cluster > 0 || e.counters != nullptr, "fused epilogue needs tile counters");
      YGG_CHECK_ARG(!e.ss_in || g->M <= kMaxRstdTokens, "too many tokens for the folded RMSNorm");
      YGG_CHECK_ARG(!e.ss_in || (e.ss_tiles >= 1 && e.norm_dim >= 1), "bad RMSNorm fold arguments");
      if (kind == kEpiStoreF32) YGG_CHECK_ARG(e.out && e.ld >= g->N, "STORE_F32 needs out / ld");
      if (kind == kEpiQkvRope)
        YGG_CHECK_ARG(e.q_out && e.cache && e.pos && e.slot && e.req && e.hd % 2 == 0 &&
                          g->N == (e.Hq + 2 * e.Hkv) * e.hd && kBM % e.hd == 0,
                      "QKV_ROPE arguments");
      if (kind == kEpiSwiglu) YGG_CHECK_ARG(e.act_out != nullptr, "SWIGLU needs act_out");
      if (kind == kEpiResid) YGG_CHECK_ARG(e.resid && e.hb && e.ss_out, "RESID needs resid / hb / ss_out");
      if (kind == kEpiArgmax) YGG_CHECK_ARG(e.out && g->M <= kArgmaxKeyOffset && (!e.ss_in || g->M <= kArgmaxKeyOffset),
                                            "ARGMAX needs out (u64 keys) and M <= 512");
      YGG_CHECK_ARG(kind != kEpiArgmax || g->cluster == 0, "ARGMAX runs on stream-K plans");
    }
    if (g->cluster > 0) {
      YGG_CHECK_ARG(kind != kEpiNone, "a cluster split-K plan needs a fused epilogue (no partials)");
      switch (kind) {
        case kEpiStoreF32: return launch_cluster_kind<kEpiStoreF32>(g, e, s);
        case kEpiQkvRope: return launch_cluster_kind<kEpiQkvRope>(g, e, s);
        case kEpiSwiglu: return launch_cluster_kind<kEpiSwiglu>(g, e, s);
        case kEpiResid: return launch_cluster_kind<kEpiResid>(g, e, s);
        default: return ygg_fail(YGG_ERR_VALUE, "unknown epilogue kind %d", kind);
      }
    }
    switch (kind) {
      case kEpiNone:
        YGG_LAUNCH_PDL(gemm_bf16_tc_kernel<kEpiNone>, dim3(g->num_ctas), dim3(kGemmThreads), smem, s, g->tmap_w,
                       g->tmap_x, p, workspace, e);
        break;
      case kEpiStoreF32:
        YGG_LAUNCH_PDL(gemm_bf16_tc_kernel<kEpiStoreF32>, dim3(g->num_ctas), dim3(kGemmThreads), smem, s, g->tmap_w,
                       g->tmap_x, p, workspace, e);
        break;
      case kEpiQkvRope:
        YGG_LAUNCH_PDL(gemm_bf16_tc_kernel<kEpiQkvRope>, dim3(g->num_ctas), dim3(kGemmThreads), smem, s, g->tmap_w,
                       g->tmap_x, p, workspace, e);
        break;
      case kEpiSwiglu:
        YGG_LAUNCH_PDL(gemm_bf16_tc_kernel<kEpiSwiglu>, dim3(g->num_ctas), dim3(kGemmThreads), smem, s, g->tmap_w,
                       g->tmap_x, p, workspace, e);
        break;
      case kEpiResid:
        YGG_LAUNCH_PDL(gemm_bf16_tc_kernel<kEpiResid>, dim3(g->num_ctas), dim3(kGemmThreads), smem, s, g->tmap_w,
                       g->tmap_x, p, workspace, e);
        break;
      case kEpiArgmax:
        YGG_LAUNCH_PDL(gemm_bf16_tc_kernel<kEpiArgmax>, dim3(g->num_ctas), dim3(kGemmThreads), smem, s, g->tmap_w,
                       g->tmap_x, p, workspace, e);
        break;
      default:
        return ygg_fail(YGG_ERR_VALUE, "unknown epilogue kind %d", kind);
    }
  } else {
    YGG_CHECK_ARG(epi == nullptr || epi->kind == kEpiNone, "fused epilogues run on the bf16 tcgen05 path only");
    dim3 grid(g->n_tiles, (g->M + kSimtBN - 1) / kSimtBN);
    YGG_LAUNCH_PDL(gemm_f32_simt_kernel, grid, dim3(256), 0, s, static_cast<const float*>(g->W),
                   static_cast<const float*>(g->X), g->M, g->N, g->K, g->BN, g->m_tiles, workspace);
  }
  return YGG_OK;
}

int ygg_argmax_reduce(const void* keys, int ntiles, int M, int32_t* out, ygg_stream_t stream) {
  YGG_CHECK_ARG(keys && out && ntiles >= 1 && M >= 1, "invalid arguments");
  YGG_LAUNCH_PDL(argmax_reduce_kernel, dim3(M), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream),
                 static_cast<const unsigned long long*>(keys), ntiles, M, out);
  return YGG_OK;
}

int ygg_gemm_plan_set_cluster(void* plan, int cluster) {
  GemmPlan* g = const_cast<GemmPlan*>(plan_of(plan));
  YGG_CHECK_ARG(g != nullptr, "invalid GEMM plan");
  YGG_CHECK_ARG(cluster >= 0 && cluster <= 16, "cluster size must be in [0, 16]");
  if (cluster == 0) {
    g->cluster = 0;
    return YGG_OK;
  }
  YGG_CHECK_ARG(g->dtype == YGG_BF16, "cluster split-K runs on the bf16 tcgen05 path only");
  YGG_CHECK_ARG(g->kb >= cluster, "fewer k-blocks than cluster CTAs");
  YGG_CHECK_ARG(cluster_stages(g, cluster) >= 2, "the receive slots leave no room for a two-stage ring");
  // every cluster must be co-resident (one wave): a second wave would double the GEMM
  const int keep = g->cluster;
  g->cluster = cluster;
  const size_t smem = cluster_smem(g);
  g->cluster = keep;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g->tiles * cluster);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int max_clusters = 0;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&max_clusters, gemm_cluster_kernel<kEpiResid>, &cfg);
  if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "cluster occupancy: %s", cudaGetErrorString(e));
  if (max_clusters < g->tiles)
    return ygg_fail(YGG_ERR_UNSUPPORTED, "%d tiles need %d co-resident clusters of %d; only %d fit", g->tiles,
                    g->tiles, cluster, max_clusters);
  g->cluster = cluster;
  return YGG_OK;
}

int ygg_gemm_plan_set_stages(void* plan, int stages) {
  GemmPlan* g = const_cast<GemmPlan*>(plan_of(plan));
  YGG_CHECK_ARG(g != nullptr && g->dtype == YGG_BF16, "invalid bf16 GEMM plan");
  YGG_CHECK_ARG(stages >= 2 && stages <= 12, "stages must be in [2, 12]");
  YGG_CHECK_ARG(kSmemExtra + static_cast<size_t>(stages) * (kBM * kBK * 2 + g->BN * kBK * 2) <= 227 * 1024,
                "ring exceeds shared memory");
  g->stages = stages;
  return YGG_OK;
}

int ygg_gemm_plan_set_layout(void* plan, int interleaved) {
  GemmPlan* g = const_cast<GemmPlan*>(plan_of(plan));
  YGG_CHECK_ARG(g != nullptr, "invalid GEMM plan");
  g->interleaved = interleaved ? 1 : 0;
  return YGG_OK;
}

int ygg_gemm_plan_set_epi_prefetch(void* plan, const void* ptr, size_t bytes) {
  GemmPlan* g = const_cast<GemmPlan*>(plan_of(plan));
  YGG_CHECK_ARG(g != nullptr, "invalid GEMM plan");
  YGG_CHECK_ARG(ptr == nullptr || (reinterpret_cast<uintptr_t>(ptr) & 15) == 0, "prefetch region must be 16-byte aligned");
  g->epi_pf = bytes ? static_cast<const char*>(ptr) : nullptr;
  g->epi_pf_bytes = g->epi_pf ? (bytes & ~static_cast<size_t>(15)) : 0;
  return YGG_OK;
}

int ygg_gemm_plan_cluster(const void* plan) {
  const GemmPlan* g = plan_of(plan);
  return g ? g->cluster : -1;
}

int ygg_gemm_run(const void* plan, float* workspace, ygg_stream_t stream) {
  const GemmPlan* g = plan_of(plan);
  YGG_CHECK_ARG(g != nullptr, "invalid GEMM plan");
  YGG_CHECK_ARG(g->cluster == 0, "a cluster split-K plan runs through ygg_gemm_fused");
  YGG_CHECK_ARG(workspace != nullptr, "null workspace");
  return gemm_launch(g, workspace, nullptr, reinterpret_cast<cudaStream_t>(stream));
}

int ygg_gemm_fused(const void* plan, float* workspace, const ygg_epilogue* epi, ygg_stream_t stream) {
  const GemmPlan* g = plan_of(plan);
  YGG_CHECK_ARG(g != nullptr, "invalid GEMM plan");
  YGG_CHECK_ARG(workspace != nullptr && epi != nullptr, "null workspace / epilogue");
  return gemm_launch(g, workspace, epi, reinterpret_cast<cudaStream_t>(stream));
}

int ygg_gemm_tiles(const void* plan) {
  const GemmPlan* g = plan_of(plan);
  return g ? g->tiles : -1;
}

int ygg_epi_store(const void* plan, const float* ws, void* out, int out_dtype, int ld_out, ygg_stream_t stream) {
  const GemmPlan* g = plan_of(plan);
  YGG_CHECK_ARG(g && ws && out, "invalid arguments");
  YGG_CHECK_ARG(ld_out >= g->N, "ld_out < N");
  EpiGeom geo = geom_of(g, 4);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  YGG_CHECK_ARG(ld_out % 8 == 0, "ld_out must be a multiple of 8");
  dim3 grid((g->N + 1023) / 1024, g->M);
  if (out_dtype == YGG_F32)
    YGG_LAUNCH_PDL(epi_store_kernel<float>, grid, dim3(kEpiThreads), 0, s, geo, ws, static_cast<float*>(out), ld_out);
  else
    YGG_LAUNCH_PDL(epi_store_kernel<__nv_bfloat16>, grid, dim3(kEpiThreads), 0, s, geo, ws,
                   static_cast<__nv_bfloat16*>(out), ld_out);
  return YGG_OK;
}

int ygg_epi_residual_norm(const void* plan, const float* ws, float* resid, const void* norm_w, float eps, void* xn_out,
                          int act_dtype, ygg_stream_t stream) {
  const GemmPlan* g = plan_of(plan);
  YGG_CHECK_ARG(g && ws && resid && norm_w && xn_out, "invalid arguments");
  YGG_CHECK_ARG(g->N % 8 == 0 && g->N / 8 <= 1024, "row wider than 8192 features");
  EpiGeom geo = geom_of(g, 5);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int threads = ((g->N / 8 + 31) / 32) * 32;
  if (act_dtype == YGG_F32)
    YGG_LAUNCH_PDL(epi_residual_norm_kernel<float>, dim3(g->M), dim3(threads), 0, s, geo, ws, resid,
                   static_cast<const float*>(norm_w), eps, static_cast<float*>(xn_out));
  else
    YGG_LAUNCH_PDL(epi_residual_norm_kernel<__nv_bfloat16>, dim3(g->M), dim3(threads), 0, s, geo, ws, resid,
                   static_cast<const __nv_bfloat16*>(norm_w), eps, static_cast<__nv_bfloat16*>(xn_out));
  return YGG_OK;
}

int ygg_epi_swiglu(const void* plan, const float* ws, void* out, int act_dtype, ygg_stream_t stream) {
  const GemmPlan* g = plan_of(plan);
  YGG_CHECK_ARG(g && ws && out, "invalid arguments");
  YGG_CHECK_ARG(g->N % 2 == 0, "gate_up width must be even");
  EpiGeom geo = geom_of(g, 6);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // Tokens per thread: 1.  (R = 4 at cfg4's 800 rows shortens this kernel 37.8 -> 34.5 us but delays the
  // down GEMM's dependency release 11 -> 43 us: net slower, measured in-graph with scripts/draft_timeline.py.)
  constexpr int R = 1;
  dim3 grid((g->N / 2 + 1023) / 1024, (g->M + R - 1) / R);
  if (act_dtype == YGG_F32)
    YGG_LAUNCH_PDL((epi_swiglu_kernel<float, R>), grid, dim3(kEpiThreads), 0, s, geo, ws, static_cast<float*>(out));
  else
    YGG_LAUNCH_PDL((epi_swiglu_kernel<__nv_bfloat16, R>), grid, dim3(kEpiThreads), 0, s, geo, ws,
                   static_cast<__nv_bfloat16*>(out));
  return YGG_OK;
}

int ygg_epi_qkv_rope(const void* plan, const float* ws, int Hq, int Hkv, int hd, float rope_theta, const int32_t* pos,
                     const int32_t* slot, const int32_t* req, void* q_out, void* cache, int S, int act_dtype,
                     const float* rope_cs, ygg_stream_t stream) {
  const GemmPlan* g = plan_of(plan);
  YGG_CHECK_ARG(g && ws && pos && slot && req && q_out && cache, "invalid arguments");
  YGG_CHECK_ARG(g->N == (Hq + 2 * Hkv) * hd, "QKV width mismatch");
  YGG_CHECK_ARG(hd % 8 == 0 && hd <= 256, "bad head dim");
  EpiGeom geo = geom_of(g, 7);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int items = (Hq + 2 * Hkv) * (hd / 8);
  dim3 grid(g->M, (items + 255) / 256);
  const float l2t = log2f(rope_theta);
  const float2* rt = reinterpret_cast<const float2*>(rope_cs);
  if (act_dtype == YGG_F32)
    YGG_LAUNCH_PDL(epi_qkv_rope_kernel<float>, grid, dim3(256), 0, s, geo, ws, Hq, Hkv, hd, l2t, pos, slot, req,
                   static_cast<float*>(q_out), static_cast<float*>(cache), S, rt);
  else
    YGG_LAUNCH_PDL(epi_qkv_rope_kernel<__nv_bfloat16>, grid, dim3(256), 0, s, geo, ws, Hq, Hkv, hd, l2t, pos, slot, req,
                   static_cast<__nv_bfloat16*>(q_out), static_cast<__nv_bfloat16*>(cache), S, rt);
  return YGG_OK;
}

}  // extern "C"
