// Row-block GEMV for decode-shaped passes (M <= 16 token rows): Y[M,N] = X[M,K] . W[N,K]^T with
// the layer epilogue fused, one launch per matmul, no split-K.
//
// Why not the stream-K tcgen05 GEMM here: at M = 8 (a draft pass over one EGT level) a 128-row UMMA
// tile leaves too few tiles to spread full-K work over 148 SMs, so the tcgen05 path splits K and
// pays a partials round trip plus a separate epilogue launch per matmul (~10 launches per layer,
// ~4 us each).  Here the unit of work is a 16-row block of W with its whole K: 2048-row matrices
// already give 128 blocks, and each block's outputs are final in registers, so RoPE + KV append,
// residual + sum of squares, SwiGLU and the logits store run straight from the accumulators.
// The work is HBM-bound (2 FLOP per weight byte per token): the tensor-core op is the legacy
// mma.sync m16n8k16 (A = 16 weight rows, B = X^T with the tokens as n), fed by ldmatrix from a
// 128B-swizzled TMA ring; its throughput is >10x what the weight stream needs.
//
// CTA = 5 warps, persistent over row blocks b = blockIdx.x, += gridDim.x:
//   warp 0 lane 0: TMA producer.  Stage = W[16 rows x 512 k] (16 KB, one 3-D box) + X[xrows x 512 k].
//                  Weight boxes are issued before griddepcontrol.wait (they never depend on the
//                  previous kernel), activations after.
//   warps 1-4: ldmatrix + mma.sync, each on two of a stage's eight 64-wide k sub-chunks with two
//              independent accumulator chains; at the end of a block the four partial accumulators are
//              summed in fixed warp order through shared memory and warp 1 runs the epilogue.
// RMSNorm is folded (gains in the weights, model.prepare_fused_ layout); the per-token rstd comes
// from the producing residual's per-block sums of squares.  QKV rows are RoPE-pair interleaved and
// gate/up rows interleaved, so rotation / gating partners are one lane-xor (4) apart.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "host_util.h"

namespace ygg {
namespace gv {

constexpr int kRows = 16;       // weight rows per block (mma M)
constexpr int kSub = 8;         // 64-wide k sub-chunks per stage
constexpr int kStageK = kSub * 64;
constexpr int kCompute = 4;                 // compute warps; warp w takes sub-chunks {2w, 2w+1} of a stage
constexpr int kThreads = 32 * (2 + kCompute);  // producer, kCompute mma warps, epilogue warp
constexpr int kMaxTok = 16;
constexpr uint32_t kMagic = 0x59474756u;  // "YGGV"

enum Epi : int { kNone = 0, kStore = 1, kQkv = 2, kSwiglu = 3, kResid = 4, kStoreTopk = 5 };

struct Params {
  int M, N, K, nblk, kchunks, stages, xrows, grid;
  const char* pf_ptr[2];  // optional L2 prefetch regions (later weights / caches), split over the CTAs
  size_t pf_bytes[2];
};

struct Epilogue {
  int kind;
  float* out;        // STORE [M][ld] f32
  int ld;
  const float* ss_in;  // [ss_blocks][M] per-block sums of squares of the un-normalised input
  int ss_blocks;
  int norm_dim;
  float eps;
  __nv_bfloat16* q_out;  // QKV
  __nv_bfloat16* cache;
  int S, Hq, Hkv, hd;
  const int32_t* pos;
  const int32_t* slot;
  const int32_t* req;
  const float2* rope_cs;
  __nv_bfloat16* act_out;  // SWIGLU [M][N/2]
  float* resid;            // RESID [M][N]
  __nv_bfloat16* hb;
  float* ss_out;           // RESID [N/16][M]
  unsigned long long* trace;  // kernel-timeline slot (profiling only) or nullptr
  TopkPartial* topk_part;     // STORE_TOPK: [M][grid] per-CTA partials (merged by ygg_topk_merge)
  int topk_k;                 // STORE_TOPK: k <= kTopkLane
  float inv_temp;             // STORE_TOPK: logits scale before the softmax / ranking
};

constexpr int kTopkLane = 8;  // per-lane candidate list of the fused top-k epilogue

// Named barriers 1..4 between the mma warps and the epilogue warp (immediate ids: a register id
// would make ptxas reserve all 16).
YGG_DEV void named_sync(int id) {
  constexpr int n = 32 * (kCompute + 1);
  switch (id) {
    case 1: asm volatile("bar.sync 1, %0;" ::"n"(n) : "memory"); break;
    case 2: asm volatile("bar.sync 2, %0;" ::"n"(n) : "memory"); break;
    case 3: asm volatile("bar.sync 3, %0;" ::"n"(n) : "memory"); break;
    default: asm volatile("bar.sync 4, %0;" ::"n"(n) : "memory"); break;
  }
}
YGG_DEV void named_arrive(int id) {
  constexpr int n = 32 * (kCompute + 1);
  switch (id) {
    case 1: asm volatile("bar.arrive 1, %0;" ::"n"(n) : "memory"); break;
    case 2: asm volatile("bar.arrive 2, %0;" ::"n"(n) : "memory"); break;
    case 3: asm volatile("bar.arrive 3, %0;" ::"n"(n) : "memory"); break;
    default: asm volatile("bar.arrive 4, %0;" ::"n"(n) : "memory"); break;
  }
}

// Insert (v, t) into a lane's sorted list (logit desc, token asc); the caller checked that it beats
// the last entry.  Static indices only, so the list stays in registers.
YGG_DEV void topk_insert(float (&lv)[kTopkLane], int (&lt)[kTopkLane], float v, int t) {
  bool done = false;
#pragma unroll
  for (int i = kTopkLane - 1; i >= 1; --i) {
    if (!done) {
      if (topk_better(v, t, lv[i - 1], lt[i - 1])) {
        lv[i] = lv[i - 1];
        lt[i] = lt[i - 1];
      } else {
        lv[i] = v;
        lt[i] = t;
        done = true;
      }
    }
  }
  if (!done) {
    lv[0] = v;
    lt[0] = t;
  }
}

struct Plan {
  uint32_t magic;
  Params p;
  size_t smem;
  size_t stage_bytes, fixed_bytes;
  alignas(64) CUtensorMap tw;
  alignas(64) CUtensorMap tx;
};

YGG_DEV void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
      : "memory");
}
YGG_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
YGG_DEV void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
YGG_DEV void mma16816(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int NT, bool TOPK>  // token tiles of 8 (1: M <= 8, 2: M <= 16); TOPK: STORE_TOPK epilogue (NT == 1)
__global__ void __launch_bounds__(kThreads, 1)
    gemv_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx, Params p, Epilogue e) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  const uint32_t w_bytes = kRows * kStageK * 2;   // 16 KB
  const uint32_t x_bytes = p.xrows * kStageK * 2; // 8 or 16 KB
  unsigned char* sw = base;
  unsigned char* sx = sw + static_cast<size_t>(S) * w_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sx + static_cast<size_t>(S) * x_bytes);
  uint64_t* empty = full + S;
  float* rstd_s = reinterpret_cast<float*>(empty + S);
  int* tok_s = reinterpret_cast<int*>(rstd_s + kMaxTok);  // [3][kMaxTok] pos, slot, req
  float* red = reinterpret_cast<float*>(tok_s + 3 * kMaxTok);  // [2][kCompute][NT][4][32] partial accumulators
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tw);
    tma_prefetch_desc(&tx);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCompute);
    }
    fence_barrier_init();
    trace_min(e.trace, 0);
  }
  __syncthreads();
  const int nb_mine = p.nblk > static_cast<int>(blockIdx.x) ? (p.nblk - 1 - blockIdx.x) / p.grid + 1 : 0;
  const int total = nb_mine * p.kchunks;
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
      // Weights never depend on the previous kernel: fill the ring before the grid dependency.
      const int pre = total < S ? total : S;
      // (block, chunk) of stage i stepped incrementally: no integer division on the issue path.
      int b = blockIdx.x, q = 0;
      auto step = [&]() {
        if (++q == p.kchunks) {
          q = 0;
          b += p.grid;
        }
      };
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], w_bytes + x_bytes);
        tma3(sw + static_cast<size_t>(i) * w_bytes, &tw, &full[i], 0, b * kRows, q * kSub, pol_w);
        step();
      }
      pdl_wait();
      for (int i = 0, qq = 0; i < pre; ++i) {
        tma3(sx + static_cast<size_t>(i) * x_bytes, &tx, &full[i], 0, 0, qq * kSub, pol_x);
        if (++qq == p.kchunks) qq = 0;
      }
      int st = pre % S;
      uint32_t ph = pre == S ? 1u : 0u;
      for (int i = pre; i < total; ++i) {
        mbar_wait(&empty[st], ph ^ 1u);
        mbar_arrive_expect_tx(&full[st], w_bytes + x_bytes);
        tma3(sw + static_cast<size_t>(st) * w_bytes, &tw, &full[st], 0, b * kRows, q * kSub, pol_w);
        tma3(sx + static_cast<size_t>(st) * x_bytes, &tx, &full[st], 0, 0, q * kSub, pol_x);
        step();
        if (++st == S) {
          st = 0;
          ph ^= 1u;
        }
      }
      for (int rg = 0; rg < 2; ++rg) {  // after this CTA's own stream: pull slices of later data into L2
        if (!p.pf_ptr[rg]) continue;
        const size_t per = ((p.pf_bytes[rg] / gridDim.x) + 255) & ~static_cast<size_t>(255);
        const size_t b0 = blockIdx.x * per, b1 = b0 + per < p.pf_bytes[rg] ? b0 + per : p.pf_bytes[rg];
        for (size_t o = b0; o < b1; o += 65536) {
          const uint32_t n = static_cast<uint32_t>(b1 - o < 65536 ? ((b1 - o) & ~static_cast<size_t>(15)) : 65536);
          if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.pf_ptr[rg] + o), "r"(n) : "memory");
        }
      }
    } else {
      pdl_wait();  // dependents may only launch once this grid is past its wait (see attn_dec.cu)
    }
    pdl_launch_dependents();
    return;
  }
  // ===== warps 1..kCompute: mma; warp kCompute + 1: epilogue of the blocks they finish =====
  if (warp <= kCompute) {
    pdl_wait();
    pdl_launch_dependents();
    if (threadIdx.x == 32) trace_min(e.trace, 1);
    const int M = p.M;
    const int cw = warp - 1;
    const uint32_t sw0 = smem_u32(sw), sx0 = smem_u32(sx);
    // ldmatrix lane roles: A (x4): row = (l & 7) + 8*((l >> 3) & 1), 16B chunk hi = l >> 4.
    const int a_row = (lane & 7) + 8 * ((lane >> 3) & 1), a_hi = lane >> 4;
    // B (x2 per token tile): token row = l & 7 (+8 for the second tile), 16B chunk hi = (l >> 3) & 1.
    const int b_row = lane & 7, b_hi = (lane >> 3) & 1;
    const int xrow_bytes = p.xrows * 128;
    int st = 0;
    uint32_t ph = 0;
    for (int bi = 0; bi < nb_mine; ++bi) {
      const int b = blockIdx.x + bi * p.grid;
      float acc[NT][4], acc2[NT][4];
  #pragma unroll
      for (int t = 0; t < NT; ++t)
  #pragma unroll
        for (int j = 0; j < 4; ++j) acc[t][j] = acc2[t][j] = 0.f;
      for (int q = 0; q < p.kchunks; ++q) {
        mbar_wait(&full[st], ph);
        const uint32_t ws = sw0 + st * w_bytes, xs = sx0 + st * x_bytes;
  #pragma unroll
        for (int uu = 0; uu < 2; ++uu) {
          const int u = 2 * cw + uu;
          const uint32_t wu = ws + u * (kRows * 128);
          const uint32_t xu = xs + u * xrow_bytes;
  #pragma unroll
          for (int s4 = 0; s4 < 4; ++s4) {
            uint32_t a0, a1, a2, a3;
            const int ja = 2 * s4 + a_hi;
            ldsm_x4(wu + a_row * 128 + ((ja ^ (a_row & 7)) << 4), a0, a1, a2, a3);
            const int jb = 2 * s4 + b_hi;
  #pragma unroll
            for (int t = 0; t < NT; ++t) {
              const int r = b_row + 8 * t;
              uint32_t b0, b1;
              ldsm_x2(xu + r * 128 + ((jb ^ (r & 7)) << 4), b0, b1);
              mma16816((s4 & 1) ? acc2[t] : acc[t], a0, a1, a2, a3, b0, b1);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (++st == S) {
          st = 0;
          ph ^= 1u;
        }
      }
      // Hand the partial accumulators to the epilogue warp through a double-buffered scratch:
      // slot bi & 1 is free again once the epilogue warp has read block bi - 2 (named barriers
      // 3 / 4 = empty, 1 / 2 = full; 128 compute + 32 epilogue threads each).
      if (bi >= 2) named_sync(3 + (bi & 1));
      float* rs = red + (bi & 1) * (kCompute * NT * 4 * 32);
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int j = 0; j < 4; ++j) rs[((cw * NT + t) * 4 + j) * 32 + lane] = acc[t][j] + acc2[t][j];
      named_arrive(1 + (bi & 1));
    }
    return;
  }
  // ===== warp kCompute + 1: epilogue (sums the compute warps' partials in fixed warp order) =====
  pdl_wait();
  pdl_launch_dependents();
  const int M = p.M;
  // Per-token inputs of the epilogue, while the mma warps stream the first block: rstd from the
  // producing residual's per-block sums of squares (lanes split the blocks, fixed-order tree
  // reduction), and the position / slot / request of each token row.
  if (e.ss_in) {
    constexpr int NTOK = 8 * NT;  // token rows this instantiation handles
    float v[NTOK];
#pragma unroll
    for (int n = 0; n < NTOK; ++n) v[n] = 0.f;
    for (int j = lane; j < e.ss_blocks; j += 32) {  // every token's load of block j in flight together
      const float* row = e.ss_in + static_cast<size_t>(j) * M;
#pragma unroll
      for (int n = 0; n < NTOK; ++n)
        if (n < M) v[n] += __ldg(row + n);
    }
    // Reduce-scatter across the lanes (halving the token set per xor step, NTOK - 1 shuffles in all
    // instead of 5 * NTOK), then full xor sums over the remaining lane bits: fixed order,
    // deterministic.  Lane l ends with token t(l) built from its high lane bits.
    int cnt = NTOK, tsel = 0;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      if (cnt > 1) {
        const int half = cnt / 2;
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < NTOK / 2; ++i) {
          if (i < half) {
            const float send = upper ? v[i] : v[i + half];
            const float recv = __shfl_xor_sync(0xffffffffu, send, o);
            v[i] = (upper ? v[i + half] : v[i]) + recv;
          }
        }
        tsel = tsel * 2 + (upper ? 1 : 0);
        cnt = half;
      } else {
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
      }
    }
    // every lane now holds the full sum of token tsel (lanes differing only in the low bits agree)
    const int low_bits = 32 / NTOK;  // lanes sharing a token
    if ((lane & (low_bits - 1)) == 0 && tsel < M) rstd_s[tsel] = rsqrtf(v[0] / static_cast<float>(e.norm_dim) + e.eps);
  }
  if (e.kind == kQkv && lane < M) {
    tok_s[lane] = __ldg(e.pos + lane);
    tok_s[kMaxTok + lane] = __ldg(e.slot + lane);
    tok_s[2 * kMaxTok + lane] = __ldg(e.req + lane);
  }
  __syncwarp();
  // STORE_TOPK (NT == 1 only): per lane and token slot q (token 2*(lane&3) + q) a running max / f64
  // sum of exp and a sorted top-kTopkLane list over this lane's rows of every block.
  constexpr int TQ = TOPK ? 2 : 1;
  float tk_m[TQ], tk_v[TQ][kTopkLane];
  double tk_s[TQ];
  int tk_t[TQ][kTopkLane];
#pragma unroll
  for (int q = 0; q < TQ; ++q) {
    tk_m[q] = -INFINITY;
    tk_s[q] = 0.0;
#pragma unroll
    for (int i = 0; i < kTopkLane; ++i) {
      tk_v[q][i] = -INFINITY;
      tk_t[q][i] = 0x7fffffff;
    }
  }
  for (int bi = 0; bi < nb_mine; ++bi) {
    const int b = blockIdx.x + bi * p.grid;
    named_sync(1 + (bi & 1));
    const float* rs = red + (bi & 1) * (kCompute * NT * 4 * 32);
    float acc[NT][4];
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < kCompute; ++w) v += rs[((w * NT + t) * 4 + j) * 32 + lane];
        acc[t][j] = v;
      }
    if (bi + 2 < nb_mine) named_arrive(3 + (bi & 1));
    if (lane == 0) trace_max(e.trace, 3);
    // ---- epilogue: acc[t] = {(row r0, tok n0), (r0, n0+1), (r0+8, n0), (r0+8, n0+1)}
    const int r0 = b * kRows + (lane >> 2);
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int n0 = t * 8 + (lane & 3) * 2;
      float v[4] = {acc[t][0], acc[t][1], acc[t][2], acc[t][3]};
      const int rr[4] = {r0, r0, r0 + 8, r0 + 8};
      const int nn[4] = {n0, n0 + 1, n0, n0 + 1};
      if (e.kind == kStore || e.kind == kStoreTopk) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          v[j] *= (e.ss_in ? rstd_s[nn[j]] : 1.f);
          if (nn[j] < M) e.out[static_cast<size_t>(nn[j]) * e.ld + rr[j]] = v[j];
        }
        if constexpr (TOPK) {
          {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int q = j & 1;
              const float x = v[j] * e.inv_temp;
              if (isnan(x)) continue;
              if (x > tk_m[q]) {
                tk_s[q] = tk_s[q] * exp(static_cast<double>(tk_m[q]) - static_cast<double>(x)) + 1.0;
                tk_m[q] = x;
              } else {
                tk_s[q] += exp(static_cast<double>(x) - static_cast<double>(tk_m[q]));
              }
              if (topk_better(x, rr[j], tk_v[q][kTopkLane - 1], tk_t[q][kTopkLane - 1]))
                topk_insert(tk_v[q], tk_t[q], x, rr[j]);
            }
          }
        }
      } else if (e.kind == kResid) {
        float sq[2] = {0.f, 0.f};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (nn[j] < M) {
            const size_t idx = static_cast<size_t>(nn[j]) * p.N + rr[j];
            const float h = e.resid[idx] + v[j];
            e.resid[idx] = h;
            e.hb[idx] = __float2bfloat16_rn(h);
            sq[j & 1] += h * h;
          }
        }
        // sum over the 16 rows of the block: lanes with equal (lane & 3) hold the same tokens
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          sq[0] += __shfl_xor_sync(0xffffffffu, sq[0], o);
          sq[1] += __shfl_xor_sync(0xffffffffu, sq[1], o);
        }
        if (lane < 4) {
          if (n0 < M) e.ss_out[static_cast<size_t>(b) * M + n0] = sq[0];
          if (n0 + 1 < M) e.ss_out[static_cast<size_t>(b) * M + n0 + 1] = sq[1];
        }
      } else {
        // SWIGLU / QKV: partner row (r ^ 1) lives in lane ^ 4.
        float o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float r = (e.ss_in && nn[j] < M) ? rstd_s[nn[j]] : 1.f;
          v[j] *= r;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = __shfl_xor_sync(0xffffffffu, v[j], 4);
        const bool even = ((lane >> 2) & 1) == 0;
        if (e.kind == kSwiglu) {
          if (even) {
            const int F = p.N / 2;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (nn[j] >= M) continue;
              const float g = v[j], u = o[j];
              e.act_out[static_cast<size_t>(nn[j]) * F + (rr[j] >> 1)] =
                  __float2bfloat16_rn(__fdividef(g, 1.f + __expf(-g)) * u);
            }
          }
        } else {  // kQkv
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (nn[j] >= M) continue;
            const int m = nn[j];
            const int R = rr[j];
            const int head = R / e.hd, pr = R % e.hd, half = e.hd / 2;
            const int pair = pr >> 1;
            const int orig = pair + (even ? 0 : half);
            float y = v[j];
            if (head < e.Hq + e.Hkv) {
              const float2 cs = __ldg(e.rope_cs + static_cast<size_t>(tok_s[m]) * half + pair);
              y = even ? (v[j] * cs.x - o[j] * cs.y) : (v[j] * cs.x + o[j] * cs.y);
            }
            const __nv_bfloat16 yb = __float2bfloat16_rn(y);
            if (head < e.Hq) {
              e.q_out[(static_cast<size_t>(m) * e.Hq + head) * e.hd + orig] = yb;
            } else {
              const bool is_v = head >= e.Hq + e.Hkv;
              const int kvh = is_v ? head - e.Hq - e.Hkv : head - e.Hq;
              const size_t cb = ((static_cast<size_t>(tok_s[2 * kMaxTok + m]) * 2 + (is_v ? 1 : 0)) * e.Hkv + kvh) *
                                static_cast<size_t>(e.S) * e.hd;
              const int sl = tok_s[kMaxTok + m];
              if (!is_v) e.cache[cb + static_cast<size_t>(sl) * e.hd + orig] = yb;
              else e.cache[cb + static_cast<size_t>(orig) * e.S + sl] = yb;  // V^T [hd][S]
            }
          }
        }
      }
    }
  }
  if constexpr (TOPK) {
    {
      // Merge the 8 lanes holding each token (equal lane & 3): (max, sum) by the xor tree, then k
      // rounds of a group tournament over the list heads (rows are distinct, so no exact ties).
#pragma unroll
      for (int q = 0; q < TQ; ++q) {
        float m = tk_m[q];
        double sm = tk_s[q];
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          const float mo = __shfl_xor_sync(0xffffffffu, m, o);
          const double so = __shfl_xor_sync(0xffffffffu, sm, o);
          const float mn = fmaxf(m, mo);
          sm = mn == -INFINITY ? 0.0
                               : sm * exp(static_cast<double>(m) - mn) + so * exp(static_cast<double>(mo) - mn);
          m = mn;
        }
        const int n = 2 * (lane & 3) + q;
        TopkPartial* out = e.topk_part + static_cast<size_t>(n) * p.grid + blockIdx.x;
        const bool leader = (lane >> 2) == 0 && n < M;
        if (leader) {
          out->max_s = m;
          out->sum_exp = sm;
        }
        for (int r = 0; r < e.topk_k; ++r) {
          float bv = tk_v[q][0];
          int bt = tk_t[q][0];
#pragma unroll
          for (int o = 4; o < 32; o <<= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
            if (topk_better(ov, ot, bv, bt)) {
              bv = ov;
              bt = ot;
            }
          }
          if (leader) {
            out->val[r] = bv;
            out->tok[r] = bt == 0x7fffffff ? -1 : bt;
          }
          if (bt != 0x7fffffff && tk_t[q][0] == bt) {  // this lane's head won: pop it
#pragma unroll
            for (int i = 0; i < kTopkLane - 1; ++i) {
              tk_v[q][i] = tk_v[q][i + 1];
              tk_t[q][i] = tk_t[q][i + 1];
            }
            tk_v[q][kTopkLane - 1] = -INFINITY;
            tk_t[q][kTopkLane - 1] = 0x7fffffff;
          }
        }
      }
    }
  }
  if (lane == 0) trace_max(e.trace, 2);
}

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) == cudaSuccess &&
        r == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(q);
  }
  return fn;
}

// [rows][K] bf16 viewed as (64 k, rows, K/64 sub-chunks); box {64, box_rows, kSub}, 128B swizzle.
static int map3(CUtensorMap* m, const void* ptr, int rows, int K, int box_rows) {
  auto enc = encoder();
  if (!enc) return ygg_fail(YGG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(K / 64)};
  cuuint64_t str[2] = {static_cast<cuuint64_t>(K) * 2, 128};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(kSub)};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, str, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return ygg_fail(YGG_ERR_CUDA, "gemv tensor map encode failed (%d)", static_cast<int>(r));
  return YGG_OK;
}

static const Plan* plan_of(const void* p) {
  const Plan* q = reinterpret_cast<const Plan*>((reinterpret_cast<uintptr_t>(p) + 63) & ~uintptr_t(63));
  return (p && q->magic == kMagic) ? q : nullptr;
}

}  // namespace gv
}  // namespace ygg

using namespace ygg;
using namespace ygg::gv;

extern "C" {

int ygg_prepare_gemv(void) {
  for (auto fn : {gemv_kernel<1, false>, gemv_kernel<2, false>, gemv_kernel<1, true>}) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "gemv attribute: %s", cudaGetErrorString(e));
  }
  return YGG_OK;
}

int ygg_gemv_set_l2_prefetch(void* plan, int region, const void* ptr, size_t bytes) {
  Plan* pl = const_cast<Plan*>(plan_of(plan));
  YGG_CHECK_ARG(pl != nullptr, "invalid gemv plan");
  YGG_CHECK_ARG(region == 0 || region == 1, "prefetch region must be 0 or 1");
  YGG_CHECK_ARG(ptr == nullptr || (reinterpret_cast<uintptr_t>(ptr) & 15) == 0, "prefetch region must be 16-byte aligned");
  pl->p.pf_ptr[region] = bytes ? static_cast<const char*>(ptr) : nullptr;
  pl->p.pf_bytes[region] = ptr ? bytes : 0;
  return YGG_OK;
}

int ygg_gemv_stream_info(const void* plan, void* weight_map, int* nblk, int* kchunks, int* stages) {
  const Plan* pl = plan_of(plan);
  YGG_CHECK_ARG(pl != nullptr && weight_map && nblk && kchunks && stages, "invalid gemv plan / outputs");
  std::memcpy(weight_map, &pl->tw, sizeof(CUtensorMap));
  *nblk = pl->p.nblk;
  *kchunks = pl->p.kchunks;
  *stages = pl->p.stages;
  return YGG_OK;
}

int ygg_gemv_grid(const void* plan) {
  const Plan* pl = plan_of(plan);
  return pl ? pl->p.grid : 0;
}

size_t ygg_gemv_plan_size(void) { return sizeof(Plan) + 64; }

int ygg_gemv_plan_init(void* plan, const void* W, const void* X, int M, int N, int K, int num_ctas) {
  YGG_CHECK_ARG(plan && W && X, "null pointer");
  YGG_CHECK_ARG(M >= 1 && M <= kMaxTok, "gemv handles 1..16 token rows");
  YGG_CHECK_ARG(N % kRows == 0 && N >= kRows, "N must be a multiple of 16");
  YGG_CHECK_ARG(K % 64 == 0 && K >= 64, "K must be a multiple of 64");
  Plan* pl = reinterpret_cast<Plan*>((reinterpret_cast<uintptr_t>(plan) + 63) & ~uintptr_t(63));
  std::memset(pl, 0, sizeof(Plan));
  pl->magic = kMagic;
  Params& p = pl->p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.nblk = N / kRows;
  p.kchunks = (K + kStageK - 1) / kStageK;
  p.xrows = M <= 8 ? 8 : 16;
  int sms = kNumSMs, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // Two CTAs per SM by default (~110 KB of ring each): a 2048-row matmul's 128-192 blocks fit one
  // wave with one block per CTA, and the next kernel's CTAs are co-resident with this one's tail,
  // so under programmatic dependent launch their weight ring fills while this kernel drains.
  constexpr int smem_kb = 110;
  int per_sm = smem_kb <= 113 ? 2 : 1;
  p.grid = num_ctas > 0 ? num_ctas : std::min(sms * per_sm, p.nblk);
  // A matrix with at most one block per SM (o / down projections: 128 blocks of 16 x K) is bound by
  // one CTA's bytes in flight: give that CTA the whole SM's ring (224 KB = 9 stages; same-box draft
  // pass 0.593 ms at 200 KB, 0.591 at 224).
  constexpr int solo_kb = 224;
  const int budget_kb = (num_ctas <= 0 && p.nblk <= sms) ? solo_kb : smem_kb;
  const size_t stage = static_cast<size_t>(kRows) * kStageK * 2 + static_cast<size_t>(p.xrows) * kStageK * 2;
  const size_t fixed = 1024 + 16 * 2 * 8 + kMaxTok * 16 + 2 * kCompute * 2 * 4 * 32 * 4 + 64;
  p.stages = static_cast<int>(std::min<size_t>(16, (static_cast<size_t>(budget_kb) * 1024 - fixed) / stage));
  YGG_CHECK_ARG(p.stages >= 2, "gemv: shared memory budget too small");
  pl->smem = fixed + static_cast<size_t>(p.stages) * stage;
  pl->stage_bytes = stage;
  pl->fixed_bytes = fixed;
  if (int rc = map3(&pl->tw, W, N, K, kRows)) return rc;
  if (int rc = map3(&pl->tx, X, M, K, p.xrows)) return rc;
  return YGG_OK;
}

int ygg_gemv_plan_set_stages(void* plan, int stages) {
  Plan* pl = const_cast<Plan*>(plan_of(plan));
  YGG_CHECK_ARG(pl != nullptr, "invalid gemv plan");
  YGG_CHECK_ARG(stages >= 2 && stages <= 16, "stages must be in [2, 16]");
  YGG_CHECK_ARG(pl->fixed_bytes + static_cast<size_t>(stages) * pl->stage_bytes <= 227 * 1024,
                "ring exceeds shared memory");
  pl->p.stages = stages;
  pl->smem = pl->fixed_bytes + static_cast<size_t>(stages) * pl->stage_bytes;
  return YGG_OK;
}

int ygg_gemv_run(const void* plan, const ygg_gemv_epilogue* ep, ygg_stream_t stream) {
  const Plan* pl = plan_of(plan);
  YGG_CHECK_ARG(pl != nullptr, "invalid gemv plan");
  YGG_CHECK_ARG(ep != nullptr, "null epilogue");
  const Params& p = pl->p;
  Epilogue e;
  std::memset(&e, 0, sizeof(e));
  e.kind = ep->kind;
  e.out = ep->out;
  e.ld = ep->ld;
  e.ss_in = ep->ss_in;
  e.ss_blocks = ep->ss_blocks;
  e.norm_dim = ep->norm_dim;
  e.eps = ep->eps;
  e.q_out = static_cast<__nv_bfloat16*>(ep->q_out);
  e.cache = static_cast<__nv_bfloat16*>(ep->cache);
  e.S = ep->S;
  e.Hq = ep->Hq;
  e.Hkv = ep->Hkv;
  e.hd = ep->hd;
  e.pos = ep->pos;
  e.slot = ep->slot;
  e.req = ep->req;
  e.rope_cs = reinterpret_cast<const float2*>(ep->rope_cs);
  e.act_out = static_cast<__nv_bfloat16*>(ep->act_out);
  e.resid = ep->resid;
  e.hb = static_cast<__nv_bfloat16*>(ep->hb);
  e.ss_out = ep->ss_out;
  e.topk_part = static_cast<TopkPartial*>(ep->topk_part);
  e.topk_k = ep->topk_k;
  e.inv_temp = ep->inv_temp;
  switch (e.kind) {
    case kStore: YGG_CHECK_ARG(e.out && e.ld >= p.N, "STORE needs out / ld"); break;
    case kStoreTopk:
      YGG_CHECK_ARG(e.out && e.ld >= p.N, "STORE_TOPK needs out / ld");
      YGG_CHECK_ARG(p.xrows == 8, "STORE_TOPK needs M <= 8 token rows");
      YGG_CHECK_ARG(e.topk_part && e.topk_k >= 1 && e.topk_k <= kTopkLane && e.topk_k <= p.N,
                    "STORE_TOPK needs topk_part and 1 <= k <= 8");
      YGG_CHECK_ARG(e.inv_temp > 0.f, "STORE_TOPK needs inv_temp > 0");
      break;
    case kResid: YGG_CHECK_ARG(e.resid && e.hb && e.ss_out, "RESID needs resid / hb / ss_out"); break;
    case kSwiglu: YGG_CHECK_ARG(e.act_out && p.N % 2 == 0, "SWIGLU needs act_out"); break;
    case kQkv:
      YGG_CHECK_ARG(e.q_out && e.cache && e.pos && e.slot && e.req && e.rope_cs && e.hd % 2 == 0 &&
                        p.N == (e.Hq + 2 * e.Hkv) * e.hd,
                    "QKV arguments");
      break;
    default: return ygg_fail(YGG_ERR_VALUE, "unknown gemv epilogue %d", e.kind);
  }
  YGG_CHECK_ARG(!e.ss_in || (e.ss_blocks >= 1 && e.norm_dim >= 1), "bad folded-RMSNorm arguments");
  e.trace = trace_next(1);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (e.kind == kStoreTopk)
    YGG_LAUNCH_PDL((gemv_kernel<1, true>), dim3(p.grid), dim3(kThreads), pl->smem, s, pl->tw, pl->tx, p, e);
  else if (p.xrows == 8)
    YGG_LAUNCH_PDL((gemv_kernel<1, false>), dim3(p.grid), dim3(kThreads), pl->smem, s, pl->tw, pl->tx, p, e);
  else
    YGG_LAUNCH_PDL((gemv_kernel<2, false>), dim3(p.grid), dim3(kThreads), pl->smem, s, pl->tw, pl->tx, p, e);
  return YGG_OK;
}

}  // extern "C"
