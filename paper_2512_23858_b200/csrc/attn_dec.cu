// Tree / prefix attention for decode-shaped passes: one CTA per (kv head, request, 64-row tile of
// query rows) walks every visible key chunk with an online softmax, so there are no split-KV
// partials and no combine launch.
//
// The tcgen05 split-KV kernel (attn_tc.cu) is built for the verify pass (T = 50 tokens x 4 heads =
// 200 query rows per kv head): there a 128-row UMMA tile is full and a separate combine is cheap.
// A draft pass has 8 tokens x 4 heads = 32 rows per kv head: 3/4 of every 128-row tile would be
// padding and the two launches cost more than the arithmetic.  Here:
//   warp 0 lane 0  TMA producer: Q tile once ([T][Gh][hd] box), then K [64 keys x hd] and V^T
//                  [hd x 64 keys] chunks (128B-swizzled) into a ring.
//   warps 1..R     16 query rows each (R = ceil(T*Gh / 16)): S = Q K^T with mma.sync m16n8k16
//                  (ldmatrix from the swizzled tiles), ancestor / prefix mask from the row's
//                  tree-mask bits, online softmax in base 2, P re-used from the S accumulators as
//                  the A operand of O += P V (the V^T cache layout is exactly the col-major B).
// Output O / l in bf16 straight into attn[m][head][hd].  Fixed key order: deterministic.
#include <cudaTypedefs.h>

#include <cmath>
#include <cstring>

#include "common.cuh"
#include "host_util.h"

namespace ygg {
namespace ad {

constexpr int kKC = 64;        // keys per chunk
constexpr int kMaxWarps = 8;   // compute warps = row warps (<= 4: 64 query rows) x key splits
constexpr int kStages = 8;
constexpr uint32_t kMagic = 0x59474144u;  // "YGAD"

struct Plan {
  uint32_t magic;
  int B, T, Hq, Hkv, hd, S, Gh, rows, warps, ksplit, stages, tpt, row_tiles, kvsplit;
  size_t smem;
  alignas(64) CUtensorMap tq;
  alignas(64) CUtensorMap tk;
  alignas(64) CUtensorMap tv;
};

struct Args {
  int T, Hq, Hkv, hd, S, Gh, rows, mask_words, ksplit, stages, tpt;  // rows = tpt * Gh (one row tile)
  int kvsplit, row_tiles;  // CTAs per (kv head, request, row tile) splitting the key chunks
  int ring_bytes;          // max(key/value ring, split-merge scratch): the barriers sit after it
  float* part;             // [B][Hkv][row_tiles][kvsplit][warps][NV][32] cross-CTA partials
  unsigned* ctr;           // [B][Hkv][row_tiles] arrival counters (monotonic)
  float scale_log2;
  const int32_t* blk_start;
  const int32_t* blk_len;
  const uint32_t* qmask;
  __nv_bfloat16* out;
};

YGG_DEV void tma2(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
YGG_DEV void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
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
YGG_DEV uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Swizzled byte offset of 16-byte chunk j of row r in a [rows][128 B] SW128 tile.
YGG_DEV uint32_t swz(int r, int j) { return static_cast<uint32_t>(r * 128 + ((j ^ (r & 7)) << 4)); }

// Visibility bits of 32 keys from absolute key kw for a query token tq (prefix always; block keys
// by the row's tree-mask bits, causal without a mask; nothing past the block).
YGG_DEV uint32_t vis_word(int kw, int bs, int bl, int tq, int mask_words, const uint32_t* mrow) {
  uint32_t pre = 0u;
  if (kw + 32 <= bs) pre = 0xffffffffu;
  else if (kw < bs) pre = (1u << (bs - kw)) - 1u;
  const int jb0 = kw - bs;
  uint32_t blk = 0u;
  if (jb0 + 32 > 0 && jb0 < bl) {
    if (mask_words == 0) {
      const int lo = jb0 < 0 ? -jb0 : 0;
      const int hi = min(31, tq - jb0);
      if (hi >= lo) blk = ((hi == 31) ? 0xffffffffu : ((1u << (hi + 1)) - 1u)) & ~((1u << lo) - 1u);
    } else if (jb0 < 0) {
      blk = __ldg(mrow) << (-jb0);
    } else {
      const int i = jb0 >> 5, s = jb0 & 31;
      const uint32_t w0 = i < mask_words ? __ldg(mrow + i) : 0u;
      const uint32_t w1 = i + 1 < mask_words ? __ldg(mrow + i + 1) : 0u;
      blk = s ? ((w0 >> s) | (w1 << (32 - s))) : w0;
    }
    const int keep = bl - jb0;
    if (keep < 32) blk &= (1u << keep) - 1u;
  }
  return pre | blk;
}

template <int HD>
__global__ void __launch_bounds__(32 * (1 + kMaxWarps), 1)
    attn_dec_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, Args a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int DCH = HD / 64;                    // 128-byte column blocks of a K / Q row
  constexpr uint32_t q_bytes = 64 * HD * 2;       // up to 64 query rows
  constexpr uint32_t k_bytes = kKC * HD * 2;      // [DCH][64 keys][128 B]
  constexpr uint32_t v_bytes = HD * kKC * 2;      // [HD rows][128 B]
  const int NS = a.stages;
  unsigned char* sq = base;
  unsigned char* sk = sq + q_bytes;
  unsigned char* sv = sk + NS * k_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sk + a.ring_bytes);
  uint64_t* empty = full + NS;
  uint64_t* qbar = empty + NS;
  const int kvh = blockIdx.x, r = blockIdx.y;
  const int rt = blockIdx.z / a.kvsplit, ks2 = blockIdx.z % a.kvsplit;  // row tile, cross-CTA key split
  const int t0 = rt * a.tpt;                                // first token of this row tile
  const int rows_cta = min(a.tpt, a.T - t0) * a.Gh;         // valid query rows of this CTA
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = (a.rows + 15) / 16;  // row warps per key split
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nw);
    }
    mbar_init(qbar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();
  const int bs = __ldg(a.blk_start + r), bl = __ldg(a.blk_len + r);
  const int nkeys = bs + bl;
  const int nch = (nkeys + kKC - 1) / kKC;
  const size_t kv_row0 = (static_cast<size_t>(r) * 2 * a.Hkv + kvh) * a.S;          // K rows of this head
  const size_t vt_row0 = ((static_cast<size_t>(r) * 2 + 1) * a.Hkv + kvh) * HD;     // V^T rows
  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(qbar, static_cast<uint32_t>(a.rows) * 128u * DCH);  // full box (OOB rows zero-filled)
      for (int dc = 0; dc < DCH; ++dc)
        tma3(sq + dc * (64 * 128), &tq, qbar, dc * 64, kvh * a.Gh, r * a.T + t0);
      for (int j = 0, c = ks2; c < nch; ++j, c += a.kvsplit) {  // this CTA's chunks, local index j
        const int st = j % NS;
        if (j >= NS) mbar_wait(&empty[st], ((j / NS) - 1) & 1);
        mbar_arrive_expect_tx(&full[st], k_bytes + v_bytes);
        for (int dc = 0; dc < DCH; ++dc)
          tma2(sk + st * k_bytes + dc * (kKC * 128), &tk, &full[st], dc * 64, static_cast<int>(kv_row0) + c * kKC);
        tma2(sv + st * v_bytes, &tv, &full[st], c * kKC, static_cast<int>(vt_row0));
      }
    }
    return;
  }
  // Compute warp (ks, rw): key split ks takes chunks ks, ks + ksplit, ...; row warp rw 16 query rows
  // (token t = row / Gh, head = kvh*Gh + row % Gh).  Splits are merged in fixed order at the end.
  const int cwi = warp - 1;
  const int ks = cwi / nw, rw = cwi % nw;
  const int qr0 = rw * 16;
  const int ra = qr0 + (lane >> 2), rb = ra + 8;  // accumulator rows of this thread
  const int ta = t0 + ra / a.Gh, tb = t0 + rb / a.Gh;
  const bool va = ra < rows_cta, vb = rb < rows_cta;
  const uint32_t* mra = a.qmask + static_cast<size_t>(r * a.T + (va ? ta : 0)) * (a.mask_words ? a.mask_words : 1);
  const uint32_t* mrb = a.qmask + static_cast<size_t>(r * a.T + (vb ? tb : 0)) * (a.mask_words ? a.mask_words : 1);
  mbar_wait(qbar, 0);
  // Q fragments for all hd k-steps (A operand), kept in registers.
  uint32_t qa[HD / 16][4];
  {
    const int arow = qr0 + (lane & 7) + 8 * ((lane >> 3) & 1), ahi = lane >> 4;
#pragma unroll
    for (int s = 0; s < HD / 16; ++s) {
      const int dc = s / 4, j = 2 * (s % 4) + ahi;
      ldsm_x4(smem_u32(sq + dc * (64 * 128)) + swz(arow, j), qa[s][0], qa[s][1], qa[s][2], qa[s][3]);
    }
  }
  float o[HD / 8][4];
#pragma unroll
  for (int n = 0; n < HD / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float ma = -INFINITY, mb = -INFINITY, la = 0.f, lb = 0.f;
  const int brow = lane & 7, bhi = (lane >> 3) & 1;
  for (int j = ks; ks2 + j * a.kvsplit < nch; j += a.ksplit) {
    const int c = ks2 + j * a.kvsplit;
    const int st = j % NS;
    const int key0 = c * kKC;
    // visibility of this thread's 16 key columns (n-tile j: keys 8j + 2*(lane&3) + {0,1}) per row
    uint32_t wa0 = 0u, wa1 = 0u, wb0 = 0u, wb1 = 0u;
    if (va) {
      wa0 = vis_word(key0, bs, bl, ta, a.mask_words, mra);
      wa1 = vis_word(key0 + 32, bs, bl, ta, a.mask_words, mra);
    }
    if (vb) {
      wb0 = vis_word(key0, bs, bl, tb, a.mask_words, mrb);
      wb1 = vis_word(key0 + 32, bs, bl, tb, a.mask_words, mrb);
    }
    mbar_wait(&full[st], (j / NS) & 1);
    const uint32_t kb = smem_u32(sk + st * k_bytes), vb_ = smem_u32(sv + st * v_bytes);
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
      const int dc = ks / 4, j = 2 * (ks % 4) + bhi;
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        uint32_t b0, b1;
        ldsm_x2(kb + dc * (kKC * 128) + swz(8 * n + brow, j), b0, b1);
        mma16816(s[n], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b0, b1);
      }
    }
    // mask + chunk row max
    float cma = -INFINITY, cmb = -INFINITY;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = 8 * n + 2 * (lane & 3) + e;  // key within the chunk
        const uint32_t wa = col < 32 ? wa0 : wa1, wb = col < 32 ? wb0 : wb1;
        const bool vis_a = (wa >> (col & 31)) & 1u, vis_b = (wb >> (col & 31)) & 1u;
        s[n][e] = vis_a ? s[n][e] * a.scale_log2 : -INFINITY;
        s[n][2 + e] = vis_b ? s[n][2 + e] * a.scale_log2 : -INFINITY;
        cma = fmaxf(cma, s[n][e]);
        cmb = fmaxf(cmb, s[n][2 + e]);
      }
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      cma = fmaxf(cma, __shfl_xor_sync(0xffffffffu, cma, off));
      cmb = fmaxf(cmb, __shfl_xor_sync(0xffffffffu, cmb, off));
    }
    const float na = fmaxf(ma, cma), nb = fmaxf(mb, cmb);
    const float fa = (na == -INFINITY) ? 1.f : exp2f(ma - na), fb = (nb == -INFINITY) ? 1.f : exp2f(mb - nb);
    ma = na;
    mb = nb;
    float sa = 0.f, sb = 0.f;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        s[n][e] = (s[n][e] == -INFINITY) ? 0.f : exp2f(s[n][e] - na);
        s[n][2 + e] = (s[n][2 + e] == -INFINITY) ? 0.f : exp2f(s[n][2 + e] - nb);
        sa += s[n][e];
        sb += s[n][2 + e];
      }
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, off);
      sb += __shfl_xor_sync(0xffffffffu, sb, off);
    }
    la = la * fa + sa;
    lb = lb * fb + sb;
#pragma unroll
    for (int n = 0; n < HD / 8; ++n) {
      o[n][0] *= fa;
      o[n][1] *= fa;
      o[n][2] *= fb;
      o[n][3] *= fb;
    }
    // O += P V: A = P (16 rows x 16 keys per k-step, from the S accumulators), B = V^T rows.
#pragma unroll
    for (int ks = 0; ks < kKC / 16; ++ks) {
      const uint32_t a0 = pack2(s[2 * ks][0], s[2 * ks][1]), a1 = pack2(s[2 * ks][2], s[2 * ks][3]);
      const uint32_t a2 = pack2(s[2 * ks + 1][0], s[2 * ks + 1][1]), a3 = pack2(s[2 * ks + 1][2], s[2 * ks + 1][3]);
      const int j = 2 * ks + bhi;
#pragma unroll
      for (int n = 0; n < HD / 8; ++n) {
        uint32_t b0, b1;
        ldsm_x2(vb_ + swz(8 * n + brow, j), b0, b1);
        mma16816(o[n], a0, a1, a2, a3, b0, b1);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  // Merge the key splits (fixed split order) through shared memory, reusing the drained ring.
  if (a.ksplit > 1) {
    asm volatile("bar.sync 1, %0;" ::"r"(32 * nw * a.ksplit) : "memory");  // ring fully consumed
    constexpr int NV = HD / 8 * 4 + 4;  // o values + (ma, mb, la, lb)
    float* xs = reinterpret_cast<float*>(sk);
    float* mine = xs + static_cast<size_t>((ks * nw + rw) * NV) * 32 + lane;
    if (ks > 0) {
#pragma unroll
      for (int n = 0; n < HD / 8; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) mine[(n * 4 + e) * 32] = o[n][e];
      mine[(NV - 4) * 32] = ma;
      mine[(NV - 3) * 32] = mb;
      mine[(NV - 2) * 32] = la;
      mine[(NV - 1) * 32] = lb;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(32 * nw * a.ksplit) : "memory");
    if (ks > 0) return;
    for (int k2 = 1; k2 < a.ksplit; ++k2) {
      const float* th = xs + static_cast<size_t>((k2 * nw + rw) * NV) * 32 + lane;
      const float m2a = th[(NV - 4) * 32], m2b = th[(NV - 3) * 32];
      const float na = fmaxf(ma, m2a), nb = fmaxf(mb, m2b);
      const float f1a = na == -INFINITY ? 0.f : exp2f(ma - na), f2a = na == -INFINITY ? 0.f : exp2f(m2a - na);
      const float f1b = nb == -INFINITY ? 0.f : exp2f(mb - nb), f2b = nb == -INFINITY ? 0.f : exp2f(m2b - nb);
#pragma unroll
      for (int n = 0; n < HD / 8; ++n) {
        o[n][0] = o[n][0] * f1a + th[(n * 4 + 0) * 32] * f2a;
        o[n][1] = o[n][1] * f1a + th[(n * 4 + 1) * 32] * f2a;
        o[n][2] = o[n][2] * f1b + th[(n * 4 + 2) * 32] * f2b;
        o[n][3] = o[n][3] * f1b + th[(n * 4 + 3) * 32] * f2b;
      }
      la = la * f1a + th[(NV - 2) * 32] * f2a;
      lb = lb * f1b + th[(NV - 1) * 32] * f2b;
      ma = na;
      mb = nb;
    }
  }
  // Cross-CTA key splits: publish this CTA's (O, m, l); the last of the group's CTAs merges all of
  // them in fixed split order (deterministic whichever CTA arrives last).
  if (a.kvsplit > 1) {
    constexpr int NV = HD / 8 * 4 + 4;
    const size_t grp = (static_cast<size_t>(r) * a.Hkv + kvh) * a.row_tiles + rt;
    const size_t gstride = static_cast<size_t>(nw) * NV * 32;
    float* mine = a.part + (grp * a.kvsplit + ks2) * gstride + static_cast<size_t>(rw) * NV * 32 + lane;
#pragma unroll
    for (int n = 0; n < HD / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) __stcg(mine + (n * 4 + e) * 32, o[n][e]);
    __stcg(mine + (NV - 4) * 32, ma);
    __stcg(mine + (NV - 3) * 32, mb);
    __stcg(mine + (NV - 2) * 32, la);
    __stcg(mine + (NV - 1) * 32, lb);
    __threadfence();
    asm volatile("bar.sync 2, %0;" ::"r"(32 * nw) : "memory");
    __shared__ int last_s;
    if (rw == 0 && lane == 0) {
      const unsigned old = atomicAdd(a.ctr + grp, 1u);
      last_s = ((old + 1u) % static_cast<unsigned>(a.kvsplit)) == 0u;
    }
    asm volatile("bar.sync 2, %0;" ::"r"(32 * nw) : "memory");
    if (!last_s) return;
    __threadfence();
    const float* base0 = a.part + grp * a.kvsplit * gstride + static_cast<size_t>(rw) * NV * 32 + lane;
    ma = __ldcg(base0 + (NV - 4) * 32);
    mb = __ldcg(base0 + (NV - 3) * 32);
    la = __ldcg(base0 + (NV - 2) * 32);
    lb = __ldcg(base0 + (NV - 1) * 32);
#pragma unroll
    for (int n = 0; n < HD / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) o[n][e] = __ldcg(base0 + (n * 4 + e) * 32);
    for (int k2 = 1; k2 < a.kvsplit; ++k2) {
      const float* th = base0 + k2 * gstride;
      const float m2a = __ldcg(th + (NV - 4) * 32), m2b = __ldcg(th + (NV - 3) * 32);
      const float na = fmaxf(ma, m2a), nb = fmaxf(mb, m2b);
      const float f1a = na == -INFINITY ? 0.f : exp2f(ma - na), f2a = na == -INFINITY ? 0.f : exp2f(m2a - na);
      const float f1b = nb == -INFINITY ? 0.f : exp2f(mb - nb), f2b = nb == -INFINITY ? 0.f : exp2f(m2b - nb);
#pragma unroll
      for (int n = 0; n < HD / 8; ++n) {
        o[n][0] = o[n][0] * f1a + __ldcg(th + (n * 4 + 0) * 32) * f2a;
        o[n][1] = o[n][1] * f1a + __ldcg(th + (n * 4 + 1) * 32) * f2a;
        o[n][2] = o[n][2] * f1b + __ldcg(th + (n * 4 + 2) * 32) * f2b;
        o[n][3] = o[n][3] * f1b + __ldcg(th + (n * 4 + 3) * 32) * f2b;
      }
      la = la * f1a + __ldcg(th + (NV - 2) * 32) * f2a;
      lb = lb * f1b + __ldcg(th + (NV - 1) * 32) * f2b;
      ma = na;
      mb = nb;
    }
  }
  // O / l -> bf16 attn[m][head][hd]
  const float ia = la > 0.f ? 1.f / la : 0.f, ib = lb > 0.f ? 1.f / lb : 0.f;
  const int ha = kvh * a.Gh + ra % a.Gh, hb = kvh * a.Gh + rb % a.Gh;
  __nv_bfloat16* oa = a.out + (static_cast<size_t>(r * a.T + ta) * a.Hq + ha) * HD;
  __nv_bfloat16* ob = a.out + (static_cast<size_t>(r * a.T + tb) * a.Hq + hb) * HD;
#pragma unroll
  for (int n = 0; n < HD / 8; ++n) {
    const int col = 8 * n + 2 * (lane & 3);
    if (va) *reinterpret_cast<uint32_t*>(oa + col) = pack2(o[n][0] * ia, o[n][1] * ia);
    if (vb) *reinterpret_cast<uint32_t*>(ob + col) = pack2(o[n][2] * ib, o[n][3] * ib);
  }
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
static int enc(CUtensorMap* m, int rank, const void* p, const cuuint64_t* dims, const cuuint64_t* str, const cuuint32_t* box) {
  auto e = encoder();
  if (!e) return ygg_fail(YGG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t es[3] = {1, 1, 1};
  CUresult rc = e(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(p), dims, str, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) return ygg_fail(YGG_ERR_CUDA, "decode attention tensor map failed (%d)", static_cast<int>(rc));
  return YGG_OK;
}
static const Plan* plan_of(const void* p) {
  const Plan* q = reinterpret_cast<const Plan*>((reinterpret_cast<uintptr_t>(p) + 63) & ~uintptr_t(63));
  return (p && q->magic == kMagic) ? q : nullptr;
}

}  // namespace ad
}  // namespace ygg

using namespace ygg;
using namespace ygg::ad;

extern "C" {

int ygg_prepare_attn_dec(void) {
  for (auto fn : {attn_dec_kernel<64>, attn_dec_kernel<128>}) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "decode attention attribute: %s", cudaGetErrorString(e));
  }
  return YGG_OK;
}

size_t ygg_attn_dec_plan_size(void) { return sizeof(Plan) + 64; }

size_t ygg_attn_dec_workspace_size(const void* plan) {
  const Plan* p = plan_of(plan);
  if (!p) return 0;
  const size_t groups = static_cast<size_t>(p->B) * p->Hkv * p->row_tiles;
  const size_t nv = static_cast<size_t>(p->hd) / 8 * 4 + 4;
  const size_t part = groups * p->kvsplit * ((p->rows + 15) / 16) * nv * 32 * sizeof(float);
  return ((part + 255) / 256) * 256 + groups * sizeof(unsigned) + 256;
}

int ygg_attn_dec_plan_init(void* plan, const void* q, const void* cache_layer, int B, int T, int Hq, int Hkv, int hd,
                           int S) {
  YGG_CHECK_ARG(plan && q && cache_layer, "null pointer");
  YGG_CHECK_ARG(hd == 64 || hd == 128, "head dim must be 64 or 128");
  YGG_CHECK_ARG(Hkv >= 1 && Hq % Hkv == 0, "bad head grouping");
  const int Gh = Hq / Hkv;
  YGG_CHECK_ARG(B >= 1 && T >= 1 && Gh <= 64 && 64 % Gh == 0, "decode attention: head group must divide 64");
  YGG_CHECK_ARG(S % 64 == 0, "cache capacity must be a multiple of 64");
  Plan* p = reinterpret_cast<Plan*>((reinterpret_cast<uintptr_t>(plan) + 63) & ~uintptr_t(63));
  std::memset(p, 0, sizeof(Plan));
  p->magic = kMagic;
  p->B = B;
  p->T = T;
  p->Hq = Hq;
  p->Hkv = Hkv;
  p->hd = hd;
  p->S = S;
  p->Gh = Gh;
  p->tpt = T < 64 / Gh ? T : 64 / Gh;   // tokens per row tile (<= 64 query rows per CTA)
  p->row_tiles = (T + p->tpt - 1) / p->tpt;
  p->rows = p->tpt * Gh;
  const int nw = (p->rows + 15) / 16;
  p->ksplit = kMaxWarps / nw;            // split the key chunks over the remaining warps
  if (hd == 128 && p->ksplit > 2) p->ksplit = 2;  // register budget of the 128-wide accumulators
  p->warps = nw * p->ksplit;
  p->stages = hd == 64 ? 8 : 4;
  if (const char* e = getenv("YGG_ATTN_DEC_STAGES")) p->stages = atoi(e) < 2 ? 2 : (atoi(e) > 8 ? 8 : atoi(e));
  // Every stage must always feed the same key-split group (chunk j -> stage j % stages, group
  // j % ksplit): otherwise a group can wait on a stage two phases ahead and the parity wait would pass
  // on a stale phase.  So stages is a multiple of ksplit.
  const int max_st = static_cast<int>((200 * 1024 - 64 * hd * 2) / (2 * kKC * hd * 2));  // smem budget
  if (p->stages > max_st) p->stages = max_st;
  p->stages = (p->stages / p->ksplit) * p->ksplit;
  if (p->stages < p->ksplit) p->stages = p->ksplit;
  // Cross-CTA key splits (merge by the last CTA of each group): off by default — same-box cfg2
  // draft pass 0.712 ms (1), 0.718 (2), 0.713 (4), 0.734 (8); verify (forced) 3.96 / 3.95 / 4.12.
  {
    int kv = 1;
    if (const char* e = getenv("YGG_ATTN_DEC_KVSPLIT")) kv = atoi(e);
    p->kvsplit = kv < 1 ? 1 : (kv > 8 ? 8 : kv);
  }
  const size_t merge = static_cast<size_t>(p->warps) * (hd / 8 * 4 + 4) * 32 * 4;
  const size_t ring = static_cast<size_t>(p->stages) * 2 * (kKC * hd * 2);
  p->smem = 1024 + 64 * hd * 2 + ((ring > merge ? ring : merge) + 15) / 16 * 16 + (2 * p->stages + 2) * 8;
  const int M = B * T;
  {  // q [M][Hq][hd]: box {64, Gh, T} -> rows (token, head-in-group); 64 rows of smem reserved
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(hd), static_cast<cuuint64_t>(Hq), static_cast<cuuint64_t>(M)};
    cuuint64_t str[2] = {static_cast<cuuint64_t>(hd) * 2, static_cast<cuuint64_t>(Hq) * hd * 2};
    cuuint32_t box[3] = {64, static_cast<cuuint32_t>(Gh), static_cast<cuuint32_t>(p->tpt)};
    if (int rc = enc(&p->tq, 3, q, dims, str, box)) return rc;
  }
  {  // K rows [(B*2*Hkv*S)][hd]: box {64, 64 keys}
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(hd), static_cast<cuuint64_t>(B) * 2 * Hkv * S};
    cuuint64_t str[1] = {static_cast<cuuint64_t>(hd) * 2};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(kKC)};
    if (int rc = enc(&p->tk, 2, cache_layer, dims, str, box)) return rc;
  }
  {  // V^T rows [(B*2*Hkv*hd)][S]: box {64 keys, hd}
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(S), static_cast<cuuint64_t>(B) * 2 * Hkv * hd};
    cuuint64_t str[1] = {static_cast<cuuint64_t>(S) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kKC), static_cast<cuuint32_t>(hd)};
    if (int rc = enc(&p->tv, 2, cache_layer, dims, str, box)) return rc;
  }
  return YGG_OK;
}

int ygg_attn_dec_run(const void* plan, const int32_t* blk_start, const int32_t* blk_len, const uint32_t* qmask,
                     int mask_words, float scale, void* out, void* workspace, ygg_stream_t stream) {
  const Plan* p = plan_of(plan);
  YGG_CHECK_ARG(p != nullptr, "invalid decode-attention plan");
  YGG_CHECK_ARG(blk_start && blk_len && out, "null pointer");
  YGG_CHECK_ARG(mask_words >= 0 && mask_words <= YGG_MAX_MASK_WORDS, "mask too wide");
  YGG_CHECK_ARG(mask_words == 0 || qmask != nullptr, "mask words without a mask");
  Args a;
  a.T = p->T;
  a.Hq = p->Hq;
  a.Hkv = p->Hkv;
  a.hd = p->hd;
  a.S = p->S;
  a.Gh = p->Gh;
  a.rows = p->rows;
  a.mask_words = mask_words;
  a.ksplit = p->ksplit;
  a.stages = p->stages;
  a.tpt = p->tpt;
  a.kvsplit = p->kvsplit;
  a.row_tiles = p->row_tiles;
  {
    const size_t merge = static_cast<size_t>(p->warps) * (p->hd / 8 * 4 + 4) * 32 * 4;
    const size_t ring = static_cast<size_t>(p->stages) * 2 * (kKC * p->hd * 2);
    a.ring_bytes = static_cast<int>(((ring > merge ? ring : merge) + 15) / 16 * 16);
  }
  YGG_CHECK_ARG(p->kvsplit == 1 || workspace != nullptr, "decode attention with key splits needs a workspace");
  {
    const size_t groups = static_cast<size_t>(p->B) * p->Hkv * p->row_tiles;
    const size_t nv = static_cast<size_t>(p->hd) / 8 * 4 + 4;
    const size_t part = groups * p->kvsplit * ((p->rows + 15) / 16) * nv * 32 * sizeof(float);
    a.part = static_cast<float*>(workspace);
    a.ctr = workspace ? reinterpret_cast<unsigned*>(static_cast<char*>(workspace) + ((part + 255) / 256) * 256) : nullptr;
  }
  a.scale_log2 = scale * 1.4426950408889634f;
  a.blk_start = blk_start;
  a.blk_len = blk_len;
  a.qmask = qmask ? qmask : reinterpret_cast<const uint32_t*>(blk_start);  // never read when mask_words == 0
  a.out = static_cast<__nv_bfloat16*>(out);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const dim3 grid(p->Hkv, p->B, p->row_tiles * p->kvsplit), block(32 * (1 + p->warps));
  if (p->hd == 64)
    YGG_LAUNCH_PDL(attn_dec_kernel<64>, grid, block, p->smem, s, p->tq, p->tk, p->tv, a);
  else
    YGG_LAUNCH_PDL(attn_dec_kernel<128>, grid, block, p->smem, s, p->tq, p->tk, p->tv, a);
  return YGG_OK;
}

}  // extern "C"
