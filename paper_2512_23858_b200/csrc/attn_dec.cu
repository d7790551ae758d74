// Tree / prefix attention for decode-shaped passes: a (1, 1, kvsplit) thread-block cluster per
// (kv head, request, 64-row tile of query rows) walks the visible key chunks with an online softmax
// (chunks interleaved over the cluster's CTAs and, inside a CTA, over ksplit warp groups); the
// partials merge in shared memory — in-CTA, then in the leader CTA through DSMEM — in fixed split
// order, so there is no combine launch and the result is deterministic.  kvsplit defaults to the
// cluster size that brings the grid to ~half the SMs (at most 4): with B = 1 only Hkv = 8 CTAs
// would otherwise carry the whole mma.sync + softmax chain.
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
// Output O / l in bf16 straight into attn[m][head][hd].
// Chunks wholly inside the committed prefix are loaded before the grid-dependency wait and skip the
// mask work; the block's chunks and Q follow the wait.
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
  int B, T, Hq, Hkv, hd, S, Gh, rows, warps, ksplit, stages, tpt, row_tiles, kvsplit, ring_bytes, slot_bytes;
  size_t smem;
  const char* pf_ptr[2];  // optional L2 prefetch regions (issued while HBM is otherwise idle)
  size_t pf_bytes[2];
  int tpf_nblk, tpf_kchunks, tpf_first;  // optional strided prefetch of a GEMV's weight chunks
  alignas(64) CUtensorMap tpf;
  alignas(64) CUtensorMap tq;
  alignas(64) CUtensorMap tk;
  alignas(64) CUtensorMap tv;
};

struct Args {
  int T, Hq, Hkv, hd, S, Gh, rows, mask_words, ksplit, stages, tpt;  // rows = tpt * Gh (one row tile)
  int warps;               // compute warps = row warps x ksplit
  int kvsplit, row_tiles;  // CTAs (one thread-block cluster) per (kv head, request, row tile)
  int ring_bytes;          // max(key/value ring, in-CTA merge scratch)
  int slot_bytes;          // cluster merge slots in the leader CTA [kvsplit - 1][warps][NV2][32] f32
  float scale_log2;
  const int32_t* blk_start;
  const int32_t* blk_len;
  const uint32_t* qmask;
  __nv_bfloat16* out;
  unsigned long long* trace;  // kernel-timeline slot (profiling only) or nullptr
  const char* pf_ptr[2];      // L2 prefetch regions (each split over the CTAs) or nullptr
  size_t pf_bytes[2];
  int tpf_nblk, tpf_kchunks, tpf_first;  // strided GEMV-chunk prefetch (tpf_nblk = 0: off)
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
YGG_DEV float ex2(float x) {  // 2^x, flush-to-zero (ex2(-inf) = 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
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

template <int HD, int KS>  // KS: in-CTA key-split groups (== Args::ksplit)
__global__ void __launch_bounds__(32 * (1 + kMaxWarps), 1)
    attn_dec_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tpf, Args a) {
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
  float* slots = reinterpret_cast<float*>(sk + a.ring_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(sk + a.ring_bytes + a.slot_bytes);
  uint64_t* empty = full + NS;
  uint64_t* qbar = empty + NS;
  uint64_t* cbar = qbar + 1;  // leader: every lane of every compute warp of the cluster has filled its slot
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
    // the leader's merge barrier completes on the transaction bytes of the other CTAs' st.async pushes:
    // (kvsplit - 1) CTAs x warps x 32 lanes x (NPW n-tiles + the (m, l) quad) x 16 B
    mbar_init(cbar, 1);
    if (a.kvsplit > 1 && ks2 == 0)
      mbar_arrive_expect_tx(cbar, static_cast<uint32_t>((a.kvsplit - 1) * a.warps * 32 * ((HD / 8) / KS + 1) * 16));
    fence_barrier_init();
    trace_min(a.trace, 0);
  }
  // Cluster members arrive on the leader's barrier: it must be initialised cluster-wide first.
  if (a.kvsplit > 1) cluster_sync();
  else __syncthreads();
  const size_t kv_row0 = (static_cast<size_t>(r) * 2 * a.Hkv + kvh) * a.S;          // K rows of this head
  const size_t vt_row0 = ((static_cast<size_t>(r) * 2 + 1) * a.Hkv + kvh) * HD;     // V^T rows
  if (warp == 0) {
    if (lane == 0) {
      // The block bounds and the committed prefix's K / V were written at least two kernels back,
      // and the kernel just before this one (gemv / epi_qkv_rope) triggers its dependents only
      // after its own grid-dependency wait, so everything two or more kernels back has completed:
      // chunks wholly inside the prefix stream in before the wait; the block's keys and Q (written
      // by the previous kernel) are loaded after it.
      const int bs = __ldg(a.blk_start + r), bl = __ldg(a.blk_len + r);
      const int nch = (bs + bl + kKC - 1) / kKC;
      auto load = [&](int j, int c) {
        const int st = j % NS;
        if (j >= NS) mbar_wait(&empty[st], ((j / NS) - 1) & 1);
        mbar_arrive_expect_tx(&full[st], k_bytes + v_bytes);
        for (int dc = 0; dc < DCH; ++dc)
          tma2(sk + st * k_bytes + dc * (kKC * 128), &tk, &full[st], dc * 64, static_cast<int>(kv_row0) + c * kKC);
        tma2(sv + st * v_bytes, &tv, &full[st], c * kKC, static_cast<int>(vt_row0));
      };
      int j = 0, c = ks2;  // this CTA's chunks, local index j
      for (; j < NS && c < nch && (c + 1) * kKC <= bs; ++j, c += a.kvsplit) load(j, c);
      pdl_wait();
      mbar_arrive_expect_tx(qbar, static_cast<uint32_t>(a.rows) * 128u * DCH);  // full box (OOB rows zero-filled)
      for (int dc = 0; dc < DCH; ++dc)
        tma3(sq + dc * (64 * 128), &tq, qbar, dc * 64, kvh * a.Gh, r * a.T + t0);
      for (; c < nch; ++j, c += a.kvsplit) load(j, c);
      if (a.tpf_nblk > 0) {
        // The next GEMV's weight chunks its ring cannot hold (chunks >= tpf_first of every 16-row
        // block), pulled into L2 through its own tensor map: one 16 KB box per instruction.
        const int ncta = static_cast<int>(gridDim.x * gridDim.y * gridDim.z);
        const int cta = static_cast<int>((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x);
        const int per_blk = a.tpf_kchunks - a.tpf_first;
        for (int i = cta; i < a.tpf_nblk * per_blk; i += ncta) {
          const int bq = i / per_blk, qq = a.tpf_first + i % per_blk;
          asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];"
                       ::"l"(reinterpret_cast<uint64_t>(&tpf)), "r"(0), "r"(bq * 16), "r"(qq * 8)
                       : "memory");
        }
      }
      for (int rg = 0; rg < 2; ++rg) {
        // After this CTA's own loads: the kernel barely touches HBM, so pull this CTA's slice of
        // later weights into L2 so that their stream starts from L2 (bulk prefetch, 64 KB each).
        if (!a.pf_ptr[rg]) continue;
        const size_t ncta = static_cast<size_t>(gridDim.x) * gridDim.y * gridDim.z;
        const size_t cta = (static_cast<size_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        const size_t per = ((a.pf_bytes[rg] / ncta) + 255) & ~static_cast<size_t>(255);
        const size_t b0 = cta * per, b1 = b0 + per < a.pf_bytes[rg] ? b0 + per : a.pf_bytes[rg];
        for (size_t o = b0; o < b1; o += 65536) {
          const uint32_t n = static_cast<uint32_t>(b1 - o < 65536 ? ((b1 - o) & ~static_cast<size_t>(15)) : 65536);
          if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.pf_ptr[rg] + o), "r"(n) : "memory");
        }
      }
    } else {
      pdl_wait();
    }
    pdl_launch_dependents();
    return;
  }
  // Block bounds were written at least two kernels back (see the producer): load them before the
  // wait, off the critical path.
  const int bs = __ldg(a.blk_start + r), bl = __ldg(a.blk_len + r);
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 32) trace_min(a.trace, 1);
  const int nkeys = bs + bl;
  const int nch = (nkeys + kKC - 1) / kKC;
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
  if (lane == 0) trace_max(a.trace, 3);
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
  // Per-thread ldmatrix offsets: row 8n + brow of a swizzled [rows][128 B] tile has (row & 7) == brow,
  // so chunk column j sits at n * 1024 + brow * 128 + ((j ^ brow) << 4) — the n part is an immediate.
  const int brow = lane & 7, bhi = (lane >> 3) & 1;
  uint32_t xoff[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) xoff[q] = static_cast<uint32_t>(brow * 128 + (((2 * q + bhi) ^ brow) << 4));
  const float sl = a.scale_log2;
  for (int j = ks; ks2 + j * a.kvsplit < nch; j += KS) {
    const int c = ks2 + j * a.kvsplit;
    const int st = j % NS;
    const int key0 = c * kKC;
    // Chunks wholly inside the committed prefix are visible to every row: no mask work at all.
    const bool in_prefix = key0 + kKC <= bs;
    // visibility of this thread's 16 key columns (n-tile j: keys 8j + 2*(lane&3) + {0,1}) per row
    uint32_t wa0 = 0u, wa1 = 0u, wb0 = 0u, wb1 = 0u;
    if (!in_prefix) {
      if (va) {
        wa0 = vis_word(key0, bs, bl, ta, a.mask_words, mra);
        wa1 = vis_word(key0 + 32, bs, bl, ta, a.mask_words, mra);
      }
      if (vb) {
        wb0 = vis_word(key0, bs, bl, tb, a.mask_words, mrb);
        wb1 = vis_word(key0 + 32, bs, bl, tb, a.mask_words, mrb);
      }
    }
    mbar_wait(&full[st], (j / NS) & 1);
    if (j == ks && lane == 0) trace_max(a.trace, 4);
    const uint32_t kb = smem_u32(sk + st * k_bytes), vb_ = smem_u32(sv + st * v_bytes);
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      const uint32_t ka = kb + (kk / 4) * (kKC * 128) + xoff[kk % 4];
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        uint32_t b0, b1;
        ldsm_x2(ka + n * 1024, b0, b1);
        mma16816(s[n], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
      }
    }
    // mask (raw scores) + chunk row max
    float cma = -INFINITY, cmb = -INFINITY;
    if (!in_prefix) {
#pragma unroll
      for (int n = 0; n < 8; ++n) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = 8 * n + 2 * (lane & 3) + e;  // key within the chunk
          const uint32_t wa = col < 32 ? wa0 : wa1, wb = col < 32 ? wb0 : wb1;
          if (!((wa >> (col & 31)) & 1u)) s[n][e] = -INFINITY;
          if (!((wb >> (col & 31)) & 1u)) s[n][2 + e] = -INFINITY;
        }
      }
    }
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      cma = fmaxf(cma, fmaxf(s[n][0], s[n][1]));
      cmb = fmaxf(cmb, fmaxf(s[n][2], s[n][3]));
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      cma = fmaxf(cma, __shfl_xor_sync(0xffffffffu, cma, off));
      cmb = fmaxf(cmb, __shfl_xor_sync(0xffffffffu, cmb, off));
    }
    // running max in scaled log2 units (scale > 0, so the max commutes with the scaling)
    const float na = fmaxf(ma, cma * sl), nb = fmaxf(mb, cmb * sl);
    const float fa = (na == -INFINITY) ? 1.f : ex2(ma - na), fb = (nb == -INFINITY) ? 1.f : ex2(mb - nb);
    const float nna = (na == -INFINITY) ? 0.f : -na, nnb = (nb == -INFINITY) ? 0.f : -nb;
    ma = na;
    mb = nb;
    float sa = 0.f, sb = 0.f;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        s[n][e] = ex2(fmaf(s[n][e], sl, nna));  // masked: -inf -> 0
        s[n][2 + e] = ex2(fmaf(s[n][2 + e], sl, nnb));
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
    if (__any_sync(0xffffffffu, fa != 1.f || fb != 1.f)) {
#pragma unroll
      for (int n = 0; n < HD / 8; ++n) {
        o[n][0] *= fa;
        o[n][1] *= fa;
        o[n][2] *= fb;
        o[n][3] *= fb;
      }
    }
    // O += P V: A = P (16 rows x 16 keys per k-step, from the S accumulators), B = V^T rows.
#pragma unroll
    for (int kk = 0; kk < kKC / 16; ++kk) {
      const uint32_t a0 = pack2(s[2 * kk][0], s[2 * kk][1]), a1 = pack2(s[2 * kk][2], s[2 * kk][3]);
      const uint32_t a2 = pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]), a3 = pack2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
      const uint32_t va_ = vb_ + xoff[kk];
#pragma unroll
      for (int n = 0; n < HD / 8; ++n) {
        uint32_t b0, b1;
        ldsm_x2(va_ + n * 1024, b0, b1);
        mma16816(o[n], a0, a1, a2, a3, b0, b1);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (j == ks && lane == 0) trace_max(a.trace, 5);
  }
  if (lane == 0) trace_max(a.trace, 6);
  // Merge.  (1) In-CTA key splits: every warp parks its (O, m, l) in the drained ring; warp (ks, rw)
  // then merges n-tiles [ks*NPW, (ks+1)*NPW) of row warp rw over the KS partials in fixed order.
  // (2) Cluster key splits: each warp writes its merged n-tiles + (m, l) into its slot in the leader
  // CTA's shared memory (DSMEM) and arrives on the leader's barrier; the leader's warps merge the
  // kvsplit slots in fixed order.  Both merges are deterministic and fully unrolled (compile-time
  // KS / NPW; the cluster loop is predicated up to 8) — they are pure latency chains otherwise.
  constexpr int NV = HD / 8 * 4 + 4;  // o values + (ma, mb, la, lb)
  constexpr int NPW = (HD / 8) / KS;
  const int n0 = ks * NPW;
  float O[NPW][4];
  float Ma = ma, Mb = mb, La = la, Lb = lb;
  if constexpr (KS > 1) {
    asm volatile("bar.sync 1, %0;" ::"r"(32 * a.warps) : "memory");  // ring fully consumed
    float* xs = reinterpret_cast<float*>(sk);
    float* mine = xs + static_cast<size_t>((ks * nw + rw) * NV) * 32 + lane;
#pragma unroll
    for (int n = 0; n < HD / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) mine[(n * 4 + e) * 32] = o[n][e];
    mine[(NV - 4) * 32] = ma;
    mine[(NV - 3) * 32] = mb;
    mine[(NV - 2) * 32] = la;
    mine[(NV - 1) * 32] = lb;
    asm volatile("bar.sync 1, %0;" ::"r"(32 * a.warps) : "memory");
    const float* b0 = xs + static_cast<size_t>(rw * NV) * 32 + lane;
    const int kstride = nw * NV * 32;
    float pm[KS][4];  // (m_a, m_b, l_a, l_b) of every partial
#pragma unroll
    for (int k2 = 0; k2 < KS; ++k2)
#pragma unroll
      for (int e = 0; e < 4; ++e) pm[k2][e] = b0[k2 * kstride + (NV - 4 + e) * 32];
    Ma = pm[0][0];
    Mb = pm[0][1];
#pragma unroll
    for (int k2 = 1; k2 < KS; ++k2) {
      Ma = fmaxf(Ma, pm[k2][0]);
      Mb = fmaxf(Mb, pm[k2][1]);
    }
    La = 0.f;
    Lb = 0.f;
#pragma unroll
    for (int k2 = 0; k2 < KS; ++k2) {
      pm[k2][0] = Ma == -INFINITY ? 0.f : ex2(pm[k2][0] - Ma);  // now the partial's weight
      pm[k2][1] = Mb == -INFINITY ? 0.f : ex2(pm[k2][1] - Mb);
      La += pm[k2][2] * pm[k2][0];
      Lb += pm[k2][3] * pm[k2][1];
    }
#pragma unroll
    for (int n = 0; n < NPW; ++n) {
      O[n][0] = O[n][1] = O[n][2] = O[n][3] = 0.f;
#pragma unroll
      for (int k2 = 0; k2 < KS; ++k2) {
        const float* tv = b0 + k2 * kstride + ((n0 + n) * 4) * 32;
        O[n][0] += tv[0] * pm[k2][0];
        O[n][1] += tv[32] * pm[k2][0];
        O[n][2] += tv[64] * pm[k2][1];
        O[n][3] += tv[96] * pm[k2][1];
      }
    }
  } else {
#pragma unroll
    for (int n = 0; n < NPW; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) O[n][e] = o[n][e];
  }
  if (a.kvsplit > 1) {
    // Slots [kvsplit - 1][warps][NPW + 1][32 lanes][4] in the leader: n-tile values, then
    // (m_a, m_b, l_a, l_b).  The leader's own partial stays in registers.
    constexpr int NV2 = (NPW + 1) * 4;
    if (ks2 != 0) {
      const uint32_t rslot = mapa_shared(
          smem_u32(slots) + static_cast<uint32_t>((((ks2 - 1) * a.warps + cwi) * NV2) * 32 + lane * 4) * 4u, 0);
      const uint32_t rbar = mapa_shared(smem_u32(cbar), 0);
      // asynchronous DSMEM stores that complete their bytes on the leader's barrier (no fence, no arrival)
#pragma unroll
      for (int n = 0; n < NPW; ++n)
        st_async_v4(rslot + n * 512u, __float_as_uint(O[n][0]), __float_as_uint(O[n][1]), __float_as_uint(O[n][2]),
                    __float_as_uint(O[n][3]), rbar);
      st_async_v4(rslot + NPW * 512u, __float_as_uint(Ma), __float_as_uint(Mb), __float_as_uint(La),
                  __float_as_uint(Lb), rbar);
      return;
    }
    mbar_wait(cbar, 0);
    const float* b0 = slots + static_cast<size_t>(cwi * NV2) * 32 + lane * 4;
    const int kstride = a.warps * NV2 * 32;
    constexpr int KV = HD == 128 ? 4 : 8;  // cluster-size cap (plan_init clamps kvsplit to it)
    float4 ml[KV];
    ml[0] = make_float4(Ma, Mb, La, Lb);
#pragma unroll
    for (int k2 = 1; k2 < KV; ++k2)
      if (k2 < a.kvsplit) ml[k2] = *reinterpret_cast<const float4*>(b0 + (k2 - 1) * kstride + NPW * 128);
#pragma unroll
    for (int k2 = 1; k2 < KV; ++k2)
      if (k2 < a.kvsplit) {
        Ma = fmaxf(Ma, ml[k2].x);
        Mb = fmaxf(Mb, ml[k2].y);
      }
    La = 0.f;
    Lb = 0.f;
#pragma unroll
    for (int k2 = 0; k2 < KV; ++k2)
      if (k2 < a.kvsplit) {
        ml[k2].x = Ma == -INFINITY ? 0.f : ex2(ml[k2].x - Ma);
        ml[k2].y = Mb == -INFINITY ? 0.f : ex2(ml[k2].y - Mb);
        La += ml[k2].z * ml[k2].x;
        Lb += ml[k2].w * ml[k2].y;
      }
#pragma unroll
    for (int n = 0; n < NPW; ++n) {
      O[n][0] *= ml[0].x;
      O[n][1] *= ml[0].x;
      O[n][2] *= ml[0].y;
      O[n][3] *= ml[0].y;
#pragma unroll
      for (int k2 = 1; k2 < KV; ++k2)
        if (k2 < a.kvsplit) {
          const float4 tv = *reinterpret_cast<const float4*>(b0 + (k2 - 1) * kstride + n * 128);
          O[n][0] += tv.x * ml[k2].x;
          O[n][1] += tv.y * ml[k2].x;
          O[n][2] += tv.z * ml[k2].y;
          O[n][3] += tv.w * ml[k2].y;
        }
    }
  }
  if (lane == 0) trace_max(a.trace, 7);
  // O / l -> bf16 attn[m][head][hd], this warp's n-tiles
  const float ia = La > 0.f ? 1.f / La : 0.f, ib = Lb > 0.f ? 1.f / Lb : 0.f;
  const int ha = kvh * a.Gh + ra % a.Gh, hb = kvh * a.Gh + rb % a.Gh;
  __nv_bfloat16* oa = a.out + (static_cast<size_t>(r * a.T + ta) * a.Hq + ha) * HD;
  __nv_bfloat16* ob = a.out + (static_cast<size_t>(r * a.T + tb) * a.Hq + hb) * HD;
#pragma unroll
  for (int n = 0; n < NPW; ++n) {
    const int col = 8 * (n0 + n) + 2 * (lane & 3);
    if (va) *reinterpret_cast<uint32_t*>(oa + col) = pack2(O[n][0] * ia, O[n][1] * ia);
    if (vb) *reinterpret_cast<uint32_t*>(ob + col) = pack2(O[n][2] * ib, O[n][3] * ib);
  }
  if (lane == 0) trace_max(a.trace, 2);
}

// Instantiations: (hd, in-CTA key splits) for 1, 2 or 4 row warps (hd 128 keeps 2 splits).
#define YGG_AD_KERNELS(X) X(64, 8) X(64, 4) X(64, 2) X(128, 2)

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
  for (auto fn : {attn_dec_kernel<64, 8>, attn_dec_kernel<64, 4>, attn_dec_kernel<64, 2>, attn_dec_kernel<128, 2>}) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "decode attention attribute: %s", cudaGetErrorString(e));
  }
  return YGG_OK;
}

size_t ygg_attn_dec_plan_size(void) { return sizeof(Plan) + 64; }

int ygg_attn_dec_set_l2_prefetch(void* plan, int region, const void* ptr, size_t bytes) {
  Plan* p = const_cast<Plan*>(plan_of(plan));
  YGG_CHECK_ARG(p != nullptr, "invalid decode-attention plan");
  YGG_CHECK_ARG(region == 0 || region == 1, "prefetch region must be 0 or 1");
  YGG_CHECK_ARG(ptr == nullptr || (reinterpret_cast<uintptr_t>(ptr) & 15) == 0, "prefetch region must be 16-byte aligned");
  p->pf_ptr[region] = bytes ? static_cast<const char*>(ptr) : nullptr;
  p->pf_bytes[region] = ptr ? bytes : 0;
  return YGG_OK;
}

int ygg_attn_dec_set_gemv_prefetch(void* plan, const void* gemv_plan) {
  Plan* p = const_cast<Plan*>(plan_of(plan));
  YGG_CHECK_ARG(p != nullptr, "invalid decode-attention plan");
  if (gemv_plan == nullptr) {
    p->tpf_nblk = 0;
    return YGG_OK;
  }
  int nblk = 0, kchunks = 0, stages = 0;
  if (int rc = ygg_gemv_stream_info(gemv_plan, &p->tpf, &nblk, &kchunks, &stages)) return rc;
  // only a GEMV whose CTAs stream one block each leaves a fixed, known tail per block
  p->tpf_first = stages;
  p->tpf_kchunks = kchunks;
  p->tpf_nblk = kchunks > stages ? nblk : 0;
  return YGG_OK;
}

size_t ygg_attn_dec_workspace_size(const void* plan) {
  // Key splits merge inside a thread-block cluster (DSMEM): no global workspace.  Measured (cfg2
  // draft, 4 splits): a global-memory merge (fence + arrival counter + last-CTA merge) cost ~5 us
  // against ~1.7 us through the leader's shared memory.
  (void)plan;
  return 0;
}

int ygg_attn_dec_plan_init(void* plan, const void* q, const void* cache_layer, int B, int T, int Hq, int Hkv, int hd,
                           int S, int kvsplit, int ksplit, int stages) {
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
  if (ksplit > 0 && ksplit * nw <= kMaxWarps && !(hd == 128 && ksplit > 2)) p->ksplit = ksplit;
  p->warps = nw * p->ksplit;
  // Key chunks are split over ksplit warp groups inside a CTA and over a (1, 1, kvsplit) cluster of
  // CTAs; the cluster's partials meet in the leader CTA's shared memory.  Default kvsplit: as many
  // CTAs as fit one wave, at most 4 (measured: cfg2 draft 8 CTAs -> 4 splits best, 8 slower; cfg2
  // verify 32 CTAs -> 4 splits 9.8 us per layer, 2 splits 11.8, 1 split 14.5).
  {
    const int ctas = B * Hkv * p->row_tiles;
    int kv = ctas >= 148 ? 1 : (148 / ctas < 4 ? 148 / ctas : 4);
    if (kvsplit > 0) kv = kvsplit;
    const int kv_cap = hd == 128 ? 4 : 8;
    p->kvsplit = kv < 1 ? 1 : (kv > kv_cap ? kv_cap : kv);
  }
  const size_t stage_bytes = 2 * static_cast<size_t>(kKC) * hd * 2;
  const size_t merge = static_cast<size_t>(p->warps) * (hd / 8 * 4 + 4) * 32 * 4;
  const size_t nv2 = static_cast<size_t>(hd / 8 / p->ksplit) * 4 + 4;
  auto smem_for = [&](int kv, int st) {
    const size_t ring = static_cast<size_t>(st) * stage_bytes;
    const size_t slots = kv > 1 ? static_cast<size_t>(kv - 1) * p->warps * nv2 * 32 * 4 : 0;
    return 1024 + 64 * static_cast<size_t>(hd) * 2 + ((ring > merge ? ring : merge) + 15) / 16 * 16 + slots +
           (2 * static_cast<size_t>(st) + 2) * 8;
  };
  const size_t budget = 220 * 1024 - 1024;  // attribute minus the static shared word
  while (p->kvsplit > 1 && smem_for(p->kvsplit, p->ksplit) > budget) --p->kvsplit;
  // Stages: every stage must always feed the same key-split group (chunk j -> stage j % stages,
  // group j % ksplit), otherwise a group can wait on a stage two phases ahead and the parity wait
  // would pass on a stale phase — so stages is a multiple of ksplit.
  // A cluster member walks ~1/kvsplit of the chunks: a ring of one stage per key-split group keeps
  // the CTA small enough to sit beside the producing GEMV's CTA (its prologue then overlaps it).
  p->stages = p->kvsplit > 1 ? p->ksplit : (hd == 64 ? 8 : 4);
  if (stages > 0) p->stages = stages > kStages ? kStages : stages;
  while (p->stages > p->ksplit && smem_for(p->kvsplit, p->stages) > budget) --p->stages;
  p->stages = (p->stages / p->ksplit) * p->ksplit;
  if (p->stages < p->ksplit) p->stages = p->ksplit;
  {
    const size_t ring = static_cast<size_t>(p->stages) * stage_bytes;
    p->ring_bytes = static_cast<int>(((ring > merge ? ring : merge) + 15) / 16 * 16);
    p->slot_bytes = p->kvsplit > 1 ? static_cast<int>(static_cast<size_t>(p->kvsplit - 1) * p->warps * nv2 * 32 * 4) : 0;
  }
  p->smem = smem_for(p->kvsplit, p->stages);
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
  a.warps = p->warps;
  a.ring_bytes = p->ring_bytes;
  a.slot_bytes = p->slot_bytes;
  (void)workspace;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.blk_start = blk_start;
  a.blk_len = blk_len;
  a.qmask = qmask ? qmask : reinterpret_cast<const uint32_t*>(blk_start);  // never read when mask_words == 0
  a.out = static_cast<__nv_bfloat16*>(out);
  a.trace = trace_next(2);
  for (int rg = 0; rg < 2; ++rg) {
    a.pf_ptr[rg] = p->pf_ptr[rg];
    a.pf_bytes[rg] = p->pf_bytes[rg];
  }
  a.tpf_nblk = p->tpf_nblk;
  a.tpf_kchunks = p->tpf_kchunks;
  a.tpf_first = p->tpf_first;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const dim3 grid(p->Hkv, p->B, p->row_tiles * p->kvsplit), block(32 * (1 + p->warps));
#define YGG_AD_LAUNCH(H, K)                                                                                    \
  if (p->hd == H && p->ksplit == K)                                                                            \
    return launch_pdl_cluster_z(attn_dec_kernel<H, K>, grid, block, p->smem, p->kvsplit, s, p->tq, p->tk, p->tv, \
                                p->tpf_nblk > 0 ? p->tpf : p->tq, a);
  YGG_AD_KERNELS(YGG_AD_LAUNCH)
#undef YGG_AD_LAUNCH
  return ygg_fail(YGG_ERR_VALUE, "decode attention: no kernel for hd %d with %d key splits", p->hd, p->ksplit);
}

}  // extern "C"
