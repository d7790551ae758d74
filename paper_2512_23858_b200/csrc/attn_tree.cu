// K2 tree attention on tcgen05 / TMEM, split over the keys inside a thread-block cluster.
//
// One (C, 1, 1) cluster per (kv head, request, row tile).  A row tile holds up to 32 query tokens of
// one request; its (token, head-in-group) query rows are spread over the four TMEM lane quarters
// (tq tokens x G heads per quarter, so every SM sub-partition's MUFU and issue slots take a share of
// the softmax).  Cluster rank ks takes the 64-key chunks ks, ks + C, ks + 2C, ... of the request's
// visible keys (committed prefix + the tree block), in rounds of NST chunks:
//   warp 8 lane 0  TMA: prefix chunks before griddepcontrol.wait (the cache was committed kernels
//                  ago), Q and the tree-block chunks after it; MMA: S_i = Q K_i^T (M=128, N=64,
//                  K=hd) into TMEM, then O = sum_i P_i V_i (M=128, N=hd, K=64) once P is in smem.
//   softmax warps  (Soft<HD>::warps: 16 at hd 128, 8 at hd 64) one thread per (row, 64/NP-key slice of a
//                  chunk): tcgen05.ld S, ancestor /
//                  prefix mask from the row's tree-mask bits, round max, exp2, bf16 P -> smem
//                  (128B-swizzled, the UMMA A operand).  Long contexts (single-CTA tiles): O accumulates
//                  in TMEM across rounds, rescaled (in TMEM) only when a row's max grows by more than 2^8
//                  over its reference; cluster tiles fold each round's O into an accumulator instead.
// Merge without a combine launch: every CTA pushes each row's unnormalised O and (max, sum) into the
// shared memory of the cluster CTA that owns the row (DSMEM stores + a release arrival on the
// owner's mbarrier); owners merge the C partials in fixed rank order (deterministic) and store bf16.
// Reference semantics: the verify forward the reference prices as latency_at(verifier, w + 1)
// (pkg/src/specsim/simulator.py:211), with the EGT ancestor mask of token_tree.py:205-218.
#include <cudaTypedefs.h>

#include <cmath>
#include <cstring>

#include <cuda_fp16.h>

#include "common.cuh"
#include "host_util.h"

namespace ygg {
namespace at {

constexpr int kKC = 64;                  // keys per chunk
constexpr int kRows = 128;               // UMMA M = TMEM lanes
// Softmax warps: NP per TMEM lane quarter, each taking a 64 / NP-key slice of every chunk (and HD / NP
// output columns in the O rescale / push).  hd 128: 16 warps (4 per quarter), which halves the per-thread
// exp2 / TMEM-load work of a round against 8 (the long-context rounds are softmax-bound); hd 64: 8.
template <int HD>
struct Soft {
  static constexpr int NP = HD == 128 ? 4 : 2;
  static constexpr int warps = 4 * NP;
  static constexpr int threads = 32 * warps;
  static constexpr int KP = kKC / NP;   // keys per thread per chunk (16 or 32)
  static constexpr int CP = HD / NP;    // O columns per thread (32)
  static_assert(CP == 32, "the O rescale / push move 32 TMEM columns per thread");
};
constexpr int kMaxThreads = 32 * 16 + 32;
constexpr uint32_t kMagic = 0x59475454u;     // "YGTT"

struct Plan {
  uint32_t magic;
  int B, T, Hq, Hkv, hd, S, G;
  int tpt, tq, row_tiles, csplit, nst, ring, tcols;
  size_t smem;
  const char* pf_ptr[2];
  size_t pf_bytes[2];
  unsigned long long* dbg;  // per-CTA checkpoint stamps (profiling only) or nullptr
  int late_trigger;         // 1: trigger the dependent launch only at the end (A/B knob)
  alignas(64) CUtensorMap tqm;
  alignas(64) CUtensorMap tk;
  alignas(64) CUtensorMap tv;
};

struct Args {
  int T, Hq, Hkv, S, G, tpt, tq, csplit, mask_words, tcols;
  int lg, lc;  // log2(G), log2(csplit)
  float scale_log2;
  const int32_t* blk_start;
  const int32_t* blk_len;
  const uint32_t* qmask;
  __nv_bfloat16* out;
  unsigned long long* trace;
  const char* pf_ptr[2];
  size_t pf_bytes[2];
  unsigned long long* dbg;
  int late_trigger;
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
YGG_DEV float ex2(float x) {  // 2^x, flush-to-zero (ex2(-inf) = 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
YGG_DEV uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
YGG_DEV void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
YGG_DEV uint32_t pack_h2(float lo, float hi) {
  __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// Issue-only TMEM load of 32 columns (no wait): the caller issues several, then tmem_wait_regs.
YGG_DEV void tmem_ld32_issue(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
YGG_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
YGG_DEV void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
YGG_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// After tmem_wait_ld: ties the 32 registers to a point after the wait, so no use moves above it.
YGG_DEV void regs_after_wait(uint32_t* r) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]),
                 "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]),
                 "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31]));
}
// 32 consecutive f32 TMEM columns of this thread's lane (two x16 loads, one wait).
YGG_DEV void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Visibility bits of 32 keys from absolute key kw for query token tq: committed prefix always; block
// keys by the row's tree-mask bits (causal without a mask); nothing at or past the block's end.
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

// NST chunks per round.  RING == NST: one round of K / V in flight and one S buffer (short contexts: the
// key split over a cluster leaves ~1 round per CTA).  RING == 2 * NST (long contexts, single-CTA tiles):
// the next round's K / V stream in while a round computes and S is double-buffered in TMEM, so round
// r + 1's Q K^T runs during round r's softmax; no cluster merge (the tile's CTA writes O itself).
template <int HD, int NST, int RING>
struct Layout {
  static constexpr bool dbl = RING > NST;
  static_assert(RING == NST || RING == 2 * NST, "ring: one or two rounds of chunks");
  static constexpr int DCH = HD / 64;
  static constexpr uint32_t q_bytes = DCH * kRows * 128;   // [DCH][128 rows][128 B]
  static constexpr uint32_t k_bytes = DCH * kKC * 128;     // one K chunk: [DCH][64 keys][128 B]
  static constexpr uint32_t v_bytes = HD * 128;            // one V^T chunk: [hd rows][64 keys x 2 B]
  static constexpr uint32_t p_bytes = kRows * 128;         // one P chunk: [128 rows][64 keys x 2 B]
  static constexpr uint32_t off_k = q_bytes;
  static constexpr uint32_t off_v = off_k + RING * k_bytes;
  static constexpr uint32_t off_p = off_v + RING * v_bytes;
  // Merge receive rows [C][128 / C][RS] of the row-normalised partial O in f16 (|O / l| <= max |V|);
  // RS = hd + 8 halves keeps row-parallel 16-byte accesses conflict-free.  Dedicated (not aliased
  // onto the ring), so a rank pushes as soon as its own rows are done.
  static constexpr int RS = HD + 8;
  static constexpr uint32_t off_recv = off_p + NST * p_bytes;
  static constexpr uint32_t off_ml = off_recv + (dbl ? 0 : kRows * RS * 2);  // f32 [C][128 / C][2] (max, sum)
  // f32 [2][NP][128] slice maxima (by round parity: a thread may start round r + 1 while a slower one of
  // its quarter still reads round r's), [NP][128] sums
  static constexpr uint32_t off_red = off_ml + kRows * 8;
  static constexpr uint32_t off_bar = off_red + 3 * Soft<HD>::NP * kRows * 4;  // k_full[RING], v_full[RING], q, s[2], p, o, recv
  static constexpr uint32_t bytes = off_bar + (2 * RING + 6) * 8 + 16;
  static constexpr int s_cols = (dbl ? 2 : 1) * NST * kKC;  // S of one round (two buffers when dbl)
  // + O: accumulated across rounds in TMEM (dbl), or a round's O + the accumulator it is folded into
  static constexpr int o_cols = (dbl ? 1 : 2) * HD;
  static constexpr int tcols = (s_cols + o_cols) <= 256 ? 256 : 512;
  static_assert(s_cols + o_cols <= 512, "TMEM budget");
};

template <int HD, int NST, int RING>
__global__ void __launch_bounds__(Soft<HD>::threads + 32, 1)
    attn_tree_kernel(const __grid_constant__ CUtensorMap tqm, const __grid_constant__ CUtensorMap tk,
                     const __grid_constant__ CUtensorMap tv, Args a) {
  using Ly = Layout<HD, NST, RING>;
  constexpr int kSoftWarps = Soft<HD>::warps, kSoftThreads = Soft<HD>::threads;
  constexpr int NP = Soft<HD>::NP, KP = Soft<HD>::KP, CP = Soft<HD>::CP;
  constexpr uint32_t kpmask = KP == 32 ? 0xffffffffu : ((1u << KP) - 1u);
  constexpr bool kHold = NST * KP <= 32;  // a round's scores stay in registers between the two passes
  constexpr int DCH = Ly::DCH;
  constexpr int RS = Ly::RS;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sq = base;
  unsigned char* sk = base + Ly::off_k;
  unsigned char* sv = base + Ly::off_v;
  unsigned char* sp = base + Ly::off_p;
  __half* recv_o = reinterpret_cast<__half*>(base + Ly::off_recv);
  float* recv_ml = reinterpret_cast<float*>(base + Ly::off_ml);
  float* red = reinterpret_cast<float*>(base + Ly::off_red);
  // K and V of a ring stage complete on separate barriers: the next round's K chunks stream into the
  // K slots as soon as this round's S = Q K^T is done (during the softmax), its V chunks as soon as
  // this round's P V is done, so the round-to-round chain no longer waits on a whole load latency.
  uint64_t* k_full = reinterpret_cast<uint64_t*>(base + Ly::off_bar);
  uint64_t* v_full = k_full + RING;
  uint64_t* q_full = v_full + RING;
  uint64_t* s_full = q_full + 1;  // [2]: one per S buffer (the second only when Ly::dbl)
  uint64_t* p_full = s_full + 2;
  uint64_t* o_full = p_full + 1;
  uint64_t* recv_bar = o_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recv_bar + 1);
  unsigned long long* dbg =
      a.dbg ? a.dbg + 16 * ((static_cast<size_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) : nullptr;
#define AT_STAMP(k) \
  if (dbg) dbg[k] = gtimer()
  const int C = a.csplit;
  const int ks = blockIdx.x, rt = blockIdx.y;
  const int kvh = blockIdx.z % a.Hkv, r = blockIdx.z / a.Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lanes_per = kRows / C;  // TMEM lanes (query rows) each cluster rank owns in the merge
  const int t0 = rt * a.tpt;
  const int tcnt = min(a.tpt, a.T - t0);
  // query row of TMEM lane lr: quarter lr / 32 holds tq tokens x G heads
  auto lane_valid = [&](int lr) {
    const int l32 = lr & 31;
    return l32 < a.tq * a.G && (lr >> 5) * a.tq + (l32 >> a.lg) < tcnt;
  };
  if (threadIdx.x == 0) {
    AT_STAMP(0);
    for (int s = 0; s < RING; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&v_full[s], 1);
    }
    mbar_init(q_full, 1);
    mbar_init(&s_full[0], 1);
    mbar_init(&s_full[1], 1);
    mbar_init(p_full, kSoftThreads);
    mbar_init(o_full, 1);
    // The merge: every rank's partial of each valid row this rank owns arrives as st.async bytes.
    int owned = 0;
    for (int ll = 0; ll < lanes_per; ++ll) owned += lane_valid(ks * lanes_per + ll) ? 1 : 0;
    mbar_init(recv_bar, 1);
    mbar_arrive_expect_tx(recv_bar, static_cast<uint32_t>(C * owned * (HD * 2 + 8)));
    fence_barrier_init();
    trace_min(a.trace, 0);
  }
  if (warp == kSoftWarps) tmem_alloc(tmem_slot, Ly::tcols);
  tc_fence_before();
  if (C > 1) cluster_sync();  // remote arrivals need every CTA's barriers initialised
  else __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) AT_STAMP(1);
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + Ly::s_cols, tAcc = Ly::dbl ? tO : tO + HD;
  // Block bounds were written at least two kernels back (the kernel just before this one triggers
  // its dependents only after its own dependency wait): read them before the wait.
  const int bs = __ldg(a.blk_start + r), bl = __ldg(a.blk_len + r);
  // causal block (no tree mask, e.g. a prefill chunk): this tile's last token sees block keys <= its own
  const int nkeys = bs + (a.mask_words == 0 ? min(bl, t0 + tcnt) : bl);
  const int nch = (nkeys + kKC - 1) / kKC;
  const int n_my = nch > ks ? (nch - ks + C - 1) >> a.lc : 0;
  const int rounds = (n_my + NST - 1) / NST;
  // this thread's query row (softmax warps): TMEM lane quarter q holds tq tokens x G heads
  const int q = warp & 3, part = warp >> 2;  // TMEM lane quarter, key / column slice (softmax warps)
  const int row = q * 32 + lane;
  const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;  // TMEM lane quarter of this warp
  const int tl = q * a.tq + (lane >> a.lg);             // token within the tile
  const bool valid = warp < kSoftWarps && lane < a.tq * a.G && tl < tcnt;
  float M = -INFINITY, l = 0.f;

  if (warp == kSoftWarps) {
    if (lane == 0) {
      const int kv_row0 = (r * 2 * a.Hkv + kvh) * a.S;        // K rows of this head
      const int vt_row0 = ((r * 2 + 1) * a.Hkv + kvh) * HD;   // V^T rows of this head
      auto load_k = [&](int j) {
        const int c = ks + j * C, st = j % RING;
        mbar_arrive_expect_tx(&k_full[st], Ly::k_bytes);
#pragma unroll
        for (int dc = 0; dc < DCH; ++dc)
          tma2(sk + st * Ly::k_bytes + dc * (kKC * 128), &tk, &k_full[st], dc * 64, kv_row0 + c * kKC);
      };
      auto load_v = [&](int j) {
        const int c = ks + j * C, st = j % RING;
        mbar_arrive_expect_tx(&v_full[st], Ly::v_bytes);
        tma2(sv + st * Ly::v_bytes, &tv, &v_full[st], c * kKC, vt_row0);
      };
      auto load = [&](int j) {
        load_k(j);
        load_v(j);
      };
      int issued = 0;
      // the committed prefix's chunks of the first round stream in before the dependency wait
      while (issued < n_my && issued < RING && (ks + issued * C + 1) * kKC <= bs) load(issued++);
      pdl_wait();
      if (!a.late_trigger) pdl_launch_dependents();
      trace_min(a.trace, 1);
      AT_STAMP(2);
      if (dbg) dbg[11] = rounds;
      const int nq = min(4, (tcnt + a.tq - 1) / a.tq);  // lane quarters holding tokens of this tile
      mbar_arrive_expect_tx(q_full, static_cast<uint32_t>(DCH * nq * 128 * a.G * a.tq));
      for (int dc = 0; dc < DCH; ++dc)
        for (int qq = 0; qq < nq; ++qq)
          tma3(sq + dc * (kRows * 128) + qq * (32 * 128), &tqm, q_full, dc * 64, kvh * a.G, r * a.T + t0 + qq * a.tq);
      while (issued < n_my && issued < RING) load(issued++);
      const uint32_t id_s = umma_idesc_bf16(kRows, kKC), id_o = umma_idesc_bf16(kRows, HD);
      mbar_wait(q_full, 0);  // always: no CTA leaves with a TMA write into its shared memory in flight
      trace_max(a.trace, 5);
      AT_STAMP(3);
      // S = Q K^T of round rr into S buffer rr & 1 (buffer 0 only unless Ly::dbl), committed on s_full[buf]
      auto s_mma = [&](int rr) {
        const int a0 = rr * NST, a1 = min(n_my, a0 + NST);
        const uint32_t sb = tS + (Ly::dbl ? (rr & 1) * NST * kKC : 0);
        for (int j = a0; j < a1; ++j) {
          const int st = j % RING;
          mbar_wait(&k_full[st], (j / RING) & 1);
          tc_fence_after();
          if (j == 0) AT_STAMP(4);
          if (j == a1 - 1 && rr == 0) AT_STAMP(5);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint64_t ad = umma_desc_sw128(smem_u32(sq + (kk / 4) * (kRows * 128)) + (kk % 4) * 32);
            const uint64_t bd = umma_desc_sw128(smem_u32(sk + st * Ly::k_bytes + (kk / 4) * (kKC * 128)) + (kk % 4) * 32);
            umma_bf16(sb + (j - a0) * kKC, ad, bd, id_s, kk > 0 ? 1u : 0u);
          }
        }
        umma_commit(&s_full[Ly::dbl ? (rr & 1) : 0]);
      };
      if (rounds > 0) s_mma(0);
      for (int rd = 0; rd < rounds; ++rd) {
        const int j0 = rd * NST, j1 = min(n_my, j0 + NST);
        // this round's K slots are free once its S MMAs completed: refill them one ring ahead.  dbl: S(rd)
        // was issued a round ago, so the refill goes out BEFORE waiting for round rd + 1's K (issued
        // after it, the refill would keep only one round of K loads in flight: ncu showed the softmax
        // warps ~30% stalled on S at cfg4)
        const int jn = Ly::dbl ? min(n_my, j1 + RING) : min(n_my, j1 + NST);
        if (Ly::dbl && rd + 1 < rounds) {
          if (j0 + RING < jn) {
            mbar_wait(&s_full[rd & 1], (rd >> 1) & 1);
            for (int j = j0 + RING; j < jn; ++j) load_k(j);
          }
          // the other S buffer was last read by round rd - 1's softmax, which this warp saw finish (p_full)
          s_mma(rd + 1);
        }
        if (rd == 0) {
          // This CTA's own loads have landed: now the kernel barely touches HBM, so pull its share of a
          // later weight stream into L2 (issued earlier, the prefetch would queue ahead of the chunk loads).
          for (int rg = 0; rg < 2; ++rg) {
            if (!a.pf_ptr[rg]) continue;
            const size_t ncta = static_cast<size_t>(gridDim.x) * gridDim.y * gridDim.z;
            const size_t cta = (static_cast<size_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
            const size_t per = ((a.pf_bytes[rg] / ncta) + 255) & ~static_cast<size_t>(255);
            const size_t b0 = cta * per, b1 = b0 + per < a.pf_bytes[rg] ? b0 + per : a.pf_bytes[rg];
            for (size_t o2 = b0; o2 < b1; o2 += 65536) {
              const uint32_t n = static_cast<uint32_t>(b1 - o2 < 65536 ? ((b1 - o2) & ~static_cast<size_t>(15)) : 65536);
              if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.pf_ptr[rg] + o2), "r"(n) : "memory");
            }
          }
        }
        if (!Ly::dbl && rd + 1 < rounds) {
          mbar_wait(&s_full[0], rd & 1);
          for (int j = j1; j < jn; ++j) load_k(j);
        }
        mbar_wait(p_full, rd & 1);
        tc_fence_after();
        trace_max(a.trace, 6);
        if (rd == 0) AT_STAMP(6);
        for (int j = j0; j < j1; ++j) {
          const int st = j % RING;
          mbar_wait(&v_full[st], (j / RING) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kKC / 16; ++kk) {
            const uint64_t ad = umma_desc_sw128(smem_u32(sp + (j - j0) * Ly::p_bytes) + kk * 32);
            const uint64_t bd = umma_desc_sw128(smem_u32(sv + st * Ly::v_bytes) + kk * 32);
            umma_bf16(tO, ad, bd, id_o, ((Ly::dbl && rd > 0) || j > j0 || kk > 0) ? 1u : 0u);
          }
        }
        umma_commit(o_full);
        if (rd + 1 < rounds) {  // ... and its V slots once its P V MMAs completed
          mbar_wait(o_full, rd & 1);
          for (int j = Ly::dbl ? j0 + RING : j1; j < jn; ++j) load_v(j);
          // non-dbl: round rd + 1's S (one S buffer: after round rd's softmax, i.e. after p_full above)
          if (!Ly::dbl) s_mma(rd + 1);
        }
      }
      // the last round's MMAs complete before the softmax warps pass o_full, i.e. before the
      // cluster barrier below: the ring is free for the merge everywhere after it
    } else {
      pdl_wait();
      if (!a.late_trigger) pdl_launch_dependents();
    }
  } else {
    // ===== softmax warps: thread = (TMEM lane row, KP-key slice of every chunk) =====
    pdl_wait();
    if (!a.late_trigger) pdl_launch_dependents();
    const int tok = rt * a.tpt + (valid ? tl : 0);
    const uint32_t* mrow = a.qmask + static_cast<size_t>(r * a.T + tok) * (a.mask_words ? a.mask_words : 1);
    const float sl = a.scale_log2;
    for (int rd = 0; rd < rounds; ++rd) {
      const int j0 = rd * NST, nj = min(n_my, j0 + NST) - j0;
      uint32_t vis[NST];
#pragma unroll
      for (int i = 0; i < NST; ++i) {
        const int kw = (ks + (j0 + i) * C) * kKC + part * KP;
        // rows past the tile (never pushed) take the prefix's all-visible word too, so fully visible
        // chunks stay on the warp-uniform fast path
        vis[i] = i >= nj ? 0u
                         : (kw + KP <= bs ? kpmask : (valid ? vis_word(kw, bs, bl, tok, a.mask_words, mrow) & kpmask : 0u));
      }
      mbar_wait(&s_full[Ly::dbl ? (rd & 1) : 0], Ly::dbl ? (rd >> 1) & 1 : rd & 1);
      tc_fence_after();
      if (threadIdx.x == 0 && rd == 0) AT_STAMP(12);
      if constexpr (Ly::dbl) {
      // ---- long contexts: O accumulates in TMEM with the lazy rescale
      const uint32_t tSr = tS + (Ly::dbl ? (rd & 1) * NST * kKC : 0);  // this round's S buffer
      // pass 1: the row max over this thread's visible scores (S kept in registers); pass 2 (after the
      // column slices exchange their maxima): P = 2^(s - ref) into the UMMA A operand
      bool full[NST];  // warp-uniform: every row of the warp sees all 32 keys (committed prefix)
#pragma unroll
      for (int i = 0; i < NST; ++i) full[i] = __all_sync(0xffffffffu, vis[i] == kpmask);
      float v[NST][KP];
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < NST; ++i) {
        if (i < nj) {
          if constexpr (KP == 32) tmem_ld32(tSr + lane_base + i * kKC + part * KP, v[i]);
          else tmem_ld16(tSr + lane_base + i * kKC + part * KP, v[i]);
          if (full[i]) {
#pragma unroll
            for (int j = 0; j < KP; ++j) mx = fmaxf(mx, v[i][j]);
          } else {
#pragma unroll
            for (int j = 0; j < KP; ++j)
              if ((vis[i] >> j) & 1u) mx = fmaxf(mx, v[i][j]);
          }
        }
      }
      float* redm = red + (rd & 1) * NP * kRows;
      redm[part * kRows + row] = mx;
      asm volatile("bar.sync %0, %1;" ::"r"(2 + q), "r"(32 * NP) : "memory");  // the NP warps of this quarter
      mx = redm[row];
#pragma unroll
      for (int pp = 1; pp < NP; ++pp) mx = fmaxf(mx, redm[pp * kRows + row]);
      // Lazy rescale: the reference max moves only when the row max grows by more than 2^8 (P <= 256 in
      // bf16 / f32 is exact enough and cannot overflow), so most rounds leave the TMEM accumulator alone.
      // The decision is the row's own (its NP threads compute the same values): rows stay independent.
      const float mnew = fmaxf(M, mx * sl);  // log2 units (scale > 0 commutes with the max)
      float alpha = 1.f;
      if (mnew > M + 8.f) {
        alpha = ex2(M - mnew);  // 0 when M = -inf
        M = mnew;
      }
      const float ref = M == -INFINITY ? 0.f : M;
      // The previous round's P V has read its P slots and accumulated: P and the accumulator are free.
      // Short rounds (NST x KP <= 32 scores per thread) keep the exponentials in registers and wait only
      // before the P stores; longer ones wait first and reload S chunk by chunk (register budget).
      auto prev_pv_done = [&]() {
        if (rd == 0) return;
        mbar_wait(o_full, (rd - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.f)) {  // warp-collective TMEM access; other rows scale by 1
          uint32_t ab[32];
          tmem_ld32_issue(tAcc + lane_base + part * CP, ab);
          tmem_wait_ld();
          regs_after_wait(ab);
#pragma unroll
          for (int c = 0; c < 32; ++c) ab[c] = __float_as_uint(__uint_as_float(ab[c]) * alpha);
          tmem_st32(tAcc + lane_base + part * CP, ab);
          tmem_wait_st();
        }
      };
      auto store_p = [&](int i) {
        const uint32_t rb = smem_u32(sp + i * Ly::p_bytes + row * 128);
#pragma unroll
        for (int u = 0; u < KP / 8; ++u)
          sts128(rb + (((part * (KP / 8) + u) ^ (row & 7)) << 4), pack2(v[i][8 * u], v[i][8 * u + 1]),
                 pack2(v[i][8 * u + 2], v[i][8 * u + 3]), pack2(v[i][8 * u + 4], v[i][8 * u + 5]),
                 pack2(v[i][8 * u + 6], v[i][8 * u + 7]));
      };
      if constexpr (!kHold) prev_pv_done();
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < NST; ++i) {
        if (i < nj) {
          if constexpr (!kHold) {
            if constexpr (KP == 32) tmem_ld32(tSr + lane_base + i * kKC + part * KP, v[i]);
            else tmem_ld16(tSr + lane_base + i * kKC + part * KP, v[i]);
          }
          if (full[i]) {
#pragma unroll
            for (int j = 0; j < KP; ++j) {
              v[i][j] = ex2(fmaf(v[i][j], sl, -ref));
              sum += v[i][j];
            }
          } else {
#pragma unroll
            for (int j = 0; j < KP; ++j) {
              v[i][j] = ((vis[i] >> j) & 1u) ? ex2(fmaf(v[i][j], sl, -ref)) : 0.f;
              sum += v[i][j];
            }
          }
          if constexpr (!kHold) store_p(i);
        }
      }
      if constexpr (kHold) {
        prev_pv_done();
#pragma unroll
        for (int i = 0; i < NST; ++i)
          if (i < nj) store_p(i);
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(p_full);
      l = l * alpha + sum;
      } else {
      // ---- cluster tiles (~one round per CTA): O of each round folded into the accumulator columns
      // (measured faster here than the TMEM accumulation: cfg2 verify 3.450 vs 3.456 ms)
      const uint32_t tSr = tS + (Ly::dbl ? (rd & 1) * NST * kKC : 0);  // this round's S buffer
      // pass 1: the row max over this thread's visible scores; pass 2 (after the two column halves
      // exchange their maxima): P = 2^(s - max) into the UMMA A operand
      bool full[NST];  // warp-uniform: every row of the warp sees all 32 keys (committed prefix)
#pragma unroll
      for (int i = 0; i < NST; ++i) full[i] = __all_sync(0xffffffffu, vis[i] == kpmask);
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < NST; ++i) {
        if (i < nj) {
          float v[KP];
          if constexpr (KP == 32) tmem_ld32(tSr + lane_base + i * kKC + part * KP, v);
          else tmem_ld16(tSr + lane_base + i * kKC + part * KP, v);
          if (full[i]) {
#pragma unroll
            for (int j = 0; j < KP; ++j) mx = fmaxf(mx, v[j]);
          } else {
#pragma unroll
            for (int j = 0; j < KP; ++j)
              if ((vis[i] >> j) & 1u) mx = fmaxf(mx, v[j]);
          }
        }
      }
      red[part * kRows + row] = mx;
      asm volatile("bar.sync %0, %1;" ::"r"(2 + q), "r"(32 * NP) : "memory");  // the NP warps of this quarter
      mx = red[row];
#pragma unroll
      for (int pp = 1; pp < NP; ++pp) mx = fmaxf(mx, red[pp * kRows + row]);
      const float mnew = fmaxf(M, mx * sl);  // log2 units (scale > 0 commutes with the max)
      const float ref = mnew == -INFINITY ? 0.f : mnew;
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < NST; ++i) {
        if (i < nj) {
          float v[KP];
          if constexpr (KP == 32) tmem_ld32(tSr + lane_base + i * kKC + part * KP, v);
          else tmem_ld16(tSr + lane_base + i * kKC + part * KP, v);
          if (full[i]) {
#pragma unroll
            for (int j = 0; j < KP; ++j) {
              const float x = fmaf(v[j], sl, -ref);
              v[j] = ex2(x);
              sum += v[j];
            }
          } else {
#pragma unroll
            for (int j = 0; j < KP; ++j) {
              const float x = fmaf(v[j], sl, -ref);
              v[j] = ((vis[i] >> j) & 1u) ? ex2(x) : 0.f;
              sum += v[j];
            }
          }
          const uint32_t rb = smem_u32(sp + i * Ly::p_bytes + row * 128);
#pragma unroll
          for (int u = 0; u < KP / 8; ++u)
            sts128(rb + (((part * (KP / 8) + u) ^ (row & 7)) << 4), pack2(v[8 * u], v[8 * u + 1]),
                   pack2(v[8 * u + 2], v[8 * u + 3]), pack2(v[8 * u + 4], v[8 * u + 5]),
                   pack2(v[8 * u + 6], v[8 * u + 7]));
        }
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(p_full);
      const float alpha = ex2(M - ref);  // 0 on the first round (M = -inf)
      l = l * alpha + sum;
      M = mnew;
      if (rounds > 1) {
        // fold this round's O into the accumulator columns (acc = acc * alpha + O_r) before the next
        // round's P V overwrites tO (its MMA waits for p_full, which this thread arrives on only after)
        mbar_wait(o_full, rd & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < CP; c += 32) {
          uint32_t ob[32], ab[32];
          tmem_ld32_issue(tO + lane_base + part * CP + c, ob);
          if (rd > 0) tmem_ld32_issue(tAcc + lane_base + part * CP + c, ab);
          tmem_wait_ld();
          regs_after_wait(ob);
          if (rd > 0) {
            regs_after_wait(ab);
#pragma unroll
            for (int i = 0; i < 32; ++i) ob[i] = __float_as_uint(fmaf(__uint_as_float(ab[i]), alpha, __uint_as_float(ob[i])));
          }
          tmem_st32(tAcc + lane_base + part * CP + c, ob);
        }
        tmem_wait_st();
      }
      }
    }
    if (threadIdx.x == 0) trace_max(a.trace, 3);
    if (threadIdx.x == 0) AT_STAMP(7);
  }
  // "Every TMEM read of the CTA is done": named barrier 1 — the softmax warps arrive (bar.arrive, they
  // need not wait) once their last TMEM read is done, the TMA / MMA warp syncs on it before the dealloc.
  auto tmem_done = [&]() {
    __syncwarp();  // reconverge the warp (its threads may come from divergent branches)
    asm volatile("bar.arrive 1, %0;" ::"r"(kSoftThreads + 32) : "memory");
  };
  if (warp == kSoftWarps) {  // the TMA / MMA warp: release TMEM once every TMEM read of the CTA is done
    tc_fence_before();
    asm volatile("bar.sync 1, %0;" ::"r"(kSoftThreads + 32) : "memory");
    tc_fence_after();
    tmem_dealloc(tmem, Ly::tcols);
    if (a.late_trigger) pdl_launch_dependents();
    return;
  }
  // ===== push this row's partial to the rank owning the row: O / l in f16 and (max, l) =====
  float* red_l = red + 2 * NP * kRows;
  red_l[part * kRows + row] = l;
  asm volatile("bar.sync %0, %1;" ::"r"(2 + q), "r"(32 * NP) : "memory");
  float ltot = red_l[row];
#pragma unroll
  for (int pp = 1; pp < NP; ++pp) ltot += red_l[pp * kRows + row];
  const float inv = ltot > 0.f ? 1.f / ltot : 0.f;
  if (Ly::dbl || C == 1) {
    // single-CTA tile (no key split): O / l straight from TMEM to the bf16 output, no merge (st.async
    // needs a cluster of at least two CTAs)
    // the last round's P V (completions are in order: earlier phases are done); without dbl, rounds > 1
    // were waited for by the fold
    if (Ly::dbl ? rounds > 0 : rounds == 1) {
      mbar_wait(o_full, (rounds - 1) & 1);
      tc_fence_after();
    }
    uint32_t ob[32];
    if (rounds > 0) {
      tmem_ld32_issue((Ly::dbl || rounds > 1 ? tAcc : tO) + lane_base + part * CP, ob);
      tmem_wait_ld();
      regs_after_wait(ob);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) ob[i] = 0u;
    }
    if (valid) {
      const int l32 = row & 31;
      const int tok = t0 + (row >> 5) * a.tq + (l32 >> a.lg);
      const int head = kvh * a.G + (l32 & (a.G - 1));
      __nv_bfloat16* dst = a.out + (static_cast<size_t>(r * a.T + tok) * a.Hq + head) * HD + part * CP;
#pragma unroll
      for (int u = 0; u < 32; u += 8) {
        uint4 ov;
        ov.x = pack2(__uint_as_float(ob[u]) * inv, __uint_as_float(ob[u + 1]) * inv);
        ov.y = pack2(__uint_as_float(ob[u + 2]) * inv, __uint_as_float(ob[u + 3]) * inv);
        ov.z = pack2(__uint_as_float(ob[u + 4]) * inv, __uint_as_float(ob[u + 5]) * inv);
        ov.w = pack2(__uint_as_float(ob[u + 6]) * inv, __uint_as_float(ob[u + 7]) * inv);
        *reinterpret_cast<uint4*>(dst + u) = ov;
      }
    }
    tc_fence_before();
    tmem_done();  // pairs with the TMA / MMA warp's: every TMEM read is done
    if (threadIdx.x == 0) {
      trace_max(a.trace, 2);
      AT_STAMP(10);
    }
    if (a.late_trigger) pdl_launch_dependents();
    return;
  }
  const int lsh = 7 - a.lc;  // log2(lanes_per)
  const int d = row >> lsh, ll = row & (lanes_per - 1);
  const uint32_t rbar = mapa_shared(smem_u32(recv_bar), d);
  const uint32_t ro = mapa_shared(smem_u32(recv_o + (static_cast<size_t>(ks * lanes_per + ll) * RS + part * CP)), d);
  if (Ly::dbl ? rounds > 0 : rounds == 1) {
    mbar_wait(o_full, (rounds - 1) & 1);
    tc_fence_after();
  }
  const uint32_t tsrc = (Ly::dbl || rounds > 1 ? tAcc : tO) + lane_base + part * CP;
#pragma unroll
  for (int c = 0; c < CP; c += 32) {
    uint32_t ob[32];
    if (rounds > 0) {
      tmem_ld32_issue(tsrc + c, ob);
      tmem_wait_ld();
      regs_after_wait(ob);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) ob[i] = 0u;
    }
    if (valid) {
#pragma unroll
      for (int u = 0; u < 32; u += 8) {
#define F(k) (__uint_as_float(ob[u + (k)]) * inv)
        st_async_v4(ro + (c + u) * 2, pack_h2(F(0), F(1)), pack_h2(F(2), F(3)), pack_h2(F(4), F(5)), pack_h2(F(6), F(7)), rbar);
#undef F
      }
    }
  }
  if (valid && part == 0)
    st_async_v2(mapa_shared(smem_u32(recv_ml + static_cast<size_t>(ks * lanes_per + ll) * 2), d), __float_as_uint(M),
                __float_as_uint(ltot), rbar);
  tc_fence_before();
  tmem_done();  // pairs with the TMA / MMA warp's: every TMEM read is done
  if (threadIdx.x == 0) AT_STAMP(8);
  // ===== owner: rows [ks * lanes_per, (ks + 1) * lanes_per): kSoftThreads / lanes_per threads per row, 8-column
  // units, the C partials combined in fixed rank order
  mbar_wait(recv_bar, 0);
  if (threadIdx.x == 0) {
    trace_max(a.trace, 4);
    AT_STAMP(9);
  }
  const int tsh = (NP == 4 ? 9 : 8) - lsh;    // log2(threads per row)
  const int ll2 = threadIdx.x >> tsh;         // owned row
  const int upart = threadIdx.x & ((1 << tsh) - 1);
  const int units = (HD / 8) >> tsh;          // 8-column units per thread
  const int lr = ks * lanes_per + ll2;        // TMEM lane of the row
  if (lane_valid(lr)) {
    const int l32 = lr & 31;
    float w[4];
    float Mg = -INFINITY;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c < C) Mg = fmaxf(Mg, recv_ml[(c * lanes_per + ll2) * 2]);
    float L = 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      w[c] = 0.f;
      if (c < C) {
        const float* ml = recv_ml + (c * lanes_per + ll2) * 2;
        w[c] = Mg == -INFINITY ? 0.f : ex2(ml[0] - Mg) * ml[1];
        L += w[c];
      }
    }
    const float il = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) w[c] *= il;
    const int tok = t0 + (lr >> 5) * a.tq + (l32 >> a.lg);
    const int head = kvh * a.G + (l32 & (a.G - 1));
    __nv_bfloat16* dst = a.out + (static_cast<size_t>(r * a.T + tok) * a.Hq + head) * HD;
    for (int u = 0; u < units; ++u) {
      const int col = (upart * units + u) * 8;
      float acc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c < C) {
          const uint4 raw = *reinterpret_cast<const uint4*>(recv_o + static_cast<size_t>(c * lanes_per + ll2) * RS + col);
          const uint32_t wv[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 x = __half22float2(*reinterpret_cast<const __half2*>(&wv[i]));
            acc[2 * i] = fmaf(w[c], x.x, acc[2 * i]);
            acc[2 * i + 1] = fmaf(w[c], x.y, acc[2 * i + 1]);
          }
        }
      }
      uint4 ov;
      ov.x = pack2(acc[0], acc[1]);
      ov.y = pack2(acc[2], acc[3]);
      ov.z = pack2(acc[4], acc[5]);
      ov.w = pack2(acc[6], acc[7]);
      *reinterpret_cast<uint4*>(dst + col) = ov;
    }
  }
  if (threadIdx.x == 0) {
    trace_max(a.trace, 2);
    AT_STAMP(10);
  }
  if (a.late_trigger) pdl_launch_dependents();
#undef AT_STAMP
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
static int enc(CUtensorMap* m, int rank, const void* p, const cuuint64_t* dims, const cuuint64_t* str,
               const cuuint32_t* box) {
  auto e = encoder();
  if (!e) return ygg_fail(YGG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t es[3] = {1, 1, 1};
  CUresult rc = e(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(p), dims, str, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) return ygg_fail(YGG_ERR_CUDA, "tree attention tensor map failed (%d)", static_cast<int>(rc));
  return YGG_OK;
}
static const Plan* plan_of(const void* p) {
  const Plan* q = reinterpret_cast<const Plan*>((reinterpret_cast<uintptr_t>(p) + 63) & ~uintptr_t(63));
  return (p && q->magic == kMagic) ? q : nullptr;
}

// Instantiations: (hd, chunks per round).
#define YGG_AT_KERNELS(X) X(64, 4, 4) X(128, 3, 3) X(128, 2, 4)

}  // namespace at
}  // namespace ygg

using namespace ygg;
using namespace ygg::at;

extern "C" {

int ygg_prepare_attn_tree(void) {
#define YGG_AT_ATTR(H, N, R)                                                                                \
  {                                                                                                         \
    cudaError_t e = cudaFuncSetAttribute(attn_tree_kernel<H, N, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                         static_cast<int>(Layout<H, N, R>::bytes + 1024));                  \
    if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "tree attention attribute: %s", cudaGetErrorString(e)); \
    e = cudaFuncSetAttribute(attn_tree_kernel<H, N, R>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);   \
    if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "tree attention cluster attribute: %s", cudaGetErrorString(e)); \
  }
  YGG_AT_KERNELS(YGG_AT_ATTR)
#undef YGG_AT_ATTR
  return YGG_OK;
}

size_t ygg_attn_tree_plan_size(void) { return sizeof(Plan) + 64; }

int ygg_attn_tree_plan_init(void* plan, const void* q, const void* cache_layer, int B, int T, int Hq, int Hkv, int hd,
                            int S, int csplit, int row_tiles) {
  YGG_CHECK_ARG(plan && q && cache_layer, "null pointer");
  YGG_CHECK_ARG(hd == 64 || hd == 128, "head dim must be 64 or 128");
  YGG_CHECK_ARG(Hkv >= 1 && Hq % Hkv == 0, "bad head grouping");
  const int G = Hq / Hkv;
  YGG_CHECK_ARG(G <= 32 && (G & (G - 1)) == 0, "tree attention: a power-of-two group of at most 32 query heads per kv head");
  YGG_CHECK_ARG(B >= 1 && T >= 1, "empty pass");
  YGG_CHECK_ARG(S % 64 == 0, "cache capacity must be a multiple of 64");
  YGG_CHECK_ARG(csplit == 0 || csplit == 1 || csplit == 2 || csplit == 4, "key split must be 1, 2 or 4 CTAs");
  Plan* p = reinterpret_cast<Plan*>((reinterpret_cast<uintptr_t>(plan) + 63) & ~uintptr_t(63));
  std::memset(p, 0, sizeof(Plan));
  p->magic = kMagic;
  p->B = B;
  p->T = T;
  p->Hq = Hq;
  p->Hkv = Hkv;
  p->hd = hd;
  p->S = S;
  p->G = G;
  // Row tiles: a lane quarter holds tq tokens x G heads (<= 32 rows), a tile four quarters.
  const int tq_max = 32 / G;
  int rt = (T + 4 * tq_max - 1) / (4 * tq_max);
  if (row_tiles > 0) {
    YGG_CHECK_ARG(row_tiles >= rt, "too few row tiles for 128 query rows each");
    rt = row_tiles;
  }
  p->tpt = (T + rt - 1) / rt;
  p->row_tiles = (T + p->tpt - 1) / p->tpt;
  p->tq = (p->tpt + 3) / 4;
  // Key split: the largest cluster (<= 4: clusters of 8 CTAs with ~180 KB of shared memory each do
  // not all fit one wave on B200's GPCs) that keeps the grid in one wave.
  int cs = csplit;
  if (cs == 0) {
    const int units = B * Hkv * p->row_tiles;
    cs = 4;
    while (cs > 1 && units * cs > 148) cs /= 2;
  }
  p->csplit = cs;
  // Dependent launch triggered at each CTA's end: the next GEMM's early CTAs otherwise slow this
  // kernel's softmax by ~1.8 us per cfg2 verify layer for no gain of their own (in-graph A/B).
  p->late_trigger = 1;
  // Round shape: clusters (short contexts, keys split over the cluster: ~one round per CTA) take 3-chunk
  // rounds at hd 128; single-CTA hd-128 tiles (batched verifies, prefill chunks: many rounds over long
  // contexts) take 2-chunk rounds over a 4-stage ring with S double-buffered in TMEM.
  if (hd == 128 && cs == 1) {
    p->nst = 2;
    p->ring = 4;
    p->smem = Layout<128, 2, 4>::bytes + 1024;
    p->tcols = Layout<128, 2, 4>::tcols;
  } else if (hd == 128) {
    p->nst = p->ring = 3;
    p->smem = Layout<128, 3, 3>::bytes + 1024;
    p->tcols = Layout<128, 3, 3>::tcols;
  } else {
    p->nst = p->ring = 4;
    p->smem = Layout<64, 4, 4>::bytes + 1024;
    p->tcols = Layout<64, 4, 4>::tcols;
  }
  const int M = B * T;
  {  // q [M][Hq][hd]: box {64, G, tq} -> one lane quarter of (token, head-in-group) rows
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(hd), static_cast<cuuint64_t>(Hq), static_cast<cuuint64_t>(M)};
    cuuint64_t str[2] = {static_cast<cuuint64_t>(hd) * 2, static_cast<cuuint64_t>(Hq) * hd * 2};
    cuuint32_t box[3] = {64, static_cast<cuuint32_t>(G), static_cast<cuuint32_t>(p->tq)};
    if (int rc = enc(&p->tqm, 3, q, dims, str, box)) return rc;
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

int ygg_attn_tree_info(const void* plan, int* csplit, int* row_tiles, int* tokens_per_tile) {
  const Plan* p = plan_of(plan);
  YGG_CHECK_ARG(p != nullptr, "invalid tree-attention plan");
  if (csplit) *csplit = p->csplit;
  if (row_tiles) *row_tiles = p->row_tiles;
  if (tokens_per_tile) *tokens_per_tile = p->tpt;
  return YGG_OK;
}

int ygg_attn_tree_set_l2_prefetch(void* plan, int region, const void* ptr, size_t bytes) {
  Plan* p = const_cast<Plan*>(plan_of(plan));
  YGG_CHECK_ARG(p != nullptr, "invalid tree-attention plan");
  YGG_CHECK_ARG(region == 0 || region == 1, "prefetch region must be 0 or 1");
  YGG_CHECK_ARG(ptr == nullptr || (reinterpret_cast<uintptr_t>(ptr) & 15) == 0, "prefetch region must be 16-byte aligned");
  p->pf_ptr[region] = bytes ? static_cast<const char*>(ptr) : nullptr;
  p->pf_bytes[region] = ptr ? (bytes & ~static_cast<size_t>(15)) : 0;
  return YGG_OK;
}

int ygg_attn_tree_set_debug(void* plan, unsigned long long* stamps) {
  Plan* p = const_cast<Plan*>(plan_of(plan));
  YGG_CHECK_ARG(p != nullptr, "invalid tree-attention plan");
  p->dbg = stamps;
  return YGG_OK;
}

int ygg_attn_tree_set_trigger(void* plan, int late) {
  Plan* p = const_cast<Plan*>(plan_of(plan));
  YGG_CHECK_ARG(p != nullptr, "invalid tree-attention plan");
  p->late_trigger = late ? 1 : 0;
  return YGG_OK;
}

int ygg_attn_tree_run(const void* plan, const int32_t* blk_start, const int32_t* blk_len, const uint32_t* qmask,
                      int mask_words, float scale, void* out, ygg_stream_t stream) {
  const Plan* p = plan_of(plan);
  YGG_CHECK_ARG(p != nullptr, "invalid tree-attention plan");
  YGG_CHECK_ARG(blk_start && blk_len && out, "null pointer");
  YGG_CHECK_ARG(mask_words >= 0 && mask_words <= YGG_MAX_MASK_WORDS, "mask too wide");
  YGG_CHECK_ARG(mask_words == 0 || qmask != nullptr, "mask words without a mask");
  Args a;
  a.T = p->T;
  a.Hq = p->Hq;
  a.Hkv = p->Hkv;
  a.S = p->S;
  a.G = p->G;
  a.lg = __builtin_ctz(static_cast<unsigned>(p->G));
  a.lc = __builtin_ctz(static_cast<unsigned>(p->csplit));
  a.tpt = p->tpt;
  a.tq = p->tq;
  a.csplit = p->csplit;
  a.mask_words = mask_words;
  a.tcols = p->tcols;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.blk_start = blk_start;
  a.blk_len = blk_len;
  a.qmask = qmask ? qmask : reinterpret_cast<const uint32_t*>(blk_start);  // never read when mask_words == 0
  a.out = static_cast<__nv_bfloat16*>(out);
  a.trace = trace_next(15);
  a.dbg = p->dbg;
  a.late_trigger = p->late_trigger;
  for (int rg = 0; rg < 2; ++rg) {
    a.pf_ptr[rg] = p->pf_ptr[rg];
    a.pf_bytes[rg] = p->pf_bytes[rg];
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const dim3 grid(p->csplit, p->row_tiles, p->Hkv * p->B), block(p->hd == 128 ? Soft<128>::threads + 32
                                                                                  : Soft<64>::threads + 32);
#define YGG_AT_LAUNCH(H, N, R)                                                                                     \
  if (p->hd == H && p->nst == N && p->ring == R)                                                                   \
    return launch_pdl_cluster_x(attn_tree_kernel<H, N, R>, grid, block, p->smem, p->csplit, s, p->tqm, p->tk, p->tv, a);
  YGG_AT_KERNELS(YGG_AT_LAUNCH)
#undef YGG_AT_LAUNCH
  return ygg_fail(YGG_ERR_VALUE, "tree attention: no kernel for hd %d", p->hd);
}

}  // extern "C"
