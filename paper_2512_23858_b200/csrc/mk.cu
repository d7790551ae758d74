// Persistent decode-shaped forward ("megakernel"): one launch runs a whole draft or verify pass.
//
// The per-kernel forward (forward.py, bf16 unfused) pays a launch + ramp + drain at each of
// ~10 kernel boundaries per layer, and HBM idles across every one of them; for a 1B draft pass
// at 8 rows that is 3x the weight-streaming floor.  Here one CTA per SM runs a static phase
// program (embed, per layer: QKV GEMM, RoPE/KV append, tree attention, combine, O GEMM,
// residual, gate|up GEMM, SwiGLU, down GEMM, residual; then the LM head) and phases are
// separated by a grid-wide arrival counter.  The weight stream does not wait on that chain:
//   warp 0 (producer)  walks this CTA's GEMM units of *every* phase in order, TMA-loading weight
//                      tiles into the smem ring as soon as a stage frees, plus an L2 prefetch
//                      look-ahead of `look` tiles; only the activation tile of a stage waits until
//                      the phase that produced it has completed grid-wide;
//   warp 1 (MMA)       single-thread tcgen05.mma issue for GEMM units (double-buffered TMEM
//                      accumulator) and the TMA + QK^T / PV MMAs of attention units;
//   warps 2-5          TMEM -> stream-K partials, the element-wise epilogue phases, the
//                      attention softmax (one thread per query row), and the chunk combine.
// GEMMs are swap-AB (weight rows = UMMA M = 128, tokens = UMMA N = BN <= 128) and split
// stream-K over the grid; partial sums are reduced by the consumer phase in fixed segment order
// (deterministic).  RMSNorm gains are folded into the next weight, and the per-row rstd comes
// from per-128-feature sums of squares written by the residual phase.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "host_util.h"

namespace ygg {
namespace mk {

constexpr int kThreads = 192;
constexpr int kBM = 128, kBK = 64;
constexpr int kKC = 64;       // attention keys per unit
constexpr int kQRows = 128;   // attention query rows per unit (UMMA M)
constexpr int kMaxRows = 128; // M = B*T
constexpr int kMaxStages = 16;
constexpr int kMaxSegTable = 1032;
constexpr int kMaxPend = 64;  // tiles one CTA touches in one GEMM phase  // tiles + 1 of the widest GEMM (vocab <= 132096)
constexpr int kSmemLimit = 227 * 1024;
constexpr uint32_t kMagic = 0x59474d4bu;  // "YGMK"

enum Kind : int { kEmbed = 0, kGemm = 1, kAttn = 3, kCombine = 4 };
// Epilogue fused into a GEMM phase, applied by the last CTA to finish each tile group ("fixup").
enum Epi : int { kEpiNone = 0, kEpiQkv = 1, kEpiResid = 2, kEpiSwiglu = 3, kEpiStore = 4 };

struct Phase {
  int kind, layer;
  int wmap, xmap;       // GEMM: tensor-map indices
  int N, K, kb, units;  // GEMM geometry (copied into the epilogue phase that reduces it)
  int seg_first;        // itab offset of seg_first[tiles + 1]
  int seg_base;         // itab offset of seg_base[G]
  int ws;               // partial buffer (0/1)
  int ss_in, ss_out;    // sums-of-squares buffers (-1 = none)
  int kmap, vmap;       // attention: this layer's K / V^T maps
  int epi;              // GEMM: fused epilogue (Epi)
  int ctr;              // GEMM: offset of this phase's tile-group arrival counters (partials published)
  int dctr;             // GEMM: offset of this phase's tile-group done counters (fixup slices finished)
  int ptot;             // GEMM: index of this phase's total done counter
  int nsegs;            // GEMM: total segments (= fixup participants summed over groups)
  int src;              // GEMM: phase that produced X (-1: gate on the grid counter instead)
  int ss_src;           // GEMM: RESID phase that produced ss_in (-1: the embed phase)
  long long cache_off;  // element offset of this layer's cache block
};

// Tensor maps live in kernel parameter space when they fit (param-space maps are what the TMA
// descriptor cache is built for); larger models fall back to the copy in global memory.
constexpr int kBankMaps = 200;
struct MapBank {
  CUtensorMap m[kBankMaps];
};

struct Args {
  const Phase* phases;
  const CUtensorMap* maps;
  const int32_t* itab;
  unsigned int* bar;
  unsigned int* ctr;  // tile-group arrival counters (monotonic; a group completes every `target` arrivals)
  unsigned int* dctr; // tile-group done counters (monotonic, +1 per participant slice per launch)
  unsigned int* ptot; // per-phase done totals
  unsigned int* lctr; // launch index of this plan (incremented by the last CTA of each launch)
  int nphases, G, M, BN, stages, look, pf_maps, bank_n;
  int attn_bytes;  // size of the attention operand region (0 in the YGG_MK_NOATTN A/B mode)
  int xflags;  // A/B only (YGG_MK_XFLAGS): 1 = skip activation loads, 2 = skip MMAs, 4 = skip partial stores
  int d, Hq, Hkv, hd, S, T, B, F, V;
  int Gh, tok_per_tile, q_tiles, chunks, mask_words, qmap;
  float eps, scale_log2;
  const __nv_bfloat16* embed;
  const int32_t* tokens;
  const int32_t* pos;
  const int32_t* slot;
  const int32_t* req;
  const int32_t* blk_start;
  const int32_t* blk_len;
  const uint32_t* qmask;
  const float2* rope_cs;
  __nv_bfloat16* cache;
  float* resid;
  __nv_bfloat16* hb;
  __nv_bfloat16* q;
  __nv_bfloat16* attn;
  __nv_bfloat16* mlp;
  float* logits;
  float* ss;  // [2][d/128][M]
  float* ws;  // [2][ws_stride]
  long long ws_stride;
  float* opart;  // [chunks][M*Hq][hd]
  float* ml;     // [chunks][M*Hq][2]
  unsigned long long* dbg;  // optional [G][nphases] %globaltimer at each phase end (profiling)
};

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
YGG_DEV const CUtensorMap* tmap(const Args& a, const MapBank& bank, int i) {
  return i < a.bank_n ? &bank.m[i] : tmap(a, bank, i);
}
YGG_DEV unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
YGG_DEV unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
YGG_DEV void fence_acq_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
YGG_DEV void red_rel_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
YGG_DEV unsigned atom_acqrel_add(unsigned* p, unsigned v) {
  unsigned o;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
  return o;
}
YGG_DEV void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
YGG_DEV void tma_prefetch_l2(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
YGG_DEV void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
YGG_DEV void tma_load_2d_plain(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
YGG_DEV void st_shared_v4(uint32_t addr, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
YGG_DEV uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// Bounded spin on the grid counter (a lost arrival traps after ~2 s instead of hanging the GPU).
YGG_DEV void wait_count(const unsigned* bar, unsigned target) {
  if (ld_rlx(bar) < target) {
    const long long t0 = clock64();
    while (ld_rlx(bar) < target) {
      if (clock64() - t0 > (1ll << 32)) __trap();
    }
  }
  fence_acq_gpu();
}
YGG_DEV void cons_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Sum of the stream-K partials of V consecutive features [n, n+V) of row m (one tile), in segment
// order (deterministic).  Loads are issued kSegBatch segments at a time so a tile split over many
// CTAs costs one L2 round trip, not one per segment.
constexpr int kSegBatch = 8;
template <int V>
YGG_DEV void part_range(const float* __restrict__ wsb, int BN, int s0, int s1, int m, int nl, float* v) {
  const float* p = wsb + static_cast<size_t>(m) * kBM + nl;
  const size_t seg_stride = static_cast<size_t>(BN) * kBM;
#pragma unroll
  for (int i = 0; i < V; ++i) v[i] = 0.f;
  for (int s = s0; s < s1; s += kSegBatch) {
    float4 x[kSegBatch][V / 4];
#pragma unroll
    for (int k = 0; k < kSegBatch; ++k) {
      const float4* q = reinterpret_cast<const float4*>(p + (s + k) * seg_stride);
#pragma unroll
      for (int i = 0; i < V / 4; ++i) x[k][i] = (s + k < s1) ? __ldcg(q + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < kSegBatch; ++k)
#pragma unroll
      for (int i = 0; i < V / 4; ++i) {
        v[4 * i] += x[k][i].x;
        v[4 * i + 1] += x[k][i].y;
        v[4 * i + 2] += x[k][i].z;
        v[4 * i + 3] += x[k][i].w;
      }
  }
}

YGG_DEV void store_bf16x8(__nv_bfloat16* dst, const float* v) {
  uint4 u;
  u.x = pack_bf16(v[0], v[1]);
  u.y = pack_bf16(v[2], v[3]);
  u.z = pack_bf16(v[4], v[5]);
  u.w = pack_bf16(v[6], v[7]);
  *reinterpret_cast<uint4*>(dst) = u;
}

// rstd of every row from the [d/128][M] sums of squares, into shared memory.
YGG_DEV void load_rstd(const Args& a, int ss_buf, float* rstd_s, int* pos_s, int* slot_s, int* req_s, int et) {
  const int nt = a.d / kBM;
  const float* ss = a.ss + static_cast<size_t>(ss_buf) * nt * a.M;
  for (int m = et; m < a.M; m += 128) {
    pos_s[m] = __ldg(a.pos + m);
    slot_s[m] = __ldg(a.slot + m);
    req_s[m] = __ldg(a.req + m);
    float s = 0.f;
    for (int t = 0; t < nt; ++t) s += __ldcg(ss + static_cast<size_t>(t) * a.M + m);
    rstd_s[m] = rsqrtf(s / static_cast<float>(a.d) + a.eps);
  }
  cons_sync();
}

// Attention unit decode: chunk-major so the live (low) chunks spread over all CTAs.
struct AttnUnit {
  int chunk, r, kvh, qt, key0, bs, bl;
  bool skip;
};
YGG_DEV AttnUnit attn_unit(const Args& a, int u) {
  AttnUnit w;
  const int per_chunk = a.B * a.Hkv * a.q_tiles;
  w.chunk = u / per_chunk;
  const int rem = u % per_chunk;
  w.r = rem / (a.Hkv * a.q_tiles);
  w.kvh = (rem / a.q_tiles) % a.Hkv;
  w.qt = rem % a.q_tiles;
  w.key0 = w.chunk * kKC;
  w.bs = __ldg(a.blk_start + w.r);
  w.bl = __ldg(a.blk_len + w.r);
  const int t0 = w.qt * a.tok_per_tile;
  const int last_tok = min(a.T - 1, t0 + a.tok_per_tile - 1);
  w.skip = w.key0 >= w.bs + w.bl || (a.mask_words == 0 && w.key0 > w.bs + last_tok);
  return w;
}

// ---------------------------------------------------------------------------
// roles
// ---------------------------------------------------------------------------
struct Smem {
  unsigned char *sa, *sb, *sq, *sk, *svt, *sp;
  uint64_t *full, *empty, *tfull, *tempty, *abar;
  uint32_t* tmem_slot;
  float* rstd_s;  // [kMaxRows]
  int* pos_s;     // [kMaxRows]
  int* slot_s;    // [kMaxRows]
  int* req_s;     // [kMaxRows]
  int* seg_s;     // [kMaxSegTable] (unused scratch)
  int* flag;      // [kMaxPend][4] deferred fixups (group, participant, parts, counter target)
};

// Producer: three cursors over this CTA's GEMM units of every phase, all in registers (local-memory
// arrays would round-trip to L2: the ring leaves almost no L1).
//   W cursor     weight tile into the next free ring stage (never waits on the phase chain)
//   X cursor     activation tile of the oldest stage whose producing phase completed grid-wide
//   look cursor  L2 prefetch of the weight tile `look` units ahead of the W cursor
struct UnitCursor {
  int p;       // phase index
  int n;       // units left in this phase's range
  int kblk, tile, kb;
  const CUtensorMap* wm;
  const CUtensorMap* xm;
};
// Advance k to the next GEMM phase with a non-empty range for this CTA; false at the end.  Unit
// coordinates are then stepped incrementally (no per-unit integer division on the issue path).
YGG_DEV bool cursor_phase(const Args& a, const MapBank& bank, UnitCursor& k, int c) {
  while (k.n <= 0) {
    if (++k.p >= a.nphases) return false;
    const Phase* P = a.phases + k.p;
    if (P->kind != kGemm) continue;
    const int units = P->units, kb = P->kb;
    const int u0 = static_cast<int>(static_cast<long long>(units) * c / a.G);
    const int u1 = static_cast<int>(static_cast<long long>(units) * (c + 1) / a.G);
    k.n = u1 - u0;
    k.kb = kb;
    k.kblk = u0 % kb;
    k.tile = u0 / kb;
    k.wm = tmap(a, bank, P->wmap);
    k.xm = tmap(a, bank, P->xmap);
  }
  return true;
}
YGG_DEV bool cursor_step(const Args& a, const MapBank& bank, UnitCursor& k, int c) {
  if (++k.kblk == k.kb) {
    k.kblk = 0;
    ++k.tile;
  }
  --k.n;
  return k.n > 0 || cursor_phase(a, bank, k, c);
}

YGG_DEV void producer(const Args& a, const MapBank& bank, const Smem& sm) {
  const int c = blockIdx.x, G = a.G, S = a.stages;
  const uint32_t a_bytes = kBM * kBK * 2, b_bytes = a.BN * kBK * 2;
  const uint32_t tx_bytes = (a.xflags & 1) ? a_bytes : a_bytes + b_bytes;
  const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
  UnitCursor w{-1, 0, 0, 0, 1, nullptr, nullptr}, x = w, l = w;
  bool w_ok = cursor_phase(a, bank, w, c);
  cursor_phase(a, bank, x, c);
  bool l_ok = cursor_phase(a, bank, l, c);
  for (int i = 0; i < a.look && l_ok; ++i) {
    tma_prefetch_l2(l.wm, l.kblk * kBK, l.tile * kBM);
    l_ok = cursor_step(a, bank, l, c);
  }
  int wstage = 0, xstage = 0, npend = 0;
  uint32_t wph = 0;
  unsigned seen = 0;
  unsigned xdep = static_cast<unsigned>(x.p) * G;  // phase x.p - 1 complete everywhere
  bool waited = false;
  unsigned L1 = 0;  // launch index + 1 (read after the grid dependency)
  // X gating source of the X cursor's phase: a GEMM's tile groups (dataflow) or the grid counter.
  int xsrc = -1, xsrc_p = -2;
  const unsigned* src_tot = nullptr;
  unsigned src_tgt = 0;
  uint64_t sat0 = 0, sat1 = 0, sat2 = 0, sat3 = 0;  // source tiles already seen final (<= 256)
  auto sat_get = [&](int f) -> bool {
    const uint64_t w = f < 64 ? sat0 : (f < 128 ? sat1 : (f < 192 ? sat2 : sat3));
    return (w >> (f & 63)) & 1ull;
  };
  auto sat_set = [&](int f) {
    const uint64_t b = 1ull << (f & 63);
    if (f < 64) sat0 |= b;
    else if (f < 128) sat1 |= b;
    else if (f < 192) sat2 |= b;
    else sat3 |= b;
  };
  auto x_source = [&]() {
    if (x.p == xsrc_p) return;
    xsrc_p = x.p;
    const Phase* P = a.phases + x.p;
    xsrc = P->src;
    sat0 = sat1 = sat2 = sat3 = 0;
    if (xsrc >= 0) {
      const Phase* Q = a.phases + xsrc;
      src_tot = a.ptot + Q->ptot;
      src_tgt = L1 * static_cast<unsigned>(Q->nsegs);
    }
  };
  // Issue X loads (oldest first) once their source is final; block only if asked.
  auto flush = [&](bool block) {
    while (npend > 0) {
      if (!waited) {
        pdl_wait();
        waited = true;
        L1 = ld_rlx(a.lctr) + 1u;
      }
      x_source();
      if (xsrc >= 0) {
        // Source GEMM's fixups all done (one counter); per-tile gating costs a load per source tile
        // on the issue path, which the single producer thread cannot afford.
        if (!sat0) {
          if (ld_rlx(src_tot) < src_tgt) {
            if (!block) return;
            const long long t0 = clock64();
            while (ld_rlx(src_tot) < src_tgt)
              if (clock64() - t0 > (1ll << 32)) __trap();
          }
          fence_acq_gpu();
          fence_async_global();
          sat0 = 1;
        }
      } else if (seen < xdep) {
        seen = ld_rlx(a.bar);
        if (seen < xdep) {
          if (!block) return;
          const long long t0 = clock64();
          while ((seen = ld_rlx(a.bar)) < xdep)
            if (clock64() - t0 > (1ll << 32)) __trap();
        }
        fence_acq_gpu();
        fence_async_global();
      }
      if (!(a.xflags & 1))
        tma_load_2d(sm.sb + static_cast<size_t>(xstage) * b_bytes, x.xm, &sm.full[xstage], x.kblk * kBK, 0, pol_x);
      if (++xstage == S) xstage = 0;
      const int xp = x.p;
      cursor_step(a, bank, x, c);
      if (x.p != xp) xdep = static_cast<unsigned>(x.p) * G;
      --npend;
    }
  };
  int cur_p = -1;
  while (w_ok) {
    if (w.p != cur_p) {
      if (a.dbg && cur_p >= 0) {
        unsigned long long tt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
        a.dbg[(2ull * G + c) * a.nphases + cur_p] = tt;  // W stream of phase cur_p fully issued
      }
      cur_p = w.p;
      if (a.pf_maps) {
        tma_prefetch_desc(w.wm);
        tma_prefetch_desc(w.xm);
      }
    }
    const uint32_t eaddr = smem_u32(&sm.empty[wstage]);
    if (!mbar_try_wait(eaddr, wph ^ 1u)) {
      const long long t0 = clock64();
      while (!mbar_try_wait(eaddr, wph ^ 1u)) {
        if (npend > 0) flush(false);
        if (clock64() - t0 > (1ll << 33)) __trap();
      }
    }
    mbar_arrive_expect_tx(&sm.full[wstage], tx_bytes);
    tma_load_2d(sm.sa + static_cast<size_t>(wstage) * a_bytes, w.wm, &sm.full[wstage], w.kblk * kBK, w.tile * kBM, pol_w);
    if (l_ok) {
      tma_prefetch_l2(l.wm, l.kblk * kBK, l.tile * kBM);
      l_ok = cursor_step(a, bank, l, c);
    }
    ++npend;
    flush(false);
    if (++wstage == S) {
      wstage = 0;
      wph ^= 1u;
    }
    w_ok = cursor_step(a, bank, w, c);
  }
  flush(true);
}

YGG_DEV void mma_role(const Args& a, const MapBank& bank, const Smem& sm, uint32_t tmem) {
  const int c = blockIdx.x, G = a.G, S = a.stages, lane = threadIdx.x & 31;
  const uint32_t a_bytes = kBM * kBK * 2, b_bytes = a.BN * kBK * 2;
  const uint32_t idesc = umma_idesc_bf16(kBM, a.BN);
  const int DCH = a.hd / 64;
  const uint32_t tS = tmem + 256, tO = tmem + 320;
  int stage = 0;
  uint32_t ph = 0;
  int acc = 0;
  uint32_t accph = 0u;  // bit i: phase parity of accumulator buffer i
  int an = 0;
  bool waited = false;
  for (int p = 0; p < a.nphases; ++p) {
    const int kind = a.phases[p].kind;
    if (kind == kGemm) {
      const int kb = a.phases[p].kb, units = a.phases[p].units;
      const int u0 = static_cast<int>(static_cast<long long>(units) * c / G);
      const int u1 = static_cast<int>(static_cast<long long>(units) * (c + 1) / G);
      if (u1 <= u0) continue;
      const int t0 = u0 / kb, t1 = (u1 - 1) / kb;
      for (int t = t0; t <= t1; ++t) {
        const int ua = max(u0, t * kb), ub = min(u1, (t + 1) * kb);
        mbar_wait(&sm.tempty[acc], ((accph >> acc) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem + static_cast<uint32_t>(acc * a.BN);
        for (int u = ua; u < ub; ++u) {
          mbar_wait(&sm.full[stage], ph);
          tc_fence_after();
          if (lane == 0 && (a.xflags & 2)) {
            mbar_arrive(&sm.empty[stage]);
          } else if (lane == 0) {
            const uint32_t aa = smem_u32(sm.sa + static_cast<size_t>(stage) * a_bytes);
            const uint32_t ba = smem_u32(sm.sb + static_cast<size_t>(stage) * b_bytes);
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              umma_bf16(d_tmem, umma_desc_sw128(aa + kk * 32), umma_desc_sw128(ba + kk * 32), idesc,
                        (u == ua && kk == 0) ? 0u : 1u);
            umma_commit(&sm.empty[stage]);
          }
          __syncwarp();
          if (++stage == S) {
            stage = 0;
            ph ^= 1u;
          }
        }
        if (lane == 0) {
          if (a.xflags & 2) mbar_arrive(&sm.tfull[acc]);
          else umma_commit(&sm.tfull[acc]);
        }
        __syncwarp();
        accph ^= 1u << acc;
        acc ^= 1;
      }
    } else if (kind == kAttn && !(a.xflags & 8)) {
      const int kmap = a.phases[p].kmap, vmap = a.phases[p].vmap;
      if (!waited) {
        pdl_wait();
        waited = true;
      }
      if (lane == 0) {
        wait_count(a.bar, static_cast<unsigned>(p) * G);
        fence_async_global();
      }
      __syncwarp();
      const int n_units = a.chunks * a.B * a.Hkv * a.q_tiles;
      for (int u = c; u < n_units; u += G) {
        const AttnUnit w = attn_unit(a, u);
        if (w.skip) continue;
        if (lane == 0) {
          const uint32_t bytes = DCH * kQRows * 128 + DCH * kKC * 128 + a.hd * 128;
          mbar_arrive_expect_tx(&sm.abar[0], bytes);
          const int t0 = w.qt * a.tok_per_tile;
          for (int dc = 0; dc < DCH; ++dc) {
            tma_load_3d(sm.sq + dc * kQRows * 128, tmap(a, bank, a.qmap), &sm.abar[0], dc * 64, w.kvh * a.Gh, w.r * a.T + t0);
            tma_load_2d_plain(sm.sk + dc * kKC * 128, tmap(a, bank, kmap), &sm.abar[0], dc * 64,
                              (w.r * 2 * a.Hkv + w.kvh) * a.S + w.key0);
          }
          tma_load_2d_plain(sm.svt, tmap(a, bank, vmap), &sm.abar[0], w.key0, ((w.r * 2 + 1) * a.Hkv + w.kvh) * a.hd);
          mbar_wait(&sm.abar[0], an & 1);
          tc_fence_after();
          const uint32_t id1 = umma_idesc_bf16(kQRows, kKC);
          for (int kk = 0; kk < a.hd / 16; ++kk)
            umma_bf16(tS, umma_desc_sw128(smem_u32(sm.sq + (kk / 4) * kQRows * 128) + (kk % 4) * 32),
                      umma_desc_sw128(smem_u32(sm.sk + (kk / 4) * kKC * 128) + (kk % 4) * 32), id1, kk > 0 ? 1u : 0u);
          umma_commit(&sm.abar[1]);
          mbar_wait(&sm.abar[2], an & 1);
          tc_fence_after();
          const uint32_t id2 = umma_idesc_bf16(kQRows, a.hd);
#pragma unroll
          for (int kk = 0; kk < kKC / 16; ++kk)
            umma_bf16(tO, umma_desc_sw128(smem_u32(sm.sp) + kk * 32), umma_desc_sw128(smem_u32(sm.svt) + kk * 32), id2,
                      kk > 0 ? 1u : 0u);
          umma_commit(&sm.abar[3]);
          mbar_wait(&sm.abar[3], an & 1);  // smem operands free for the next unit
        }
        __syncwarp();
        ++an;
      }
    }
  }
}

// Visibility bits of 32 keys starting at absolute key kw for one query row: prefix keys
// (< bs) always, block keys by the row's tree-mask bit (causal when no mask), none past the block.
YGG_DEV uint32_t vis_word(int kw, int bs, int bl, int tq, bool row_valid, int mask_words, const uint32_t* mrow) {
  if (!row_valid) return 0u;
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

// Partial sums of K items at once (rows m[k], tile-local features nl[k]..+8), segments in order;
// SB segments' loads for all K items are in flight together (one L2 round trip per SB segments).
template <int K, int SB>
YGG_DEV void sumk(const float* __restrict__ wsb, int BN, int s0, int s1, const int* m, const int* nl, float (*v)[8]) {
  const size_t seg_stride = static_cast<size_t>(BN) * kBM;
  const float* p[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    p[k] = wsb + static_cast<size_t>(m[k]) * kBM + nl[k];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[k][j] = 0.f;
  }
  for (int s = s0; s < s1; s += SB) {
    float4 x[SB][K][2];
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      const bool ok = s + b < s1;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const float4* q = reinterpret_cast<const float4*>(p[k] + (s + b) * seg_stride);
        x[b][k][0] = ok ? __ldcg(q) : make_float4(0.f, 0.f, 0.f, 0.f);
        x[b][k][1] = ok ? __ldcg(q + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int b = 0; b < SB; ++b)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        v[k][0] += x[b][k][0].x; v[k][1] += x[b][k][0].y; v[k][2] += x[b][k][0].z; v[k][3] += x[b][k][0].w;
        v[k][4] += x[b][k][1].x; v[k][5] += x[b][k][1].y; v[k][6] += x[b][k][1].z; v[k][7] += x[b][k][1].w;
      }
  }
}

// Gate (segments [s0,s1)) and up ([q0,q1)) partial sums of K items, both ranges' loads in flight together.
template <int K, int SB>
YGG_DEV void sum_gu(const float* __restrict__ wsb, int BN, int s0, int s1, int q0, int q1, const int* m, const int* nl,
                    float (*v)[8], float (*u)[8]) {
  const size_t seg_stride = static_cast<size_t>(BN) * kBM;
  const float* p[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    p[k] = wsb + static_cast<size_t>(m[k]) * kBM + nl[k];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[k][j] = u[k][j] = 0.f;
  }
  const int ns = s1 - s0, nq = q1 - q0, n = ns > nq ? ns : nq;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int b0 = 0; b0 < n; b0 += SB) {
    float4 x[SB][K][4];
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      const bool okg = b0 + b < ns, oku = b0 + b < nq;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const float4* qg = reinterpret_cast<const float4*>(p[k] + (s0 + b0 + b) * seg_stride);
        const float4* qu = reinterpret_cast<const float4*>(p[k] + (q0 + b0 + b) * seg_stride);
        x[b][k][0] = okg ? __ldcg(qg) : z;
        x[b][k][1] = okg ? __ldcg(qg + 1) : z;
        x[b][k][2] = oku ? __ldcg(qu) : z;
        x[b][k][3] = oku ? __ldcg(qu + 1) : z;
      }
    }
#pragma unroll
    for (int b = 0; b < SB; ++b)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        v[k][0] += x[b][k][0].x; v[k][1] += x[b][k][0].y; v[k][2] += x[b][k][0].z; v[k][3] += x[b][k][0].w;
        v[k][4] += x[b][k][1].x; v[k][5] += x[b][k][1].y; v[k][6] += x[b][k][1].z; v[k][7] += x[b][k][1].w;
        u[k][0] += x[b][k][2].x; u[k][1] += x[b][k][2].y; u[k][2] += x[b][k][2].z; u[k][3] += x[b][k][2].w;
        u[k][4] += x[b][k][3].x; u[k][5] += x[b][k][3].y; u[k][6] += x[b][k][3].z; u[k][7] += x[b][k][3].w;
      }
  }
}

// Fused epilogue of rows [row0, row1) of one tile group (this participant's slice).  Thread item =
// (row m, 8 consecutive features); the 16 items of a row sit in 16 consecutive lanes, so RoPE pairs
// (feature f, f +- hd/2: same head, same tile) are one shuffle apart and the per-tile sum of squares
// is a 16-lane reduction.  Two items per thread per pass; partials summed in segment order.
template <int EPI, int IP, int SB>
YGG_DEV void fixup(const Args& a, const Smem& sm, int t, const float* wsb, int s0, int s1, int q0, int q1, int ss_out,
                   long long cache_off, int et, int row0, int row1) {
  const int M = a.M, BN = a.BN, lane = threadIdx.x & 31;
  const int items = (row1 - row0) * 16;
  for (int i0 = 0; i0 < items; i0 += 128 * IP) {
    int mm[4], nl[4];
    bool live[4];
#pragma unroll
    for (int k = 0; k < IP; ++k) {
      const int i = i0 + k * 128 + et;
      live[k] = i < items;
      mm[k] = live[k] ? row0 + (i >> 4) : row0;
      nl[k] = (i & 15) * 8;
    }
    float v[4][8];
    float2 cs[4][8];
    if (EPI == kEpiQkv) {
      const int half = a.hd / 2;
#pragma unroll
      for (int k = 0; k < IP; ++k) {
        const int n = t * kBM + nl[k];
        const int idx0 = n % a.hd;
        const bool rope = n / a.hd < a.Hq + a.Hkv;
        const float2* cp = a.rope_cs + static_cast<size_t>(sm.pos_s[mm[k]]) * half + (idx0 % half);
#pragma unroll
        for (int j = 0; j < 8; ++j) cs[k][j] = rope ? __ldg(cp + j) : make_float2(1.f, 0.f);
      }
    }
    float4 rx[4][2];
    if (EPI == kEpiResid) {
#pragma unroll
      for (int k = 0; k < IP; ++k) {
        const float4* rp = reinterpret_cast<const float4*>(a.resid + static_cast<size_t>(mm[k]) * a.d + t * kBM + nl[k]);
        rx[k][0] = __ldcg(rp);
        rx[k][1] = __ldcg(rp + 1);
      }
    }
    float u[4][8];
    if (EPI == kEpiSwiglu) sum_gu<IP, SB>(wsb, BN, s0, s1, q0, q1, mm, nl, v, u);
    else sumk<IP, SB>(wsb, BN, s0, s1, mm, nl, v);
#pragma unroll
    for (int k = 0; k < IP; ++k) {
      const int m = mm[k];
      const int n = t * kBM + nl[k];
      if (EPI == kEpiQkv) {
        const float r = sm.rstd_s[m];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[k][j] *= r;
        const int hd = a.hd, half = hd / 2;
        const int head = n / hd, idx0 = n % hd;
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = __shfl_xor_sync(0xffffffffu, v[k][j], hd / 16);
        const bool first = idx0 < half;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          v[k][j] = first ? (v[k][j] * cs[k][j].x - o[j] * cs[k][j].y) : (v[k][j] * cs[k][j].x + o[j] * cs[k][j].y);
        if (live[k]) {
          if (head < a.Hq) {
            store_bf16x8(a.q + (static_cast<size_t>(m) * a.Hq + head) * hd + idx0, v[k]);
          } else {
            const bool is_v = head >= a.Hq + a.Hkv;
            const int kvh = is_v ? head - a.Hq - a.Hkv : head - a.Hq;
            const int rq = sm.req_s[m], sl = sm.slot_s[m];
            __nv_bfloat16* base = a.cache + cache_off +
                                  ((static_cast<size_t>(rq) * 2 + (is_v ? 1 : 0)) * a.Hkv + kvh) * static_cast<size_t>(a.S) * hd;
            if (!is_v) {
              store_bf16x8(base + static_cast<size_t>(sl) * hd + idx0, v[k]);
            } else {  // V^T [hd][S]
#pragma unroll
              for (int j = 0; j < 8; ++j) base[static_cast<size_t>(idx0 + j) * a.S + sl] = __float2bfloat16_rn(v[k][j]);
            }
          }
        }
      } else if (EPI == kEpiResid) {
        float sq = 0.f;
        v[k][0] += rx[k][0].x; v[k][1] += rx[k][0].y; v[k][2] += rx[k][0].z; v[k][3] += rx[k][0].w;
        v[k][4] += rx[k][1].x; v[k][5] += rx[k][1].y; v[k][6] += rx[k][1].z; v[k][7] += rx[k][1].w;
        if (live[k]) {
          float4* rp = reinterpret_cast<float4*>(a.resid + static_cast<size_t>(m) * a.d + n);
          __stcg(rp, make_float4(v[k][0], v[k][1], v[k][2], v[k][3]));
          __stcg(rp + 1, make_float4(v[k][4], v[k][5], v[k][6], v[k][7]));
          store_bf16x8(a.hb + static_cast<size_t>(m) * a.d + n, v[k]);
#pragma unroll
          for (int j = 0; j < 8; ++j) sq += v[k][j] * v[k][j];
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (live[k] && (lane & 15) == 0)
          __stcg(a.ss + (static_cast<size_t>(ss_out) * (a.d / kBM) + t) * M + m, sq);
      } else if (EPI == kEpiSwiglu) {
        const float r = sm.rstd_s[m];
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float g = v[k][j] * r;
          o[j] = __fdividef(g, 1.f + __expf(-g)) * (u[k][j] * r);
        }
        if (live[k]) store_bf16x8(a.mlp + static_cast<size_t>(m) * a.F + n, o);
      } else if (EPI == kEpiStore) {
        if (live[k]) {
          const float r = sm.rstd_s[m];
          float4* dst = reinterpret_cast<float4*>(a.logits + static_cast<size_t>(m) * a.V + n);
          __stcg(dst, make_float4(v[k][0] * r, v[k][1] * r, v[k][2] * r, v[k][3] * r));
          __stcg(dst + 1, make_float4(v[k][4] * r, v[k][5] * r, v[k][6] * r, v[k][7] * r));
        }
      }
    }
  }
}

YGG_DEV void fixup_any(int epi, const Args& a, const Smem& sm, int t, const float* wsb, const int* pe, int ss_out,
                       long long cache_off, int et, int row0, int row1) {
  const int s0 = pe[4], s1 = pe[5], q0 = pe[6], q1 = pe[7];
  // Few items: one item per thread with every segment in flight; many: two items, 8-segment batches.
  const bool few = (row1 - row0) * 16 <= 128;
#define YGG_FX(E, I, B) fixup<E, I, B>(a, sm, t, wsb, s0, s1, q0, q1, ss_out, cache_off, et, row0, row1)
  switch (epi) {
    case kEpiQkv: if (few) YGG_FX(kEpiQkv, 1, 16); else YGG_FX(kEpiQkv, 2, 8); break;
    case kEpiResid: if (few) YGG_FX(kEpiResid, 1, 16); else YGG_FX(kEpiResid, 2, 8); break;
    case kEpiSwiglu: if (few) YGG_FX(kEpiSwiglu, 1, 8); else YGG_FX(kEpiSwiglu, 2, 4); break;
    default: if (few) YGG_FX(kEpiStore, 1, 16); else YGG_FX(kEpiStore, 2, 8); break;
  }
#undef YGG_FX
}

YGG_DEV void consumer(const Args& a, const Smem& sm, uint32_t tmem) {
  const int c = blockIdx.x, G = a.G, M = a.M, BN = a.BN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int et = threadIdx.x - 64;       // 0..127
  const int quarter = warp & 3;          // TMEM lane quarter of this warp
  const int row = quarter * 32 + lane;   // TMEM lane = feature row (GEMM) / query row (attention)
  const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
  const uint32_t tS = tmem + 256, tO = tmem + 320;
  const int stride = G * 128;
  int acc = 0;
  uint32_t accph = 0u;
  int an = 0;
  pdl_wait();
  const unsigned L1 = ld_rlx(a.lctr) + 1u;  // launch index + 1: targets of the monotonic done counters
  for (int p = 0; p < a.nphases; ++p) {
    const Phase* PP = a.phases + p;
    const int kind = PP->kind;
    if (kind != kGemm && p > 0) {
      if (et == 0) wait_count(a.bar, static_cast<unsigned>(p) * G);
      cons_sync();
    }
    if (kind == kGemm) {
      const int kb = PP->kb, units = PP->units, epi = PP->epi, ss_in = PP->ss_in, ss_out = PP->ss_out;
      const long long cache_off = PP->cache_off;
      const int* sf = a.itab + PP->seg_first;
      unsigned* ctr = a.ctr + PP->ctr;
      float* wsb = a.ws + PP->ws * a.ws_stride;
      const int half_t = a.F / kBM;
      bool have_rstd = false;
      const int ss_src = PP->ss_src;
      auto need_rstd = [&]() {
        if (!have_rstd && ss_in >= 0) {
          // ss_in is complete once every fixup slice of the producing RESID phase is done (or the
          // embed phase, for the first layer); X tiles alone do not imply it under dataflow gating.
          if (et == 0) {
            if (ss_src >= 0) {
              const Phase* Q = a.phases + ss_src;
              wait_count(a.ptot + Q->ptot, L1 * static_cast<unsigned>(Q->nsegs));
            } else {
              wait_count(a.bar, static_cast<unsigned>(G));
            }
          }
          cons_sync();
          load_rstd(a, ss_in, sm.rstd_s, sm.pos_s, sm.slot_s, sm.req_s, et);
          have_rstd = true;
        }
      };
      const int u0 = static_cast<int>(static_cast<long long>(units) * c / G);
      const int u1 = static_cast<int>(static_cast<long long>(units) * (c + 1) / G);
      if (u1 > u0) {
        const int t0 = u0 / kb, t1 = (u1 - 1) / kb;
        const int sbase = __ldg(a.itab + PP->seg_base + c);
        int npend_ = 0;
        for (int t = t0; t <= t1; ++t) {
          const int seg = sbase + (t - t0);
          const int nseg = __ldg(sf + t + 1) - __ldg(sf + t);
          mbar_wait(&sm.tfull[acc], (accph >> acc) & 1u);
          tc_fence_after();
          const uint32_t taddr = tmem + lane_base + static_cast<uint32_t>(acc * BN);
          if (epi == kEpiStore && nseg == 1) {
            // Whole tile on this CTA: logits straight from TMEM (thread = vocabulary row).
            need_rstd();
            float* dst = a.logits + static_cast<size_t>(t) * kBM + row;
            for (int c0 = 0; c0 < BN; c0 += 16) {
              float v[16];
              tmem_ld16(taddr + c0, v);
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (c0 + j < M) __stcg(dst + static_cast<size_t>(c0 + j) * a.V, v[j] * sm.rstd_s[c0 + j]);
            }
            tc_fence_before();
            mbar_arrive(&sm.tempty[acc]);
            accph ^= 1u << acc;
            acc ^= 1;
            continue;
          }
          float* dst = wsb + static_cast<size_t>(seg) * BN * kBM + row;
          for (int c0 = 0; c0 < BN; c0 += 16) {
            float v[16];
            tmem_ld16(taddr + c0, v);
            if (a.xflags & 4) continue;
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (c0 + j < M) __stcg(dst + static_cast<size_t>(c0 + j) * kBM, v[j]);
          }
          tc_fence_before();
          mbar_arrive(&sm.tempty[acc]);
          accph ^= 1u << acc;
          acc ^= 1;
          if (a.dbg && et == 0 && t == t1) {
            unsigned long long tt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
            a.dbg[(static_cast<size_t>(G) + c) * a.nphases + p] = tt;  // last partial drained from TMEM
          }
          if (epi == kEpiNone) continue;
          // Record the tile group this partial belongs to; arrivals are published in one batch below.
          if (et == 0) {
            int g = t, j = seg - __ldg(sf + t), nparts = nseg;
            if (epi == kEpiSwiglu) {
              g = t % half_t;
              const int ng = __ldg(sf + g + 1) - __ldg(sf + g);
              const int nu = __ldg(sf + g + half_t + 1) - __ldg(sf + g + half_t);
              nparts = ng + nu;
              if (t >= half_t) j += ng;
            }
            int* pe = sm.flag + 8 * npend_;
            pe[0] = g;
            pe[1] = j;
            pe[2] = nparts;
            pe[4] = __ldg(sf + g);
            pe[5] = __ldg(sf + g + 1);
            pe[6] = (epi == kEpiSwiglu) ? __ldg(sf + g + half_t) : 0;
            pe[7] = (epi == kEpiSwiglu) ? __ldg(sf + g + half_t + 1) : 0;
          }
          ++npend_;
          if (t == t0) need_rstd();  // rstd / positions (inputs of earlier phases) while partials drain
        }
        if (npend_ > 0) {
          // Publish every partial of this range (one release per group, in parallel), then wait for
          // each group's other participants; every participant finishes a row slice of the group.
          cons_sync();
          if (et < npend_) {
            int* pe = sm.flag + 8 * et;
            fence_acq_gpu();
            unsigned old;
            asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr + pe[0]) : "memory");
            const unsigned np = static_cast<unsigned>(pe[2]);
            wait_count(ctr + pe[0], (old / np + 1u) * np);
          }
          cons_sync();
          if (a.dbg && et == 0) {
            unsigned long long tt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
            a.dbg[(3ull * G + c) * a.nphases + p] = tt;  // all of this CTA's tile groups complete
          }
          long long fx0 = clock64();
          int fx_items = 0;
          for (int i = 0; i < npend_; ++i) {
            const int* pe = sm.flag + 8 * i;
            const int g = pe[0], j = pe[1], nparts = pe[2];
            const int r0 = static_cast<int>(static_cast<long long>(M) * j / nparts);
            const int r1 = static_cast<int>(static_cast<long long>(M) * (j + 1) / nparts);
            if (r1 > r0) fixup_any(epi, a, sm, g, wsb, pe, ss_out, cache_off, et, r0, r1);
            fx_items += (r1 - r0) * 16;
          }
          // Publish the finished slices: per-group done counters gate the next GEMM's X tiles.
          fence_async_global();
          cons_sync();
          if (et < npend_) {
            const int* pe = sm.flag + 8 * et;
            red_rel_add(a.dctr + PP->dctr + pe[0], 1u);
            red_rel_add(a.ptot + PP->ptot, 1u);
          }
          if (a.dbg && et == 0) {
            a.dbg[(6ull * G + c) * a.nphases + p] = static_cast<unsigned long long>(clock64() - fx0);
            a.dbg[(7ull * G + c) * a.nphases + p] = static_cast<unsigned long long>(fx_items) * 1000ull + npend_;
          }
        }
      }
    } else if (kind == kEmbed) {
      const int d8 = a.d / 8, items = M * d8;
      const int nt = a.d / kBM;
      float* ss = a.ss + static_cast<size_t>(PP->ss_out) * nt * M;
      for (int i0 = c * 128; i0 < items; i0 += stride) {
        const int i = i0 + et;
        const bool live = i < items;
        const int m = live ? i / d8 : 0, n = live ? (i % d8) * 8 : 0;
        float h[8];
        float sq = 0.f;
        if (live) {
          const int tok = __ldg(a.tokens + m);
          const uint4 u = __ldg(reinterpret_cast<const uint4*>(a.embed + static_cast<size_t>(tok) * a.d + n));
          const uint32_t wv[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&wv[k]);
            h[2 * k] = __bfloat162float(b.x);
            h[2 * k + 1] = __bfloat162float(b.y);
          }
          float4* wp = reinterpret_cast<float4*>(a.resid + static_cast<size_t>(m) * a.d + n);
          __stcg(wp, make_float4(h[0], h[1], h[2], h[3]));
          __stcg(wp + 1, make_float4(h[4], h[5], h[6], h[7]));
          store_bf16x8(a.hb + static_cast<size_t>(m) * a.d + n, h);
#pragma unroll
          for (int k = 0; k < 8; ++k) sq += h[k] * h[k];
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (live && (lane & 15) == 0) __stcg(ss + static_cast<size_t>(n / kBM) * M + m, sq);
      }
    } else if (kind == kAttn && !(a.xflags & 8)) {
      const int n_units = a.chunks * a.B * a.Hkv * a.q_tiles;
      const size_t rows_all = static_cast<size_t>(M) * a.Hq;
      for (int u = c; u < n_units; u += G) {
        const AttnUnit w = attn_unit(a, u);
        if (w.skip) continue;
        const int t0 = w.qt * a.tok_per_tile;
        const int tq = t0 + row / a.Gh;
        const int head = w.kvh * a.Gh + row % a.Gh;
        const bool row_valid = tq < a.T;
        const int m = w.r * a.T + tq;
        const uint32_t* mrow = a.qmask + static_cast<size_t>(row_valid ? m : 0) * a.mask_words;
        const uint32_t vis0 = vis_word(w.key0, w.bs, w.bl, tq, row_valid, a.mask_words, mrow);
        const uint32_t vis1 = vis_word(w.key0 + 32, w.bs, w.bl, tq, row_valid, a.mask_words, mrow);
        mbar_wait(&sm.abar[1], an & 1);
        tc_fence_after();
        float mx = -INFINITY;
#pragma unroll
        for (int c0 = 0; c0 < kKC; c0 += 16) {
          float v[16];
          tmem_ld16(tS + lane_base + c0, v);
          const uint32_t bits = (c0 < 32 ? vis0 : vis1) >> (c0 & 31);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if ((bits >> j) & 1u) mx = fmaxf(mx, v[j] * a.scale_log2);
        }
        float l = 0.f;
        const uint32_t rbase = smem_u32(sm.sp + row * 128);
#pragma unroll
        for (int c0 = 0; c0 < kKC; c0 += 16) {
          float v[16];
          tmem_ld16(tS + lane_base + c0, v);
          const uint32_t bits = (c0 < 32 ? vis0 : vis1) >> (c0 & 31);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            v[j] = ((bits >> j) & 1u) ? exp2f(v[j] * a.scale_log2 - mx) : 0.f;
            l += v[j];
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int uu = c0 / 8 + h;
            const float* p8 = v + 8 * h;
            st_shared_v4(rbase + ((uu ^ (row & 7)) << 4), pack_bf16(p8[0], p8[1]), pack_bf16(p8[2], p8[3]),
                         pack_bf16(p8[4], p8[5]), pack_bf16(p8[6], p8[7]));
          }
        }
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(&sm.abar[2]);
        mbar_wait(&sm.abar[3], an & 1);
        tc_fence_after();
        const size_t orow = static_cast<size_t>(m) * a.Hq + head;
        float* op = a.opart + (static_cast<size_t>(w.chunk) * rows_all + (row_valid ? orow : 0)) * a.hd;
        for (int c0 = 0; c0 < a.hd; c0 += 16) {
          float o[16];
          tmem_ld16(tO + lane_base + c0, o);
          if (row_valid) {
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              __stcg(reinterpret_cast<float4*>(op + c0 + j), make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]));
          }
        }
        if (row_valid)
          __stcg(reinterpret_cast<float2*>(a.ml + (static_cast<size_t>(w.chunk) * rows_all + orow) * 2),
                 make_float2(mx, l));
        tc_fence_before();
        ++an;
      }
    } else if (kind == kCombine) {
      // Merge chunk partials in fixed chunk order; every chunk's loads of a batch are in flight at once.
      const int rows = M * a.Hq;
      const int nw = G * 4;
      const int DPL = a.hd / 32;  // 2 or 4
      constexpr int CB = 8;
      for (int rr = c * 4 + (et >> 5); rr < rows; rr += nw) {
        const int r = (rr / a.Hq) / a.T;
        const int nch = (__ldg(a.blk_start + r) + __ldg(a.blk_len + r) + kKC - 1) / kKC;
        float Mx = -INFINITY;
        for (int c0 = 0; c0 < nch; c0 += CB) {
          float mv[CB];
#pragma unroll
          for (int k = 0; k < CB; ++k)
            mv[k] = (c0 + k < nch) ? __ldcg(a.ml + (static_cast<size_t>(c0 + k) * rows + rr) * 2) : -INFINITY;
#pragma unroll
          for (int k = 0; k < CB; ++k) Mx = fmaxf(Mx, mv[k]);
        }
        float accv[4] = {0.f, 0.f, 0.f, 0.f};
        float L = 0.f;
        if (Mx != -INFINITY) {
          for (int c0 = 0; c0 < nch; c0 += CB) {
            float2 mlv[CB];
            float4 ov[CB];
#pragma unroll
            for (int k = 0; k < CB; ++k) {
              const bool ok = c0 + k < nch;
              const size_t base = static_cast<size_t>(c0 + k) * rows + rr;
              mlv[k] = ok ? __ldcg(reinterpret_cast<const float2*>(a.ml + base * 2)) : make_float2(-INFINITY, 0.f);
              const float* o = a.opart + base * a.hd + lane * DPL;
              if (!ok) ov[k] = make_float4(0.f, 0.f, 0.f, 0.f);
              else if (DPL == 4) ov[k] = __ldcg(reinterpret_cast<const float4*>(o));
              else {
                const float2 x = __ldcg(reinterpret_cast<const float2*>(o));
                ov[k] = make_float4(x.x, x.y, 0.f, 0.f);
              }
            }
#pragma unroll
            for (int k = 0; k < CB; ++k) {
              if (mlv[k].x == -INFINITY) continue;
              const float wgt = exp2f(mlv[k].x - Mx);
              L += wgt * mlv[k].y;
              accv[0] += wgt * ov[k].x;
              accv[1] += wgt * ov[k].y;
              accv[2] += wgt * ov[k].z;
              accv[3] += wgt * ov[k].w;
            }
          }
        }
        const float inv = L > 0.f ? 1.f / L : 0.f;
        __nv_bfloat16* dst = a.attn + static_cast<size_t>(rr) * a.hd + lane * DPL;
        if (DPL == 4) {
          uint2 u;
          u.x = pack_bf16(accv[0] * inv, accv[1] * inv);
          u.y = pack_bf16(accv[2] * inv, accv[3] * inv);
          *reinterpret_cast<uint2*>(dst) = u;
        } else {
          *reinterpret_cast<uint32_t*>(dst) = pack_bf16(accv[0] * inv, accv[1] * inv);
        }
      }
    }
    // Publish this CTA's writes of phase p (generic stores, read later by TMA or other SMs).
    if (a.dbg && et == 0) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      a.dbg[(4ull * G + c) * a.nphases + p] = tt;  // work of phase p done
    }
    fence_async_global();
    cons_sync();
    if (a.dbg && et == 0) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      a.dbg[(5ull * G + c) * a.nphases + p] = tt;  // after the proxy fence + CTA barrier
    }
    if (et == 0) {
      // Counter semantics: value >= (p+1)*G  <=>  every CTA finished phase p.  GEMM phases do not
      // wait for phase p-1 up front (their data dependency is carried by the TMA ring), so a CTA
      // must not publish phase p before phase p-1 is complete everywhere.
      if (kind == kGemm && p > 0) wait_count(a.bar, static_cast<unsigned>(p) * G);
      if (a.dbg) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.dbg[static_cast<size_t>(c) * a.nphases + p] = t;
      }
      if (p == a.nphases - 1) {
        const unsigned old = atom_acqrel_add(a.bar, 1u);
        if (old == static_cast<unsigned>(a.nphases) * G - 1u) {  // last CTA: reset for the next launch
          atomicExch(a.bar, 0u);
          atomicAdd(a.lctr, 1u);
        }
      } else {
        red_rel_add(a.bar, 1u);
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) mk_kernel(const __grid_constant__ Args a, const __grid_constant__ MapBank bank) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = a.stages;
  const int DCH = a.hd / 64;
  Smem sm;
  sm.sa = base;
  sm.sb = sm.sa + static_cast<size_t>(S) * kBM * kBK * 2;
  sm.sq = sm.sb + static_cast<size_t>(S) * a.BN * kBK * 2;
  sm.sk = sm.sq + DCH * kQRows * 128;
  sm.svt = sm.sk + DCH * kKC * 128;
  sm.sp = sm.svt + a.hd * 128;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm.sq + a.attn_bytes);
  sm.full = bars;
  sm.empty = bars + S;
  sm.tfull = bars + 2 * S;
  sm.tempty = sm.tfull + 2;
  sm.abar = sm.tempty + 2;
  sm.tmem_slot = reinterpret_cast<uint32_t*>(sm.abar + 4);
  sm.rstd_s = reinterpret_cast<float*>(sm.tmem_slot + 4);
  sm.pos_s = reinterpret_cast<int*>(sm.rstd_s + kMaxRows);
  sm.slot_s = sm.pos_s + kMaxRows;
  sm.req_s = sm.slot_s + kMaxRows;
  sm.seg_s = sm.req_s + kMaxRows;
  sm.flag = sm.seg_s + kMaxSegTable;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.tfull[i], 1);
      mbar_init(&sm.tempty[i], 128);
    }
    mbar_init(&sm.abar[0], 1);
    mbar_init(&sm.abar[1], 1);
    mbar_init(&sm.abar[2], 128);
    mbar_init(&sm.abar[3], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(sm.tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *sm.tmem_slot;
  if (warp == 0) {
    if (lane == 0) producer(a, bank, sm);
  } else if (warp == 1) {
    mma_role(a, bank, sm, tmem);
  } else {
    consumer(a, sm, tmem);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  pdl_launch_dependents();
}

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
struct Plan {
  uint32_t magic;
  Args args;
  MapBank bank;
  int grid;
  size_t smem;
};

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static int encode(CUtensorMap* map, int rank, const void* ptr, const cuuint64_t* dims, const cuuint64_t* strides,
                  const cuuint32_t* box) {
  auto fn = encoder();
  if (!fn) return ygg_fail(YGG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t es[3] = {1, 1, 1};
  CUresult rc = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) return ygg_fail(YGG_ERR_CUDA, "persistent forward: tensor map encode failed (%d)", (int)rc);
  return YGG_OK;
}
static int map2d(CUtensorMap* m, const void* p, long long rows, long long cols, int box_rows, int box_cols = 64) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t str[1] = {static_cast<cuuint64_t>(cols) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  return encode(m, 2, p, dims, str, box);
}

// Static geometry shared by query and init.
struct Geo {
  int G, M, BN, stages, look;
  int nphases, nmaps, itab_len, nctr;
  size_t ws_floats;  // per buffer
  size_t part_bytes;
  size_t table_bytes;
  size_t smem;
  int chunks, q_tiles, tok_per_tile, Gh;
};

static int num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return kNumSMs;
  return n > 0 ? n : kNumSMs;
}

static int check_desc(const ygg_mk_desc* d) {
  YGG_CHECK_ARG(d != nullptr, "null descriptor");
  YGG_CHECK_ARG(d->n_layers >= 1 && d->B >= 1 && d->T >= 1, "bad layer / row counts");
  const int M = d->B * d->T;
  if (M > kMaxRows) return ygg_fail(YGG_ERR_UNSUPPORTED, "persistent forward handles <= %d rows (got %d)", kMaxRows, M);
  YGG_CHECK_ARG(d->head_dim == 64 || d->head_dim == 128, "head dim must be 64 or 128");
  YGG_CHECK_ARG(d->n_kv_heads >= 1 && d->n_heads % d->n_kv_heads == 0, "bad head grouping");
  YGG_CHECK_ARG(kQRows % (d->n_heads / d->n_kv_heads) == 0, "group size must divide 128");
  const int qkv = (d->n_heads + 2 * d->n_kv_heads) * d->head_dim;
  YGG_CHECK_ARG(d->d_model % 128 == 0 && qkv % 128 == 0 && d->ffn % 128 == 0 && d->vocab % 128 == 0,
                "matmul widths must be multiples of 128");
  YGG_CHECK_ARG((d->n_heads * d->head_dim) % 64 == 0 && d->ffn % 64 == 0, "matmul depths must be multiples of 64");
  YGG_CHECK_ARG(d->S % 64 == 0 && d->S >= 64, "cache capacity must be a multiple of 64");
  YGG_CHECK_ARG(d->mask_words >= 0 && d->mask_words <= YGG_MAX_MASK_WORDS, "mask too wide");
  YGG_CHECK_ARG(d->vocab / 128 + 1 <= kMaxSegTable && (d->n_heads + 2 * d->n_kv_heads) * d->head_dim / 128 + 1 <= kMaxSegTable &&
                    2 * d->ffn / 128 + 1 <= kMaxSegTable,
                "GEMM too wide for the persistent forward's segment table");
  return YGG_OK;
}

static size_t attn_smem_bytes(int hd) {
  if (getenv("YGG_MK_NOATTN")) return 0;  // A/B only: attention phases become no-ops (wrong results)
  return (hd / 64) * kQRows * 128 + (hd / 64) * kKC * 128 + hd * 128 + kQRows * 128;
}

static int geometry(const ygg_mk_desc* d, Geo* g) {
  if (int rc = check_desc(d)) return rc;
  g->G = d->num_ctas > 0 ? std::min(d->num_ctas, num_sms()) : num_sms();
  g->M = d->B * d->T;
  g->BN = (g->M + 15) / 16 * 16;
  static const int env_look = [] {
    const char* s = getenv("YGG_MK_LOOK");
    return s ? atoi(s) : -1;
  }();
  g->look = d->lookahead >= 0 ? d->lookahead : (env_look >= 0 ? env_look : 0);
  const size_t fixed = 1024 + attn_smem_bytes(d->head_dim) + (2 * kMaxStages + 8) * 8 + 16 + kMaxRows * 16 +
                       kMaxSegTable * 4 + kMaxPend * 32;
  const size_t stage = static_cast<size_t>(kBM) * kBK * 2 + static_cast<size_t>(g->BN) * kBK * 2;
  int st = static_cast<int>((kSmemLimit - fixed) / stage);
  g->stages = std::min(kMaxStages, st);
  if (const char* cap = getenv("YGG_MK_STAGES")) g->stages = std::max(2, std::min(g->stages, atoi(cap)));  // A/B
  if (g->stages < 2) return ygg_fail(YGG_ERR_UNSUPPORTED, "persistent forward: shared memory too small");
  g->smem = fixed + g->stages * stage;
  g->Gh = d->n_heads / d->n_kv_heads;
  g->tok_per_tile = kQRows / g->Gh;
  g->q_tiles = (d->T + g->tok_per_tile - 1) / g->tok_per_tile;
  g->chunks = (d->S + kKC - 1) / kKC;
  const int L = d->n_layers;
  g->nphases = 1 + 6 * L + 1;
  g->nmaps = 6 * L + 1 + 4;
  // Segments per GEMM: sum over CTAs of tiles touched, <= tiles + G.
  const int qkv = (d->n_heads + 2 * d->n_kv_heads) * d->head_dim;
  const int Ns[5] = {qkv, d->d_model, 2 * d->ffn, d->d_model, d->vocab};
  size_t max_seg = 0;
  int itab = 0;
  for (int i = 0; i < 5; ++i) {
    const int tiles = Ns[i] / kBM;
    max_seg = std::max(max_seg, static_cast<size_t>(tiles + g->G));
    itab += (tiles + 1 + g->G) * (i == 4 ? 1 : L);
  }
  g->itab_len = itab;
  g->nctr = 0;
  for (int i = 0; i < 5; ++i) g->nctr += (Ns[i] / kBM) * (i == 4 ? 1 : L);
  g->ws_floats = max_seg * g->BN * kBM;
  g->part_bytes = static_cast<size_t>(g->chunks) * g->M * d->n_heads * (d->head_dim + 2) * sizeof(float);
  g->table_bytes = static_cast<size_t>(g->nmaps) * sizeof(CUtensorMap) + static_cast<size_t>(g->nphases) * sizeof(Phase) +
                   static_cast<size_t>(g->itab_len) * 4 + static_cast<size_t>(g->nctr) * 8 +
                   static_cast<size_t>(g->nphases) * 4 + 192;
  return YGG_OK;
}

static const Plan* plan_of(const void* p) {
  const Plan* q = reinterpret_cast<const Plan*>((reinterpret_cast<uintptr_t>(p) + 63) & ~uintptr_t(63));
  return (p && q->magic == kMagic) ? q : nullptr;
}

}  // namespace mk
}  // namespace ygg

using namespace ygg;
using namespace ygg::mk;

extern "C" {

int ygg_prepare_mk(void) {
  cudaError_t e = cudaFuncSetAttribute(mk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
  if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "persistent forward attribute: %s", cudaGetErrorString(e));
  return YGG_OK;
}

size_t ygg_mk_plan_size(void) { return sizeof(Plan) + 64; }

int ygg_mk_query(const ygg_mk_desc* desc, size_t* table_bytes, size_t* ws_bytes, size_t* attn_part_bytes) {
  Geo g;
  if (int rc = geometry(desc, &g)) return rc;
  if (table_bytes) *table_bytes = g.table_bytes;
  if (ws_bytes) *ws_bytes = 2 * g.ws_floats * sizeof(float);
  if (attn_part_bytes) *attn_part_bytes = g.part_bytes;
  return YGG_OK;
}

int ygg_mk_plan_init(void* plan_mem, const ygg_mk_desc* d, void* table_dev, size_t table_bytes) {
  Geo g;
  if (int rc = geometry(d, &g)) return rc;
  YGG_CHECK_ARG(plan_mem && table_dev, "null plan / table");
  YGG_CHECK_ARG(table_bytes >= g.table_bytes, "table buffer too small");
  YGG_CHECK_ARG((reinterpret_cast<uintptr_t>(table_dev) & 127) == 0, "table buffer must be 128-byte aligned");
  YGG_CHECK_ARG(d->wqkv && d->wo && d->wgu && d->wdown && d->embed && d->lm_head, "null weight pointer");
  YGG_CHECK_ARG(d->tokens && d->pos && d->slot && d->req && d->blk_start && d->blk_len && d->rope_cs && d->cache,
                "null row input");
  YGG_CHECK_ARG(d->mask_words == 0 || d->qmask, "mask words without a mask");
  YGG_CHECK_ARG(d->resid && d->hb && d->q && d->attn && d->mlp && d->logits && d->ss && d->ws && d->attn_part,
                "null activation buffer");
  const int L = d->n_layers, M = g.M, G = g.G, hd = d->head_dim;
  const int qkv = (d->n_heads + 2 * d->n_kv_heads) * hd, qdim = d->n_heads * hd;
  std::vector<CUtensorMap> maps(g.nmaps);
  std::vector<Phase> phases;
  std::vector<int32_t> itab;
  phases.reserve(g.nphases);
  itab.reserve(g.itab_len);
  // maps: [6 per layer: qkv, o, gu, down, K, V^T] [lm] [X: hb, attn, mlp] [Q]
  const int lm_map = 6 * L, xm_hb = lm_map + 1, xm_attn = lm_map + 2, xm_mlp = lm_map + 3, qmap = lm_map + 4;
  const long long kv_rows = static_cast<long long>(d->B) * 2 * d->n_kv_heads;
  for (int l = 0; l < L; ++l) {
    if (int rc = map2d(&maps[6 * l + 0], d->wqkv[l], qkv, d->d_model, kBM)) return rc;
    if (int rc = map2d(&maps[6 * l + 1], d->wo[l], d->d_model, qdim, kBM)) return rc;
    if (int rc = map2d(&maps[6 * l + 2], d->wgu[l], 2LL * d->ffn, d->d_model, kBM)) return rc;
    if (int rc = map2d(&maps[6 * l + 3], d->wdown[l], d->d_model, d->ffn, kBM)) return rc;
    const void* cl = static_cast<const __nv_bfloat16*>(d->cache) + l * d->layer_stride;
    if (int rc = map2d(&maps[6 * l + 4], cl, kv_rows * d->S, hd, kKC)) return rc;          // K rows [.., S][hd]
    if (int rc = map2d(&maps[6 * l + 5], cl, kv_rows * hd, d->S, hd, kKC)) return rc;       // V^T rows [.., hd][S]
  }
  if (int rc = map2d(&maps[lm_map], d->lm_head, d->vocab, d->d_model, kBM)) return rc;
  if (int rc = map2d(&maps[xm_hb], d->hb, M, d->d_model, g.BN)) return rc;
  if (int rc = map2d(&maps[xm_attn], d->attn, M, qdim, g.BN)) return rc;
  if (int rc = map2d(&maps[xm_mlp], d->mlp, M, d->ffn, g.BN)) return rc;
  {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(hd), static_cast<cuuint64_t>(d->n_heads), static_cast<cuuint64_t>(M)};
    cuuint64_t str[2] = {static_cast<cuuint64_t>(hd) * 2, static_cast<cuuint64_t>(d->n_heads) * hd * 2};
    cuuint32_t box[3] = {64, static_cast<cuuint32_t>(g.Gh), static_cast<cuuint32_t>(g.tok_per_tile)};
    if (int rc = encode(&maps[qmap], 3, d->q, dims, str, box)) return rc;
  }
  int wsbuf = 0;
  int nctr = 0;
  bool too_many_tiles = false;
  int nptot = 0;
  auto gemm = [&](int layer, int wmap, int xmap, int N, int K, int epi, int ss_in, int ss_out, int src,
                  int ss_src) -> int {
    Phase P;
    std::memset(&P, 0, sizeof(P));
    P.kind = kGemm;
    P.layer = layer;
    P.wmap = wmap;
    P.xmap = xmap;
    P.N = N;
    P.K = K;
    P.kb = K / kBK;
    const int tiles = N / kBM;
    P.units = tiles * P.kb;
    P.ws = wsbuf;
    wsbuf ^= 1;
    P.epi = epi;
    P.ss_in = ss_in;
    P.ss_out = ss_out;
    P.cache_off = static_cast<long long>(std::min(layer, L - 1)) * d->layer_stride;
    P.ctr = nctr;
    P.dctr = nctr;  // done counters live in a parallel array (same offsets)
    nctr += tiles;
    P.ptot = nptot++;
    P.src = getenv("YGG_MK_DATAFLOW") ? src : -1;  // dataflow X gating (A/B; grid counter by default)
    P.ss_src = ss_src;
    std::vector<int> count(tiles, 0), sbase(G, 0);
    if ((P.units + G - 1) / G / P.kb + 2 > kMaxPend) too_many_tiles = true;
    int seg = 0;
    for (int c = 0; c < G; ++c) {
      const long long u0 = static_cast<long long>(P.units) * c / G, u1 = static_cast<long long>(P.units) * (c + 1) / G;
      sbase[c] = seg;
      if (u1 > u0) {
        const int t0 = static_cast<int>(u0 / P.kb), t1 = static_cast<int>((u1 - 1) / P.kb);
        for (int t = t0; t <= t1; ++t) ++count[t];
        seg += t1 - t0 + 1;
      }
    }
    P.seg_first = static_cast<int>(itab.size());
    int accn = 0;
    for (int t = 0; t < tiles; ++t) {
      itab.push_back(accn);
      accn += count[t];
    }
    itab.push_back(accn);
    P.seg_base = static_cast<int>(itab.size());
    for (int c = 0; c < G; ++c) itab.push_back(sbase[c]);
    P.nsegs = seg;
    phases.push_back(P);
    return static_cast<int>(phases.size()) - 1;
  };
  {
    Phase E;
    std::memset(&E, 0, sizeof(E));
    E.kind = kEmbed;
    E.ss_in = -1;
    E.ss_out = 0;
    phases.push_back(E);
  }
  // Per layer: QKV(+rstd, RoPE, q / KV append) | attention | combine | O(+residual, ss) |
  // gate|up(+rstd, SwiGLU) | down(+residual, ss).  ss buffer 0 feeds QKV and the LM head, 1 feeds gate|up.
  int prev_down = -1;
  for (int l = 0; l < L; ++l) {
    gemm(l, 6 * l + 0, xm_hb, qkv, d->d_model, kEpiQkv, 0, -1, prev_down, prev_down);
    {
      Phase A;
      std::memset(&A, 0, sizeof(A));
      A.kind = kAttn;
      A.layer = l;
      A.kmap = 6 * l + 4;
      A.vmap = 6 * l + 5;
      A.ss_in = A.ss_out = -1;
      A.cache_off = static_cast<long long>(l) * d->layer_stride;
      phases.push_back(A);
      A.kind = kCombine;
      phases.push_back(A);
    }
    const int po = gemm(l, 6 * l + 1, xm_attn, d->d_model, qdim, kEpiResid, -1, 1, -1, -1);
    const int pg = gemm(l, 6 * l + 2, xm_hb, 2 * d->ffn, d->d_model, kEpiSwiglu, 1, -1, po, po);
    prev_down = gemm(l, 6 * l + 3, xm_mlp, d->d_model, d->ffn, kEpiResid, -1, 0, pg, -1);
  }
  gemm(L, lm_map, xm_hb, d->vocab, d->d_model, kEpiStore, 0, -1, prev_down, prev_down);
  if (too_many_tiles) return ygg_fail(YGG_ERR_UNSUPPORTED, "persistent forward: too many tiles per CTA in one GEMM");
  if (static_cast<int>(phases.size()) != g.nphases || static_cast<int>(itab.size()) > g.itab_len || nctr > g.nctr)
    return ygg_fail(YGG_ERR_VALUE, "persistent forward: internal program size mismatch");
  // Device table: maps | phases | itab | tile-group counters | barrier counter.
  std::vector<unsigned char> blob(g.table_bytes, 0);
  size_t off = 0;
  std::memcpy(blob.data() + off, maps.data(), maps.size() * sizeof(CUtensorMap));
  const size_t maps_off = off;
  off += maps.size() * sizeof(CUtensorMap);
  const size_t ph_off = off;
  std::memcpy(blob.data() + off, phases.data(), phases.size() * sizeof(Phase));
  off += static_cast<size_t>(g.nphases) * sizeof(Phase);
  const size_t it_off = off;
  std::memcpy(blob.data() + off, itab.data(), itab.size() * 4);
  off += static_cast<size_t>(g.itab_len) * 4;
  const size_t ctr_off = off;
  off += static_cast<size_t>(g.nctr) * 4;
  const size_t dctr_off = off;
  off += static_cast<size_t>(g.nctr) * 4;
  const size_t ptot_off = off;
  off += static_cast<size_t>(g.nphases) * 4;
  const size_t lctr_off = off;
  off += 4;
  const size_t bar_off = (off + 63) / 64 * 64;
  if (bar_off + 4 > g.table_bytes) return ygg_fail(YGG_ERR_VALUE, "persistent forward: table overflow");
  cudaError_t e = cudaMemcpy(table_dev, blob.data(), g.table_bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "persistent forward table upload: %s", cudaGetErrorString(e));
  Plan* pl = reinterpret_cast<Plan*>((reinterpret_cast<uintptr_t>(plan_mem) + 63) & ~uintptr_t(63));
  std::memset(pl, 0, sizeof(Plan));
  pl->magic = kMagic;
  pl->grid = G;
  pl->smem = g.smem;
  Args& a = pl->args;
  const bool use_bank = !getenv("YGG_MK_GLOBAL_MAPS");
  a.bank_n = use_bank ? std::min(static_cast<int>(maps.size()), kBankMaps) : 0;
  if (static_cast<int>(maps.size()) > kBankMaps) a.bank_n = 0;  // all-or-nothing keeps the lookup uniform
  for (int i = 0; i < a.bank_n; ++i) pl->bank.m[i] = maps[i];
  unsigned char* tb = static_cast<unsigned char*>(table_dev);
  a.maps = reinterpret_cast<const CUtensorMap*>(tb + maps_off);
  a.phases = reinterpret_cast<const Phase*>(tb + ph_off);
  a.itab = reinterpret_cast<const int32_t*>(tb + it_off);
  a.bar = reinterpret_cast<unsigned*>(tb + bar_off);
  a.ctr = reinterpret_cast<unsigned*>(tb + ctr_off);
  a.dctr = reinterpret_cast<unsigned*>(tb + dctr_off);
  a.ptot = reinterpret_cast<unsigned*>(tb + ptot_off);
  a.lctr = reinterpret_cast<unsigned*>(tb + lctr_off);
  a.nphases = g.nphases;
  if (const char* stop = getenv("YGG_MK_STOP")) a.nphases = std::max(1, std::min(g.nphases, atoi(stop)));  // debugging
  a.G = G;
  a.M = M;
  a.BN = g.BN;
  a.stages = g.stages;
  a.look = g.look;
  a.pf_maps = getenv("YGG_MK_PFMAP") ? atoi(getenv("YGG_MK_PFMAP")) : 1;
  a.xflags = getenv("YGG_MK_XFLAGS") ? atoi(getenv("YGG_MK_XFLAGS")) : 0;
  if (getenv("YGG_MK_NOATTN")) a.xflags |= 8;
  a.attn_bytes = static_cast<int>(attn_smem_bytes(hd));
  a.d = d->d_model;
  a.Hq = d->n_heads;
  a.Hkv = d->n_kv_heads;
  a.hd = hd;
  a.S = d->S;
  a.T = d->T;
  a.B = d->B;
  a.F = d->ffn;
  a.V = d->vocab;
  a.Gh = g.Gh;
  a.tok_per_tile = g.tok_per_tile;
  a.q_tiles = g.q_tiles;
  a.chunks = g.chunks;
  a.mask_words = d->mask_words;
  a.qmap = qmap;
  a.eps = d->eps;
  a.scale_log2 = d->attn_scale * 1.4426950408889634f;
  a.embed = static_cast<const __nv_bfloat16*>(d->embed);
  a.tokens = d->tokens;
  a.pos = d->pos;
  a.slot = d->slot;
  a.req = d->req;
  a.blk_start = d->blk_start;
  a.blk_len = d->blk_len;
  a.qmask = d->qmask;
  a.rope_cs = reinterpret_cast<const float2*>(d->rope_cs);
  a.cache = static_cast<__nv_bfloat16*>(d->cache);
  a.resid = d->resid;
  a.hb = static_cast<__nv_bfloat16*>(d->hb);
  a.q = static_cast<__nv_bfloat16*>(d->q);
  a.attn = static_cast<__nv_bfloat16*>(d->attn);
  a.mlp = static_cast<__nv_bfloat16*>(d->mlp);
  a.logits = d->logits;
  a.ss = d->ss;
  a.ws = d->ws;
  a.ws_stride = static_cast<long long>(g.ws_floats);
  a.opart = d->attn_part;
  a.ml = d->attn_part + static_cast<size_t>(g.chunks) * M * d->n_heads * hd;
  a.dbg = reinterpret_cast<unsigned long long*>(d->dbg);
  return YGG_OK;
}

int ygg_mk_run(const void* plan, ygg_stream_t stream) {
  const Plan* p = plan_of(plan);
  YGG_CHECK_ARG(p != nullptr, "invalid persistent-forward plan");
  YGG_LAUNCH_PDL(mk_kernel, dim3(p->grid), dim3(kThreads), p->smem, reinterpret_cast<cudaStream_t>(stream), p->args,
                 p->bank);
  return YGG_OK;
}

}  // extern "C"
