// Tree kernels of the speculative step: EGT expansion (K1), mask (K7), knapsack prune (K6),
// acceptance walk (K5) and KV compaction.  Compiled with --fmad=false: every f64 expression
// here must round exactly like the CPython float arithmetic of the reference.
//
// Reference (pkg/src/specsim/): egt.py:65-114 (candidates, grow_step), egt.py:150-282
// (SubtreeKnapsack, prune_verify), acceptance.py:176-184 (path_products), acceptance.py:221-241
// (sample_with_probs), token_tree.py:146-168 (subtree), token_tree.py:205-218 (build_mask),
// latency.py:68-82,154-161 (latency_at, tree_speedup).
#include "common.cuh"
#include "host_util.h"

#include <cfloat>
#include <cmath>

namespace ygg {

constexpr double kSiblingTol = 1e-9;  // token_tree.py:31
enum : int32_t { kFlagShortfall = 1, kFlagContract = 2, kFlagCapacity = 4, kFlagStopped = 8, kFlagIndex = 16 };

// ===========================================================================
// K1a: softmax + top-k per row (DrafterDistribution.candidates realised on draft logits).
// Phase 1: each CTA scans a chunk of one row: chunk max, f64 sum of exp, local top-k by
// (logit desc, token asc).  Phase 2: one CTA per row merges chunks deterministically.
// ===========================================================================
constexpr int kTopkChunk = 4096;
constexpr int kTopkThreads = 256;
using TopkChunkOut = TopkPartial;

YGG_DEV bool better(float va, int ta, float vb, int tb) { return topk_better(va, ta, vb, tb); }
YGG_DEV unsigned long long topk_key(float v, int tok) {  // larger key == better (v desc, tok asc)
  const uint32_t b = __float_as_uint(v + 0.0f);  // -0 -> +0: equal values order by token, like better()
  const uint32_t ord = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return (static_cast<unsigned long long>(ord) << 32) | static_cast<uint32_t>(~static_cast<uint32_t>(tok));
}
YGG_DEV float key_val(unsigned long long key) {
  const uint32_t ord = static_cast<uint32_t>(key >> 32);
  return __uint_as_float((ord & 0x80000000u) ? (ord & 0x7fffffffu) : ~ord);
}
YGG_DEV int key_tok(unsigned long long key) { return static_cast<int>(~static_cast<uint32_t>(key)); }
constexpr unsigned long long kNoKey = 0ull;  // below every real key (even -inf with token 2^31 - 1)
YGG_DEV unsigned long long warp_max_key(unsigned long long key) {
  const uint32_t hi = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(key >> 32));
  const uint32_t lo = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(key >> 32) == hi ? static_cast<uint32_t>(key) : 0u);
  return (static_cast<unsigned long long>(hi) << 32) | lo;
}

template <typename T>
__global__ void __launch_bounds__(kTopkThreads) topk_phase1(const T* __restrict__ logits, int V, int ld, int k,
                                                            float inv_temp, int nchunks, TopkChunkOut* out) {
  pdl_wait();
  const int row = blockIdx.y, chunk = blockIdx.x;
  const int begin = chunk * kTopkChunk, end = min(V, begin + kTopkChunk);
  __shared__ float sv[kTopkChunk];
  __shared__ float red_f[kTopkThreads / 32];
  __shared__ double red_d[kTopkThreads / 32];
  __shared__ int red_i[kTopkThreads / 32];
  const T* src = logits + static_cast<size_t>(row) * ld;
  constexpr int kPer = kTopkChunk / kTopkThreads;
  float lmax = -INFINITY;
  {
    float xv[kPer];  // all of this thread's loads in flight together
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = begin + threadIdx.x + j * kTopkThreads;
      xv[j] = i < end ? to_f32(src[i]) * inv_temp : -INFINITY;
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = begin + threadIdx.x + j * kTopkThreads;
      if (i < end) sv[i - begin] = xv[j];
      lmax = fmaxf(lmax, xv[j]);
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  lmax = warp_max(lmax);
  if (lane == 0) red_f[warp] = lmax;
  __syncthreads();
  float cmax = red_f[0];
  for (int w = 1; w < kTopkThreads / 32; ++w) cmax = fmaxf(cmax, red_f[w]);
  double s = 0.0;
  for (int i = begin + threadIdx.x; i < end; i += blockDim.x) s += exp(static_cast<double>(sv[i - begin]) - cmax);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red_d[warp] = s;
  __syncthreads();
  TopkChunkOut* o = out + static_cast<size_t>(row) * nchunks + chunk;
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < kTopkThreads / 32; ++w) tot += red_d[w];
    o->max_s = cmax;
    o->sum_exp = tot;
  }
  // Top-k of the chunk by a tournament over 64-bit keys ordered exactly like better() (logit desc,
  // token asc; NaN excluded): every thread keeps its 16 elements as keys, its best and second best;
  // each warp pops its k best with two redux.sync max reductions per round — a lane's next key after
  // a pop is its cached second best, or (third pop onwards, rare) the largest of its keys below the
  // popped one (keys are unique) — then warp 0 pops the chunk's k best over the 8 warps' lists.
  constexpr int NW = kTopkThreads / 32;
  __shared__ unsigned long long wsel[NW][kTopkMaxK];
  unsigned long long mk[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int i = begin + threadIdx.x + j * kTopkThreads;
    const float v = i < end ? sv[i - begin] : __int_as_float(0x7fc00000);
    mk[j] = isnan(v) ? kNoKey : topk_key(v, i);
  }
  unsigned long long cur = kNoKey, second = kNoKey;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const unsigned long long x = mk[j];
    if (x > cur) {
      second = cur;
      cur = x;
    } else if (x > second) {
      second = x;
    }
  }
  int pops = 0;
  for (int r = 0; r < k; ++r) {
    const unsigned long long win = warp_max_key(cur);
    if (lane == 0) wsel[warp][r] = win;
    if (win != kNoKey && cur == win) {  // keys are unique (distinct indices): exactly one lane pops
      if (++pops == 1) {
        cur = second;
      } else {
        unsigned long long nb = kNoKey;
#pragma unroll
        for (int j = 0; j < kPer; ++j)
          if (mk[j] < win && mk[j] > nb) nb = mk[j];
        cur = nb;
      }
    }
  }
  __syncthreads();
  if (warp == 0) {
    int hp = 0;
    unsigned long long ck = lane < NW ? wsel[lane][0] : kNoKey;
    for (int r = 0; r < k; ++r) {
      const unsigned long long win = warp_max_key(ck);
      if (lane == 0) {
        o->val[r] = win == kNoKey ? -INFINITY : key_val(win);
        o->tok[r] = win == kNoKey ? -1 : key_tok(win);
      }
      if (win != kNoKey && ck == win) {
        ++hp;
        ck = hp < k ? wsel[lane][hp] : kNoKey;
      }
    }
  }
  pdl_launch_dependents();
}

__global__ void __launch_bounds__(kTopkThreads) topk_phase2(const TopkChunkOut* __restrict__ chunks, int nchunks,
                                                            int k, int32_t* out_tok, double* out_prob,
                                                            float* out_stats) {
  pdl_wait();
  const int row = blockIdx.x;
  const TopkChunkOut* c = chunks + static_cast<size_t>(row) * nchunks;
  extern __shared__ unsigned char smem_raw[];
  float* cv = reinterpret_cast<float*>(smem_raw);
  int* ct = reinterpret_cast<int*>(cv + nchunks * k);
  __shared__ float gmax_s;
  __shared__ double z_s;
  __shared__ float sel_v[kTopkMaxK];
  __shared__ int sel_t[kTopkMaxK];
  const int n = nchunks * k;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    cv[i] = c[i / k].val[i % k];
    ct[i] = c[i / k].tok[i % k];
  }
  if (threadIdx.x == 0) {
    float m = -INFINITY;
    for (int j = 0; j < nchunks; ++j) m = fmaxf(m, c[j].max_s);
    double z = 0.0;  // fixed chunk order => deterministic
    for (int j = 0; j < nchunks; ++j) z += c[j].sum_exp * exp(static_cast<double>(c[j].max_s) - m);
    gmax_s = m;
    z_s = z;
  }
  __syncthreads();
  // Rank every candidate by (logit desc, token asc); the first k win.
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int ti = ct[i];
    if (ti < 0) continue;
    float vi = cv[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      int tj = ct[j];
      if (tj >= 0 && better(cv[j], tj, vi, ti)) ++rank;
    }
    if (rank < k) { sel_v[rank] = vi; sel_t[rank] = ti; }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double m = gmax_s;
    double e[kTopkMaxK];
    double topsum = 0.0;
    for (int r = 0; r < k; ++r) {
      e[r] = exp(static_cast<double>(sel_v[r]) - m);
      topsum += e[r];
    }
    const double z = fmax(z_s, topsum);  // rounding guard: sum(top-k probs) <= 1
    double p[kTopkMaxK];
    int t[kTopkMaxK];
    for (int r = 0; r < k; ++r) { p[r] = e[r] / z; t[r] = sel_t[r]; }
    // Final order (prob desc, token asc): exp is monotone, so only equal-prob runs can move.
    for (int a = 1; a < k; ++a) {
      double pa = p[a];
      int ta = t[a];
      int b = a - 1;
      while (b >= 0 && (p[b] < pa || (p[b] == pa && t[b] > ta))) { p[b + 1] = p[b]; t[b + 1] = t[b]; --b; }
      p[b + 1] = pa;
      t[b + 1] = ta;
    }
    for (int r = 0; r < k; ++r) {
      out_tok[static_cast<size_t>(row) * k + r] = t[r];
      out_prob[static_cast<size_t>(row) * k + r] = p[r];
    }
    if (out_stats) {
      out_stats[2 * row] = static_cast<float>(m);
      out_stats[2 * row + 1] = static_cast<float>(m + log(z_s));
    }
  }
  pdl_launch_dependents();
}

// Phase 2 for <= 512 chunks (thread t owns chunks t and t + 256).  One round of vector loads stages
// every chunk's stats and sorted list (lists in shared memory); block max, then the f64 normaliser
// sum_j sum_exp_j * exp(max_j - M) (per-thread terms, warp xor tree, warps in order: fixed order,
// deterministic).  Candidates are packed into 64-bit keys ordered exactly like (logit desc, token
// asc), so a tournament round is two redux.sync max reductions instead of a shuffle tree: each warp
// pops its k best over its chunk heads, then warp 0 pops the block's k best over the warps' lists.
constexpr int kMergeOwn = 2;

struct L2Regions {  // weights of the next pass to pull into L2 while the merge / grow leave HBM idle
  const char* ptr[4];
  unsigned long long bytes[4];
};

__global__ void __launch_bounds__(kTopkThreads) topk_merge_kernel(const TopkPartial* __restrict__ chunks, int nchunks,
                                                                  int k, int32_t* out_tok, double* out_prob,
                                                                  float* out_stats, unsigned long long* trace,
                                                                  L2Regions pf, int stage) {
  if (threadIdx.x == 0) { trace_min(trace, 0); trace_max(trace, 6); }
  pdl_wait();
  if (threadIdx.x == 0) { trace_min(trace, 1); trace_max(trace, 7); }
  if (threadIdx.x < 4 && pf.ptr[threadIdx.x]) {  // one thread per region, slices over the CTAs
    const int rg = threadIdx.x;
    const size_t per = ((pf.bytes[rg] / gridDim.x) + 255) & ~static_cast<size_t>(255);
    const size_t b0 = blockIdx.x * per, b1 = b0 + per < pf.bytes[rg] ? b0 + per : pf.bytes[rg];
    for (size_t o = b0; o < b1; o += 65536) {
      const uint32_t n = static_cast<uint32_t>(b1 - o < 65536 ? ((b1 - o) & ~static_cast<size_t>(15)) : 65536);
      if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf.ptr[rg] + o), "r"(n) : "memory");
    }
  }
  const int row = blockIdx.x;
  const TopkPartial* c = chunks + static_cast<size_t>(row) * nchunks;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  constexpr int NW = kTopkThreads / 32;
  __shared__ float red_f[NW];
  __shared__ double red_d[NW];
  __shared__ float sel_v[kTopkMaxK];
  __shared__ int sel_t[kTopkMaxK];
  __shared__ unsigned long long wsel[NW][kTopkMaxK];
  extern __shared__ __align__(16) unsigned long long merge_keys[];  // [nchunks][k] candidate keys
  // stage: this row's partials ([nchunks] x 272 B, contiguous) arrive in shared memory by one bulk
  // copy — the TMA engine streams them instead of every thread waiting on its own L2 round trips.
  if (stage) {
    __shared__ __align__(8) uint64_t sbar;
    TopkPartial* sp = reinterpret_cast<TopkPartial*>(merge_keys + ((static_cast<size_t>(nchunks) * k + 1) & ~static_cast<size_t>(1)));
    if (t == 0) {
      mbar_init(&sbar, 1);
      fence_barrier_init();
      const uint32_t bytes = static_cast<uint32_t>(nchunks) * static_cast<uint32_t>(sizeof(TopkPartial));
      mbar_arrive_expect_tx(&sbar, bytes);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(smem_u32(sp)), "l"(reinterpret_cast<uint64_t>(c)), "r"(bytes), "r"(smem_u32(&sbar))
          : "memory");
    }
    __syncthreads();
    mbar_wait(&sbar, 0);
    c = sp;
  }
  float cm[kMergeOwn];
  double cs[kMergeOwn];
  float lm = -INFINITY;
  // Every load of both owned chunks issued before any is used (k <= 8: two float4 + two int4 per
  // chunk; larger k falls back to a loop).
  float4 v4[kMergeOwn][2];
  int4 t4[kMergeOwn][2];
#pragma unroll
  for (int o = 0; o < kMergeOwn; ++o) {
    const int j = t + o * kTopkThreads;
    cm[o] = -INFINITY;
    cs[o] = 0.0;
    if (j < nchunks) {
      const TopkPartial* cj = c + j;
      cm[o] = stage ? cj->max_s : __ldcg(&cj->max_s);
      cs[o] = stage ? cj->sum_exp : __ldcg(&cj->sum_exp);
      if (k <= 8) {  // val / tok are 16-byte aligned in TopkPartial
        v4[o][0] = stage ? *reinterpret_cast<const float4*>(cj->val) : __ldcg(reinterpret_cast<const float4*>(cj->val));
        t4[o][0] = stage ? *reinterpret_cast<const int4*>(cj->tok) : __ldcg(reinterpret_cast<const int4*>(cj->tok));
        if (k > 4) {
          v4[o][1] = stage ? *reinterpret_cast<const float4*>(cj->val + 4) : __ldcg(reinterpret_cast<const float4*>(cj->val + 4));
          t4[o][1] = stage ? *reinterpret_cast<const int4*>(cj->tok + 4) : __ldcg(reinterpret_cast<const int4*>(cj->tok + 4));
        }
      }
    }
  }
#pragma unroll
  for (int o = 0; o < kMergeOwn; ++o) {
    const int j = t + o * kTopkThreads;
    if (j < nchunks) {
      unsigned long long* dst = merge_keys + static_cast<size_t>(j) * k;
      if (k <= 8) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const float vv[4] = {v4[o][hh].x, v4[o][hh].y, v4[o][hh].z, v4[o][hh].w};
          const int tt[4] = {t4[o][hh].x, t4[o][hh].y, t4[o][hh].z, t4[o][hh].w};
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (4 * hh + u < k) dst[4 * hh + u] = tt[u] < 0 ? kNoKey : topk_key(vv[u], tt[u]);
        }
      } else {
        const TopkPartial* cj = c + j;
        for (int r = 0; r < k; ++r) dst[r] = cj->tok[r] < 0 ? kNoKey : topk_key(cj->val[r], cj->tok[r]);
      }
    }
    lm = fmaxf(lm, cm[o]);
  }
  const float wm = warp_max(lm);
  if (lane == 0) red_f[warp] = wm;
  __syncthreads();
  if (t == 0) trace_max(trace, 3);
  float gm = red_f[0];
  for (int w = 1; w < NW; ++w) gm = fmaxf(gm, red_f[w]);
  double z = 0.0;
#pragma unroll
  for (int o = 0; o < kMergeOwn; ++o)
    if (cm[o] != -INFINITY) z += cs[o] * exp(static_cast<double>(cm[o]) - static_cast<double>(gm));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  if (lane == 0) red_d[warp] = z;
  if (t == 0) trace_max(trace, 4);
  // (1) per-warp tournament over the heads of the lanes' chunk lists
  int h[kMergeOwn];
  unsigned long long hk[kMergeOwn];
#pragma unroll
  for (int o = 0; o < kMergeOwn; ++o) {
    const int j = t + o * kTopkThreads;
    h[o] = 0;
    hk[o] = j < nchunks ? merge_keys[static_cast<size_t>(j) * k] : kNoKey;
  }
  for (int r = 0; r < k; ++r) {
    unsigned long long best = hk[0];
#pragma unroll
    for (int o = 1; o < kMergeOwn; ++o) best = hk[o] > best ? hk[o] : best;
    const unsigned long long win = warp_max_key(best);
    if (lane == 0) wsel[warp][r] = win;
    if (win == kNoKey) continue;  // warp-uniform
#pragma unroll
    for (int o = 0; o < kMergeOwn; ++o) {
      if (hk[o] == win) {  // keys are unique (distinct tokens): exactly one lane / chunk pops
        const int j = t + o * kTopkThreads;
        ++h[o];
        hk[o] = h[o] < k ? merge_keys[static_cast<size_t>(j) * k + h[o]] : kNoKey;
      }
    }
  }
  __syncthreads();
  // (2) warp 0: lanes 0..NW-1 each own one warp's sorted winners
  if (warp == 0) {
    int hp = 0;
    unsigned long long ck = lane < NW ? wsel[lane][0] : kNoKey;
    for (int r = 0; r < k; ++r) {
      const unsigned long long win = warp_max_key(ck);
      if (lane == 0) {
        sel_v[r] = key_val(win);
        sel_t[r] = win == kNoKey ? -1 : key_tok(win);
      }
      if (win != kNoKey && ck == win) {
        ++hp;
        ck = hp < k ? wsel[lane][hp] : kNoKey;
      }
    }
  }
  __syncthreads();
  if (t == 0) trace_max(trace, 5);
  // Probabilities and final order, one thread per selected candidate: p = e / max(Z, sum of the
  // top-k e) (rounding guard: the top-k probabilities never sum above 1), then each entry's rank
  // under (prob desc, token asc) — exp is monotone, so only equal-probability runs move.
  __shared__ double sel_e[kTopkMaxK];
  __shared__ double s_zz, s_zs;
  __shared__ int s_kk;
  if (t < k) sel_e[t] = sel_t[t] >= 0 ? exp(static_cast<double>(sel_v[t]) - static_cast<double>(gm)) : 0.0;
  __syncthreads();
  if (t == 0) {
    double zs = 0.0;
    for (int w = 0; w < NW; ++w) zs += red_d[w];
    double topsum = 0.0;
    int kk = 0;
    for (int r = 0; r < k; ++r) {
      if (sel_t[r] < 0) break;
      topsum += sel_e[r];
      ++kk;
    }
    s_zs = zs;
    s_zz = fmax(zs, topsum);
    s_kk = kk;
  }
  __syncthreads();
  if (t < k) {
    const int kk = s_kk;
    if (t < kk) {
      const double pt = sel_e[t] / s_zz;
      const int tt = sel_t[t];
      int rank = 0;
      for (int j = 0; j < kk; ++j) {
        const double pj = sel_e[j] / s_zz;
        if (pj > pt || (pj == pt && sel_t[j] < tt)) ++rank;
      }
      out_tok[static_cast<size_t>(row) * k + rank] = tt;
      out_prob[static_cast<size_t>(row) * k + rank] = pt;
    } else {
      out_tok[static_cast<size_t>(row) * k + t] = -1;
      out_prob[static_cast<size_t>(row) * k + t] = 0.0;
    }
  }
  if (t == 0 && out_stats) {
    out_stats[2 * row] = static_cast<float>(gm);
    out_stats[2 * row + 1] = static_cast<float>(static_cast<double>(gm) + log(s_zs));
  }
  pdl_launch_dependents();
  if (threadIdx.x == 0) trace_max(trace, 2);
}

// ===========================================================================
// K1b: one grow_step per request (egt.py:83-114).
// ===========================================================================
constexpr int kGrowThreads = 256;
constexpr int kGrowMaxCand = 1024;
constexpr int kGrowMaxFront = 256;

__global__ void __launch_bounds__(kGrowThreads) grow_level_kernel(ygg_tree t, int Fmax, int k, int w_draft,
                                                                  const int32_t* __restrict__ cand_tok,
                                                                  const double* __restrict__ cand_prob,
                                                                  const int32_t* __restrict__ cand_n,
                                                                  unsigned long long* trace) {
  if (threadIdx.x == 0) trace_min(trace, 0);
  const int b = blockIdx.x;
  __shared__ double sc[kGrowMaxCand];
  __shared__ int spar[kGrowMaxCand];
  __shared__ int srank[kGrowMaxCand];
  __shared__ int sslot[kGrowMaxCand];  // (frontier row, rank) packed
  __shared__ int s_n, s_ok, s_added;
  __shared__ int s_apar[kGrowMaxCand];     // attached nodes by rank: parent, surrogate prob
  __shared__ double s_aprob[kGrowMaxCand];
  __shared__ int s_fn, s_size0, s_flags;
  __shared__ int s_cnt[kGrowMaxFront], s_par[kGrowMaxFront], s_off[kGrowMaxFront + 1];
  __shared__ double s_cum[kGrowMaxFront];
  int32_t* flags = t.flags + b;
  const size_t tb = static_cast<size_t>(b) * t.cap;
  const int32_t* frontier = t.frontier + tb;
  // One round of independent loads: the tree header (thread 0) and, speculatively for every
  // possible frontier row f < Fmax (thread f), its candidate count, its k probabilities (contract
  // check: range, descending, running sum — _checked_candidates, egt.py:65-80), its parent node and
  // the parent's path probability.  Nothing below re-reads global candidate data.
  if (threadIdx.x == 0) {
    s_ok = 1;
    s_fn = t.frontier_n[b];
    s_size0 = t.size[b];
    s_flags = *flags;
  }
  const int fmax = min(Fmax, kGrowMaxFront);
  if (threadIdx.x < fmax) {
    const int f = threadIdx.x;
    const int cnt = cand_n ? cand_n[static_cast<size_t>(b) * Fmax + f] : k;
    const int parent = frontier[f];
    s_cnt[f] = cnt;
    s_par[f] = parent;
    s_cum[f] = (parent >= 0 && parent < t.cap) ? t.cum[tb + parent] : 0.0;
  }
  // The header, frontier rows and candidate counts come from kernels long done (the previous grow /
  // the level inputs); only the candidate probabilities come from the merge just before: wait here.
  pdl_wait();
  if (threadIdx.x == 0) trace_min(trace, 1);
  __syncthreads();
  const int fn = s_fn, size0 = s_size0;
  if (s_flags & kFlagStopped) return;
  if (threadIdx.x < min(fn, fmax)) {
    const int f = threadIdx.x;
    const int cnt = s_cnt[f];
    const double* pr = cand_prob + (static_cast<size_t>(b) * Fmax + f) * k;
    double total = 0.0, prev = INFINITY;
    bool bad = cnt < 0 || cnt > k;
    for (int r = 0; r < cnt && !bad; ++r) {
      double p = pr[r];
      if (!(p >= 0.0 && p <= 1.0)) bad = true;
      if (p > prev) bad = true;
      prev = p;
      total = total + p;
    }
    if (total > 1.0 + kSiblingTol) bad = true;
    if (bad) atomicExch(&s_ok, 0);
  }
  if (threadIdx.x == 0) {  // candidate offsets of the frontier rows, from shared memory
    int acc = 0;
    for (int f = 0; f < fn && f < kGrowMaxFront; ++f) {
      s_off[f] = acc;
      acc += s_cnt[f];
    }
    s_off[min(fn, kGrowMaxFront)] = acc;
    s_n = min(acc, kGrowMaxCand);
  }
  __syncthreads();
  if (!s_ok) {
    if (threadIdx.x == 0) atomicOr(flags, kFlagContract);
    return;
  }
  // Scored candidates in (frontier row, rank) order, one thread per candidate slot.
  for (int i = threadIdx.x; i < fn * k; i += blockDim.x) {
    const int f = i / k, r = i % k;
    if (f >= kGrowMaxFront) continue;
    const int cnt = s_off[f + 1] - s_off[f];
    const int n = s_off[f] + r;
    if (r >= cnt || n >= kGrowMaxCand) continue;
    sc[n] = s_cum[f] * cand_prob[(static_cast<size_t>(b) * Fmax + f) * k + r];
    spar[n] = s_par[f];
    sslot[n] = f * k + r;
  }
  __syncthreads();
  const int n = s_n;
  // Rank by (-score, parent, rank); equal keys cannot occur (parent, rank) unique.
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double si = sc[i];
    const int pi = spar[i], ri = sslot[i] % k;
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double sj = sc[j];
      const int pj = spar[j], rj = sslot[j] % k;
      if (sj > si || (sj == si && (pj < pi || (pj == pi && rj < ri)))) ++rank;
    }
    srank[i] = rank;
  }
  __syncthreads();
  const int added = min(n, w_draft);
  if (threadIdx.x == 0) {
    s_added = added;
    if (size0 + added > t.cap) atomicOr(flags, kFlagCapacity);
  }
  __syncthreads();
  if (size0 + added > t.cap) return;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int r = srank[i];
    if (r >= added) continue;
    const int idx = size0 + r;
    const int parent = spar[i];
    const int f = sslot[i] / k, rk = sslot[i] % k;
    const size_t ci = (static_cast<size_t>(b) * Fmax + f) * k + rk;
    const double pr = cand_prob[ci];
    t.token[tb + idx] = cand_tok[ci];
    t.parent[tb + idx] = parent;
    t.depth[tb + idx] = t.depth[tb + parent] + 1;
    t.prob[tb + idx] = pr;
    t.cum[tb + idx] = sc[i];
    s_apar[r] = parent;
    s_aprob[r] = pr;
    uint32_t* row = t.mask + (tb + idx) * t.mask_words;
    const uint32_t* prow = t.mask + (tb + parent) * t.mask_words;
    for (int w = 0; w < t.mask_words; ++w) row[w] = prow[w] | ((idx >> 5) == w ? (1u << (idx & 31)) : 0u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // add_child sibling-sum check in insertion order (token_tree.py:79-83).
    for (int i = 0; i < added; ++i) {
      const int p = s_apar[i];
      double s = 0.0;
      for (int j = 0; j < i; ++j)
        if (s_apar[j] == p) s = s + s_aprob[j];
      if (s + s_aprob[i] > 1.0 + kSiblingTol) atomicOr(flags, kFlagContract);
    }
    int32_t* fr = t.frontier + tb;
    for (int i = 0; i < added; ++i) fr[i] = size0 + i;
    if (added > 0) t.frontier_n[b] = added;
    t.size[b] = size0 + added;
    int fl = 0;
    if (added < w_draft) fl |= kFlagShortfall;
    if (added == 0) fl |= kFlagStopped;  // grow_egt breaks when nothing was added (egt.py:145-146)
    if (fl) atomicOr(flags, fl);
  }
  pdl_launch_dependents();
  if (threadIdx.x == 0) trace_max(trace, 2);
}

// ===========================================================================
// K7: build_mask (token_tree.py:205-218): row(i) = row(parent) | bit(i), one warp per tree.
// ===========================================================================
__global__ void build_mask_kernel(ygg_tree t) {
  pdl_wait();
  const int b = blockIdx.x, lane = threadIdx.x;
  const size_t tb = static_cast<size_t>(b) * t.cap;
  const int n = t.size[b];
  for (int i = 0; i < t.cap; ++i) {
    const int p = (i < n) ? t.parent[tb + i] : -1;
    if (i < n && i > 0 && !(p >= 0 && p < i)) {
      if (lane == 0) atomicOr(t.flags + b, kFlagIndex);
    }
    if (lane < t.mask_words) {
      uint32_t v = 0;
      if (i < n) {
        if (i > 0 && p >= 0 && p < i) v = t.mask[(tb + p) * t.mask_words + lane];
        if ((i >> 5) == lane) v |= 1u << (i & 31);
      }
      t.mask[(tb + i) * t.mask_words + lane] = v;
    }
    __syncwarp();
  }
  pdl_launch_dependents();
}

// ===========================================================================
// K6: path_products + SubtreeKnapsack + latency-aware prune + pick (egt.py:150-282).
// ===========================================================================
YGG_DEV double latency_at_dev(const ygg_profile& p, int width) {
  // latency.py:68-82, operation order preserved (compiled without FMA contraction).
  if (width <= p.width[0]) return p.latency_us[0];
  const int n = p.n;
  if (width >= p.width[n - 1]) {
    const double w0 = p.width[n - 2], l0 = p.latency_us[n - 2];
    const double w1 = p.width[n - 1], l1 = p.latency_us[n - 1];
    const double slope = (l1 - l0) / (w1 - w0);
    return l1 + slope * static_cast<double>(width - p.width[n - 1]);
  }
  int hi = 0;
  while (hi < n && p.width[hi] <= width) ++hi;  // bisect_right
  const double l0 = p.latency_us[hi - 1], l1 = p.latency_us[hi];
  return l0 + (l1 - l0) * static_cast<double>(width - p.width[hi - 1]) /
                  static_cast<double>(p.width[hi] - p.width[hi - 1]);
}

YGG_DEV double tree_speedup_dev(const ygg_profile_pair& pp, double aal, int w_draft, int d_draft, int w_verify) {
  // latency.py:154-161: aal * T_v(1) / (D * T_d(W) + T_v(w_verify + 1))
  const double draft_cost = static_cast<double>(d_draft) * latency_at_dev(pp.drafter, w_draft);
  const double verify_cost = latency_at_dev(pp.verifier, w_verify + 1);
  return aal * latency_at_dev(pp.verifier, 1) / (draft_cost + verify_cost);
}

constexpr int kKnapThreads = 256;

__global__ void __launch_bounds__(kKnapThreads) knapsack_prune_kernel(
    ygg_tree t, const double* __restrict__ probs, const ygg_profile_pair* __restrict__ prof, ygg_prune_args args,
    int32_t* keep_idx, int32_t* new_idx, int32_t* w_verify, double* expected_aal, double* speedup,
    double* aal_at_cap, double* speedup_at_cap, double* best_out, uint8_t* alloc_out) {
  pdl_wait();
  const int b = blockIdx.x;
  const size_t tb = static_cast<size_t>(b) * t.cap;
  const int N = t.size[b];
  const int cap = min(args.max_verify, N);
  const int R = cap + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* best = reinterpret_cast<double*>(smem_raw);                       // [N][R]
  double* gain = best + static_cast<size_t>(N) * R;                         // [N]
  double* tmp = gain + N;                                                   // [R] ping-pong row
  double* spv = tmp + R;                                                    // [R] Eq.3 per size
  uint8_t* alloc = reinterpret_cast<uint8_t*>(spv + R);                     // [N][R] (indexed by child)
  int* par = reinterpret_cast<int*>(alloc + ((static_cast<size_t>(N) * R + 15) & ~size_t(15)));  // [N]
  int* sz = par + N;                                                        // [N]
  int* stack = sz + N;                                                      // [2N]
  int* head_asc = stack + 2 * N;                                            // first child (index order)
  int* next_asc = head_asc + N;
  int* head_desc = next_asc + N;                                            // first child (reverse order)
  int* next_desc = head_desc + N;
  __shared__ int s_best_k;
  __shared__ double s_best_speed;

  {
    // Stage parents and node probabilities in shared memory with every thread (one round trip),
    // so thread 0's in-order product chain below reads on-chip operands only.
    const double* pr = probs ? probs + tb : t.prob + tb;
    const double* tab = args.node_table ? args.node_table + tb : nullptr;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      par[i] = t.parent[tb + i];
      const double c = tab ? tab[i] : -1.0;
      gain[i] = c >= 0.0 ? c : pr[i];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // path_products (acceptance.py:176-184) and subtree sizes (egt.py:225-229).
    if (!args.probs_are_gains) {
      for (int i = 1; i < N; ++i) gain[i] = gain[par[i]] * gain[i];
    }
    for (int i = 0; i < N; ++i) sz[i] = 1;
    for (int v = N - 1; v >= 1; --v) sz[par[v]] += sz[v];
    // child lists: ascending index (= insertion order, the merge order) and descending (pick)
    for (int i = 0; i < N; ++i) head_asc[i] = head_desc[i] = -1;
    for (int c = N - 1; c >= 1; --c) {
      next_asc[c] = head_asc[par[c]];
      head_asc[par[c]] = c;
    }
    for (int c = 1; c < N; ++c) {
      next_desc[c] = head_desc[par[c]];
      head_desc[par[c]] = c;
    }
  }
  __syncthreads();
  // Bottom-up merge (egt.py:175-196).  Thread s owns target size s; k ascending and the strict
  // '>' reproduce the reference's first-maximum tie rule exactly.
  // Rows ping-pong between the node's slot and `tmp`, so each child merge is one barrier.
  for (int v = N - 1; v >= 0; --v) {
    double* row = best + static_cast<size_t>(v) * R;
    const int s = threadIdx.x;
    if (s < R) row[s] = (s == 1) ? gain[v] : -INFINITY;
    __syncthreads();
    double* src = row;
    double* dst = tmp;
    for (int c = head_asc[v]; c >= 0; c = next_asc[c]) {  // children in insertion (= index) order
      const double* crow = best + static_cast<size_t>(c) * R;
      const int top_c = min(sz[c], cap);
      if (s < R) {
        double m = s >= 1 ? src[s] : 0.0;
        int a = 0;
        if (s >= 1) {
#pragma unroll 4
          for (int kk = max(1, s - top_c); kk <= s - 1; ++kk) {
            const double rk = src[kk];
            if (rk == -INFINITY) continue;
            const double value = rk + crow[s - kk];
            if (value > m) { m = value; a = s - kk; }
          }
        }
        dst[s] = s >= 1 ? m : src[0];
        alloc[static_cast<size_t>(c) * R + s] = static_cast<uint8_t>(a);
      }
      __syncthreads();
      double* t2 = src;
      src = dst;
      dst = t2;
    }
    if (src != row) {  // the last merge landed in tmp
      if (s < R) row[s] = src[s];
      __syncthreads();
    }
  }
  if (best_out || alloc_out) {
    // Optional export of the whole DP (SubtreeKnapsack.best_row / pick on the host).
    const size_t ob = static_cast<size_t>(b) * t.cap * (args.max_verify + 1);
    const int RO = args.max_verify + 1;
    for (int i = threadIdx.x; i < N * RO; i += blockDim.x) {
      const int v = i / RO, s = i % RO;
      if (best_out) best_out[ob + i] = (s < R) ? best[static_cast<size_t>(v) * R + s] : -INFINITY;
      if (alloc_out) alloc_out[ob + i] = (s < R) ? alloc[static_cast<size_t>(v) * R + s] : 0;
    }
  }
  {  // Eq.3 for every size at once; thread 0 then scans them in the reference's order
    const int kk = threadIdx.x;
    if (args.fixed_k <= 0 && kk >= 1 && kk <= cap && best[kk] != -INFINITY)
      spv[kk] = tree_speedup_dev(*prof, 1.0 + best[kk], args.w_draft, args.d_draft, kk);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const ygg_profile_pair pp = *prof;
    int best_k = 0;
    double best_speed = -INFINITY;
    const double* root = best;
    const bool shape_ok = cap <= 1 + args.d_draft * args.w_draft;
    if (args.fixed_k > 0) {
      best_k = min(args.fixed_k, cap);
      best_speed = shape_ok ? tree_speedup_dev(pp, 1.0 + root[best_k], args.w_draft, args.d_draft, best_k) : NAN;
    } else {
      for (int kk = 1; kk <= cap; ++kk) {  // egt.py:261-273 (speedups precomputed in parallel)
        if (root[kk] == -INFINITY) continue;
        const double sp = spv[kk];
        if (sp > best_speed + 1e-12) { best_k = kk; best_speed = sp; }
      }
    }
    if (!shape_ok) atomicOr(t.flags + b, kFlagContract);
    s_best_k = best_k;
    s_best_speed = best_speed;
    w_verify[b] = best_k;
    expected_aal[b] = 1.0 + root[best_k];
    speedup[b] = best_speed;
    if (aal_at_cap) aal_at_cap[b] = 1.0 + root[cap];
    if (speedup_at_cap)
      speedup_at_cap[b] = shape_ok ? tree_speedup_dev(pp, 1.0 + root[cap], args.w_draft, args.d_draft, cap) : NAN;
  }
  __syncthreads();
  // pick(best_k) (egt.py:206-222): peel the recorded allocations in reverse merge order.
  uint8_t* keep = reinterpret_cast<uint8_t*>(next_desc + N);  // [N] flags
  for (int i = threadIdx.x; i < N; i += blockDim.x) keep[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    int sp = 0;
    stack[sp++] = 0;
    stack[sp++] = s_best_k;
    while (sp > 0) {
      const int kk = stack[--sp];
      const int v = stack[--sp];
      keep[v] = 1;
      int remaining = kk;
      for (int c = head_desc[v]; c >= 0; c = next_desc[c]) {  // children in reverse index order
        const int taken = alloc[static_cast<size_t>(c) * R + remaining];
        if (taken) {
          stack[sp++] = c;
          stack[sp++] = taken;
          remaining -= taken;
        }
      }
    }
    int j = 0;
    for (int i = 0; i < N; ++i) {
      new_idx[tb + i] = keep[i] ? j : -1;
      if (keep[i]) keep_idx[tb + j++] = i;
    }
    for (int i = N; i < t.cap; ++i) new_idx[tb + i] = -1;
    for (int i = j; i < t.cap; ++i) keep_idx[tb + i] = -1;
  }
  pdl_launch_dependents();
}

// path_products (acceptance.py:176-184): out[0] = p[0]; out[i] = out[parent(i)] * p[i], index order.
__global__ void path_products_kernel(ygg_tree t, const double* __restrict__ probs, double* __restrict__ out) {
  pdl_wait();
  pdl_launch_dependents();
  const int b = blockIdx.x;
  if (threadIdx.x != 0) return;
  const size_t tb = static_cast<size_t>(b) * t.cap;
  const int n = t.size[b];
  const double* p = probs ? probs + tb : t.prob + tb;
  if (n > 0) out[tb] = p[0];
  for (int i = 1; i < n; ++i) out[tb + i] = out[tb + t.parent[tb + i]] * p[i];
}

// TokenTree.subtree (token_tree.py:146-168): kept nodes in ascending old order.
constexpr int kSubtreeMax = 1024;  // largest pruned-tree capacity handled on chip
__global__ void subtree_kernel(ygg_tree in, ygg_tree out, const int32_t* __restrict__ keep_idx,
                               const int32_t* __restrict__ new_idx) {
  // Everything staged through shared memory in a few parallel rounds: kept count by a block count,
  // gathered rows, ancestor-or-self mask rows by walking each node's (on-chip) parent chain, and
  // the frontier (deepest level, index order) from on-chip depths.
  pdl_wait();
  const int b = blockIdx.x;
  const size_t ib = static_cast<size_t>(b) * in.cap, ob = static_cast<size_t>(b) * out.cap;
  __shared__ int s_par[kSubtreeMax], s_dep[kSubtreeMax];
  __shared__ int s_n, s_md;
  if (threadIdx.x == 0) {
    s_n = 0;
    s_md = 0;
  }
  __syncthreads();
  int local = 0;
  for (int i = threadIdx.x; i < in.cap; i += blockDim.x) local += keep_idx[ib + i] >= 0 ? 1 : 0;
  if (local) atomicAdd(&s_n, local);
  __syncthreads();
  const int n = min(s_n, out.cap);  // kept indices are packed first, -1 after
  for (int i = threadIdx.x; i < out.cap; i += blockDim.x) {
    int p = -1, d = 0;
    if (i < n) {
      const int o = keep_idx[ib + i];
      const int op = in.parent[ib + o];
      p = op < 0 ? -1 : new_idx[ib + op];
      d = in.depth[ib + o];
      out.token[ob + i] = in.token[ib + o];
      out.prob[ob + i] = in.prob[ib + o];
      out.cum[ob + i] = in.cum[ib + o];
      atomicMax(&s_md, d);
    } else {
      out.token[ob + i] = 0;
      out.prob[ob + i] = 0.0;
      out.cum[ob + i] = 0.0;
    }
    out.parent[ob + i] = p;
    out.depth[ob + i] = d;
    s_par[i] = p;
    s_dep[i] = d;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < out.cap; i += blockDim.x) {
    uint32_t* row = out.mask + (ob + i) * out.mask_words;
    for (int w = 0; w < out.mask_words; ++w) {
      uint32_t bits = 0u;
      if (i < n)
        for (int v = i, steps = 0; v >= 0 && v < n && steps <= i; v = s_par[v], ++steps)  // bounded walk
          if ((v >> 5) == w) bits |= 1u << (v & 31);
      row[w] = bits;
    }
  }
  if (threadIdx.x == 0) {
    const int md = s_md;
    int fnn = 0;
    for (int i = 0; i < n; ++i)
      if (s_dep[i] == md) out.frontier[ob + fnn++] = i;
    out.frontier_n[b] = fnn;
    out.size[b] = n;
    out.flags[b] = 0;
  }
  pdl_launch_dependents();
}

// ===========================================================================
// K5: acceptance walk (acceptance.py:221-241) + greedy / sampled realisations.
// ===========================================================================
constexpr int kAcceptThreads = 1024;
constexpr int kAcceptWarps = kAcceptThreads / 32;
constexpr int kAcceptSmemNodes = 256;  // trees up to this size are walked from shared memory

// 4 consecutive logits as f32 (through L2: the LM head just wrote them)
template <typename T>
YGG_DEV void ld4(const T* p, float* o);
template <>
YGG_DEV void ld4<float>(const float* p, float* o) {
  const float4 q = __ldcg(reinterpret_cast<const float4*>(p));
  o[0] = q.x; o[1] = q.y; o[2] = q.z; o[3] = q.w;
}
template <>
YGG_DEV void ld4<__nv_bfloat16>(const __nv_bfloat16* p, float* o) {
  const uint2 u = __ldcg(reinterpret_cast<const uint2*>(p));
  const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u.x), b = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
  o[0] = __bfloat162float(a.x); o[1] = __bfloat162float(a.y); o[2] = __bfloat162float(b.x); o[3] = __bfloat162float(b.y);
}
constexpr int kAcceptUnroll = 8;  // 4-logit loads in flight per thread

// log-sum-exp of row lr / T by the whole block (SAMPLE without precomputed row stats): f32 max, f32
// per-thread sums of exp(x - max) combined in f64 in fixed order.  Every thread returns the value.
// vec: 4-logit loads (V % 4 == 0, row 4-element aligned), kAcceptUnroll of them in flight per thread.
template <typename T>
YGG_DEV double block_row_lse(const T* __restrict__ lr, int V, float inv_temp, bool vec, float* redf, double* redd) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float m = -INFINITY;
  const int nq = V >> 2;
  if (vec) {
    for (int i = threadIdx.x; i < nq; i += kAcceptUnroll * kAcceptThreads) {
      float q[kAcceptUnroll][4];
#pragma unroll
      for (int u = 0; u < kAcceptUnroll; ++u) {
        const int j = i + u * kAcceptThreads;
        if (j < nq) ld4(lr + 4 * j, q[u]);
        else q[u][0] = q[u][1] = q[u][2] = q[u][3] = -INFINITY;
      }
#pragma unroll
      for (int u = 0; u < kAcceptUnroll; ++u)
#pragma unroll
        for (int k = 0; k < 4; ++k) m = fmaxf(m, q[u][k] * inv_temp);
    }
  } else {
    for (int v = threadIdx.x; v < V; v += kAcceptThreads) m = fmaxf(m, to_f32(lr[v]) * inv_temp);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) redf[warp] = m;
  __syncthreads();
  float gm = redf[0];
  for (int w = 1; w < kAcceptWarps; ++w) gm = fmaxf(gm, redf[w]);
  float sf = 0.f;
  if (vec) {
    for (int i = threadIdx.x; i < nq; i += kAcceptUnroll * kAcceptThreads) {
      float q[kAcceptUnroll][4];
#pragma unroll
      for (int u = 0; u < kAcceptUnroll; ++u) {
        const int j = i + u * kAcceptThreads;
        if (j < nq) ld4(lr + 4 * j, q[u]);
        else q[u][0] = q[u][1] = q[u][2] = q[u][3] = -INFINITY;
      }
#pragma unroll
      for (int u = 0; u < kAcceptUnroll; ++u)
#pragma unroll
        for (int k = 0; k < 4; ++k) sf += __expf(q[u][k] * inv_temp - gm);
    }
  } else {
    for (int v = threadIdx.x; v < V; v += kAcceptThreads) sf += __expf(to_f32(lr[v]) * inv_temp - gm);
  }
  double sd = sf;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sd += __shfl_xor_sync(0xffffffffu, sd, o);
  if (lane == 0) redd[warp] = sd;
  __syncthreads();
  double tot = 0.0;
  for (int w = 0; w < kAcceptWarps; ++w) tot += redd[w];
  __syncthreads();  // redf / redd are reused by the next call
  return static_cast<double>(gm) + log(tot);
}

// One block per request.  The walk (thread 0) follows acceptance.py:221-241; in SAMPLE mode without
// row stats the block computes each walked row's log-sum-exp on demand (<= depth + 1 rows per request
// instead of a stats pass over every verify row).
template <typename T>
__global__ void __launch_bounds__(kAcceptThreads) accept_kernel(
    ygg_tree t, int mode, const double* __restrict__ probs, const double* __restrict__ uniforms, int n_uniform,
    const int32_t* __restrict__ row_argmax, const T* __restrict__ logits, int V, int ld,
    const float* __restrict__ row_stats, float inv_temp, int32_t* path, int32_t* path_len, int32_t* accepted_len,
    int32_t* bonus, int32_t* n_draws) {
  pdl_wait();
  const int b = blockIdx.x;
  const size_t tb = static_cast<size_t>(b) * t.cap;
  const int N = t.size[b];
  const int rows = t.cap + 1;  // verify rows per request: [confirmed, node 0, node 1, ...]
  const bool ondemand = mode == YGG_ACCEPT_SAMPLE && row_stats == nullptr;
  // 4-logit vector loads: every row starts 4-element aligned
  const bool vec = logits != nullptr && (V & 3) == 0 && (ld & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(logits) & (4 * sizeof(T) - 1)) == 0;
  __shared__ int s_have, s_took, s_prow, s_stop_row, s_lse_row, s_excl[64], s_nexcl, s_owner;
  __shared__ double s_u2, s_lse;
  __shared__ float s_redf[kAcceptWarps];
  __shared__ double s_redd[kAcceptWarps], s_scan[kAcceptWarps];
  auto lse_of = [&](int prow) -> double {  // thread 0 only
    if (ondemand) return s_lse;
    return row_stats ? static_cast<double>(row_stats[2 * (static_cast<size_t>(b) * rows + prow) + 1]) : 0.0;
  };
  int len = 0, cursor = -1, draw_i = 0, excl_n = 0;  // walk state (thread 0)
  // the walk's node scans read the tree from shared memory (one coalesced load) instead of one
  // dependent global load per node per visited group
  __shared__ int32_t s_parent[kAcceptSmemNodes], s_token[kAcceptSmemNodes];
  const bool smem_tree = N <= kAcceptSmemNodes;
  if (smem_tree) {
    for (int i = threadIdx.x; i < N; i += kAcceptThreads) {
      s_parent[i] = t.parent[tb + i];
      s_token[i] = t.token[tb + i];
    }
  }
  const int32_t* parent = smem_tree ? s_parent : t.parent + tb;
  const int32_t* token = smem_tree ? s_token : t.token + tb;
  if (threadIdx.x == 0) s_lse_row = -1;
  __syncthreads();
  while (true) {
    if (threadIdx.x == 0) {
      // group = [0] if cursor is None else children(cursor)
      const int first = cursor < 0 ? 0 : cursor + 1;
      bool any = false;
      for (int c = first; c < N; ++c) {
        if (cursor < 0 ? c == 0 : parent[c] == cursor) { any = true; break; }
      }
      s_have = any;
      s_prow = cursor < 0 ? 0 : 1 + cursor;
    }
    __syncthreads();
    if (!s_have) break;
    if (ondemand) {
      const int prow = s_prow;
      const double l = block_row_lse(logits + (static_cast<size_t>(b) * rows + prow) * ld, V, inv_temp, vec, s_redf, s_redd);
      if (threadIdx.x == 0) {
        s_lse = l;
        s_lse_row = prow;
      }
    }
    if (threadIdx.x == 0) {
      const int prow = cursor < 0 ? 0 : 1 + cursor;
      const int first = cursor < 0 ? 0 : cursor + 1;
      const double draw = (mode == YGG_ACCEPT_GREEDY) ? 0.5
                          : (draw_i < n_uniform ? uniforms[static_cast<size_t>(b) * n_uniform + draw_i] : 1.0);
      ++draw_i;
      const double lse = mode == YGG_ACCEPT_SAMPLE ? lse_of(prow) : 0.0;
      double cumulative = 0.0;
      int chosen = -1;
      excl_n = 0;
      for (int c = first; c < N; ++c) {
        if (!(cursor < 0 ? c == 0 : parent[c] == cursor)) continue;
        double p;
        if (mode == YGG_ACCEPT_PROBS) {
          p = probs[tb + c];
        } else if (mode == YGG_ACCEPT_GREEDY) {
          p = (token[c] == row_argmax[static_cast<size_t>(b) * rows + prow]) ? 1.0 : 0.0;
        } else {
          const size_t r = static_cast<size_t>(b) * rows + prow;
          const float l = to_f32(logits[r * ld + token[c]]) * inv_temp;
          p = exp(static_cast<double>(l) - lse);
        }
        if (excl_n < 64) s_excl[excl_n++] = token[c];
        cumulative += p;
        if (draw < cumulative) { chosen = c; break; }
        if (cursor < 0) break;  // the root group has a single member
      }
      if (chosen >= 0) {
        path[tb + len++] = chosen;
        cursor = chosen;
        excl_n = 0;
      }
      s_took = chosen >= 0;
    }
    __syncthreads();
    if (!s_took) break;
  }
  if (threadIdx.x == 0) {
    s_stop_row = (cursor < 0 ? 0 : 1 + cursor);
    s_nexcl = excl_n;
    s_u2 = (n_uniform > 0 && uniforms) ? uniforms[static_cast<size_t>(b) * n_uniform + (n_uniform - 1)] : 0.5;
    s_owner = -1;
    path_len[b] = len;
    accepted_len[b] = len + 1;
    if (n_draws) n_draws[b] = draw_i;
    for (int i = len; i < t.cap; ++i) path[tb + i] = -1;
  }
  __syncthreads();
  if (mode == YGG_ACCEPT_GREEDY) {
    if (threadIdx.x == 0 && bonus) bonus[b] = row_argmax[static_cast<size_t>(b) * rows + s_stop_row];
  } else if (mode == YGG_ACCEPT_SAMPLE && bonus) {
    // Residual bonus: sample p(.|stop row) with the rejected children removed (inverse CDF in token
    // order).  Together with the walk this emits exactly p(.|prefix).  Each warp owns a contiguous
    // slice read in coalesced 4-token groups; the slice masses (f64 sums of the f32 exponentials) are
    // scanned in fixed order, and the last warp whose slice starts at or below the target rescans its
    // slice in token order (warp prefix sums, 128 tokens per step).
    const int stop = s_stop_row;
    const size_t r = static_cast<size_t>(b) * rows + stop;
    double lse;
    if (ondemand) {
      if (s_lse_row == stop) {
        lse = s_lse;  // written by thread 0 before the barrier above
      } else {
        lse = block_row_lse(logits + r * ld, V, inv_temp, vec, s_redf, s_redd);
      }
    } else {
      lse = row_stats[2 * r + 1];
    }
    const T* lr = logits + r * ld;
    const int nex = s_nexcl;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nq = (V + 3) >> 2;                                  // 4-token groups
    const int per_w = (nq + kAcceptWarps - 1) / kAcceptWarps;    // groups per warp slice (contiguous)
    const int g0 = min(nq, warp * per_w), g1 = min(nq, g0 + per_w);
    auto load_group = [&](int j, float* x) {
      if (vec) {
        ld4(lr + 4 * j, x);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = 4 * j + k < V ? to_f32(lr[4 * j + k]) : 0.f;
      }
    };
    // probabilities of group j's tokens (0: excluded or past the end)
    auto group_probs = [&](int j, const float* x, double* p) {
      unsigned ex = 0;
      for (int e = 0; e < nex; ++e) {
        const unsigned d = static_cast<unsigned>(s_excl[e] - 4 * j);
        if (d < 4u) ex |= 1u << d;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        p[k] = (4 * j + k < V && !((ex >> k) & 1u))
                   ? static_cast<double>(__expf(static_cast<float>(static_cast<double>(x[k] * inv_temp) - lse)))
                   : 0.0;
    };
    // pass 1: this warp's slice mass (coalesced groups, kAcceptUnroll loads in flight per lane)
    double lm = 0.0;
    for (int base = g0; base < g1; base += 32 * kAcceptUnroll) {
      float x[kAcceptUnroll][4];
#pragma unroll
      for (int u = 0; u < kAcceptUnroll; ++u) {
        const int j = base + u * 32 + lane;
        if (j < g1) load_group(j, x[u]);
      }
#pragma unroll
      for (int u = 0; u < kAcceptUnroll; ++u) {
        const int j = base + u * 32 + lane;
        if (j < g1) {
          double p[4];
          group_probs(j, x[u], p);
          lm += (p[0] + p[1]) + (p[2] + p[3]);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lm += __shfl_xor_sync(0xffffffffu, lm, o);
    if (lane == 0) s_scan[warp] = lm;
    __syncthreads();
    double prefix = 0.0, total = 0.0;
    for (int w = 0; w < kAcceptWarps; ++w) {
      if (w < warp) prefix += s_scan[w];
      total += s_scan[w];
    }
    const double target = s_u2 * total;
    // the slice holding the target: the last one with mass that starts at or below it (fixed order)
    if (lane == 0 && lm > 0.0 && prefix <= target) atomicMax(&s_owner, warp);
    __syncthreads();
    if (warp == s_owner) {
      // pass 2 (one warp): token-order scan of the slice, 128 tokens per step
      const double rest = target - prefix;
      double acc = 0.0;
      int pick = -1, last_ok = -1;
      for (int base = g0; base < g1 && pick < 0; base += 32) {
        const int j = base + lane;
        float x[4] = {0.f, 0.f, 0.f, 0.f};
        double p[4] = {0.0, 0.0, 0.0, 0.0};
        if (j < g1) {
          load_group(j, x);
          group_probs(j, x, p);
        }
        const double ls = (p[0] + p[1]) + (p[2] + p[3]);
        double incl = ls;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        int lv = -1;  // this lane's last token with mass
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (p[k] > 0.0) lv = 4 * j + k;
        const unsigned cross = __ballot_sync(0xffffffffu, acc + incl > rest);
        if (cross) {
          const int fl = __ffs(cross) - 1;
          int pk = -1;
          if (lane == fl) {
            double a = acc + (incl - ls);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              a += p[k];
              if (pk < 0 && p[k] > 0.0 && a > rest) pk = 4 * j + k;
            }
            if (pk < 0) pk = lv;  // rounding at the group's end: its last token with mass
          }
          pick = __shfl_sync(0xffffffffu, pk, fl);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lv = max(lv, __shfl_xor_sync(0xffffffffu, lv, o));
        if (lv >= 0) last_ok = lv;
        acc += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) bonus[b] = pick >= 0 ? pick : last_ok;  // rounding at the slice's end: its last token
    } else if (threadIdx.x == 0 && s_owner < 0) {
      bonus[b] = 0;  // no mass anywhere (every token excluded or underflowed)
    }
  }
  pdl_launch_dependents();
}

// ===========================================================================
// Acceptance statistics per grown-tree position (calibrated acceptance for the Eq.3 objective).
// ===========================================================================
__global__ void accept_stats_kernel(ygg_tree vt, const int32_t* __restrict__ keep_idx, int keep_cap,
                                    const int32_t* __restrict__ path, const int32_t* __restrict__ path_len,
                                    uint32_t* __restrict__ counts) {
  pdl_wait();
  pdl_launch_dependents();
  const int b = blockIdx.x;
  const size_t tb = static_cast<size_t>(b) * vt.cap;
  const int N = vt.size[b];
  const int n = path_len[b];
  __shared__ unsigned char on_path[256];
  for (int i = threadIdx.x; i < N; i += blockDim.x) on_path[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) on_path[path[tb + i]] = 1;
  __syncthreads();
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    const int p = vt.parent[tb + j];
    if (p >= 0 && !on_path[p]) continue;  // parent rejected: this node was never tested
    const int g = keep_idx[static_cast<size_t>(b) * keep_cap + j];
    atomicAdd(counts + 2 * g, 1u);
    if (on_path[j]) atomicAdd(counts + 2 * g + 1, 1u);
  }
}

// Feature tap: the target's hidden state at each request's last accepted row (the bonus's context).
__global__ void feature_tap_kernel(const __nv_bfloat16* __restrict__ hidden, int T, int d,
                                   const int32_t* __restrict__ path, int path_cap,
                                   const int32_t* __restrict__ path_len, float* __restrict__ out) {
  pdl_wait();
  pdl_launch_dependents();
  const int b = blockIdx.x;
  const int n = path_len[b];
  const int stop = n > 0 ? 1 + path[static_cast<size_t>(b) * path_cap + n - 1] : 0;
  const __nv_bfloat16* src = hidden + (static_cast<size_t>(b) * T + stop) * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) out[static_cast<size_t>(b) * d + i] = __bfloat162float(src[i]);
}

// ===========================================================================
// KV compaction of the accepted path (new; the map is derived from accepted_path).
// ===========================================================================
template <typename T>
__global__ void kv_compact_kernel(T* cache, int B, int Hkv, int S, int hd, long long layer_stride,
                                  const int32_t* __restrict__ base, const int32_t* __restrict__ path,
                                  const int32_t* __restrict__ path_len, int path_cap,
                                  const int32_t* __restrict__ keep_idx, int keep_cap,
                                  const int32_t* __restrict__ node_depth, int depth_cap, int skip_depth) {
  pdl_wait();
  const int layer = blockIdx.y, b = blockIdx.z;
  const int kvh = blockIdx.x;  // over 2*Hkv
  const int n = path_len[b];
  if (n <= 0) return;
  T* head = cache + layer * layer_stride + (static_cast<size_t>(b) * 2 * Hkv + kvh) * static_cast<size_t>(S) * hd;
  // K rows are [S][hd]; V is stored transposed [hd][S] (see attn_tc.cu).
  const bool vt = kvh >= Hkv;
  const size_t s_stride = vt ? 1 : static_cast<size_t>(hd);
  const size_t d_stride = vt ? static_cast<size_t>(S) : 1;
  const int p0 = base[b] + 1;
  constexpr int kMaxPath = 64;
  // The move list (source node per accepted position, or -1) resolved once per CTA, one thread per
  // path entry, instead of every thread chasing path -> keep_idx -> depth serially.  Paths longer
  // than kMaxPath go in chunks: a chunk's destinations (< its first position) never overlap a later
  // chunk's sources (source node >= path position), and inside a chunk every read precedes the writes.
  __shared__ int s_src[kMaxPath];
  for (int c0 = 0; c0 < n; c0 += kMaxPath) {
    const int np = (n - c0) < kMaxPath ? (n - c0) : kMaxPath;
    __syncthreads();
    for (int i = threadIdx.x; i < np; i += blockDim.x) {
      const int node = path[static_cast<size_t>(b) * path_cap + c0 + i];
      const int src_node = keep_idx ? keep_idx[static_cast<size_t>(b) * keep_cap + node] : node;
      const bool skip = (node_depth && node_depth[static_cast<size_t>(b) * depth_cap + src_node] >= skip_depth) ||
                        src_node == c0 + i;
      s_src[i] = skip ? -1 : src_node;
    }
    __syncthreads();
    for (int d = threadIdx.x; d < hd; d += blockDim.x) {
      T vals[kMaxPath];
      int dst[kMaxPath];
      int m = 0;
      for (int i = 0; i < np; ++i) {
        const int src_node = s_src[i];
        if (src_node < 0) continue;
        vals[m] = head[static_cast<size_t>(p0 + src_node) * s_stride + d * d_stride];
        dst[m] = p0 + c0 + i;
        ++m;
      }
      for (int j = 0; j < m; ++j) head[static_cast<size_t>(dst[j]) * s_stride + d * d_stride] = vals[j];
    }
  }
}

}  // namespace ygg

using namespace ygg;

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int ygg_prepare_tree(void) {
  cudaError_t e = cudaFuncSetAttribute(knapsack_prune_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "knapsack attribute: %s", cudaGetErrorString(e));
  e = cudaFuncSetAttribute(topk_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e != cudaSuccess) return ygg_fail(YGG_ERR_CUDA, "top-k merge attribute: %s", cudaGetErrorString(e));
  return YGG_OK;
}

size_t ygg_topk_workspace(int rows, int V, int k) {
  const int nchunks = (V + kTopkChunk - 1) / kTopkChunk;
  return static_cast<size_t>(rows) * nchunks * sizeof(TopkChunkOut);
}

int ygg_topk_softmax(const void* logits, int dtype, int rows, int V, int ld, int k, float temperature,
                     int32_t* out_tok, double* out_prob, float* out_stats, void* workspace, size_t workspace_bytes,
                     ygg_stream_t stream) {
  YGG_CHECK_ARG(rows >= 0 && V >= 1 && ld >= V, "bad logits shape");
  YGG_CHECK_ARG(k >= 1 && k <= kTopkMaxK && k <= V, "k must be in [1, 32] and <= V");
  YGG_CHECK_ARG(temperature > 0.f, "temperature must be > 0");
  YGG_CHECK_ARG(workspace_bytes >= ygg_topk_workspace(rows, V, k), "workspace too small");
  if (rows == 0) return YGG_OK;
  const int nchunks = (V + kTopkChunk - 1) / kTopkChunk;
  auto* ws = static_cast<TopkChunkOut*>(workspace);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const float inv_t = 1.0f / temperature;
  if (dtype == YGG_F32)
    YGG_LAUNCH_PDL(topk_phase1<float>, dim3(nchunks, rows), dim3(kTopkThreads), 0, s,
                   static_cast<const float*>(logits), V, ld, k, inv_t, nchunks, ws);
  else if (dtype == YGG_BF16)
    YGG_LAUNCH_PDL(topk_phase1<__nv_bfloat16>, dim3(nchunks, rows), dim3(kTopkThreads), 0, s,
                   static_cast<const __nv_bfloat16*>(logits), V, ld, k, inv_t, nchunks, ws);
  else
    return ygg_fail(YGG_ERR_VALUE, "unknown dtype");
  if (nchunks <= kTopkThreads * kMergeOwn) {
    const size_t keys = (static_cast<size_t>(nchunks) * k + 1) / 2 * 2 * 8;
    const size_t staged = keys + static_cast<size_t>(nchunks) * sizeof(TopkPartial);
    const int stage = staged <= 200 * 1024 ? 1 : 0;
    YGG_LAUNCH_PDL(topk_merge_kernel, dim3(rows), dim3(kTopkThreads), stage ? staged : keys, s,
                   static_cast<const TopkPartial*>(ws),
                   nchunks, k, out_tok, out_prob, out_stats, trace_next(10), L2Regions{}, stage);
    return YGG_OK;
  }
  const size_t smem = static_cast<size_t>(nchunks) * k * (sizeof(float) + sizeof(int));
  YGG_CHECK_ARG(smem <= 48 * 1024, "too many candidates for phase 2");
  YGG_LAUNCH_PDL(topk_phase2, dim3(rows), dim3(kTopkThreads), smem, s, ws, nchunks, k, out_tok, out_prob, out_stats);
  return YGG_OK;
}

size_t ygg_topk_partial_bytes(int rows, int nchunks) {
  return static_cast<size_t>(rows < 0 ? 0 : rows) * (nchunks < 0 ? 0 : nchunks) * sizeof(TopkPartial);
}

int ygg_topk_merge(const void* partials, int rows, int nchunks, int k, int32_t* out_tok, double* out_prob,
                   float* out_stats, ygg_stream_t stream) {
  return ygg_topk_merge_l2(partials, rows, nchunks, k, out_tok, out_prob, out_stats, nullptr, 0, stream);
}

int ygg_topk_merge_l2(const void* partials, int rows, int nchunks, int k, int32_t* out_tok, double* out_prob,
                      float* out_stats, const ygg_l2_region* regions, int n_regions, ygg_stream_t stream) {
  YGG_CHECK_ARG(partials && out_tok && out_prob, "null pointer");
  YGG_CHECK_ARG(n_regions >= 0 && n_regions <= 4 && (n_regions == 0 || regions != nullptr), "at most 4 L2 regions");
  L2Regions pf;
  for (int i = 0; i < 4; ++i) {
    pf.ptr[i] = i < n_regions && regions[i].bytes ? static_cast<const char*>(regions[i].ptr) : nullptr;
    pf.bytes[i] = pf.ptr[i] ? regions[i].bytes : 0;
    YGG_CHECK_ARG(!pf.ptr[i] || (reinterpret_cast<uintptr_t>(pf.ptr[i]) & 15) == 0, "L2 region must be 16-byte aligned");
  }
  YGG_CHECK_ARG(rows >= 0 && nchunks >= 1 && nchunks <= kTopkThreads * kMergeOwn, "nchunks must be in [1, 512]");
  YGG_CHECK_ARG(k >= 1 && k <= kTopkMaxK, "k must be in [1, 32]");
  YGG_CHECK_ARG(static_cast<size_t>(nchunks) * k * 8 <= 200 * 1024, "too many candidates to merge");
  if (rows == 0) return YGG_OK;
  const size_t keys = (static_cast<size_t>(nchunks) * k + 1) / 2 * 2 * 8;
  const size_t staged = keys + static_cast<size_t>(nchunks) * sizeof(TopkPartial);
  const int stage = staged <= 200 * 1024 ? 1 : 0;
  YGG_LAUNCH_PDL(topk_merge_kernel, dim3(rows), dim3(kTopkThreads), stage ? staged : keys,
                 reinterpret_cast<cudaStream_t>(stream),
                 static_cast<const TopkPartial*>(partials), nchunks, k, out_tok, out_prob, out_stats, trace_next(10), pf,
                 stage);
  return YGG_OK;
}

static int check_tree(const ygg_tree& t) {
  YGG_CHECK_ARG(t.B >= 1 && t.cap >= 1 && t.cap <= 32 * YGG_MAX_MASK_WORDS, "tree capacity out of range");
  YGG_CHECK_ARG(t.mask_words == (t.cap + 31) / 32, "mask_words must equal ceil(cap/32)");
  YGG_CHECK_ARG(t.token && t.parent && t.depth && t.prob && t.cum && t.mask && t.size && t.frontier &&
                    t.frontier_n && t.flags,
                "tree pointers must be non-null");
  return YGG_OK;
}

int ygg_egt_grow_level(ygg_tree tree, int Fmax, int k, int w_draft, const int32_t* cand_tok, const double* cand_prob,
                       const int32_t* cand_n, ygg_stream_t stream) {
  if (int rc = check_tree(tree)) return rc;
  YGG_CHECK_ARG(w_draft >= 1, "w_draft must be >= 1");
  YGG_CHECK_ARG(k >= 1 && Fmax >= 1 && Fmax <= kGrowThreads && Fmax * k <= kGrowMaxCand, "candidate grid too large");
  YGG_CHECK_ARG(cand_tok && cand_prob, "candidate pointers must be non-null");
  YGG_LAUNCH_PDL(grow_level_kernel, dim3(tree.B), dim3(kGrowThreads), 0, reinterpret_cast<cudaStream_t>(stream),
                 tree, Fmax, k, w_draft, cand_tok, cand_prob, cand_n, trace_next(11));
  return YGG_OK;
}

int ygg_build_mask(ygg_tree tree, ygg_stream_t stream) {
  if (int rc = check_tree(tree)) return rc;
  YGG_LAUNCH_PDL(build_mask_kernel, dim3(tree.B), dim3(32), 0, reinterpret_cast<cudaStream_t>(stream), tree);
  return YGG_OK;
}

static size_t knap_smem(int N, int cap) {
  const size_t R = cap + 1;
  size_t bytes = N * R * sizeof(double) + N * sizeof(double) + 2 * R * sizeof(double);
  bytes += (N * R + 15) & ~size_t(15);
  bytes += 2 * N * sizeof(int) + 2 * N * sizeof(int) + 4 * N * sizeof(int) + N;
  return bytes + 64;
}

int ygg_knapsack_prune(ygg_tree tree, const double* probs, const ygg_profile_pair* profiles_dev, ygg_prune_args args,
                       int32_t* keep_idx, int32_t* new_idx, int32_t* w_verify, double* expected_aal, double* speedup,
                       double* aal_at_cap, double* speedup_at_cap, double* best_table, uint8_t* alloc_table,
                       ygg_stream_t stream) {
  if (int rc = check_tree(tree)) return rc;
  YGG_CHECK_ARG(args.max_verify >= 1, "max_size must be >= 1");
  YGG_CHECK_ARG(args.d_draft >= 1 && args.w_draft >= 1, "d_draft and w_draft must be >= 1");
  YGG_CHECK_ARG(args.max_verify < kKnapThreads, "max_verify must be < 256");
  YGG_CHECK_ARG(profiles_dev && keep_idx && new_idx && w_verify && expected_aal && speedup, "null output");
  const size_t smem = knap_smem(tree.cap, std::min(args.max_verify, tree.cap));
  YGG_CHECK_ARG(smem <= 220 * 1024, "tree too large for the on-chip knapsack");
  YGG_LAUNCH_PDL(knapsack_prune_kernel, dim3(tree.B), dim3(kKnapThreads), smem, reinterpret_cast<cudaStream_t>(stream),
                 tree, probs, profiles_dev, args, keep_idx, new_idx, w_verify, expected_aal, speedup, aal_at_cap,
                 speedup_at_cap, best_table, alloc_table);
  return YGG_OK;
}

int ygg_accept_stats(ygg_tree vtree, const int32_t* keep_idx, int keep_cap, const int32_t* path,
                     const int32_t* path_len, uint32_t* counts, ygg_stream_t stream) {
  YGG_CHECK_ARG(keep_idx && path && path_len && counts, "null pointer");
  YGG_CHECK_ARG(vtree.cap <= 256 && keep_cap >= vtree.cap, "verify trees are limited to 256 nodes");
  YGG_LAUNCH_PDL(accept_stats_kernel, dim3(vtree.B), dim3(128), 0, reinterpret_cast<cudaStream_t>(stream), vtree,
                 keep_idx, keep_cap, path, path_len, counts);
  return YGG_OK;
}

int ygg_feature_tap(const void* hidden, int T, int d, const int32_t* path, int path_cap, const int32_t* path_len,
                    int B, float* out, ygg_stream_t stream) {
  YGG_CHECK_ARG(hidden && path && path_len && out && T >= 1 && d >= 1 && B >= 1, "invalid arguments");
  YGG_LAUNCH_PDL(feature_tap_kernel, dim3(B), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream),
                 static_cast<const __nv_bfloat16*>(hidden), T, d, path, path_cap, path_len, out);
  return YGG_OK;
}

int ygg_path_products(ygg_tree tree, const double* probs, double* out, ygg_stream_t stream) {
  if (int rc = check_tree(tree)) return rc;
  YGG_CHECK_ARG(out != nullptr, "null output");
  YGG_LAUNCH_PDL(path_products_kernel, dim3(tree.B), dim3(32), 0, reinterpret_cast<cudaStream_t>(stream), tree, probs,
                 out);
  return YGG_OK;
}

int ygg_tree_subtree(ygg_tree in, ygg_tree out, const int32_t* keep_idx, const int32_t* new_idx,
                     ygg_stream_t stream) {
  if (int rc = check_tree(in)) return rc;
  if (int rc = check_tree(out)) return rc;
  YGG_CHECK_ARG(in.B == out.B && out.cap >= 1, "tree batch mismatch");
  YGG_CHECK_ARG(out.cap <= kSubtreeMax, "pruned tree capacity too large");
  YGG_LAUNCH_PDL(subtree_kernel, dim3(in.B), dim3(128), 0, reinterpret_cast<cudaStream_t>(stream), in, out, keep_idx,
                 new_idx);
  return YGG_OK;
}

int ygg_accept(ygg_tree tree, int mode, const double* probs, const double* uniforms, int n_uniform,
               const int32_t* row_argmax, const void* logits, int logits_dtype, int V, int ld, const float* row_stats,
               float temperature, int32_t* path, int32_t* path_len, int32_t* accepted_len, int32_t* bonus,
               int32_t* n_draws, ygg_stream_t stream) {
  if (int rc = check_tree(tree)) return rc;
  YGG_CHECK_ARG(path && path_len && accepted_len, "null output");
  if (mode == YGG_ACCEPT_PROBS) {
    YGG_CHECK_ARG(probs && uniforms && n_uniform >= 1, "PROBS mode needs probs and uniforms");
  } else if (mode == YGG_ACCEPT_GREEDY) {
    YGG_CHECK_ARG(row_argmax != nullptr, "GREEDY mode needs row_argmax");
  } else if (mode == YGG_ACCEPT_SAMPLE) {
    // row_stats may be null: the kernel then computes the walked rows' log-sum-exp itself
    YGG_CHECK_ARG(logits && uniforms && n_uniform >= 2 && temperature > 0.f && V >= 1 && ld >= V,
                  "SAMPLE mode needs logits and uniforms");
  } else {
    return ygg_fail(YGG_ERR_VALUE, "unknown accept mode");
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const float inv_t = temperature > 0.f ? 1.0f / temperature : 1.0f;
  if (logits_dtype == YGG_BF16)
    YGG_LAUNCH_PDL(accept_kernel<__nv_bfloat16>, dim3(tree.B), dim3(kAcceptThreads), 0, s, tree, mode, probs, uniforms,
                   n_uniform, row_argmax, static_cast<const __nv_bfloat16*>(logits), V, ld, row_stats, inv_t, path,
                   path_len, accepted_len, bonus, n_draws);
  else
    YGG_LAUNCH_PDL(accept_kernel<float>, dim3(tree.B), dim3(kAcceptThreads), 0, s, tree, mode, probs, uniforms,
                   n_uniform, row_argmax, static_cast<const float*>(logits), V, ld, row_stats, inv_t, path, path_len,
                   accepted_len, bonus, n_draws);
  return YGG_OK;
}

int ygg_kv_compact(void* cache, int dtype, int layers, int B, int Hkv, int S, int hd, long long layer_stride,
                   const int32_t* base, const int32_t* path, const int32_t* path_len, int path_cap,
                   const int32_t* keep_idx, int keep_cap, const int32_t* node_depth, int depth_cap, int skip_depth,
                   ygg_stream_t stream) {
  YGG_CHECK_ARG(cache && base && path && path_len, "null pointer");
  YGG_CHECK_ARG(layers >= 1 && B >= 1 && Hkv >= 1 && S >= 1 && hd >= 1, "bad cache shape");
  dim3 grid(2 * Hkv, layers, B);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int threads = hd >= 128 ? 128 : 64;
  if (dtype == YGG_BF16)
    YGG_LAUNCH_PDL(kv_compact_kernel<__nv_bfloat16>, grid, dim3(threads), 0, s, static_cast<__nv_bfloat16*>(cache), B,
                   Hkv, S, hd, layer_stride, base, path, path_len, path_cap, keep_idx, keep_cap, node_depth, depth_cap,
                   skip_depth);
  else
    YGG_LAUNCH_PDL(kv_compact_kernel<float>, grid, dim3(threads), 0, s, static_cast<float*>(cache), B, Hkv, S, hd,
                   layer_stride, base, path, path_len, path_cap, keep_idx, keep_cap, node_depth, depth_cap, skip_depth);
  return YGG_OK;
}

}  // extern "C"
