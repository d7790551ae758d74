/*
 * ygg.h — C ABI of the B200-native Yggdrasil speculative-decoding step (libygg.so).
 *
 * Every entry point takes raw device pointers, plain integer shapes and a cudaStream_t,
 * returns 0 (YGG_OK) or a ygg_status code, never allocates device memory on the hot path,
 * never synchronises the stream, and is reentrant (all state is caller-owned).  Argument
 * errors map to the reference's conventions: YGG_ERR_VALUE ~ ValueError,
 * YGG_ERR_INDEX ~ IndexError (reference: pkg/src/specsim/token_tree.py:76-77,
 * egt.py:65-80, cli.py:338-351).  ygg_last_error() returns a thread-local message.
 *
 * Reference interfaces replaced (all paths relative to the reference's pkg/src/specsim/):
 *   ygg_topk_softmax / ygg_egt_grow_level  -> DrafterDistribution.candidates + grow_step
 *                                             (egt.py:52-114), build_mask row update (token_tree.py:205-218)
 *   ygg_build_mask                         -> build_mask (token_tree.py:205-218)
 *   ygg_knapsack_prune                     -> path_products + SubtreeKnapsack + prune_verify + TokenTree.subtree
 *                                             (acceptance.py:176-184, egt.py:150-282, token_tree.py:146-168)
 *   ygg_accept                             -> sample_with_probs / VerificationOutcome (acceptance.py:208-241)
 *   ygg_kv_compact                         -> (new) KV compaction of the accepted path; map = accepted_path
 *   ygg_gemm_*, ygg_attention, ygg_rmsnorm, ygg_qkv_rope_kv, ... -> the verify / draft forwards the
 *                                             reference prices as latency_at(...) (simulator.py:202-214)
 *   ygg_stamp                              -> (new) on-device stage timer feeding LatencyProfile /
 *                                             StageProfiles tables (latency.py:164-190, scheduler.py:82-103)
 */
#ifndef YGG_H_
#define YGG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* ygg_stream_t; /* == cudaStream_t */

typedef enum {
  YGG_OK = 0,
  YGG_ERR_VALUE = 1,       /* invalid argument value (ValueError) */
  YGG_ERR_INDEX = 2,       /* node index out of range (IndexError) */
  YGG_ERR_CUDA = 3,        /* CUDA runtime / driver failure */
  YGG_ERR_UNSUPPORTED = 4  /* shape outside the compiled envelope */
} ygg_status;

typedef enum { YGG_F32 = 0, YGG_BF16 = 1 } ygg_dtype;

#define YGG_MAX_BREAKPOINTS 32
#define YGG_MAX_MASK_WORDS 8 /* trees up to 256 nodes */

/* Piecewise-linear width->latency curve (reference LatencyProfile, latency.py:34-82). */
typedef struct {
  int32_t n;
  int32_t width[YGG_MAX_BREAKPOINTS];
  double latency_us[YGG_MAX_BREAKPOINTS];
} ygg_profile;

/* Reference ProfilePair (latency.py:130-134).  Lives in device memory so the on-device
 * profiler can refresh it without re-capturing graphs. */
typedef struct {
  ygg_profile drafter;
  ygg_profile verifier;
} ygg_profile_pair;

/* Batched draft trees, structure-of-arrays, one tree per request.  Mirrors TokenTree
 * (token_tree.py:34-197): node 0 is the root, parent[i] < i, depth = parent depth + 1. */
typedef struct {
  int32_t B;          /* requests */
  int32_t cap;        /* node capacity per tree */
  int32_t mask_words; /* u32 words per mask row (ceil(cap/32)) */
  int32_t* token;     /* [B, cap] */
  int32_t* parent;    /* [B, cap]; -1 for the root */
  int32_t* depth;     /* [B, cap] */
  double* prob;       /* [B, cap] surrogate (drafter) probability */
  double* cum;        /* [B, cap] product of surrogates root..node, in path order */
  uint32_t* mask;     /* [B, cap, mask_words] ancestor-or-self bit rows (build_mask) */
  int32_t* size;      /* [B] node count */
  int32_t* frontier;  /* [B, cap] newest-level node indices, ascending */
  int32_t* frontier_n;/* [B] */
  int32_t* flags;     /* [B] bit0 shortfall, bit1 candidate contract violated, bit2 capacity */
} ygg_tree;

/* Per-request sequence state of the generate loop (device memory).  hist[b][0..P[b]) are
 * confirmed tokens whose KV is in the target cache; hist[b][P[b]] is the pending bonus token. */
typedef struct {
  int32_t B;        /* requests */
  int32_t S;        /* history / KV capacity per request */
  int32_t* hist;    /* [B, S] */
  int32_t* P;       /* [B] */
  int32_t* n_gen;   /* [B] tokens generated so far */
  int32_t* acc_log; /* [B, log_cap] accepted_len per step (ring), may be NULL */
  int32_t* step;    /* [1] step counter */
  int32_t log_cap;
  int32_t p_limit;  /* commit never advances P[b] past p_limit (the tree / scratch slots of the next
                       step must fit in S); 0 = S - 1 */
  int32_t* gen_limit; /* [B] a request with n_gen >= gen_limit[b] is finished and frozen; may be NULL */
  int32_t* status;  /* [B] bit0 finished (gen_limit reached), bit1 frozen at p_limit; may be NULL */
} ygg_seq;

/* ---------------- library ---------------- */
int ygg_version(void);
const char* ygg_last_error(void);
/* Number of SMs and compute capability of the current device; fails unless sm_100. */
int ygg_device_check(int* num_sms, int* cc_major, int* cc_minor);

/* ---------------- K1: EGT expansion (egt.py:52-114) ---------------- */
/* Softmax(logits/temperature) top-k per row.  Ties ordered (prob desc, token asc).
 * logits: [rows, ld] f32 or bf16.  out_tok [rows,k], out_prob [rows,k] (f64 of the f32 value),
 * out_stats [rows,2] (row max, log-sum-exp) or NULL.  workspace >= ygg_topk_workspace(rows,V,k). */
size_t ygg_topk_workspace(int rows, int V, int k);
/* Merge per-chunk top-k partials [rows][nchunks] (nchunks <= 512; written by the LM-head GEMV's
 * STORE_TOPK epilogue) into the same outputs as ygg_topk_softmax. */
size_t ygg_topk_partial_bytes(int rows, int nchunks);
int ygg_topk_merge(const void* partials, int rows, int nchunks, int k, int32_t* out_tok, double* out_prob,
                   float* out_stats, ygg_stream_t stream);
/* Same, and the merge also pulls up to 4 regions into L2 (the next pass's first weights) while it
 * and the following tree kernels leave HBM idle. */
typedef struct {
  const void* ptr;
  uint64_t bytes;
} ygg_l2_region;
int ygg_topk_merge_l2(const void* partials, int rows, int nchunks, int k, int32_t* out_tok, double* out_prob,
                      float* out_stats, const ygg_l2_region* regions, int n_regions, ygg_stream_t stream);
int ygg_topk_softmax(const void* logits, int dtype, int rows, int V, int ld, int k, float temperature,
                     int32_t* out_tok, double* out_prob, float* out_stats, void* workspace,
                     size_t workspace_bytes, ygg_stream_t stream);

/* One grow_step per tree: candidates [B, Fmax, k] (rank order, counts in cand_n [B, Fmax]
 * or NULL = all k) for frontier rows; attaches the global top-w_draft by
 * (score desc, parent asc, rank asc), score = cum[parent] * prob (f64), in score order. */
int ygg_egt_grow_level(ygg_tree tree, int Fmax, int k, int w_draft, const int32_t* cand_tok,
                       const double* cand_prob, const int32_t* cand_n, ygg_stream_t stream);

/* K7: full mask rebuild from parent links (build_mask). */
int ygg_build_mask(ygg_tree tree, ygg_stream_t stream);

/* ---------------- K6: knapsack + latency-aware prune (egt.py:150-282) ---------------- */
typedef struct {
  int32_t max_verify;  /* knapsack cap = min(max_verify, size) */
  int32_t d_draft;     /* TreeShape.d_draft for Eq.3 */
  int32_t w_draft;     /* TreeShape.w_draft for Eq.3 */
  int32_t fixed_k;     /* >0: skip the objective and keep exactly min(fixed_k, cap) nodes */
  int32_t probs_are_gains; /* 1: `probs` already holds the per-node gains (SubtreeKnapsack(tree, gains, k)) */
  const double* node_table; /* optional [B, cap] calibrated acceptance per node position (an ExplicitAcceptance,
                               acceptance.py:106-129, keyed by the grown-tree index); entries < 0 fall back to
                               `probs` / tree.prob; NULL = off */
} ygg_prune_args;

/* probs [B, cap] f64 acceptance probabilities (freeze_probs); NULL = use tree.prob.
 * Outputs: keep_idx [B, cap] kept old indices ascending (-1 padded), new_idx [B, cap] (-1 dropped),
 * w_verify [B], expected_aal [B], speedup [B], aal_at_cap [B] (1+best(root,cap)), speedup_at_cap [B];
 * optional best_table [B, cap, max_verify+1] f64 and alloc_table (u8, same shape, indexed by the
 * merged child) export the DP for SubtreeKnapsack.best_row / pick. */
int ygg_knapsack_prune(ygg_tree tree, const double* probs, const ygg_profile_pair* profiles_dev,
                       ygg_prune_args args, int32_t* keep_idx, int32_t* new_idx, int32_t* w_verify,
                       double* expected_aal, double* speedup, double* aal_at_cap, double* speedup_at_cap,
                       double* best_table, uint8_t* alloc_table, ygg_stream_t stream);

/* Acceptance statistics of one step, per grown-tree node position (pooled over requests): for every
 * verified node whose parent was accepted (the root always), counts[2g] += 1 (tested) and, if it was
 * accepted itself, counts[2g+1] += 1, where g = keep_idx[b][j] is the verified node's grown index.
 * counts [keep_cap][2] u32 (caller zeroes).  Feeds the calibrated node_table of ygg_knapsack_prune. */
int ygg_accept_stats(ygg_tree vtree, const int32_t* keep_idx, int keep_cap, const int32_t* path,
                     const int32_t* path_len, uint32_t* counts, ygg_stream_t stream);

/* Depth-predictor feature tap: the target's last-token hidden state of each
 * request — row `stop` of the verify's final-norm output, stop = 0 (bonus row) when nothing was
 * accepted, else 1 + the last accepted node — copied as f32 to out [B, d].  hidden [B*T, d] bf16. */
int ygg_feature_tap(const void* hidden, int T, int d, const int32_t* path, int path_cap, const int32_t* path_len,
                    int B, float* out, ygg_stream_t stream);

/* path_products (acceptance.py:176-184): out[b,0] = p[b,0]; out[b,i] = out[b,parent(i)] * p[b,i] (f64,
 * index order); probs NULL = tree.prob. */
int ygg_path_products(ygg_tree tree, const double* probs, double* out, ygg_stream_t stream);

/* Gather the pruned tree (TokenTree.subtree) into `out` from `in` using keep_idx/new_idx. */
int ygg_tree_subtree(ygg_tree in, ygg_tree out, const int32_t* keep_idx, const int32_t* new_idx,
                     ygg_stream_t stream);

/* ---------------- K5: acceptance walk (acceptance.py:221-241) ---------------- */
typedef enum {
  YGG_ACCEPT_PROBS = 0,  /* reference semantics: probs[B,cap] f64 + uniforms */
  YGG_ACCEPT_GREEDY = 1, /* prob(child)=1 iff token == argmax(target row of parent) */
  YGG_ACCEPT_SAMPLE = 2  /* prob(child)=softmax(target/T) at parent row; residual bonus */
} ygg_accept_mode;

/* Walk the tree from above the root; one uniform per visited group (uniforms [B, n_uniform]).
 * Target rows: row 0 = the confirmed/bonus token, row 1+i = tree node i (verify order).
 * row_argmax [B, rows] (GREEDY), logits [B*rows, ld] + row_stats [B*rows, 2] (SAMPLE; row_stats may
 * be NULL: the kernel then computes the log-sum-exp of the rows it walks itself).
 * Outputs: path [B, cap] (accepted node indices), path_len [B], accepted_len [B] = path_len+1,
 * bonus [B] (GREEDY/SAMPLE: next confirmed token), n_draws [B] uniforms consumed by the walk (or NULL). */
int ygg_accept(ygg_tree tree, int mode, const double* probs, const double* uniforms, int n_uniform,
               const int32_t* row_argmax, const void* logits, int logits_dtype, int V, int ld,
               const float* row_stats, float temperature, int32_t* path, int32_t* path_len,
               int32_t* accepted_len, int32_t* bonus, int32_t* n_draws, ygg_stream_t stream);

/* ---------------- KV cache + sequence bookkeeping ---------------- */
/* Per request: move K/V of accepted nodes to contiguous slots after the confirmed token.
 * cache layout per layer: [B, 2, Hkv, S, hd] (dtype); layer stride in elements.
 * src slot of accepted node i = base[b] + 1 + map(path[b,i]) where map = keep_idx (or identity
 * if keep_idx NULL); dst = base[b] + 1 + i.  Nodes with depth >= skip_depth are not moved. */
int ygg_kv_compact(void* cache, int dtype, int layers, int B, int Hkv, int S, int hd, long long layer_stride,
                   const int32_t* base, const int32_t* path, const int32_t* path_len, int path_cap,
                   const int32_t* keep_idx, int keep_cap, const int32_t* node_depth, int depth_cap,
                   int skip_depth, ygg_stream_t stream);

/* ---------------- dense forward ops ---------------- */
size_t ygg_gemm_plan_size(void);
/* Weight-streaming GEMM plan: Y[M,N] = X[M,K] . W[N,K]^T written as per-tile partials
 * ws[seg][Mpad][128] f32 (seg_first[N/128+1] on device).  bf16 -> tcgen05/TMA, f32 -> SIMT. */
int ygg_gemm_plan_init(void* plan, int dtype, const void* W, const void* X, int M, int N, int K, int num_ctas,
                       int32_t* seg_first_dev, int* num_segments, size_t* workspace_bytes);
int ygg_gemm_run(const void* plan, float* workspace, ygg_stream_t stream);

/* Fused epilogues of the bf16 tcgen05 GEMM: the last CTA to finish an output tile reduces its
 * stream-K partials in fixed order and applies the op (one launch per linear layer).  RMSNorm is
 * folded: its gain is pre-multiplied into W and, when ss_in is given, every output row (token) m is
 * scaled by rsqrt(sum_t ss_in[t][m] / norm_dim + eps).  Weight row layouts: QKV_ROPE rows are
 * permuted per head so RoPE pairs (i, i+hd/2) are adjacent; SWIGLU rows interleave gate/up. */
typedef enum {
  YGG_EPI_NONE = 0,      /* partials only (ygg_gemm_run) */
  YGG_EPI_STORE_F32 = 1, /* out[m][n] = y (logits) */
  YGG_EPI_QKV_ROPE = 2,  /* RoPE at pos[m]; q -> q_out [M,Hq,hd]; k -> K rows, v -> V^T of the cache */
  YGG_EPI_SWIGLU = 3,    /* act_out[m][j] = silu(gate_j) * up_j */
  YGG_EPI_RESID = 4,     /* resid[m][n] += y; hb = bf16(resid); ss_out[n/128][m] = per-tile sum of squares */
  YGG_EPI_ARGMAX = 5     /* greedy LM head: no logits; out (as u64 [N/128][M]) = per 128-row tile and token the
                            key (ordered f32 max << 32 | ~index) of its first maximum; ygg_argmax_reduce */
} ygg_epi_kind;

typedef struct {
  int32_t kind;
  const float* ss_in;
  int32_t ss_tiles;
  int32_t norm_dim;
  float eps;
  float* out;
  int32_t ld;
  void* q_out;
  void* cache;
  int32_t S, Hq, Hkv, hd;
  float rope_theta;
  const int32_t* pos;
  const int32_t* slot;
  const int32_t* req;
  void* act_out;
  float* resid;
  void* hb;
  float* ss_out;
  int32_t* counters; /* [tiles] zero-initialised arrival counters (self-resetting) */
  unsigned long long* dbg; /* optional per-CTA timer stamps [num_ctas][8] (profiling only), or NULL */
  const float* rope_cs;    /* optional [positions][hd/2][2] (cos, sin) table for QKV_ROPE, or NULL */
} ygg_epilogue;

int ygg_gemm_fused(const void* plan, float* workspace, const ygg_epilogue* epi, ygg_stream_t stream);
/* Row argmax from the ARGMAX epilogue's per-tile keys [ntiles][M]: out[m] = index of the first maximum
 * over all tiles (the same value row_stats returns on the stored logits). */
int ygg_argmax_reduce(const void* keys, int ntiles, int M, int32_t* out, ygg_stream_t stream);
/* Cluster split-K (bf16): one thread-block cluster of `cluster` CTAs per 128-row output tile, the tile's
 * K range split evenly over them, the partials reduced through DSMEM into the cluster's leader, which
 * applies the fused epilogue (no workspace partials, no counters).  Fails with YGG_ERR_UNSUPPORTED
 * unless every tile's cluster is co-resident in one wave.  cluster = 0 restores stream-K.  Such a plan
 * runs only through ygg_gemm_fused. */
int ygg_gemm_plan_set_cluster(void* plan, int cluster);
int ygg_gemm_plan_cluster(const void* plan);
/* Row layout of W for this plan's separate QKV / SwiGLU epilogue kernels: interleaved != 0 = the fused
 * layout (model.prepare_fused_: RoPE pair (i, i + hd/2) of a head at rows (2i, 2i + 1); gate j / up j
 * at rows 2j / 2j + 1), so passes over fused-layout weights that do not take the GEMV (prefill chunks,
 * batched draft levels) run the per-kernel epilogues.  Default 0 (standard row order). */
int ygg_gemm_plan_set_layout(void* plan, int interleaved);
/* TMA ring depth override of a bf16 stream-K plan (2..12 stages, <= 227 KB of shared memory). */
int ygg_gemm_plan_set_stages(void* plan, int stages);
/* L2 prefetch issued by this plan's separate epilogue kernel (ygg_epi_*): right after its dependency
 * wait every CTA pulls its share of [ptr, ptr + bytes) into L2 — a later weight stream, fetched while
 * HBM would otherwise idle.  bytes = 0 turns it off.  Results are unaffected. */
int ygg_gemm_plan_set_epi_prefetch(void* plan, const void* ptr, size_t bytes);
int ygg_gemm_tiles(const void* plan);
/* Embedding gather for the fused path: resid (f32), hb (bf16) and per-128-feature-tile sums of
 * squares ss_out [d/128][M] (the first layer's folded RMSNorm input). */
int ygg_embed_fused(const void* table, int V, int d, const int32_t* tokens, int M, float* resid, void* hb,
                    float* ss_out, ygg_stream_t stream);

/* Epilogues over GEMM partials (all deterministic fixed-order segment sums). */
int ygg_epi_store(const void* plan, const float* ws, void* out, int out_dtype, int ld_out, ygg_stream_t stream);
int ygg_epi_residual_norm(const void* plan, const float* ws, float* resid, const void* norm_w, float eps,
                          void* xn_out, int act_dtype, ygg_stream_t stream);
int ygg_epi_swiglu(const void* plan, const float* ws, void* out, int act_dtype, ygg_stream_t stream);
/* QKV epilogue: RoPE on q,k at pos[m]; q -> q_out [M, Hq, hd]; k -> K rows, v -> V^T of the cache at
 * slot[m] of request req[m].  rope_cs: optional [positions][hd/2][2] (cos, sin) table, else sincosf. */
int ygg_epi_qkv_rope(const void* plan, const float* ws, int Hq, int Hkv, int hd, float rope_theta,
                     const int32_t* pos, const int32_t* slot, const int32_t* req, void* q_out, void* cache,
                     int S, int act_dtype, const float* rope_cs, ygg_stream_t stream);

int ygg_embed(const void* table, int dtype, int V, int d, const int32_t* tokens, int M, float* resid_out,
              ygg_stream_t stream);
int ygg_rmsnorm(const float* x, const void* w, int dtype, int M, int d, float eps, void* out, ygg_stream_t stream);
/* ygg_embed followed by ygg_rmsnorm in one launch (table, norm gains and activations share dtype). */
int ygg_embed_rmsnorm(const void* table, const void* norm_w, int dtype, int V, int d, const int32_t* tokens, int M,
                      float eps, float* resid_out, void* xn_out, ygg_stream_t stream);

/* Tree/prefix attention.  q [M, Hq, hd]; per query row m of request r, mask row
 * qmask[m, mask_words] over the request's block; keys [0, blk_start[r]) always visible,
 * keys blk_start[r] + j visible iff bit j (qmask NULL: causal block).  Rows of request r are
 * the contiguous range [r*M/B, (r+1)*M/B).  out [M, Hq*hd]. */
int ygg_attention(const void* q, const void* cache, int dtype, int M, int B, int Hq, int Hkv, int hd, int S,
                  const int32_t* blk_start, const int32_t* blk_len, const uint32_t* qmask, int mask_words,
                  float scale, void* out, ygg_stream_t stream);

/* K2 on tcgen05 (bf16): split-KV tree attention.  Cache layout per layer: [B, 2, Hkv, S, hd]
 * where the kv=0 half holds K rows [S][hd] and the kv=1 half holds V transposed [hd][S]
 * (S % 64 == 0).  Plan = TMA tensor maps for q and one layer's cache; partials >= partial_bytes. */
size_t ygg_attn_plan_size(void);
int ygg_attn_plan_init(void* plan, const void* q, const void* cache_layer, int B, int M, int Hq, int Hkv, int hd,
                       int S, size_t* partial_bytes);
int ygg_attention_tc(const void* plan, const int32_t* blk_start, const int32_t* blk_len, const uint32_t* qmask,
                     int mask_words, float scale, float* partials, void* out, ygg_stream_t stream);

/* Per-row max / argmax / log-sum-exp(x/temperature) over logits [rows, ld]. */
int ygg_row_stats(const void* logits, int dtype, int rows, int V, int ld, float temperature, int32_t* argmax,
                  float* stats, ygg_stream_t stream);

int ygg_gemm_seg_table_len(const void* plan);

/* ---------------- step bookkeeping (no host sync) ---------------- */
/* Draft pass 0 inputs: rows [hist[P-1], hist[P]] per request (R rows, padded). */
int ygg_pass0_inputs(ygg_seq seq, int R, int tree_cap, int32_t* tokens, int32_t* pos, int32_t* slot, int32_t* req,
                     uint32_t* qmask, int mask_words, int32_t* blk_start, int32_t* blk_len, ygg_stream_t stream);
/* Reset each tree to its root = top-1 candidate of pass-0 row `row` (DrafterDistribution.root()). */
int ygg_init_roots(ygg_tree tree, const int32_t* cand_tok, const double* cand_prob, int k, int R, int row,
                   ygg_stream_t stream);
/* Draft pass inputs for the newest tree level (frontier rows, padded to R; cand_n [B,R]). */
int ygg_level_inputs(ygg_tree tree, ygg_seq seq, int R, int k, int32_t* tokens, int32_t* pos, int32_t* slot,
                     int32_t* req, uint32_t* qmask, int mask_words, int32_t* blk_start, int32_t* blk_len,
                     int32_t* cand_n, ygg_stream_t stream);
/* Verify inputs: bonus row + pruned tree rows, T = vtree.cap + 1 rows per request. */
int ygg_verify_inputs(ygg_tree vtree, ygg_seq seq, int32_t* tokens, int32_t* pos, int32_t* slot, int32_t* req,
                      uint32_t* qmask, int mask_words, int32_t* blk_start, int32_t* blk_len, ygg_stream_t stream);
/* Append accepted tokens + bonus, advance P, log accepted_len; emit [B, emit_cap] (optional) receives
 * [count, tokens..., -1 padding] of this step for host streaming. */
int ygg_commit(ygg_seq seq, ygg_tree vtree, const int32_t* path, const int32_t* path_len, const int32_t* bonus,
               int32_t* emit, int emit_cap, ygg_stream_t stream);

/* ---------------- K8: on-device stage timer ---------------- */
int ygg_stamp(unsigned long long* slot, ygg_stream_t stream);

/* In-graph kernel timeline (profiling only).  While armed, every launch of a traced kernel
 * (gemv = 1, decode attention = 2) takes the next slot of buf[slots][8] — {first CTA start, first
 * return from the grid-dependency wait, last CTA end, kernel checkpoints 3..7 (latest over CTAs)},
 * written with %globaltimer atomics; the caller initialises fields 0 and 1 to ~0, the rest to 0.  Arming with slots = 0 disarms.
 * ygg_trace_used returns the number of slots taken and copies their kernel ids. */
/* The armed state is per host thread (thread_local): only launches issued by the arming thread are traced. */
int ygg_trace_arm(unsigned long long* buf, int slots);
int ygg_trace_used(int* kernel_ids, int cap);

/* ---------------- Row-block GEMV (decode passes, 1..16 token rows) ----------------
 * Y = X . W^T with the layer epilogue fused; one launch per matmul, full K per 16-row block of W
 * (no split-K partials).  Weights in the fused layout (model.prepare_fused_): RMSNorm gains folded,
 * QKV rows RoPE-pair interleaved, gate/up rows interleaved.  ss_in / ss_out are per-block sums of
 * squares of the un-normalised residual ([blocks][M]); the consumer applies rstd. */
typedef enum {
  YGG_GEMV_STORE = 1, YGG_GEMV_QKV = 2, YGG_GEMV_SWIGLU = 3, YGG_GEMV_RESID = 4,
  YGG_GEMV_STORE_TOPK = 5  /* STORE + per-CTA top-k partials of every token row (M <= 8, k <= 8) */
} ygg_gemv_kind;
typedef struct {
  int32_t kind;
  float* out;            /* STORE: [M][ld] f32 */
  int32_t ld;
  const float* ss_in;    /* [ss_blocks][M] or NULL (no folded RMSNorm) */
  int32_t ss_blocks;
  int32_t norm_dim;
  float eps;
  void* q_out;           /* QKV: q [M][Hq][hd] bf16 */
  void* cache;           /* QKV: this layer's [B][2][Hkv][S][hd] block (V transposed) */
  int32_t S, Hq, Hkv, hd;
  const int32_t* pos; const int32_t* slot; const int32_t* req;
  const float* rope_cs;  /* [positions][hd/2][2] */
  void* act_out;         /* SWIGLU: [M][N/2] bf16 */
  float* resid;          /* RESID: [M][N] f32, updated in place */
  void* hb;              /* RESID: bf16 copy of the residual */
  float* ss_out;         /* RESID: [N/16][M] */
  void* topk_part;       /* STORE_TOPK: >= ygg_topk_partial_bytes(M, ygg_gemv_grid(plan)) bytes */
  int32_t topk_k;        /* STORE_TOPK: 1..8 */
  float inv_temp;        /* STORE_TOPK: 1 / temperature applied to the logits before softmax / ranking */
} ygg_gemv_epilogue;
size_t ygg_gemv_plan_size(void);
int ygg_gemv_grid(const void* plan);  /* CTAs of the plan = top-k chunks per row of STORE_TOPK */
/* The plan's weight tensor map (CUtensorMap, 128 bytes: box {64, 16 rows, 8 k-chunks of 64}) and
 * stream geometry (16-row blocks, 512-wide k chunks per block, ring stages). */
int ygg_gemv_stream_info(const void* plan, void* weight_map, int* nblk, int* kchunks, int* stages);
/* Optional: after streaming its own weights every CTA pulls its slices of up to two regions
 * [ptr, ptr + bytes) into L2 (later weights / the next attention's cache; region 0 or 1, issued in
 * that order; bytes = 0 disables the region). */
int ygg_gemv_set_l2_prefetch(void* plan, int region, const void* ptr, size_t bytes);
int ygg_gemv_plan_init(void* plan, const void* W, const void* X, int M, int N, int K, int num_ctas);
/* Ring depth override (2..16 stages of 16 weight rows x 512 k; default: the shared-memory budget). */
int ygg_gemv_plan_set_stages(void* plan, int stages);
int ygg_gemv_run(const void* plan, const ygg_gemv_epilogue* epi, ygg_stream_t stream);

/* ---------------- Decode attention (tree / draft / verify passes) ----------------
 * One CTA per (kv head, request, 64-row tile of (token, head) query rows) walks every visible key
 * chunk with an online softmax (no split-KV partials, no combine launch); prefix keys always visible,
 * block keys by the row's tree-mask bits (causal when mask_words == 0).  q [B*T][Hq][hd]; cache_layer as for ygg_attn_plan_init;
 * out [B*T][Hq][hd] bf16.  kvsplit = CTAs per cluster splitting the keys (0 = automatic: as many as
 * fit one wave, at most 4; capped at 4 for hd 128 and 8 for hd 64); ksplit = key-split warp groups
 * inside a CTA (0 = automatic: 8 warps / row warps, at most 2 for hd 128).  The partials merge in
 * fixed order, so two plans with the same (kvsplit, ksplit) reduce identically whatever their row
 * count (the lossless-greedy identity between a tree verify and AR decoding relies on it); stages = key /
 * value ring stages (0 = automatic; rounded down to a multiple of ksplit, shrunk to fit shared memory). */
size_t ygg_attn_dec_plan_size(void);
int ygg_attn_dec_plan_init(void* plan, const void* q, const void* cache_layer, int B, int T, int Hq, int Hkv, int hd,
                           int S, int kvsplit, int ksplit, int stages);
/* Launch order contract (programmatic dependent launch): K / V chunks wholly inside the committed
 * prefix (keys < blk_start) and blk_start / blk_len are read BEFORE the grid-dependency wait, so they
 * must have been written at least two kernels earlier on the stream and the kernel immediately
 * before this launch must not trigger its dependents before its own grid-dependency wait (every
 * libygg kernel that precedes it in a pass obeys this; a non-PDL kernel always does).
 * workspace: >= ygg_attn_dec_workspace_size(plan) bytes (currently 0; may be NULL).  The key chunks of
 * each (kv head, request, row tile) are split over a thread-block cluster of CTAs and merged in the
 * leader CTA's shared memory in fixed split order (YGG_ATTN_DEC_KVSPLIT overrides the cluster size). */
size_t ygg_attn_dec_workspace_size(const void* plan);
/* Optional: every launch of this plan also pulls up to two regions [ptr, ptr + bytes) into L2 (each
 * split over its CTAs, issued after the CTA's own loads) — later weights, streamed while the
 * attention leaves HBM idle.  region 0 or 1; bytes = 0 disables the region. */
int ygg_attn_dec_set_l2_prefetch(void* plan, int region, const void* ptr, size_t bytes);
/* Optional: every launch also pulls into L2 the weight chunks of a row-block GEMV plan that its ring
 * cannot hold (chunks >= its stage count of every block), through the GEMV's own tensor map — for a
 * GEMV whose CTAs stream one block each.  gemv_plan = NULL disables. */
int ygg_attn_dec_set_gemv_prefetch(void* plan, const void* gemv_plan);
int ygg_attn_dec_run(const void* plan, const int32_t* blk_start, const int32_t* blk_len, const uint32_t* qmask,
                     int mask_words, float scale, void* out, void* workspace, ygg_stream_t stream);

/* K2 tree attention on tcgen05 / TMEM (csrc/attn_tree.cu) for tree / decode passes: the same
 * visibility and arguments as ygg_attn_dec_run: committed prefix + ancestor mask over the tree block;
 * S = Q K^T and O = P V on the tensor cores with S / O in TMEM, one (csplit, 1, 1) thread-block
 * cluster per (kv head, request, row tile of <= 32 tokens), the keys split over the cluster's CTAs in
 * 64-key chunks and merged through DSMEM in fixed rank order (deterministic, no combine launch, no
 * workspace).  csplit in {0 (automatic: the largest of 4, 2, 1 keeping the grid in one wave), 1, 2, 4};
 * row_tiles = 0 picks the fewest tiles.  Same launch-order contract as ygg_attn_dec_run. */
size_t ygg_attn_tree_plan_size(void);
int ygg_attn_tree_plan_init(void* plan, const void* q, const void* cache_layer, int B, int T, int Hq, int Hkv, int hd,
                            int S, int csplit, int row_tiles);
int ygg_attn_tree_info(const void* plan, int* csplit, int* row_tiles, int* tokens_per_tile);
int ygg_attn_tree_set_l2_prefetch(void* plan, int region, const void* ptr, size_t bytes);
/* Profiling only: every launch writes 16 %globaltimer checkpoints per CTA into stamps (NULL = off). */
int ygg_attn_tree_set_debug(void* plan, unsigned long long* stamps);
/* A/B knob: late = 0 triggers the dependent launch right after the dependency wait (the next kernel's
 * prologue overlaps this one); late = 1 (the plan default, measured faster) only when each CTA ends. */
int ygg_attn_tree_set_trigger(void* plan, int late);
int ygg_attn_tree_run(const void* plan, const int32_t* blk_start, const int32_t* blk_len, const uint32_t* qmask,
                      int mask_words, float scale, void* out, ygg_stream_t stream);


#ifdef __cplusplus
}
#endif
#endif /* YGG_H_ */
