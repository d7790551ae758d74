// Device-side bookkeeping of the speculative step, so a whole step replays from a CUDA graph
// with no host synchronisation: every data-dependent quantity (prefix length P, bonus token,
// tree tensors, accepted lengths) lives in device memory and these kernels turn it into the
// static-shape inputs of the next forward pass.
//
// Conventions (reference simulator.py:9-14):
//   hist[b][0..P) are confirmed tokens with KV in the target cache, hist[b][P] is the pending
//   bonus token.  A tree node i of the grown (draft) tree lives at draft slot P+1+i, position
//   P+1+depth(i); verify row 0 is the bonus at slot P, row 1+i is pruned node i at slot P+1+i.
#include "common.cuh"
#include "host_util.h"

namespace ygg {

// Draft pass 0: rows [hist[P-1], hist[P]] at positions/slots P-1, P (causal), padding rows
// write scratch slots beyond the tree region and attend only to the prefix.
__global__ void pass0_inputs_kernel(ygg_seq seq, int R, int tree_cap, int32_t* tokens, int32_t* pos, int32_t* slot,
                                    int32_t* req, uint32_t* qmask, int mask_words, int32_t* blk_start,
                                    int32_t* blk_len) {
  pdl_wait();
  pdl_launch_dependents();
  const int b = blockIdx.x;
  const int P = seq.P[b];
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    const int m = b * R + r;
    req[m] = b;
    int tok, p, s;
    if (r < 2) {
      p = P - 1 + r;
      tok = seq.hist[static_cast<size_t>(b) * seq.S + p];
      s = p;
    } else {
      tok = 0;
      p = P;
      s = P + 1 + tree_cap + r;
    }
    tokens[m] = tok;
    pos[m] = p;
    slot[m] = s;
    for (int w = 0; w < mask_words; ++w) {
      uint32_t v = 0;
      if (w == 0 && r < 2) v = (r == 0) ? 1u : 3u;
      qmask[static_cast<size_t>(m) * mask_words + w] = v;
    }
  }
  if (threadIdx.x == 0) {
    blk_start[b] = P - 1;
    blk_len[b] = 2;
  }
}

// Roots from draft pass 0 (DrafterDistribution.root(), egt.py:56-58): the top-1 candidate of
// the bonus row (row 1 of pass 0).  Resets each tree to the single root node.
__global__ void init_roots_kernel(ygg_tree t, const int32_t* __restrict__ cand_tok,
                                  const double* __restrict__ cand_prob, int k, int R, int row) {
  pdl_wait();
  pdl_launch_dependents();
  const int b = blockIdx.x;
  const size_t tb = static_cast<size_t>(b) * t.cap;
  for (int i = threadIdx.x; i < t.cap; i += blockDim.x) {
    for (int w = 0; w < t.mask_words; ++w) t.mask[(tb + i) * t.mask_words + w] = 0u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const size_t ci = (static_cast<size_t>(b) * R + row) * k;
    t.token[tb] = cand_tok[ci];
    t.prob[tb] = cand_prob[ci];
    t.cum[tb] = cand_prob[ci];  // path_prob(root) = 1.0 * s_root (egt.py:102-104)
    t.parent[tb] = -1;
    t.depth[tb] = 0;
    t.mask[tb * t.mask_words] = 1u;
    t.size[b] = 1;
    t.frontier[tb] = 0;
    t.frontier_n[b] = 1;
    t.flags[b] = 0;
  }
}

// Draft pass over the newest level: rows = frontier nodes (padded to R), block = tree nodes so far.
__global__ void level_inputs_kernel(ygg_tree t, ygg_seq seq, int R, int k, int32_t* tokens, int32_t* pos,
                                    int32_t* slot, int32_t* req, uint32_t* qmask, int mask_words,
                                    int32_t* blk_start, int32_t* blk_len, int32_t* cand_n,
                                    unsigned long long* trace) {
  if (threadIdx.x == 0) trace_min(trace, 0);
  pdl_wait();
  if (threadIdx.x == 0) trace_min(trace, 1);
  pdl_launch_dependents();
  const int b = blockIdx.x;
  const size_t tb = static_cast<size_t>(b) * t.cap;
  const int P = seq.P[b];
  const int fn = (t.flags[b] & 8) ? 0 : t.frontier_n[b];  // stopped trees draft nothing
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    const int m = b * R + r;
    req[m] = b;
    if (r < fn) {
      const int node = t.frontier[tb + r];
      tokens[m] = t.token[tb + node];
      pos[m] = P + 1 + t.depth[tb + node];
      slot[m] = P + 1 + node;
      for (int w = 0; w < mask_words; ++w)
        qmask[static_cast<size_t>(m) * mask_words + w] = (w < t.mask_words) ? t.mask[(tb + node) * t.mask_words + w] : 0u;
      cand_n[m] = k;
    } else {
      tokens[m] = 0;
      pos[m] = P + 1;
      slot[m] = P + 1 + t.cap + r;
      for (int w = 0; w < mask_words; ++w) qmask[static_cast<size_t>(m) * mask_words + w] = 0u;
      cand_n[m] = 0;
    }
  }
  if (threadIdx.x == 0) {
    blk_start[b] = P + 1;
    blk_len[b] = t.size[b];
  }
  if (threadIdx.x == 0) trace_max(trace, 2);
}

// Verify rows: row 0 = bonus (slot P), row 1+i = pruned node i (slot P+1+i); mask over the
// T = cap+1 verify slots = bit 0 | (tree row << 1).
__global__ void verify_inputs_kernel(ygg_tree t, ygg_seq seq, int32_t* tokens, int32_t* pos, int32_t* slot,
                                     int32_t* req, uint32_t* qmask, int mask_words, int32_t* blk_start,
                                     int32_t* blk_len) {
  pdl_wait();
  pdl_launch_dependents();
  const int b = blockIdx.x;
  const int T = t.cap + 1;
  const size_t tb = static_cast<size_t>(b) * t.cap;
  const int P = seq.P[b];
  const int n = t.size[b];
  for (int r = threadIdx.x; r < T; r += blockDim.x) {
    const int m = b * T + r;
    req[m] = b;
    uint32_t* mrow = qmask + static_cast<size_t>(m) * mask_words;
    if (r == 0) {
      tokens[m] = seq.hist[static_cast<size_t>(b) * seq.S + P];
      pos[m] = P;
      slot[m] = P;
      for (int w = 0; w < mask_words; ++w) mrow[w] = (w == 0) ? 1u : 0u;
    } else {
      const int i = r - 1;
      slot[m] = P + r;
      if (i < n) {
        tokens[m] = t.token[tb + i];
        pos[m] = P + 1 + t.depth[tb + i];
        const uint32_t* trow = t.mask + (tb + i) * t.mask_words;
        for (int w = 0; w < mask_words; ++w) {
          const uint32_t lo = (w < t.mask_words) ? trow[w] : 0u;
          const uint32_t carry = (w >= 1 && w - 1 < t.mask_words) ? (trow[w - 1] >> 31) : 0u;
          mrow[w] = (lo << 1) | carry | (w == 0 ? 1u : 0u);
        }
      } else {
        tokens[m] = 0;
        pos[m] = P + 1;
        for (int w = 0; w < mask_words; ++w) mrow[w] = ((r >> 5) == w) ? (1u << (r & 31)) : 0u;
      }
    }
  }
  if (threadIdx.x == 0) {
    blk_start[b] = P;
    blk_len[b] = T;
  }
}

// Commit an accepted path: append the accepted tokens + bonus to the history, advance P,
// record accepted_len (lagged host readback feeds the depth predictor).  A request that has reached
// its generation limit, or whose next prefix would pass seq.p_limit (the next step's tree and scratch
// slots must stay inside the S-slot cache), is frozen: nothing is appended, P stays, emit count 0.
__global__ void commit_kernel(ygg_seq seq, ygg_tree vt, const int32_t* __restrict__ path,
                              const int32_t* __restrict__ path_len, const int32_t* __restrict__ bonus,
                              int32_t* __restrict__ emit, int emit_cap) {
  pdl_wait();
  pdl_launch_dependents();
  const int b = threadIdx.x;
  const int step = seq.step[0];
  if (b < seq.B) {
    const size_t tb = static_cast<size_t>(b) * vt.cap;
    const int P = seq.P[b];
    const int a = path_len[b];
    const int limit = seq.p_limit > 0 ? seq.p_limit : seq.S - 1;
    const bool finished = seq.gen_limit && seq.n_gen[b] >= seq.gen_limit[b];
    const bool full = !finished && P + 1 + a > limit;
    int32_t* em = emit ? emit + static_cast<size_t>(b) * emit_cap : nullptr;
    if (finished || full) {
      if (seq.status) seq.status[b] |= (finished ? 1 : 0) | (full ? 2 : 0);
      if (em) {
        em[0] = 0;
        for (int i = 0; i < emit_cap - 1; ++i) em[1 + i] = -1;
      }
    } else {
      int32_t* h = seq.hist + static_cast<size_t>(b) * seq.S;
      for (int i = 0; i < a; ++i) h[P + 1 + i] = vt.token[tb + path[tb + i]];
      h[P + 1 + a] = bonus[b];
      if (em) {  // per-step emitted tokens for host streaming: [count, tokens...]
        em[0] = 1 + a;
        for (int i = 0; i < emit_cap - 1; ++i) em[1 + i] = (i <= a) ? h[P + 1 + i] : -1;
      }
      seq.P[b] = P + 1 + a;
      seq.n_gen[b] += 1 + a;
      if (seq.status && seq.gen_limit && seq.n_gen[b] >= seq.gen_limit[b]) seq.status[b] |= 1;
    }
    if (seq.acc_log && seq.log_cap > 0)
      seq.acc_log[static_cast<size_t>(b) * seq.log_cap + (step % seq.log_cap)] = (finished || full) ? 0 : 1 + a;
  }
  __syncthreads();
  if (b == 0) seq.step[0] = step + 1;
}

}  // namespace ygg

using namespace ygg;

extern "C" {

int ygg_pass0_inputs(ygg_seq seq, int R, int tree_cap, int32_t* tokens, int32_t* pos, int32_t* slot, int32_t* req,
                     uint32_t* qmask, int mask_words, int32_t* blk_start, int32_t* blk_len, ygg_stream_t stream) {
  YGG_CHECK_ARG(R >= 2 && mask_words >= 1, "pass 0 needs R >= 2 rows and a mask");
  YGG_LAUNCH_PDL(pass0_inputs_kernel, dim3(seq.B), dim3(64), 0, reinterpret_cast<cudaStream_t>(stream), seq, R,
                 tree_cap, tokens, pos, slot, req, qmask, mask_words, blk_start, blk_len);
  return YGG_OK;
}

int ygg_init_roots(ygg_tree tree, const int32_t* cand_tok, const double* cand_prob, int k, int R, int row,
                   ygg_stream_t stream) {
  YGG_CHECK_ARG(cand_tok && cand_prob && k >= 1 && row < R, "invalid arguments");
  YGG_LAUNCH_PDL(init_roots_kernel, dim3(tree.B), dim3(128), 0, reinterpret_cast<cudaStream_t>(stream), tree, cand_tok,
                 cand_prob, k, R, row);
  return YGG_OK;
}

int ygg_level_inputs(ygg_tree tree, ygg_seq seq, int R, int k, int32_t* tokens, int32_t* pos, int32_t* slot,
                     int32_t* req, uint32_t* qmask, int mask_words, int32_t* blk_start, int32_t* blk_len,
                     int32_t* cand_n, ygg_stream_t stream) {
  YGG_CHECK_ARG(mask_words >= tree.mask_words, "query mask narrower than the tree mask");
  YGG_LAUNCH_PDL(level_inputs_kernel, dim3(tree.B), dim3(64), 0, reinterpret_cast<cudaStream_t>(stream), tree, seq, R,
                 k, tokens, pos, slot, req, qmask, mask_words, blk_start, blk_len, cand_n, trace_next(13));
  return YGG_OK;
}

int ygg_verify_inputs(ygg_tree vtree, ygg_seq seq, int32_t* tokens, int32_t* pos, int32_t* slot, int32_t* req,
                      uint32_t* qmask, int mask_words, int32_t* blk_start, int32_t* blk_len, ygg_stream_t stream) {
  YGG_CHECK_ARG(mask_words * 32 >= vtree.cap + 1, "verify mask too narrow");
  YGG_LAUNCH_PDL(verify_inputs_kernel, dim3(vtree.B), dim3(128), 0, reinterpret_cast<cudaStream_t>(stream), vtree, seq,
                 tokens, pos, slot, req, qmask, mask_words, blk_start, blk_len);
  return YGG_OK;
}

int ygg_commit(ygg_seq seq, ygg_tree vtree, const int32_t* path, const int32_t* path_len, const int32_t* bonus,
               int32_t* emit, int emit_cap, ygg_stream_t stream) {
  YGG_CHECK_ARG(path && path_len && bonus, "invalid arguments");
  YGG_CHECK_ARG(seq.B <= 1024, "too many requests");
  YGG_LAUNCH_PDL(commit_kernel, dim3(1), dim3(seq.B), 0, reinterpret_cast<cudaStream_t>(stream), seq, vtree, path,
                 path_len, bonus, emit, emit_cap);
  return YGG_OK;
}

}  // extern "C"
