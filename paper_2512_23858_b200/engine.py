"""The speculative-decoding step on the GPU: EGT draft -> prune -> tree verify -> accept -> compact.

One ``SpecDecoder.step`` is the north-star hot path, realising the
reference iteration (pkg/src/specsim/simulator.py:305-338) with real models:

  draft pass 0   : draft forward over [x_{P-1}, bonus]; root = top-1 of the bonus row
                   (DrafterDistribution.root(), egt.py:56-58; "the root rides along with the
                   previous bonus", simulator.py:9-11)
  draft pass 1..D: draft forward over the newest level with the tree mask, softmax top-k per
                   row (K1a) and one global top-W grow_step per tree (K1b, egt.py:83-114)
  prune          : path products + SubtreeKnapsack + Eq.3 objective from the device latency
                   table (K6, egt.py:150-282), TokenTree.subtree relabel (token_tree.py:146-168)
  verify         : target forward over [bonus, pruned nodes] with the ancestor mask (K2-K4)
  accept         : greedy / sampled acceptance walk (K5, acceptance.py:221-241)
  compact+commit : accepted K/V moved to contiguous slots in both caches, P advanced

Every data-dependent value stays on the device, so the whole step is captured once per static
shape (D, W, max_verify, B) as a CUDA graph and replayed with no host synchronisation.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .device_tree import DeviceTrees, SeqState
from .forward import Forward, new_cache, prefill_causal
from .model import ModelConfig
from .plan import ForwardPlan

GREEDY, SAMPLE = "greedy", "sample"


@dataclass
class StepShape:
    depth: int          # D: draft levels past the root
    width: int          # W: nodes per level
    expansion_k: int = 8
    max_verify: int = 64
    fixed_verify: int = 0  # >0: prune to exactly this many nodes (static verify width)

    def __post_init__(self):
        if self.depth < 1 or self.width < 1 or self.expansion_k < 1:
            raise ValueError("depth, width and expansion_k must be >= 1")
        if self.depth + 1 > 64:  # an accepted path holds <= depth + 1 nodes (KV compaction bound)
            raise ValueError("depth must be <= 63")
        if self.expansion_k > 32:
            raise ValueError("expansion_k must be <= 32")
        if self.max_verify < 1:
            raise ValueError("max_verify must be >= 1")


class SpecDecoder:
    def __init__(
        self,
        target_cfg: ModelConfig,
        target_w: dict,
        draft_cfg: ModelConfig,
        draft_w: dict,
        shape: StepShape,
        batch: int = 1,
        max_seq: int = 2048,
        act_dtype: torch.dtype = torch.bfloat16,
        mode: str = GREEDY,
        temperature: float = 1.0,
        profiles=None,
        prefill_len: int = 0,
        device="cuda",
        plan: ForwardPlan | None = None,
        share: "SpecDecoder | None" = None,
        scratch: int = 0,
        calibrate: bool = False,
        feature_tap: bool = False,
        overlap_compaction: bool = False,
    ):
        """``share``: another decoder whose sequence state, KV caches and prefill forwards this one
        uses (one decoding state, several captured step shapes: runtime.AdaptiveDecoder); ``scratch``:
        tree / padding slots to reserve past the prefix (default this shape's); ``calibrate``: the
        Eq.3 objective uses per-position acceptance rates measured on the device (set_node_table)
        instead of the draft's surrogate probabilities wherever a rate is known."""
        L.require_device()
        if target_cfg.vocab != draft_cfg.vocab:
            raise ValueError("target and draft must share a vocabulary")
        if mode not in (GREEDY, SAMPLE):
            raise ValueError(f"mode must be {GREEDY!r} or {SAMPLE!r}")
        self.tc, self.dc = target_cfg, draft_cfg
        self.tw, self.dw = target_w, draft_w
        self.shape = shape
        self.B = batch
        self.mode, self.temperature = mode, float(temperature)
        self.act_dtype = act_dtype
        D, W, k = shape.depth, shape.width, shape.expansion_k
        self.tree_cap = 1 + D * W
        self.vcap = min(shape.max_verify, self.tree_cap)
        self.T = self.vcap + 1
        self.R = max(W, 2)
        scratch = max(scratch, self.tree_cap + self.R + 8)
        dev = torch.device(device)
        self.dev = dev
        if share is not None:
            if share.B != batch or share.tc is not target_cfg or share.dc is not draft_cfg:
                raise ValueError("a shared decoding state needs the same batch and models")
            if share.S - share.seq.p_limit < scratch:
                raise ValueError("the shared state reserves too few scratch slots for this shape")
            self.S, self.seq, self.tcache, self.dcache = share.S, share.seq, share.tcache, share.dcache
        else:
            self.S = (max_seq + scratch + 63) // 64 * 64
            # commit freezes a request rather than let the next step's tree / scratch slots pass S
            self.seq = SeqState(batch, self.S, device=dev, p_limit=self.S - scratch)
            self.tcache = new_cache(target_cfg, batch, self.S, act_dtype, dev)
            self.dcache = new_cache(draft_cfg, batch, self.S, act_dtype, dev)
        tmw = max(1, (self.T + 31) // 32)
        dmw = max(1, (self.tree_cap + 31) // 32)
        self.plan = plan
        dplan = plan or ForwardPlan()
        if dplan.tree_attn is None:  # draft levels keep the mma.sync decode attention (plan.py: tree_attn)
            dplan = dataclasses.replace(dplan, tree_attn=False)
        self.draft = Forward(draft_cfg, draft_w, self.dcache, batch, self.R, dmw, act_dtype, plan=dplan)
        # The verify always runs the target's tree-pass families (stream-K GEMM, decode attention), never
        # the draft's row-block GEMV even when B * T <= 16: the GEMV needs the fused weight layout (it
        # would rewrite the shared target weights in place) and would round differently from ARDecoder,
        # the oracle of the lossless-greedy identity.
        self.verify = Forward(target_cfg, target_w, self.tcache, batch, self.T, tmw, act_dtype, gemv=False, plan=plan,
                              lm_argmax=mode == GREEDY)
        self.grown = DeviceTrees(batch, self.tree_cap, dev)
        self.vtree = DeviceTrees(batch, self.vcap, dev)
        i32 = dict(dtype=torch.int32, device=dev)
        f64 = dict(dtype=torch.float64, device=dev)
        rows = batch * self.R
        self.cand_tok = torch.zeros(rows, k, **i32)
        self.cand_prob = torch.zeros(rows, k, **f64)
        self.cand_n = torch.zeros(rows, **i32)
        self.topk_ws = torch.empty(int(L.lib().ygg_topk_workspace(max(rows, 1), draft_cfg.vocab, k)),
                                   dtype=torch.uint8, device=dev)
        # Draft top-k straight from the LM-head GEMV epilogue (per-CTA partials + one merge launch).
        self.topk_fused = self.draft.fuse_topk(k)
        self.keep_idx = torch.zeros(batch, self.tree_cap, **i32)
        self.new_idx = torch.zeros(batch, self.tree_cap, **i32)
        self.w_verify = torch.zeros(batch, **i32)
        self.exp_aal = torch.zeros(batch, **f64)
        self.speedup = torch.zeros(batch, **f64)
        self.row_argmax = torch.zeros(batch * self.T, **i32)
        self.path = torch.zeros(batch, self.vcap, **i32)
        self.path_len = torch.zeros(batch, **i32)
        self.acc_len = torch.zeros(batch, **i32)
        self.bonus = torch.zeros(batch, **i32)
        self.emit = torch.zeros(batch, D + 3, **i32)
        self.n_uniform = D + 3
        self.uniforms = torch.full((batch, self.n_uniform), 0.5, **f64)
        self._u_host = [torch.full((batch, self.n_uniform), 0.5, dtype=torch.float64).pin_memory() for _ in range(2)]
        self._u_ev = [torch.cuda.Event(), torch.cuda.Event()]
        self._u_used = [False, False]
        self._u_next = 0
        self.set_profiles(profiles)
        self.prefill_len = prefill_len
        self._prefill_fwd = share._prefill_fwd if share is not None else {}
        self._prefill_side = None  # side stream of the draft prefill (created on first use)
        # root candidate probabilities of the step's pass 0 (depth-predictor features)
        self.root_probs = torch.zeros(batch, k, **f64)
        # calibrated acceptance (ExplicitAcceptance by grown-tree position): device counts of tested /
        # accepted per position, and the table the prune objective reads (< 0: surrogate probability)
        self.calibrate = calibrate
        self.accept_counts = torch.zeros(self.tree_cap, 2, dtype=torch.int32, device=dev)
        # the target's last-token hidden state per request (depth-predictor feature)
        self.feature_tap = feature_tap and act_dtype == torch.bfloat16
        self.hidden_tap = torch.zeros(batch, target_cfg.d_model, dtype=torch.float32, device=dev)
        # Two-lane step (the reference's stage overlap, scheduler.py:224-268, on the GPU): the target KV
        # compaction of step i only has to land before the verify of step i+1, so it runs on a side
        # stream concurrently with step i+1's draft phase instead of on the critical path.
        self.overlap_compaction = overlap_compaction
        self._side = torch.cuda.Stream(device=dev) if overlap_compaction else None
        self.compact_base = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.node_table = torch.full((batch, self.tree_cap), -1.0, **f64)
        self.graph = None
        self.step_count = 0

    # ------------------------------------------------------------------
    def set_profiles(self, profiles) -> None:
        """Device copy of the latency table (ProfilePair) that drives the Eq.3 objective."""
        if profiles is None:
            d_bp, v_bp = ((1, 1.0), (64, 1.0)), ((1, 1.0), (64, 1.0))
        else:
            d_bp, v_bp = profiles.drafter.breakpoints, profiles.verifier.breakpoints
        raw = L.profile_pair_bytes(d_bp, v_bp)
        host = torch.frombuffer(bytearray(raw), dtype=torch.uint8)
        if not hasattr(self, "profiles_dev"):
            self.profiles_dev = torch.empty(len(raw), dtype=torch.uint8, device=self.dev)
        self.profiles_dev.copy_(host)

    # ------------------------------------------------------------------
    def _prefill_forward(self, cfg, w, cache, n: int) -> Forward:
        key = (cfg.name, n, id(cache))
        f = self._prefill_fwd.get(key)
        if f is None:
            f = Forward(cfg, w, cache, self.B, n, 0, self.act_dtype, plan=self.plan)
            self._prefill_fwd[key] = f
        return f

    def prefill(self, prompts: torch.Tensor) -> None:
        """Causal prefill of both models over ``prompts`` [B, P0]; the bonus is the target argmax."""
        B, P0 = prompts.shape
        if B != self.B:
            raise ValueError(f"expected {self.B} prompts, got {B}")
        if P0 + self.tree_cap + self.R + 8 > self.S:
            raise ValueError("prompt too long for the cache")
        lib = L.lib()
        s = L.stream_ptr()
        prompts_d = prompts.to(self.dev, torch.int32)
        self.seq.hist.zero_()
        self.seq.hist[:, :P0] = prompts_d
        # The two models' prefills are independent: the draft's runs on a side stream, filling the SMs the
        # target's latency-bound kernels (attention, epilogues, dependency gaps) leave idle.
        main = torch.cuda.current_stream(self.dev)
        if self._prefill_side is None:
            self._prefill_side = torch.cuda.Stream(self.dev)
        side = self._prefill_side
        side.wait_stream(main)
        with torch.cuda.stream(side):
            prefill_causal(self.dc, self.dw, self.dcache, prompts_d, self.act_dtype, False, self._prefill_fwd,
                           plan=self.plan)
        last = prefill_causal(self.tc, self.tw, self.tcache, prompts_d, self.act_dtype, True, self._prefill_fwd,
                              plan=self.plan)
        am = torch.zeros(B, dtype=torch.int32, device=self.dev)
        L.check(lib.ygg_row_stats(last.data_ptr(), L.YGG_F32, B, self.tc.vocab, self.tc.vocab, 1.0, am.data_ptr(),
                                  None, s))
        self.seq.hist[torch.arange(B, device=self.dev), P0] = am
        main.wait_stream(side)
        self.seq.P.fill_(P0)
        self.seq.n_gen.fill_(1)
        self.seq.step.zero_()
        self.seq.status.zero_()
        self.seq.gen_limit.fill_(2**31 - 1)
        self.path_len.zero_()  # no pending (deferred) compaction

    # ------------------------------------------------------------------
    def prefill_slot(self, b: int, prompt: torch.Tensor, n_tokens: int, chunk: int = 64) -> None:
        """Admit one request into slot ``b`` while the other slots keep their state (continuous
        batching): causal prefill of ``prompt`` [P0] into slot b's region of both caches in fixed
        ``chunk``-row passes (one set of plans per slot, whatever the prompt length; the last chunk is
        padded — its padding rows only write KV past the prefix), the bonus = target argmax of the last
        prompt row, and slot b's sequence state reset with generation limit ``n_tokens``."""
        P0 = int(prompt.numel())
        if not 0 <= b < self.B:
            raise IndexError(f"slot {b} out of range")
        if P0 < 1 or P0 + n_tokens + self.shape.depth + 2 > self.seq.p_limit or P0 + chunk > self.S:
            raise ValueError("prompt + generation do not fit the slot's cache")
        lib = L.lib()
        dev = self.dev
        toks = torch.zeros(((P0 + chunk - 1) // chunk) * chunk, dtype=torch.int32, device=dev)
        toks[:P0] = prompt.to(dev, torch.int32)
        bonus = torch.zeros(1, dtype=torch.int32, device=dev)
        for cfg, w, cache in ((self.tc, self.tw, self.tcache), (self.dc, self.dw, self.dcache)):
            view = cache[:, b : b + 1]
            nchunk = toks.numel() // chunk
            for c in range(nchunk):
                final = c == nchunk - 1
                key = ("slot", b, cfg.name, chunk, final and cfg is self.tc)
                f = self._prefill_fwd.get(key)
                if f is None:
                    f = Forward(cfg, w, view, 1, chunk, 0, self.act_dtype, logits=final and cfg is self.tc, gemv=False,
                                decode_attn=False, plan=self.plan)
                    self._prefill_fwd[key] = f
                f.tokens.copy_(toks[c * chunk : (c + 1) * chunk])
                pos = torch.arange(c * chunk, (c + 1) * chunk, dtype=torch.int32, device=dev)
                f.pos.copy_(pos)
                f.slot.copy_(pos)
                f.blk_start.fill_(c * chunk)
                f.blk_len.fill_(chunk)
                f.run()
                if final and cfg is self.tc:
                    r = (P0 - 1) - c * chunk
                    L.check(lib.ygg_row_stats(f.logits[r:].data_ptr(), L.YGG_F32, 1, cfg.vocab, cfg.vocab, 1.0,
                                              bonus.data_ptr(), None, L.stream_ptr()))
        self.path_len[b] = 0  # no deferred compaction of the slot's previous request
        sq = self.seq
        sq.hist[b].zero_()
        sq.hist[b, :P0] = toks[:P0]
        sq.hist[b, P0] = bonus[0]
        sq.P[b] = P0
        sq.n_gen[b] = 1
        sq.status[b] = 0
        sq.gen_limit[b] = n_tokens

    def park_slot(self, b: int) -> None:
        """Mark slot b idle: a valid dummy state (P = 1) that the commit kernel keeps frozen."""
        self.path_len[b] = 0
        sq = self.seq
        sq.hist[b].zero_()
        sq.P[b] = 1
        sq.n_gen[b] = 0
        sq.gen_limit[b] = 0
        sq.status[b] = 1

    # ------------------------------------------------------------------
    def _draft_topk(self, rows: int, k: int, s) -> None:
        """Candidates of every draft row (DrafterDistribution.candidates, egt.py:65-80)."""
        lib, dr = L.lib(), self.draft
        if self.topk_fused:
            L.check(lib.ygg_topk_merge(dr.topk_part.data_ptr(), rows, dr.topk_chunks, k, self.cand_tok.data_ptr(),
                                       self.cand_prob.data_ptr(), None, s))
        else:
            L.check(lib.ygg_topk_softmax(dr.logits.data_ptr(), L.YGG_F32, rows, self.dc.vocab, self.dc.vocab, k, 1.0,
                                         self.cand_tok.data_ptr(), self.cand_prob.data_ptr(), None,
                                         self.topk_ws.data_ptr(), self.topk_ws.numel(), s))

    def _launch_step(self, stream=None, stamp=None) -> None:
        """Enqueue one step.  ``stamp(i)`` (K8 profiler) is called at the stage boundaries
        0 | pass0 | 1 | draft levels | 2 | prune | 3 | verify forward | 4 | accept+compact+commit | 5."""
        if stamp is None:
            stamp = lambda i: None  # noqa: E731
        stamp(0)
        lib = L.lib()
        s = L.stream_ptr(stream)
        chk = L.check
        sh = self.shape
        D, W, k = sh.depth, sh.width, sh.expansion_k
        dr, vf, g, vt = self.draft, self.verify, self.grown, self.vtree
        rows = self.B * self.R
        tc, dc = self.tc, self.dc
        main = stream if stream is not None else torch.cuda.current_stream(self.dev)
        if self.overlap_compaction:
            # lane 2: the previous step's target KV compaction (base = its pre-commit prefix length)
            self._side.wait_stream(main)
            chk(lib.ygg_kv_compact(self.tcache.data_ptr(), L.dtype_code(self.act_dtype), tc.n_layers, self.B,
                                   tc.n_kv_heads, self.S, tc.head_dim, self.tcache.stride(0),
                                   self.compact_base.data_ptr(), self.path.data_ptr(), self.path_len.data_ptr(),
                                   self.vcap, None, 0, None, 0, 0, L.stream_ptr(self._side)))
        # ---- draft pass 0: [x_{P-1}, bonus] -> root
        chk(lib.ygg_pass0_inputs(self.seq.struct, self.R, self.tree_cap, dr.tokens.data_ptr(), dr.pos.data_ptr(),
                                 dr.slot.data_ptr(), dr.req.data_ptr(), dr.qmask.data_ptr(), dr.mask_words,
                                 dr.blk_start.data_ptr(), dr.blk_len.data_ptr(), s))
        dr.run(stream)
        self._draft_topk(rows, k, s)
        chk(lib.ygg_init_roots(g.struct, self.cand_tok.data_ptr(), self.cand_prob.data_ptr(), k, self.R, 1, s))
        with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream()):
            self.root_probs.copy_(self.cand_prob.view(self.B, self.R, k)[:, 1, :])
        stamp(1)
        # ---- draft passes 1..D: grow one level each
        for lvl in range(D):
            chk(lib.ygg_level_inputs(g.struct, self.seq.struct, self.R, k, dr.tokens.data_ptr(), dr.pos.data_ptr(),
                                     dr.slot.data_ptr(), dr.req.data_ptr(), dr.qmask.data_ptr(), dr.mask_words,
                                     dr.blk_start.data_ptr(), dr.blk_len.data_ptr(), self.cand_n.data_ptr(), s))
            dr.run(stream)
            self._draft_topk(rows, k, s)
            chk(lib.ygg_egt_grow_level(g.struct, self.R, k, W, self.cand_tok.data_ptr(), self.cand_prob.data_ptr(),
                                       self.cand_n.data_ptr(), s))
        stamp(2)
        # ---- prune (latency-aware objective or fixed width)
        args = L.YggPruneArgs(sh.max_verify, D, W, sh.fixed_verify, 0,
                              self.node_table.data_ptr() if self.calibrate else None)
        chk(lib.ygg_knapsack_prune(g.struct, None, self.profiles_dev.data_ptr(), args, self.keep_idx.data_ptr(),
                                   self.new_idx.data_ptr(), self.w_verify.data_ptr(), self.exp_aal.data_ptr(),
                                   self.speedup.data_ptr(), None, None, None, None, s))
        chk(lib.ygg_tree_subtree(g.struct, vt.struct, self.keep_idx.data_ptr(), self.new_idx.data_ptr(), s))
        stamp(3)
        # ---- verify
        if self.overlap_compaction:
            main.wait_stream(self._side)  # join: the target prefix is compacted
        chk(lib.ygg_verify_inputs(vt.struct, self.seq.struct, vf.tokens.data_ptr(), vf.pos.data_ptr(),
                                  vf.slot.data_ptr(), vf.req.data_ptr(), vf.qmask.data_ptr(), vf.mask_words,
                                  vf.blk_start.data_ptr(), vf.blk_len.data_ptr(), s))
        vf.run(stream)
        stamp(4)
        if self.mode == GREEDY:
            vf.argmax_rows(self.row_argmax, s)  # fused LM-head argmax keys (bf16) / logits scan (f32)
            chk(lib.ygg_accept(vt.struct, L.YGG_ACCEPT_GREEDY, None, None, 0, self.row_argmax.data_ptr(), None,
                               L.YGG_F32, self.tc.vocab, self.tc.vocab, None, 1.0, self.path.data_ptr(),
                               self.path_len.data_ptr(), self.acc_len.data_ptr(), self.bonus.data_ptr(), None, s))
        else:  # self.uniforms is filled by set_uniforms() on the stream, before the replay
            # no row-stats pass: the accept kernel computes the log-sum-exp of the rows it walks
            # (<= depth + 1 per request; cfg4: 0.79 -> ~0.03 ms per step)
            chk(lib.ygg_accept(vt.struct, L.YGG_ACCEPT_SAMPLE, None, self.uniforms.data_ptr(), self.n_uniform,
                               None, vf.logits.data_ptr(), L.YGG_F32, self.tc.vocab, self.tc.vocab,
                               None, self.temperature, self.path.data_ptr(),
                               self.path_len.data_ptr(), self.acc_len.data_ptr(), self.bonus.data_ptr(), None, s))
        if self.feature_tap:
            chk(lib.ygg_feature_tap(vf.xn.data_ptr(), self.T, self.tc.d_model, self.path.data_ptr(), self.vcap,
                                    self.path_len.data_ptr(), self.B, self.hidden_tap.data_ptr(), s))
        if self.calibrate:
            chk(lib.ygg_accept_stats(vt.struct, self.keep_idx.data_ptr(), self.tree_cap, self.path.data_ptr(),
                                     self.path_len.data_ptr(), self.accept_counts.data_ptr(), s))
        # ---- KV compaction (target: verify order; draft: grown-tree slots, leaves never drafted)
        if self.overlap_compaction:
            with torch.cuda.stream(main):
                self.compact_base.copy_(self.seq.P)  # deferred to the next step's lane 2
        else:
            chk(lib.ygg_kv_compact(self.tcache.data_ptr(), L.dtype_code(self.act_dtype), tc.n_layers, self.B,
                                   tc.n_kv_heads, self.S, tc.head_dim, self.tcache.stride(0), self.seq.P.data_ptr(),
                                   self.path.data_ptr(), self.path_len.data_ptr(), self.vcap, None, 0, None, 0, 0, s))
        chk(lib.ygg_kv_compact(self.dcache.data_ptr(), L.dtype_code(self.act_dtype), dc.n_layers, self.B,
                               dc.n_kv_heads, self.S, dc.head_dim, self.dcache.stride(0), self.seq.P.data_ptr(),
                               self.path.data_ptr(), self.path_len.data_ptr(), self.vcap, self.keep_idx.data_ptr(),
                               self.tree_cap, g.depth.data_ptr(), self.tree_cap, D, s))
        chk(lib.ygg_commit(self.seq.struct, vt.struct, self.path.data_ptr(), self.path_len.data_ptr(),
                           self.bonus.data_ptr(), self.emit.data_ptr(), self.emit.shape[1], s))
        stamp(5)

    # ------------------------------------------------------------------
    def node_rates(self, prior: float = 4.0) -> np.ndarray:
        """Calibrated acceptance per grown-tree position from the device counts (host sync):
        p_i = (accepted_i + m r_d) / (tested_i + m) with r_d the pooled rate of i's EGT level (depth
        d = level of position i: nodes 1 + (d-1) W .. d W) and m = ``prior``; -1 where neither the
        position nor its level has been tested (the objective then keeps the surrogate probability)."""
        c = self.accept_counts.cpu().numpy().astype(np.float64)
        W, D = self.shape.width, self.shape.depth
        out = np.full(self.tree_cap, -1.0)
        last = None
        for d in range(D + 1):
            lo, hi = (0, 1) if d == 0 else (1 + (d - 1) * W, 1 + d * W)
            tested, acc = c[lo:hi, 0], c[lo:hi, 1]
            if tested.sum() > 0:
                last = acc.sum() / tested.sum()
            if last is None:
                continue
            out[lo:hi] = (acc + prior * last) / (tested + prior)
        return out

    def set_node_table(self, rates) -> None:
        """Load per-position acceptance rates (same for every request) into the prune objective's
        table; takes effect from the next step (stream-ordered copy, no re-capture)."""
        t = torch.as_tensor(np.asarray(rates, dtype=np.float64)).reshape(1, -1).expand(self.B, -1)
        self.node_table.copy_(t)

    # ------------------------------------------------------------------
    def set_uniforms(self, step_index: int, seed: int, stream=None) -> None:
        """Acceptance uniforms of the next step from default_rng([seed, step]) (simulator.py:306).

        The host fills one of two pinned buffers and enqueues its H2D copy into the device buffer the
        step graph reads, on the launching stream, so the copy lands after the previous step and before
        the next replay.  Before a pinned buffer is rewritten, the event recorded after its previous copy
        is awaited: the host may run many steps ahead without overwriting uniforms still in flight."""
        slot = self._u_next % 2
        self._u_next += 1
        ev = self._u_ev[slot]
        if self._u_used[slot]:
            ev.synchronize()
        rng = np.random.default_rng([seed, step_index])
        self._u_host[slot].copy_(torch.from_numpy(rng.random((self.B, self.n_uniform))))
        st = stream if stream is not None else torch.cuda.current_stream(self.dev)
        with torch.cuda.stream(st):
            self.uniforms.copy_(self._u_host[slot], non_blocking=True)
            ev.record(st)
        self._u_used[slot] = True

    def capture(self) -> None:
        """Capture one step as a CUDA graph (static shapes, device-resident control)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            # warm-up launch outside capture is not needed: kernels are plain launches; but the
            # caching allocator must not allocate inside the captured region.
            pass
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._launch_step()
        self.graph = g

    def step(self, use_graph: bool = True) -> None:
        if use_graph:
            if self.graph is None:
                raise RuntimeError("call capture() first")
            self.graph.replay()
        else:
            self._launch_step()
        self.step_count += 1

    def read_emitted(self, host_out: torch.Tensor) -> None:
        """Async D2H of this step's emitted tokens ([count, tokens...] per request) into pinned memory."""
        host_out.copy_(self.emit, non_blocking=True)

    def generated(self, b: int = 0) -> list[int]:
        P0 = self.prefill_len
        n = int(self.seq.n_gen[b])
        return self.seq.hist[b, P0 : P0 + n].cpu().tolist()

    def generate(self, prompts: torch.Tensor, n_tokens: int, use_graph: bool = True, sync_every: int = 8,
                 seed: int = 0):
        """Public generate loop: prefill, then steps until every request has n_tokens.

        Each request stops on the device once it has n_tokens (commit freezes it: no more history, no
        KV movement past its prefix), so requests that accept fast never run past the cache while the
        slowest catches up; the host polls the finished flags every ``sync_every`` steps."""
        B, P0 = prompts.shape
        D = self.shape.depth
        # every step appends at most D + 2 tokens; a request may overshoot n_tokens by D + 1 before it
        # freezes, and the next step's tree / scratch slots sit past the prefix
        if P0 + n_tokens + D + 2 > self.seq.p_limit:
            raise ValueError(f"prompt {P0} + {n_tokens} generated tokens do not fit the cache (max_seq too small: "
                             f"prefix limit {self.seq.p_limit})")
        self.prefill_len = P0
        self.prefill(prompts)
        self.seq.gen_limit.fill_(n_tokens)
        self.seq.status.zero_()
        if use_graph and self.graph is None:
            self.capture()
        steps = 0
        while True:
            if steps % sync_every == 0:
                st = self.seq.status.cpu()
                if bool((st != 0).all()):
                    if bool((st & 2).any()):
                        raise RuntimeError("a request reached the cache capacity before n_tokens")
                    break
            if self.mode == SAMPLE:
                self.set_uniforms(steps, seed)
            self.step(use_graph)
            steps += 1
        return [self.generated(b)[:n_tokens] for b in range(self.B)], steps


class ARDecoder:
    """Plain greedy autoregressive decoding through the same kernels (baseline and oracle
    for the lossless-greedy identity: speculative output == AR output)."""

    def __init__(self, cfg: ModelConfig, w: dict, batch: int = 1, max_seq: int = 2048,
                 act_dtype: torch.dtype = torch.bfloat16, device="cuda", plan: ForwardPlan | None = None):
        L.require_device()
        self.cfg, self.w, self.B = cfg, w, batch
        self.S = (max_seq + 8 + 63) // 64 * 64
        self.act_dtype = act_dtype
        self.dev = torch.device(device)
        self.cache = new_cache(cfg, batch, self.S, act_dtype, self.dev)
        # AR is the oracle of the lossless-greedy identity, so it runs the same kernel families as the
        # verify pass (stream-K GEMM and the cluster decode attention of tree passes that fit one
        # wave), not the draft's GEMV.
        self.plan = plan
        self.fwd = Forward(cfg, w, self.cache, batch, 1, 1, act_dtype, gemv=False, plan=plan)
        self.fwd.qmask.fill_(1)
        self.argmax = torch.zeros(batch, dtype=torch.int32, device=self.dev)
        self.P = torch.zeros(batch, dtype=torch.int32, device=self.dev)
        self.graph = None

    def _launch(self, stream=None):
        lib = L.lib()
        s = L.stream_ptr(stream)
        f = self.fwd
        f.tokens.copy_(self.argmax)
        f.pos.copy_(self.P)
        f.slot.copy_(self.P)
        f.blk_start.copy_(self.P)
        f.run(stream)
        L.check(lib.ygg_row_stats(f.logits.data_ptr(), L.YGG_F32, self.B, self.cfg.vocab, self.cfg.vocab, 1.0,
                                  self.argmax.data_ptr(), None, s))
        self.P.add_(1)

    def generate(self, prompts: torch.Tensor, n_tokens: int, use_graph: bool = True) -> list:
        B, P0 = prompts.shape
        pd = prompts.to(self.dev, torch.int32)
        last = prefill_causal(self.cfg, self.w, self.cache, pd, self.act_dtype, True, plan=self.plan)
        L.check(L.lib().ygg_row_stats(last.data_ptr(), L.YGG_F32, B, self.cfg.vocab, self.cfg.vocab, 1.0,
                                      self.argmax.data_ptr(), None, L.stream_ptr()))
        self.P.fill_(P0)
        self.fwd.blk_len.fill_(1)
        out = [self.argmax.clone()]
        if use_graph and self.graph is None:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._launch()
            self.graph = g
            # capture does not execute; nothing advanced yet
        for _ in range(n_tokens - 1):
            if use_graph:
                self.graph.replay()
            else:
                self._launch()
            out.append(self.argmax.clone())
        return torch.stack(out, 1).cpu().tolist()
