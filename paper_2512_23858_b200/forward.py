"""One static-shape Llama forward over the C ABI (K3 GEMM + K4 epilogues + K2 attention).

A ``Forward`` owns its activation buffers, GEMM plans (TMA descriptors are built once
against these fixed buffers) and per-row inputs (tokens, positions, KV slots, tree masks),
so a pass is a fixed sequence of kernel launches that CUDA-graph capture records verbatim.
It realises the verifier / drafter forward the reference only prices
(``latency_at(profiles.verifier, w_verify + 1)``, pkg/src/specsim/simulator.py:211-213).

bf16 default (10 launches per layer): tcgen05 stream-K GEMM writing f32 partials, then a
vectorised epilogue kernel (RoPE + KV append from a host RoPE table / residual + cluster-DSMEM
RMSNorm / SwiGLU), and the tcgen05 split-KV tree attention + combine.

bf16 with ForwardPlan(fused_epilogues=True) (6 launches per layer): every epilogue fused into its GEMM —
  GEMM(qkv, x=hb)  + rstd + RoPE + q / KV-cache append      (YGG_EPI_QKV_ROPE)
  GEMM(o)          + residual add, hb, per-tile sum-of-squares (YGG_EPI_RESID)
  GEMM(gate|up, x=hb) + rstd + SwiGLU                        (YGG_EPI_SWIGLU)
  GEMM(down)       + residual add, hb, sum-of-squares          (YGG_EPI_RESID)
with RMSNorm gains folded into the next weights (model.prepare_fused_) and the per-token rstd
applied by the consuming GEMM's epilogue.  Same results; today slower, because the split-tile
fixups sit on each GEMM's critical path.

f32 (parity path): SIMT GEMM + the same separate epilogue kernels + SIMT attention.  The
residual stream is f32 in every path.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import math

import torch

from . import _lib as L
from .model import ModelConfig, prepare_fused_, rope_table
from .plan import DEFAULT, ForwardPlan


class GemmPlan:
    """Host-side plan (TMA tensor maps + stream-K segment table) for Y = X . W^T."""

    def __init__(self, W: torch.Tensor, X: torch.Tensor, M: int, num_ctas: int = 0):
        lib = L.lib()
        N, K = W.shape
        self.M, self.N, self.K = M, N, K
        self.dtype = L.dtype_code(W.dtype)
        self._mem = C.create_string_buffer(int(lib.ygg_gemm_plan_size()))
        mp = (M + 15) // 16 * 16
        bn = min(mp, 256)
        tiles = (N // 128) * ((M + bn - 1) // bn)
        self.tiles = tiles
        self.seg_table = torch.zeros(tiles + 1 + 160, dtype=torch.int32, device=W.device)
        nseg, wsb = C.c_int(), C.c_size_t()
        L.check(
            lib.ygg_gemm_plan_init(
                self._mem, self.dtype, W.data_ptr(), X.data_ptr(), M, N, K, num_ctas, self.seg_table.data_ptr(),
                C.byref(nseg), C.byref(wsb)
            )
        )
        self.segments = nseg.value
        self.ws_bytes = wsb.value
        self.W, self.X = W, X  # keep alive
        self.epi = None  # L.YggEpilogue for the fused path
        self.cluster = 0  # > 0: cluster split-K (Forward._try_cluster)

    @property
    def handle(self):
        return self._mem


class AttnPlan:
    """TMA tensor maps for the tcgen05 split-KV attention over one layer's cache."""

    def __init__(self, q: torch.Tensor, cache_layer_ptr: int, B: int, M: int, cfg: ModelConfig, S: int):
        lib = L.lib()
        self._mem = C.create_string_buffer(int(lib.ygg_attn_plan_size()))
        pb = C.c_size_t()
        L.check(lib.ygg_attn_plan_init(self._mem, q.data_ptr(), cache_layer_ptr, B, M, cfg.n_heads,
                                       cfg.n_kv_heads, cfg.head_dim, S, C.byref(pb)))
        self.partial_bytes = pb.value

    @property
    def handle(self):
        return self._mem


class Forward:
    def __init__(
        self,
        cfg: ModelConfig,
        weights: dict,
        cache: torch.Tensor,
        B: int,
        R: int,
        mask_words: int,
        act_dtype: torch.dtype,
        logits: bool = True,
        num_ctas: int = 0,
        gemv: bool | None = None,
        decode_attn: bool | None = None,
        plan: ForwardPlan | None = None,
        lm_argmax: bool = False,
        last_logits: bool = False,
    ):
        """``last_logits``: the LM head runs on each request's last row only (``logits`` is [B, V]) — a
        prefill chunk needs nothing else, and the [B*R, V] head is most of a chunk's wasted work."""
        L.require_device()
        plan = plan or DEFAULT
        self.plan = plan
        self.cfg, self.cache = cfg, cache
        self.B, self.R, self.M = B, R, B * R
        self.mask_words = mask_words
        self.act_dtype = act_dtype
        self.act = L.dtype_code(act_dtype)
        # bf16 default: plain stream-K GEMM + separate vectorised epilogue kernels (faster today);
        # plan.fused_epilogues selects the fused-epilogue GEMMs (same results, tested).
        bf16 = act_dtype == torch.bfloat16
        if gemv is None:
            gemv = True if plan.gemv is None else plan.gemv
        if decode_attn is None:
            decode_attn = True if plan.decode_attn is None else plan.decode_attn
        # Decode passes of <= 16 rows: row-block GEMV with fused epilogues (csrc/gemv.cu); needs the
        # fused weight layout, which then also routes every other bf16 forward on these weights
        # (prefill, verify) through the fused-epilogue GEMM.
        self.gemv = bool(gemv) and bf16 and logits and B * R <= 16 and mask_words <= L.MAX_MASK_WORDS
        self.layout_fused = bf16 and (plan.fused_epilogues or self.gemv or weights.get("_layout") == "fused")
        if self.layout_fused:
            prepare_fused_(weights, cfg)
        # Non-GEMV passes over fused-layout weights (draft prefill chunks, batched draft levels) run the
        # per-kernel epilogues with the layout flag (ygg_gemm_plan_set_layout) unless the plan asks for the
        # fused-epilogue GEMMs (measured slower at M = 512: DESIGN.md §4).
        self.fused = self.layout_fused and (self.gemv or plan.fused_epilogues or plan.fused_layout_gemm)
        self.w = weights
        dev = cache.device
        M, d = self.M, cfg.d_model
        i32 = dict(dtype=torch.int32, device=dev)
        # per-row inputs (written by the step bookkeeping kernels)
        self.tokens = torch.zeros(M, **i32)
        self.pos = torch.zeros(M, **i32)
        self.slot = torch.zeros(M, **i32)
        self.req = torch.arange(M, **i32) // R
        self.qmask = torch.zeros(M, max(mask_words, 1), dtype=torch.int32, device=dev)
        self.blk_start = torch.zeros(B, **i32)
        self.blk_len = torch.zeros(B, **i32)
        # activations
        self.resid = torch.zeros(M, d, dtype=torch.float32, device=dev)
        self.xn = torch.zeros(M, d, dtype=act_dtype, device=dev)  # f32 path: normalised input; bf16: hb
        self.q = torch.zeros(M, cfg.q_dim, dtype=act_dtype, device=dev)
        self.attn = torch.zeros(M, cfg.q_dim, dtype=act_dtype, device=dev)
        self.mlp = torch.zeros(M, cfg.ffn, dtype=act_dtype, device=dev)
        self.last_logits = bool(last_logits and logits)
        self.logits = (torch.zeros(B if self.last_logits else M, cfg.vocab, dtype=torch.float32, device=dev)
                       if logits else None)
        self.xn_last = torch.zeros(B, d, dtype=act_dtype, device=dev) if self.last_logits else None
        self.layer_stride = cache.stride(0)
        self.S = cache.shape[4]
        self.scale = 1.0 / math.sqrt(cfg.head_dim)
        self.plans = []
        ws = 0
        for lw in weights["layers"]:
            p = {
                "qkv": GemmPlan(lw["wqkv"], self.xn, M, num_ctas),
                "o": GemmPlan(lw["wo"], self.attn, M, num_ctas),
                "gu": GemmPlan(lw["wgu"], self.xn, M, num_ctas),
                "down": GemmPlan(lw["wdown"], self.mlp, M, num_ctas),
            }
            self.plans.append(p)
            ws = max(ws, *(q.ws_bytes for q in p.values()))
        self.lm_plan = (GemmPlan(weights["lm_head"], self.xn_last if self.last_logits else self.xn,
                                 B if self.last_logits else M, num_ctas) if logits else None)
        if self.lm_plan:
            ws = max(ws, self.lm_plan.ws_bytes)
        self.ws = torch.empty(max(ws // 4, 1), dtype=torch.float32, device=dev)
        self.attn_plans = None
        if act_dtype == torch.bfloat16 and mask_words <= L.MAX_MASK_WORDS:
            es = cache.element_size()
            self.attn_plans = [AttnPlan(self.q, cache.data_ptr() + li * self.layer_stride * es, B, M, cfg, self.S)
                               for li in range(cfg.n_layers)]
            self.attn_part = torch.empty(self.attn_plans[0].partial_bytes // 4 + 1, dtype=torch.float32, device=dev)
        self.rope_cs = rope_table(cfg, self.S + 64, dev)
        # Decode attention (csrc/attn_dec.cu: clusters of CTAs per (kv head, request, 64-row tile), no
        # split-KV partials / combine launch) for draft levels and AR (one kv head's rows fit one tile)
        # and for tree passes whose row tiles fit one wave (the cfg2 verify: 50 tokens x 4 heads = 4
        # tiles x 8 kv heads; measured in-graph 9.8 us per layer vs 13.8 for tcgen05 split-KV +
        # combine).  Prefill and wide batched verifies keep the split-KV tcgen05 kernel.
        self.ad_plans = None
        gh = cfg.n_heads // cfg.n_kv_heads
        tree_fits = mask_words > 0 and (B * cfg.n_kv_heads * ((R * gh + 63) // 64) <= 148 or plan.decode_attn_wide)
        if (decode_attn and act_dtype == torch.bfloat16 and mask_words <= L.MAX_MASK_WORDS
                and (R * gh <= 64 or tree_fits)):
            lib = L.lib()
            es = cache.element_size()
            self.ad_plans = []
            for li in range(cfg.n_layers):
                mem = C.create_string_buffer(int(lib.ygg_attn_dec_plan_size()))
                L.check(lib.ygg_attn_dec_plan_init(mem, self.q.data_ptr(), cache.data_ptr() + li * self.layer_stride * es,
                                                   B, R, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, self.S,
                                                   plan.attn_kvsplit, plan.attn_ksplit, plan.attn_stages))
                self.ad_plans.append(mem)
            self.ad_ws = torch.zeros(int(lib.ygg_attn_dec_workspace_size(self.ad_plans[0])) // 4 + 64,
                                     dtype=torch.float32, device=dev)
        # tcgen05 / TMEM tree attention (csrc/attn_tree.cu): S and O on the tensor cores, keys split over
        # a thread-block cluster, merged through DSMEM; replaces the decode attention when planned.
        self.at_plans = None
        use_tree = plan.tree_attn if plan.tree_attn is not None else not self.gemv
        # causal passes (prefill chunks, no tree mask) take it too: one CTA per (kv head, request, 32-token
        # row tile) that walks only the keys its last token sees, instead of split-KV + combine launches
        causal_tree = mask_words == 0 and plan.prefill_tree_attn and act_dtype == torch.bfloat16
        tree_pass = use_tree and act_dtype == torch.bfloat16 and 0 < mask_words <= L.MAX_MASK_WORDS
        if (tree_pass or causal_tree) and gh <= 32 and gh & (gh - 1) == 0:
            lib = L.lib()
            es = cache.element_size()
            self.at_plans = []
            for li in range(cfg.n_layers):
                mem = C.create_string_buffer(int(lib.ygg_attn_tree_plan_size()))
                L.check(lib.ygg_attn_tree_plan_init(mem, self.q.data_ptr(), cache.data_ptr() + li * self.layer_stride * es,
                                                    B, R, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, self.S,
                                                    plan.tree_csplit, plan.tree_row_tiles))
                self.at_plans.append(mem)
        # Unfused bf16 LM head: whole output tiles go straight from TMEM to the f32 logits and only the
        # split stream-K tiles are reduced (in fixed segment order, by their participants) — the
        # [M, V] f32 partials round trip and the separate store epilogue disappear.  Same values.
        self.lm_epi = None
        # Greedy verify (lm_argmax): the LM head stores no logits, only per-128-row-tile keys of each
        # token's first maximum (YGG_EPI_ARGMAX), reduced by ygg_argmax_reduce.
        self.lm_argmax = bool(lm_argmax and bf16 and self.lm_plan is not None and M <= 512 and not self.last_logits)
        if self.lm_argmax:
            self.lm_keys = torch.zeros(cfg.vocab // 128, M, dtype=torch.int64, device=dev)
        if bf16 and not self.fused and self.lm_plan is not None and (plan.lm_store_fused or self.lm_argmax):
            self.lm_counters = torch.zeros(self.lm_plan.tiles, dtype=torch.int32, device=dev)
            e = L.YggEpilogue()
            e.kind = L.YGG_EPI_ARGMAX if self.lm_argmax else L.YGG_EPI_STORE_F32
            e.counters = self.lm_counters.data_ptr()
            e.out = self.lm_keys.data_ptr() if self.lm_argmax else self.logits.data_ptr()
            e.ld = cfg.vocab
            self.lm_epi = e
        if self.fused:
            self._setup_fused()
        elif self.layout_fused:
            for p in self.plans:
                L.check(L.lib().ygg_gemm_plan_set_layout(p["qkv"].handle, 1))
                L.check(L.lib().ygg_gemm_plan_set_layout(p["gu"].handle, 1))
        if self.gemv:
            self._setup_gemv()
        self._setup_attn_l2_prefetch()
        if not self.gemv and not self.fused and bf16:
            self._setup_epi_l2_prefetch()

    # ------------------------------------------------------------------
    def _setup_gemv(self) -> None:
        """Row-block GEMV plans + epilogues (csrc/gemv.cu) for a <= 16-row decode pass."""
        lib, cfg, M = L.lib(), self.cfg, self.M
        dev = self.cache.device
        d = cfg.d_model
        self.ss_e = torch.zeros(d // 128, M, dtype=torch.float32, device=dev)  # embed: per 128 features
        self.ss_ga = torch.zeros(d // 16, M, dtype=torch.float32, device=dev)  # after down: per 16 rows
        self.ss_gb = torch.zeros(d // 16, M, dtype=torch.float32, device=dev)  # after o-proj
        es = self.cache.element_size()
        eps = float(cfg.norm_eps)

        def plan(W, X):
            mem = C.create_string_buffer(int(lib.ygg_gemv_plan_size()))
            N, K = W.shape
            L.check(lib.ygg_gemv_plan_init(mem, W.data_ptr(), X.data_ptr(), M, N, K, 0))
            return mem

        def epi(kind, **kw):
            e = L.YggGemvEpilogue()
            e.kind = kind
            for k, v in kw.items():
                setattr(e, k, v)
            return e

        self.gv = []
        for li, lw in enumerate(self.w["layers"]):
            ss_in, blocks = (self.ss_e, d // 128) if li == 0 else (self.ss_ga, d // 16)
            cache_l = self.cache.data_ptr() + li * self.layer_stride * es
            self.gv.append([
                (plan(lw["wqkv"], self.xn),
                 epi(L.YGG_GEMV_QKV, ss_in=ss_in.data_ptr(), ss_blocks=blocks, norm_dim=d, eps=eps,
                     q_out=self.q.data_ptr(), cache=cache_l, S=self.S, Hq=cfg.n_heads, Hkv=cfg.n_kv_heads,
                     hd=cfg.head_dim, pos=self.pos.data_ptr(), slot=self.slot.data_ptr(), req=self.req.data_ptr(),
                     rope_cs=self.rope_cs.data_ptr())),
                (plan(lw["wo"], self.attn),
                 epi(L.YGG_GEMV_RESID, resid=self.resid.data_ptr(), hb=self.xn.data_ptr(),
                     ss_out=self.ss_gb.data_ptr())),
                (plan(lw["wgu"], self.xn),
                 epi(L.YGG_GEMV_SWIGLU, ss_in=self.ss_gb.data_ptr(), ss_blocks=d // 16, norm_dim=d, eps=eps,
                     act_out=self.mlp.data_ptr())),
                (plan(lw["wdown"], self.mlp),
                 epi(L.YGG_GEMV_RESID, resid=self.resid.data_ptr(), hb=self.xn.data_ptr(),
                     ss_out=self.ss_ga.data_ptr())),
            ])
        # Latency-bound GEMVs pull a share of the layer's later weight streams into L2 while HBM would
        # otherwise idle (plan.draft_qkv_l2 / draft_o_l2; sizes derived from the matrix sizes).
        for li, lw in enumerate(self.w["layers"]):
            for (pl, _), regs, first in ((self.gv[li][0], self.plan.draft_qkv_l2, 1),
                                         (self.gv[li][1], self.plan.draft_o_l2, 0)):
                for j, rg in enumerate(regs[: 2 - first]):
                    W = lw[rg.target]
                    off, n = rg.region(W, self.plan.l2_bytes)
                    if n > 0:
                        L.check(lib.ygg_gemv_set_l2_prefetch(pl, first + j, W.data_ptr() + off, n))
        ss_last, blocks_last = (self.ss_ga, d // 16) if cfg.n_layers > 0 else (self.ss_e, d // 128)
        self.gv_lm = (plan(self.w["lm_head"], self.xn),
                      epi(L.YGG_GEMV_STORE, out=self.logits.data_ptr(), ld=cfg.vocab, ss_in=ss_last.data_ptr(),
                          ss_blocks=blocks_last, norm_dim=d, eps=eps))

    def _setup_attn_l2_prefetch(self) -> None:
        """While the decode attention of layer l runs, HBM is nearly idle: it pulls the start of a later
        weight stream of the layer into L2 — for the draft the down projection (its GEMV CTAs cannot be
        resident during the gate|up stream; the O projection already sits in the GEMV ring), for the
        verify the start of gate|up (plan.draft_attn_l2 / verify_attn_l2)."""
        if self.ad_plans is None:
            return
        lib = L.lib()
        regions = self.plan.draft_attn_l2 if self.gemv else self.plan.verify_attn_l2
        for li, plan in enumerate(self.ad_plans):
            for j, rg in enumerate(regions[:2]):
                W = self.w["layers"][li][rg.target]
                off, n = rg.region(W, self.plan.l2_bytes)
                L.check(lib.ygg_attn_dec_set_l2_prefetch(plan, j, W.data_ptr() + off if n > 0 else None, n))
                if self.at_plans is not None:
                    L.check(lib.ygg_attn_tree_set_l2_prefetch(self.at_plans[li], j, W.data_ptr() + off if n > 0 else None,
                                                              n))

    def _setup_epi_l2_prefetch(self) -> None:
        """The separate epilogue kernels of a verify / prefill pass idle HBM too: each pulls a region of a
        later weight stream into L2 (plan.verify_epi_l2: (GEMM name, L2Prefetch) pairs)."""
        lib = L.lib()
        layers = self.w["layers"]
        for li, p in enumerate(self.plans):
            for name, rg in self.plan.verify_epi_l2:
                lj = li + (1 if rg.next_layer else 0)
                if lj >= len(layers):
                    continue
                W = layers[lj][rg.target]
                off, n = rg.region(W, self.plan.l2_bytes)
                L.check(lib.ygg_gemm_plan_set_epi_prefetch(p[name].handle, W.data_ptr() + off if n > 0 else None, n))

    def fuse_topk(self, k: int, temperature: float = 1.0) -> bool:
        """Draft GEMV pass: have the LM-head epilogue also emit per-CTA top-k partials of every row
        (STORE_TOPK; merged by ``ygg_topk_merge``), replacing the top-k scan of the logits.  Only
        for <= 8 rows and k <= 8; returns whether it is on."""
        if not (self.gemv and self.M <= 8 and 1 <= k <= 8) or not self.plan.topk_fused:
            return False
        lib = L.lib()
        plan, e = self.gv_lm
        self.topk_chunks = int(lib.ygg_gemv_grid(plan))
        self.topk_part = torch.empty(int(lib.ygg_topk_partial_bytes(self.M, self.topk_chunks)), dtype=torch.uint8,
                                     device=self.cache.device)
        e.kind = L.YGG_GEMV_STORE_TOPK
        e.topk_part = self.topk_part.data_ptr()
        e.topk_k = k
        e.inv_temp = 1.0 / temperature
        return True

    def _attend(self, li: int, qm, s) -> None:
        """bf16 attention of layer li: decode kernel when planned, else split-KV tcgen05 + combine."""
        lib = L.lib()
        if self.at_plans is not None:
            L.check(lib.ygg_attn_tree_run(self.at_plans[li], self.blk_start.data_ptr(), self.blk_len.data_ptr(), qm,
                                          self.mask_words, self.scale, self.attn.data_ptr(), s))
        elif self.ad_plans is not None:
            L.check(lib.ygg_attn_dec_run(self.ad_plans[li], self.blk_start.data_ptr(), self.blk_len.data_ptr(), qm,
                                         self.mask_words, self.scale, self.attn.data_ptr(), self.ad_ws.data_ptr(), s))
        else:
            L.check(lib.ygg_attention_tc(self.attn_plans[li].handle, self.blk_start.data_ptr(), self.blk_len.data_ptr(),
                                         qm, self.mask_words, self.scale, self.attn_part.data_ptr(),
                                         self.attn.data_ptr(), s))

    def _run_gemv(self, stream) -> None:
        lib, cfg = L.lib(), self.cfg
        s = L.stream_ptr(stream)
        chk = L.check
        chk(lib.ygg_embed_fused(self.w["embed"].data_ptr(), cfg.vocab, cfg.d_model, self.tokens.data_ptr(), self.M,
                                self.resid.data_ptr(), self.xn.data_ptr(), self.ss_e.data_ptr(), s))
        qm = self.qmask.data_ptr() if self.mask_words > 0 else None
        for li, ops in enumerate(self.gv):
            (pq, eq), (po, eo), (pg, eg), (pd, ed) = ops
            chk(lib.ygg_gemv_run(pq, C.byref(eq), s))
            self._attend(li, qm, s)
            chk(lib.ygg_gemv_run(po, C.byref(eo), s))
            chk(lib.ygg_gemv_run(pg, C.byref(eg), s))
            chk(lib.ygg_gemv_run(pd, C.byref(ed), s))
        chk(lib.ygg_gemv_run(self.gv_lm[0], C.byref(self.gv_lm[1]), s))

    # ------------------------------------------------------------------
    def _setup_fused(self) -> None:
        cfg, M, d = self.cfg, self.M, self.cfg.d_model
        dev = self.cache.device
        nt = d // 128
        self.ss_a = torch.zeros(nt, M, dtype=torch.float32, device=dev)
        self.ss_b = torch.zeros(nt, M, dtype=torch.float32, device=dev)
        # One arrival-counter array per plan: the counters are monotonic epochs (launch L of a plan
        # moves a split tile's counter from L*nseg to (L+1)*nseg), so plans must never share them.
        plans = [p for layer in self.plans for p in layer.values()] + ([self.lm_plan] if self.lm_plan else [])
        offs, total = [], 0
        for p in plans:
            offs.append(total)
            total += p.tiles
        self.counters = torch.zeros(max(total, 1), dtype=torch.int32, device=dev)
        counter_ptr = {id(p): self.counters.data_ptr() + 4 * o for p, o in zip(plans, offs)}
        eps = float(cfg.norm_eps)
        es = self.cache.element_size()
        cur = {"plan": None}

        def epi(kind, **kw):
            e = L.YggEpilogue()
            e.kind = kind
            e.counters = counter_ptr[id(cur["plan"])]
            for k, v in kw.items():
                setattr(e, k, v)
            return e

        if self.plan.cluster_split_k:
            for p in self.plans:
                for name in ("qkv", "o", "gu", "down"):
                    self._try_cluster(p[name])
        for li, p in enumerate(self.plans):
            cache_l = self.cache.data_ptr() + li * self.layer_stride * es
            cur["plan"] = p["qkv"]
            p["qkv"].epi = epi(L.YGG_EPI_QKV_ROPE, ss_in=self.ss_a.data_ptr(), ss_tiles=nt, norm_dim=d, eps=eps,
                               q_out=self.q.data_ptr(), cache=cache_l, S=self.S, Hq=cfg.n_heads, Hkv=cfg.n_kv_heads,
                               hd=cfg.head_dim, rope_theta=cfg.rope_theta, pos=self.pos.data_ptr(),
                               slot=self.slot.data_ptr(), req=self.req.data_ptr(), rope_cs=self.rope_cs.data_ptr())
            cur["plan"] = p["o"]
            p["o"].epi = epi(L.YGG_EPI_RESID, resid=self.resid.data_ptr(), hb=self.xn.data_ptr(),
                             ss_out=self.ss_b.data_ptr())
            cur["plan"] = p["gu"]
            p["gu"].epi = epi(L.YGG_EPI_SWIGLU, ss_in=self.ss_b.data_ptr(), ss_tiles=nt, norm_dim=d, eps=eps,
                              act_out=self.mlp.data_ptr())
            cur["plan"] = p["down"]
            p["down"].epi = epi(L.YGG_EPI_RESID, resid=self.resid.data_ptr(), hb=self.xn.data_ptr(),
                                ss_out=self.ss_a.data_ptr())
        if self.last_logits:
            self.ss_last = torch.zeros(nt, self.B, dtype=torch.float32, device=dev)
        if self.lm_plan:
            cur["plan"] = self.lm_plan
            lm_ss = self.ss_last if self.last_logits else self.ss_a
            self.lm_plan.epi = epi(L.YGG_EPI_ARGMAX if self.lm_argmax else L.YGG_EPI_STORE_F32, ss_in=lm_ss.data_ptr(),
                                   ss_tiles=nt, norm_dim=d, eps=eps,
                                   out=(self.lm_keys if self.lm_argmax else self.logits).data_ptr(), ld=cfg.vocab)

    def _try_cluster(self, gp: GemmPlan) -> None:
        """Cluster split-K for a GEMM whose tiles, times a cluster of 2-4 CTAs, fill one wave."""
        lib = L.lib()
        sms = torch.cuda.get_device_properties(self.cache.device).multi_processor_count
        gp.cluster = 0
        for cs in (4, 3, 2):
            if gp.tiles * cs <= sms and lib.ygg_gemm_plan_set_cluster(gp.handle, cs) == L.YGG_OK:
                gp.cluster = cs
                return

    def argmax_rows(self, out: torch.Tensor, stream_ptr) -> None:
        """Row argmax of this pass's logits into ``out`` [M] int32: from the fused LM-head keys when the
        pass was built with lm_argmax, else by scanning the stored logits (row_stats)."""
        lib = L.lib()
        if self.lm_argmax:
            L.check(lib.ygg_argmax_reduce(self.lm_keys.data_ptr(), self.cfg.vocab // 128, self.M, out.data_ptr(),
                                          stream_ptr))
        else:
            L.check(lib.ygg_row_stats(self.logits.data_ptr(), L.YGG_F32, self.M, self.cfg.vocab, self.cfg.vocab, 1.0,
                                      out.data_ptr(), None, stream_ptr))

    def weight_bytes(self) -> int:
        """Algorithmic HBM bytes of the matmul weights streamed per pass."""
        total = 0
        for p in self.plans:
            total += sum(q.W.numel() * q.W.element_size() for q in p.values())
        if self.lm_plan:
            total += self.lm_plan.W.numel() * self.lm_plan.W.element_size()
        return total

    def gemm_calls(self):
        """(plan, epilogue) of every GEMM launch of one pass, in order (for per-launch timing)."""
        out = []
        for p in self.plans:
            out += [p["qkv"], p["o"], p["gu"], p["down"]]
        if self.lm_plan:
            out.append(self.lm_plan)
        return out

    def launch_gemm(self, plan: GemmPlan, stream_ptr) -> None:
        lib = L.lib()
        if self.fused:
            L.check(lib.ygg_gemm_fused(plan.handle, self.ws.data_ptr(), C.byref(plan.epi), stream_ptr))
        else:
            L.check(lib.ygg_gemm_run(plan.handle, self.ws.data_ptr(), stream_ptr))

    def run(self, stream: torch.cuda.Stream | None = None) -> None:
        if self.gemv:
            self._run_gemv(stream)
        elif self.fused:
            self._run_fused(stream)
        else:
            self._run_unfused(stream)

    def _gather_last(self, stream) -> None:
        """last_logits: each request's last row of the LM-head input (and, fused, of its sums of squares)."""
        with torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext():
            self.xn_last.copy_(self.xn.view(self.B, self.R, -1)[:, -1])
            if self.fused:
                nt = self.ss_a.shape[0]
                self.ss_last.copy_(self.ss_a.view(nt, self.B, self.R)[:, :, -1])

    def _run_fused(self, stream, stamps: torch.Tensor | None = None) -> None:
        """``stamps`` (int64 [>= 6*layers+3], debug only): a %globaltimer stamp kernel is enqueued
        after every launch, giving in-graph per-kernel durations."""
        lib, cfg = L.lib(), self.cfg
        s = L.stream_ptr(stream)
        chk = L.check
        ws = self.ws.data_ptr()
        k = [0]

        def stamp():
            if stamps is not None:
                chk(lib.ygg_stamp(stamps.data_ptr() + 8 * k[0], s))
                k[0] += 1

        stamp()
        chk(lib.ygg_embed_fused(self.w["embed"].data_ptr(), cfg.vocab, cfg.d_model, self.tokens.data_ptr(), self.M,
                                self.resid.data_ptr(), self.xn.data_ptr(), self.ss_a.data_ptr(), s))
        stamp()
        qm = self.qmask.data_ptr() if self.mask_words > 0 else None
        for li, p in enumerate(self.plans):
            chk(lib.ygg_gemm_fused(p["qkv"].handle, ws, C.byref(p["qkv"].epi), s))
            stamp()
            self._attend(li, qm, s)
            stamp()
            chk(lib.ygg_gemm_fused(p["o"].handle, ws, C.byref(p["o"].epi), s))
            stamp()
            chk(lib.ygg_gemm_fused(p["gu"].handle, ws, C.byref(p["gu"].epi), s))
            stamp()
            chk(lib.ygg_gemm_fused(p["down"].handle, ws, C.byref(p["down"].epi), s))
            stamp()
        if self.lm_plan is not None:
            if self.last_logits:
                self._gather_last(stream)
            chk(lib.ygg_gemm_fused(self.lm_plan.handle, ws, C.byref(self.lm_plan.epi), s))
            stamp()

    def _run_unfused(self, stream, stamps: torch.Tensor | None = None) -> None:
        lib, cfg = L.lib(), self.cfg
        s = L.stream_ptr(stream)
        chk = L.check
        w = self.w
        M = self.M
        k = [0]

        def stamp():
            if stamps is not None:
                chk(lib.ygg_stamp(stamps.data_ptr() + 8 * k[0], s))
                k[0] += 1

        stamp()
        wdt = L.dtype_code(w["embed"].dtype)
        n0 = w["layers"][0]["attn_norm"]
        if wdt == self.act and L.dtype_code(n0.dtype) == self.act:  # one launch: embedding + first norm
            chk(lib.ygg_embed_rmsnorm(w["embed"].data_ptr(), n0.data_ptr(), self.act, cfg.vocab, cfg.d_model,
                                      self.tokens.data_ptr(), M, cfg.norm_eps, self.resid.data_ptr(),
                                      self.xn.data_ptr(), s))
        else:
            chk(lib.ygg_embed(w["embed"].data_ptr(), wdt, cfg.vocab, cfg.d_model, self.tokens.data_ptr(), M,
                              self.resid.data_ptr(), s))
            chk(lib.ygg_rmsnorm(self.resid.data_ptr(), n0.data_ptr(), self.act, M, cfg.d_model, cfg.norm_eps,
                                self.xn.data_ptr(), s))
        ws = self.ws.data_ptr()
        nl = len(self.plans)
        qm = self.qmask.data_ptr() if self.mask_words > 0 else None
        for li, (p, lw) in enumerate(zip(self.plans, w["layers"])):
            cache_l = self.cache.data_ptr() + li * self.layer_stride * self.cache.element_size()
            chk(lib.ygg_gemm_run(p["qkv"].handle, ws, s))
            chk(lib.ygg_epi_qkv_rope(p["qkv"].handle, ws, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim,
                                     cfg.rope_theta, self.pos.data_ptr(), self.slot.data_ptr(),
                                     self.req.data_ptr(), self.q.data_ptr(), cache_l, self.S, self.act,
                                     self.rope_cs.data_ptr(), s))
            stamp()
            if self.attn_plans is not None:
                self._attend(li, qm, s)
            else:
                chk(lib.ygg_attention(self.q.data_ptr(), cache_l, self.act, M, self.B, cfg.n_heads, cfg.n_kv_heads,
                                      cfg.head_dim, self.S, self.blk_start.data_ptr(), self.blk_len.data_ptr(),
                                      qm, self.mask_words, self.scale, self.attn.data_ptr(), s))
            stamp()
            chk(lib.ygg_gemm_run(p["o"].handle, ws, s))
            chk(lib.ygg_epi_residual_norm(p["o"].handle, ws, self.resid.data_ptr(), lw["mlp_norm"].data_ptr(),
                                          cfg.norm_eps, self.xn.data_ptr(), self.act, s))
            stamp()
            chk(lib.ygg_gemm_run(p["gu"].handle, ws, s))
            chk(lib.ygg_epi_swiglu(p["gu"].handle, ws, self.mlp.data_ptr(), self.act, s))
            stamp()
            chk(lib.ygg_gemm_run(p["down"].handle, ws, s))
            nxt = w["layers"][li + 1]["attn_norm"] if li + 1 < nl else w["final_norm"]
            chk(lib.ygg_epi_residual_norm(p["down"].handle, ws, self.resid.data_ptr(), nxt.data_ptr(),
                                          cfg.norm_eps, self.xn.data_ptr(), self.act, s))
            stamp()
        if self.lm_plan is not None:
            if self.last_logits:
                self._gather_last(stream)
            if self.lm_epi is not None:
                chk(lib.ygg_gemm_fused(self.lm_plan.handle, ws, C.byref(self.lm_epi), s))
            else:
                chk(lib.ygg_gemm_run(self.lm_plan.handle, ws, s))
                chk(lib.ygg_epi_store(self.lm_plan.handle, ws, self.logits.data_ptr(), L.YGG_F32, cfg.vocab, s))
            stamp()


def prefill_causal(cfg: ModelConfig, w: dict, cache: torch.Tensor, prompts: torch.Tensor, act_dtype: torch.dtype,
                   want_logits: bool, cache_fwd: dict | None = None, max_rows: int = 2048,
                   plan: ForwardPlan | None = None) -> torch.Tensor | None:
    """Causal prefill of ``prompts`` [B, P0] (device int32) into ``cache``, in chunks of at most
    ``max_rows`` rows per launch (each chunk attends to the earlier chunks as its prefix), so 2k-token
    prompts at batch 8-16 (cfg4 / cfg5) never materialise [B*P0, V] logits or partials.  Returns the
    f32 logits of each request's last prompt position [B, V] when ``want_logits`` (else None)."""
    B, P0 = prompts.shape
    chunk = max(1, min(P0, max_rows // B))
    dev = prompts.device
    fwd = cache_fwd if cache_fwd is not None else {}
    last = None
    for c0 in range(0, P0, chunk):
        n = min(chunk, P0 - c0)
        final = c0 + n == P0
        key = (cfg.name, n, id(cache), final and want_logits)
        f = fwd.get(key)
        if f is None:
            f = Forward(cfg, w, cache, B, n, 0, act_dtype, logits=final and want_logits, gemv=False,
                        decode_attn=False, plan=plan, last_logits=True)
            fwd[key] = f
        f.tokens.copy_(prompts[:, c0:c0 + n].reshape(-1))
        pos = torch.arange(c0, c0 + n, dtype=torch.int32, device=dev).repeat(B)
        f.pos.copy_(pos)
        f.slot.copy_(pos)
        f.blk_start.fill_(c0)
        f.blk_len.fill_(n)
        f.run()
        if final and want_logits:
            last = f.logits
    return last


def new_cache(cfg: ModelConfig, B: int, S: int, dtype: torch.dtype, device) -> torch.Tensor:
    """KV cache [layers, B, 2, Hkv, S, hd]: the kv=0 half holds K rows [S][hd] (per-head contiguous key
    streams); the kv=1 half holds V transposed, [hd][S], so both attention MMAs read K-major tiles.
    S is rounded up to a multiple of 64 (TMA row alignment)."""
    S = (S + 63) // 64 * 64
    return torch.zeros(cfg.n_layers, B, 2, cfg.n_kv_heads, S, cfg.head_dim, dtype=dtype, device=device)
