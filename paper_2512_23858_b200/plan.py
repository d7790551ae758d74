"""Typed per-forward kernel plan: which kernel family runs each part of a pass and how much of the
later weight streams each latency-bound kernel pulls into L2 while HBM would otherwise idle.

Everything the round-1 code read from ``YGG_*`` environment variables at plan time is a field
here; a ``Forward`` takes one ``ForwardPlan`` (default: ``ForwardPlan()``, the measured-best
choices below).  L2-prefetch sizes are derived from the matrix sizes of the model being run, not
fixed byte counts: each is a fraction of the target matrix, capped by a share of the L2.

Measured on cfg2 (same-box A/Bs), which the fractions reproduce at the 1B draft / 8B
target sizes:
  draft QKV GEMV      -> the first quarter of gate|up      (16 MB of 64: pass 0.570 -> 0.563 ms)
  draft O GEMV        -> the next quarter of gate|up       (16 MB: 0.625 -> 0.615 ms)
  draft attention     -> the first 3/8 of down             (12 MB of 32: 0.634 -> 0.627 ms)
  verify attention    -> the first tenth of gate|up        (24 MB of 235: verify 3.578 -> 3.464 ms)
                         + the first quarter of O            (8 MB of 34: 4-14 us per verify in five
                                                              same-box A/Bs, scripts/verify_plan_ab.py)
A kernel that pulls more than it leaves idle slows itself as much as the next kernel gains, so every
region is also capped at a quarter of the L2 (31.5 MB on B200).
"""

from __future__ import annotations

from dataclasses import dataclass, field

L2_BYTES_B200 = 126 * (1 << 20)


@dataclass(frozen=True)
class L2Prefetch:
    """One kernel's L2 pull: ``fraction`` of matrix ``target`` starting at ``offset_fraction``."""

    target: str               # weight name in the layer dict (wqkv / wo / wgu / wdown)
    fraction: float
    offset_fraction: float = 0.0
    next_layer: bool = False  # the matrix of the following layer (nothing after the last layer)

    def region(self, W, l2_bytes: int) -> tuple[int, int]:
        """(byte offset, byte count) of the region inside ``W``."""
        total = W.numel() * W.element_size()
        cap = l2_bytes // 4
        off = min(int(self.offset_fraction * total), cap) & ~255 if self.offset_fraction else 0
        n = min(int(self.fraction * total), cap, total - off) & ~255
        return off, max(n, 0)


@dataclass(frozen=True)
class ForwardPlan:
    # kernel families (None = automatic by shape: bf16 passes of <= 16 rows take the row-block GEMV;
    # the decode attention for passes whose row tiles fit one wave)
    gemv: bool | None = None
    decode_attn: bool | None = None
    fused_epilogues: bool = False   # fused-epilogue GEMMs for every non-GEMV bf16 pass (fused weight layout)
    fused_layout_gemm: bool = False  # non-GEMV passes over weights already in the fused layout (the draft's
    #                                  prefill chunks): fused-epilogue GEMMs instead of stream-K GEMM + the
    #                                  layout-aware epilogue kernels (512-row chunk of the 1B draft: 3.7 vs 2.0 ms)
    cluster_split_k: bool = True    # fused-epilogue GEMMs whose tiles x cluster fill one wave run as cluster
    #                                 split-K with a DSMEM reduction (csrc/gemm.cu gemm_cluster_kernel)
    lm_store_fused: bool = True     # LM-head logits straight from TMEM (no partials round trip)
    topk_fused: bool = True         # draft top-k partials from the LM-head GEMV epilogue
    decode_attn_wide: bool = False  # the decode attention also for tree passes whose row tiles exceed a wave
    #                                 (measured slower than the tree attention: cfg4 verify 20.2 vs 17.4 ms,
    #                                 cfg5 94.0 vs 91.8 ms; scripts/cfg_plan_ab.py)
    attn_kvsplit: int = 0           # decode attention cluster size (0 = automatic)
    attn_ksplit: int = 0            # decode attention key-split warp groups per CTA (0 = automatic)
    attn_stages: int = 0            # decode attention K/V ring stages (0 = automatic)
    tree_attn: bool | None = None   # tcgen05 / TMEM tree attention (csrc/attn_tree.cu) instead of the
    #                                 mma.sync decode attention wherever the latter would run; None =
    #                                 automatic: verify / AR passes (measured at parity in the cfg2 verify
    #                                 graph, 3.498 vs 3.491 ms), not draft passes (32 query rows per kv head:
    #                                 cfg2 GEMV pass 0.604 vs 0.565 ms; cfg4 batched levels 39.3 vs 36.0 ms
    #                                 per step) — SpecDecoder builds its draft forward with tree_attn=False
    prefill_tree_attn: bool = True  # causal passes (prefill chunks) on the tree attention too (causal tiles
    #                                 stop at their last token's key) instead of split-KV tcgen05 + combine
    tree_csplit: int = 0            # its key-split cluster size (0 = automatic)
    tree_row_tiles: int = 0         # its row tiles per (kv head, request) (0 = fewest)
    # L2 prefetch issued by latency-bound kernels (see module docstring)
    draft_qkv_l2: tuple = (L2Prefetch("wgu", 0.25),)
    draft_o_l2: tuple = (L2Prefetch("wgu", 0.25, 0.25),)
    draft_attn_l2: tuple = (L2Prefetch("wdown", 0.375),)
    verify_attn_l2: tuple = (L2Prefetch("wgu", 0.1), L2Prefetch("wo", 0.25))
    # (GEMM, region) pairs: the separate epilogue kernel of that GEMM (verify / prefill passes) pulls the
    # region into L2 after its dependency wait (csrc/gemm.cu epi_l2_prefetch)
    verify_epi_l2: tuple = ()
    l2_bytes: int = field(default=L2_BYTES_B200)


DEFAULT = ForwardPlan()
