"""ctypes binding of libygg.so (the C ABI declared in include/ygg.h).

There is no fallback: if the shared library is missing or was built for another
architecture every entry point raises.  Status codes map onto the reference's error
conventions (pkg/src/specsim/token_tree.py:76-77 IndexError, egt.py:65-80 ValueError).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import torch

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["YGG_LIB_PATH"]) if os.environ.get("YGG_LIB_PATH") else _HERE / "libygg.so"  # A/B builds

YGG_OK, YGG_ERR_VALUE, YGG_ERR_INDEX, YGG_ERR_CUDA, YGG_ERR_UNSUPPORTED = range(5)
YGG_F32, YGG_BF16 = 0, 1
YGG_ACCEPT_PROBS, YGG_ACCEPT_GREEDY, YGG_ACCEPT_SAMPLE = 0, 1, 2
MAX_BREAKPOINTS = 32
MAX_MASK_WORDS = 8

FLAG_SHORTFALL, FLAG_CONTRACT, FLAG_CAPACITY, FLAG_STOPPED, FLAG_INDEX = 1, 2, 4, 8, 16

i32p = C.POINTER(C.c_int32)
u32p = C.POINTER(C.c_uint32)
f64p = C.POINTER(C.c_double)
f32p = C.POINTER(C.c_float)
vp = C.c_void_p


class YggTree(C.Structure):
    _fields_ = [
        ("B", C.c_int32),
        ("cap", C.c_int32),
        ("mask_words", C.c_int32),
        ("token", vp),
        ("parent", vp),
        ("depth", vp),
        ("prob", vp),
        ("cum", vp),
        ("mask", vp),
        ("size", vp),
        ("frontier", vp),
        ("frontier_n", vp),
        ("flags", vp),
    ]


class YggSeq(C.Structure):
    _fields_ = [
        ("B", C.c_int32),
        ("S", C.c_int32),
        ("hist", vp),
        ("P", vp),
        ("n_gen", vp),
        ("acc_log", vp),
        ("step", vp),
        ("log_cap", C.c_int32),
        ("p_limit", C.c_int32),
        ("gen_limit", vp),
        ("status", vp),
    ]


class YggProfile(C.Structure):
    _fields_ = [
        ("n", C.c_int32),
        ("width", C.c_int32 * MAX_BREAKPOINTS),
        ("latency_us", C.c_double * MAX_BREAKPOINTS),
    ]


class YggProfilePair(C.Structure):
    _fields_ = [("drafter", YggProfile), ("verifier", YggProfile)]


class YggPruneArgs(C.Structure):
    _fields_ = [
        ("max_verify", C.c_int32),
        ("d_draft", C.c_int32),
        ("w_draft", C.c_int32),
        ("fixed_k", C.c_int32),
        ("probs_are_gains", C.c_int32),
        ("node_table", vp),
    ]


class YggEpilogue(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("ss_in", vp), ("ss_tiles", C.c_int32), ("norm_dim", C.c_int32), ("eps", C.c_float),
        ("out", vp), ("ld", C.c_int32), ("q_out", vp), ("cache", vp), ("S", C.c_int32), ("Hq", C.c_int32),
        ("Hkv", C.c_int32), ("hd", C.c_int32), ("rope_theta", C.c_float), ("pos", vp), ("slot", vp), ("req", vp),
        ("act_out", vp), ("resid", vp), ("hb", vp), ("ss_out", vp), ("counters", vp), ("dbg", vp),
        ("rope_cs", vp),
    ]


class YggGemvEpilogue(C.Structure):
    """ygg_gemv_epilogue (include/ygg.h)."""

    _fields_ = [
        ("kind", C.c_int32), ("out", vp), ("ld", C.c_int32), ("ss_in", vp), ("ss_blocks", C.c_int32),
        ("norm_dim", C.c_int32), ("eps", C.c_float), ("q_out", vp), ("cache", vp), ("S", C.c_int32),
        ("Hq", C.c_int32), ("Hkv", C.c_int32), ("hd", C.c_int32), ("pos", vp), ("slot", vp), ("req", vp),
        ("rope_cs", vp), ("act_out", vp), ("resid", vp), ("hb", vp), ("ss_out", vp),
        ("topk_part", vp), ("topk_k", C.c_int32), ("inv_temp", C.c_float),
    ]


class YggL2Region(C.Structure):
    """ygg_l2_region (include/ygg.h): a byte range to pull into L2."""

    _fields_ = [("ptr", vp), ("bytes", C.c_uint64)]


YGG_GEMV_STORE, YGG_GEMV_QKV, YGG_GEMV_SWIGLU, YGG_GEMV_RESID, YGG_GEMV_STORE_TOPK = 1, 2, 3, 4, 5

YGG_EPI_NONE, YGG_EPI_STORE_F32, YGG_EPI_QKV_ROPE, YGG_EPI_SWIGLU, YGG_EPI_RESID, YGG_EPI_ARGMAX = range(6)

# name -> (restype, argtypes)
_SIGS: dict[str, tuple] = {
    "ygg_version": (C.c_int, []),
    "ygg_last_error": (C.c_char_p, []),
    "ygg_device_check": (C.c_int, [C.POINTER(C.c_int)] * 3),
    "ygg_topk_workspace": (C.c_size_t, [C.c_int, C.c_int, C.c_int]),
    "ygg_topk_softmax": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, vp, vp, vp, vp,
                                   C.c_size_t, vp]),
    "ygg_egt_grow_level": (C.c_int, [YggTree, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp]),
    "ygg_build_mask": (C.c_int, [YggTree, vp]),
    "ygg_knapsack_prune": (C.c_int, [YggTree, vp, vp, YggPruneArgs, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "ygg_accept_stats": (C.c_int, [YggTree, vp, C.c_int, vp, vp, vp, vp]),
    "ygg_feature_tap": (C.c_int, [vp, C.c_int, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp]),
    "ygg_tree_subtree": (C.c_int, [YggTree, YggTree, vp, vp, vp]),
    "ygg_path_products": (C.c_int, [YggTree, vp, vp, vp]),
    "ygg_accept": (C.c_int, [YggTree, C.c_int, vp, vp, C.c_int, vp, vp, C.c_int, C.c_int, C.c_int, vp, C.c_float,
                             vp, vp, vp, vp, vp, vp]),
    "ygg_kv_compact": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_longlong, vp, vp, vp,
                                 C.c_int, vp, C.c_int, vp, C.c_int, C.c_int, vp]),
    "ygg_gemm_plan_size": (C.c_size_t, []),
    "ygg_gemm_plan_init": (C.c_int, [vp, C.c_int, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp,
                                     C.POINTER(C.c_int), C.POINTER(C.c_size_t)]),
    "ygg_gemm_seg_table_len": (C.c_int, [vp]),
    "ygg_gemm_run": (C.c_int, [vp, vp, vp]),
    "ygg_argmax_reduce": (C.c_int, [vp, C.c_int, C.c_int, vp, vp]),
    "ygg_gemm_plan_set_cluster": (C.c_int, [vp, C.c_int]),
    "ygg_gemm_plan_cluster": (C.c_int, [vp]),
    "ygg_gemm_plan_set_epi_prefetch": (C.c_int, [vp, vp, C.c_size_t]),
    "ygg_gemm_plan_set_layout": (C.c_int, [vp, C.c_int]),
    "ygg_gemm_plan_set_stages": (C.c_int, [vp, C.c_int]),
    "ygg_gemm_fused": (C.c_int, [vp, vp, C.POINTER(YggEpilogue), vp]),
    "ygg_gemm_tiles": (C.c_int, [vp]),
    "ygg_embed_fused": (C.c_int, [vp, C.c_int, C.c_int, vp, C.c_int, vp, vp, vp, vp]),
    "ygg_epi_store": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, vp]),
    "ygg_epi_residual_norm": (C.c_int, [vp, vp, vp, vp, C.c_float, vp, C.c_int, vp]),
    "ygg_epi_swiglu": (C.c_int, [vp, vp, vp, C.c_int, vp]),
    "ygg_epi_qkv_rope": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_float, vp, vp, vp, vp, vp, C.c_int, C.c_int,
                                   vp, vp]),
    "ygg_embed": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp, C.c_int, vp, vp]),
    "ygg_rmsnorm": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_float, vp, vp]),
    "ygg_embed_rmsnorm": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_float, vp, vp, vp]),
    "ygg_attention": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp,
                                C.c_int, C.c_float, vp, vp]),
    "ygg_attn_plan_size": (C.c_size_t, []),
    "ygg_attn_plan_init": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.POINTER(C.c_size_t)]),
    "ygg_attention_tc": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_float, vp, vp, vp]),
    "ygg_row_stats": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, vp, vp, vp]),
    "ygg_pass0_inputs": (C.c_int, [YggSeq, C.c_int, C.c_int, vp, vp, vp, vp, vp, C.c_int, vp, vp, vp]),
    "ygg_init_roots": (C.c_int, [YggTree, vp, vp, C.c_int, C.c_int, C.c_int, vp]),
    "ygg_level_inputs": (C.c_int, [YggTree, YggSeq, C.c_int, C.c_int, vp, vp, vp, vp, vp, C.c_int, vp, vp, vp, vp]),
    "ygg_verify_inputs": (C.c_int, [YggTree, YggSeq, vp, vp, vp, vp, vp, C.c_int, vp, vp, vp]),
    "ygg_commit": (C.c_int, [YggSeq, YggTree, vp, vp, vp, vp, C.c_int, vp]),
    "ygg_stamp": (C.c_int, [vp, vp]),
    "ygg_trace_arm": (C.c_int, [vp, C.c_int]),
    "ygg_trace_used": (C.c_int, [vp, C.c_int]),
    "ygg_attn_dec_plan_size": (C.c_size_t, []),
    "ygg_attn_dec_plan_init": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.c_int]),
    "ygg_attn_dec_workspace_size": (C.c_size_t, [vp]),
    "ygg_attn_dec_run": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_float, vp, vp, vp]),
    "ygg_gemv_plan_size": (C.c_size_t, []),
    "ygg_gemv_plan_init": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int]),
    "ygg_gemv_run": (C.c_int, [vp, C.POINTER(YggGemvEpilogue), vp]),
    "ygg_gemv_plan_set_stages": (C.c_int, [vp, C.c_int]),
    "ygg_gemv_grid": (C.c_int, [vp]),
    "ygg_gemv_set_l2_prefetch": (C.c_int, [vp, C.c_int, vp, C.c_size_t]),
    "ygg_attn_dec_set_l2_prefetch": (C.c_int, [vp, C.c_int, vp, C.c_size_t]),
    "ygg_attn_dec_set_gemv_prefetch": (C.c_int, [vp, vp]),
    "ygg_attn_tree_plan_size": (C.c_size_t, []),
    "ygg_attn_tree_plan_init": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_int]),
    "ygg_attn_tree_info": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ygg_attn_tree_set_l2_prefetch": (C.c_int, [vp, C.c_int, vp, C.c_size_t]),
    "ygg_attn_tree_set_debug": (C.c_int, [vp, vp]),
    "ygg_attn_tree_set_trigger": (C.c_int, [vp, C.c_int]),
    "ygg_attn_tree_run": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_float, vp, vp]),
    "ygg_gemv_stream_info": (C.c_int, [vp, vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ygg_topk_partial_bytes": (C.c_size_t, [C.c_int, C.c_int]),
    "ygg_topk_merge": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp]),
    "ygg_topk_merge_l2": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, C.c_int, vp]),
}

EXPORTED = tuple(_SIGS)

# Kernels launched by one successful call (used to count device launches per step).
KERNELS_PER_CALL = {
    "ygg_topk_softmax": 2, "ygg_egt_grow_level": 1, "ygg_build_mask": 1, "ygg_knapsack_prune": 1,
    "ygg_tree_subtree": 1, "ygg_path_products": 1, "ygg_accept": 1, "ygg_kv_compact": 1, "ygg_gemm_run": 1, "ygg_gemm_fused": 1, "ygg_embed_fused": 1, "ygg_epi_store": 1,
    "ygg_epi_residual_norm": 1, "ygg_epi_swiglu": 1, "ygg_epi_qkv_rope": 1, "ygg_embed": 1, "ygg_rmsnorm": 1, "ygg_embed_rmsnorm": 1,
    "ygg_attention": 1, "ygg_attention_tc": 2, "ygg_row_stats": 1, "ygg_pass0_inputs": 1, "ygg_init_roots": 1, "ygg_level_inputs": 1,
    "ygg_verify_inputs": 1, "ygg_commit": 1, "ygg_stamp": 1, "ygg_gemv_run": 1, "ygg_attn_dec_run": 1, "ygg_attn_tree_run": 1, "ygg_topk_merge": 1, "ygg_topk_merge_l2": 1,
}
launches = {"count": 0}


class _Counted:
    __slots__ = ("fn", "k")

    def __init__(self, fn, k):
        self.fn, self.k = fn, k

    def __call__(self, *a):
        rc = self.fn(*a)
        if rc == 0:
            launches["count"] += self.k
        return rc


class _Lib:
    pass


_lib = None


def load():
    """Load libygg.so and bind every entry point (no device work is done here)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)"
            )
        raw = C.CDLL(str(LIB_PATH))
        lib = _Lib()
        lib._raw = raw
        for name, (res, args) in _SIGS.items():
            fn = getattr(raw, name)
            fn.restype = res
            fn.argtypes = args
            setattr(lib, name, _Counted(fn, KERNELS_PER_CALL[name]) if name in KERNELS_PER_CALL else fn)
        _lib = lib
    return _lib


def lib():
    return load()


def check(rc: int) -> None:
    if rc == YGG_OK:
        return
    msg = (lib().ygg_last_error() or b"").decode(errors="replace")
    if rc == YGG_ERR_VALUE:
        raise ValueError(msg)
    if rc == YGG_ERR_INDEX:
        raise IndexError(msg)
    raise RuntimeError(f"libygg error {rc}: {msg}")


_device_checked = False


def require_device() -> None:
    """Fail loudly unless a B200 (sm_100) is present; the kernels have no other path."""
    global _device_checked
    if _device_checked:
        return
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2512_23858_b200 needs a CUDA B200 device (sm_100a); no CPU fallback exists")
    n, ma, mi = C.c_int(), C.c_int(), C.c_int()
    check(lib().ygg_device_check(C.byref(n), C.byref(ma), C.byref(mi)))
    _device_checked = True


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return YGG_F32
    if dt == torch.bfloat16:
        return YGG_BF16
    raise ValueError(f"unsupported dtype {dt}")


def make_profile(breakpoints) -> YggProfile:
    p = YggProfile()
    pts = list(breakpoints)
    if not 2 <= len(pts) <= MAX_BREAKPOINTS:
        raise ValueError(f"profile needs 2..{MAX_BREAKPOINTS} breakpoints, got {len(pts)}")
    p.n = len(pts)
    for i, (w, lat) in enumerate(pts):
        p.width[i] = int(w)
        p.latency_us[i] = float(lat)
    return p


def profile_pair_bytes(drafter_bps, verifier_bps) -> bytes:
    pp = YggProfilePair(make_profile(drafter_bps), make_profile(verifier_bps))
    return bytes(pp)


if os.environ.get("YGG_EAGER_LOAD"):
    load()
