"""Equal-growth tree drafting and verification-width pruning (API of pkg/src/specsim/egt.py),
executed by the device kernels.

``grow_step`` gathers candidates from the caller's ``DrafterDistribution`` plugin (host, as in the
reference, egt.py:52-80) and runs the global top-W selection on the GPU (K1 ``ygg_egt_grow_level``),
appending the attached nodes to the host ``TokenTree``.  ``SubtreeKnapsack`` / ``prune_verify`` /
``select_width`` run the f64 tree-knapsack and Eq.3 objective on the GPU (K6
``ygg_knapsack_prune``).  Every tie rule matches the reference bit-for-bit (tests/golden/).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Protocol, Sequence, runtime_checkable

import numpy as np
import torch

from . import _lib as L
from . import device_tree
from .acceptance import AcceptanceModel, SurrogateAcceptance, freeze_probs
from .latency import ProfilePair, SpeedupInputs, TreeShape, tree_speedup
from .token_tree import SIBLING_SUM_TOL, TokenTree, new_tree


@dataclass(frozen=True)
class EgtConfig:
    candidate_widths: tuple[int, ...] = (1, 2, 4, 8)
    max_depth: int = 16
    max_verify: int = 64
    expansion_k: int = 8

    def __post_init__(self) -> None:
        if not self.candidate_widths:
            raise ValueError("candidate_widths must be non-empty")
        if any(w < 1 for w in self.candidate_widths):
            raise ValueError(f"candidate widths must be >= 1: {self.candidate_widths}")
        if list(self.candidate_widths) != sorted(set(self.candidate_widths)):
            raise ValueError(f"candidate widths must be sorted and distinct: {self.candidate_widths}")
        if self.max_depth < 1:
            raise ValueError(f"max_depth {self.max_depth} must be >= 1")
        if self.max_verify < 1:
            raise ValueError(f"max_verify {self.max_verify} must be >= 1")
        if self.expansion_k < 1:
            raise ValueError(f"expansion_k {self.expansion_k} must be >= 1")


@runtime_checkable
class DrafterDistribution(Protocol):
    def root(self) -> tuple[int, float]:
        ...

    def candidates(self, tree: TokenTree, node: int, k: int) -> Sequence[tuple[int, float]]:
        ...


def _checked_candidates(drafter, tree, node, k) -> list[tuple[int, float]]:
    out = list(drafter.candidates(tree, node, k))
    total, prev = 0.0, float("inf")
    for _, p in out:
        if not 0.0 <= p <= 1.0:
            raise ValueError(f"candidate probability {p} for node {node} out of range")
        if p > prev:
            raise ValueError(f"candidate probabilities for node {node} must be descending")
        prev = p
        total += p
    if total > 1.0 + SIBLING_SUM_TOL:
        raise ValueError(f"candidate probabilities for node {node} sum to {total}")
    return out


def grow_step(tree: TokenTree, drafter: DrafterDistribution, w_draft: int, expansion_k: int = 8) -> list[int]:
    """Attach up to ``w_draft`` leaves under the newest level (global top-W on the GPU)."""
    if w_draft < 1:
        raise ValueError(f"w_draft {w_draft} must be >= 1")
    frontier = tree.levels[-1]
    if not frontier:
        raise ValueError("frontier is empty")
    cands = [_checked_candidates(drafter, tree, node, expansion_k) for node in frontier]
    kmax = max(1, max(len(c) for c in cands))
    F = len(frontier)
    tok = torch.zeros(1, F, kmax, dtype=torch.int32)
    prob = torch.zeros(1, F, kmax, dtype=torch.float64)
    cnt = torch.zeros(1, F, dtype=torch.int32)
    for f, cl in enumerate(cands):
        cnt[0, f] = len(cl)
        for r, (t, p) in enumerate(cl):
            tok[0, f, r] = int(t)
            prob[0, f, r] = float(p)
    n0 = len(tree)
    dt = device_tree.upload(tree, n0 + w_draft)
    tok_d, prob_d, cnt_d = tok.cuda(), prob.cuda(), cnt.cuda()
    L.check(L.lib().ygg_egt_grow_level(dt.struct, F, kmax, w_draft, tok_d.data_ptr(), prob_d.data_ptr(),
                                       cnt_d.data_ptr(), L.stream_ptr()))
    flags = int(dt.flags[0])
    if flags & L.FLAG_CONTRACT:
        raise ValueError("candidate lists violate the drafter contract")
    n1 = int(dt.size[0])
    added = []
    if n1 > n0:
        toks = dt.token[0, n0:n1].cpu().tolist()
        pars = dt.parent[0, n0:n1].cpu().tolist()
        probs = dt.prob[0, n0:n1].cpu().tolist()
        for t, p, q in zip(toks, pars, probs):
            added.append(tree.add_child(p, t, q))
    return added


@dataclass(frozen=True)
class GrowthResult:
    tree: TokenTree
    shortfall: bool


def grow_egt(tree: TokenTree, drafter: DrafterDistribution, d_draft: int, w_draft: int,
             expansion_k: int = 8) -> GrowthResult:
    if d_draft < 1:
        raise ValueError(f"d_draft {d_draft} must be >= 1")
    short = False
    for _ in range(d_draft):
        if not tree.levels[-1]:
            short = True
            break
        added = grow_step(tree, drafter, w_draft, expansion_k)
        if len(added) < w_draft:
            short = True
        if not added:
            break
    return GrowthResult(tree=tree, shortfall=short)


def _dev_profiles(profiles: ProfilePair | None) -> torch.Tensor:
    if profiles is None:
        bp = ((1, 1.0), (2, 1.0))
        raw = L.profile_pair_bytes(bp, bp)
    else:
        raw = L.profile_pair_bytes(profiles.drafter.breakpoints, profiles.verifier.breakpoints)
    return torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()


class _Knap:
    """One K6 launch on a host tree; returns every output plus the exported DP tables."""

    def __init__(self, tree: TokenTree, probs: np.ndarray, max_verify: int, profiles: ProfilePair | None,
                 d_draft: int, w_draft: int, fixed_k: int = 0, tables: bool = False, gains: bool = False):
        if max_verify < 1:
            raise ValueError(f"max_size {max_verify} must be >= 1")
        dt = device_tree.upload(tree)
        cap = dt.cap
        self.N = len(tree)
        self.cap = min(max_verify, self.N)
        mv = min(max_verify, 255)
        p = torch.zeros(1, cap, dtype=torch.float64)
        p[0, : self.N] = torch.as_tensor(np.asarray(probs, dtype=np.float64))
        p = p.cuda()
        pp = _dev_profiles(profiles)
        i32 = dict(dtype=torch.int32, device="cuda")
        f64 = dict(dtype=torch.float64, device="cuda")
        self.keep = torch.zeros(1, cap, **i32)
        self.new = torch.zeros(1, cap, **i32)
        self.wv = torch.zeros(1, **i32)
        self.aal = torch.zeros(1, **f64)
        self.sp = torch.zeros(1, **f64)
        self.aal_cap = torch.zeros(1, **f64)
        self.sp_cap = torch.zeros(1, **f64)
        self.best = torch.full((1, cap, mv + 1), float("-inf"), **f64) if tables else None
        self.alloc = torch.zeros(1, cap, mv + 1, dtype=torch.uint8, device="cuda") if tables else None
        args = L.YggPruneArgs(mv, max(d_draft, 1), max(w_draft, 1), fixed_k, 1 if gains else 0)
        L.check(L.lib().ygg_knapsack_prune(
            dt.struct, p.data_ptr(), pp.data_ptr(), args, self.keep.data_ptr(), self.new.data_ptr(),
            self.wv.data_ptr(), self.aal.data_ptr(), self.sp.data_ptr(), self.aal_cap.data_ptr(),
            self.sp_cap.data_ptr(), self.best.data_ptr() if tables else None,
            self.alloc.data_ptr() if tables else None, L.stream_ptr()))
        self.flags = int(dt.flags[0])


def _subtree_sizes(tree: TokenTree) -> list[int]:
    sizes = [1] * len(tree)
    for v in range(len(tree) - 1, 0, -1):
        sizes[tree.parent(v)] += sizes[v]
    return sizes


class SubtreeKnapsack:
    """best(v, k): max total gain of a connected subtree rooted at v with k nodes (GPU DP)."""

    def __init__(self, tree: TokenTree, gains: np.ndarray, max_size: int) -> None:
        if max_size < 1:
            raise ValueError(f"max_size {max_size} must be >= 1")
        if len(gains) != len(tree):
            raise ValueError(f"need one gain per node, got {len(gains)} for {len(tree)}")
        self.tree = tree
        self.gains = np.asarray(gains, dtype=np.float64)
        self.max_size = min(max_size, len(tree))
        k = _Knap(tree, self.gains, max_size, None, 1, 1, tables=True, gains=True)
        self._best = k.best[0, : len(tree), : self.max_size + 1].cpu().numpy()
        self._alloc = k.alloc[0, : len(tree), : self.max_size + 1].cpu().numpy()
        self._kids = [tree.children(v) for v in range(len(tree))]

    def best(self, v: int, k: int) -> float:
        if not 1 <= k <= self.max_size:
            raise ValueError(f"size {k} out of range [1, {self.max_size}]")
        return float(self._best[v][k])

    def best_row(self, v: int) -> np.ndarray:
        return self._best[v].copy()

    def pick(self, k: int) -> set[int]:
        if not 1 <= k <= self.max_size or self._best[0][k] == -np.inf:
            raise ValueError(f"no connected root subtree of size {k}")
        keep: set[int] = set()
        stack = [(0, k)]
        while stack:
            v, kk = stack.pop()
            keep.add(v)
            rem = kk
            for c in reversed(self._kids[v]):
                taken = int(self._alloc[c][rem])
                if taken:
                    stack.append((c, taken))
                    rem -= taken
        return keep


@dataclass(frozen=True)
class PruneResult:
    tree: TokenTree
    w_verify: int
    kept: tuple[int, ...]
    expected_aal: float
    speedup: float


def prune_verify(tree: TokenTree, model: AcceptanceModel, profiles: ProfilePair, d_draft: int, w_draft: int,
                 max_verify: int) -> PruneResult:
    """Latency-aware verification budget + optimal connected subtree (K6 on the GPU)."""
    probs = freeze_probs(model, tree)
    k = _Knap(tree, probs, max_verify, profiles, d_draft, w_draft)
    if k.flags & L.FLAG_CONTRACT:
        TreeShape(w_draft=w_draft, d_draft=d_draft, w_verify=k.cap)  # raises the reference ValueError
    kept = tuple(i for i in k.keep[0].cpu().tolist() if i >= 0)
    pruned, _ = tree.subtree(kept)
    return PruneResult(tree=pruned, w_verify=int(k.wv[0]), kept=kept, expected_aal=float(k.aal[0]),
                       speedup=float(k.sp[0]))


def select_width(config: EgtConfig, depth: int, drafter: DrafterDistribution, profiles: ProfilePair,
                 model: AcceptanceModel | None = None) -> int:
    if not 1 <= depth <= config.max_depth:
        raise ValueError(f"depth {depth} outside [1, {config.max_depth}]")
    model = model if model is not None else SurrogateAcceptance()
    best_w, best_v = config.candidate_widths[0], -np.inf
    for w in config.candidate_widths:
        tree = new_tree(*drafter.root())
        grow_egt(tree, drafter, depth, w, config.expansion_k)
        k = _Knap(tree, freeze_probs(model, tree), config.max_verify, profiles, depth, w)
        value = float(k.sp_cap[0])
        if value > best_v + 1e-12:
            best_w, best_v = w, value
    return best_w


def depth_decay_aal(p0: float, gamma: float, w_draft: int, d_draft: int) -> float:
    """Closed-form AAL of the concentrated growth limit under a depth-rank model (egt.py:321-345)."""
    from .acceptance import DepthDecayAcceptance

    if not 0.0 <= p0 <= 1.0:
        raise ValueError(f"p0 {p0} must be in [0, 1]")
    if not 0.0 <= gamma <= 1.0:
        raise ValueError(f"gamma {gamma} must be in [0, 1]")
    if w_draft < 1 or d_draft < 1:
        raise ValueError("w_draft and d_draft must be >= 1")
    top = DepthDecayAcceptance.rank_share(0, w_draft)
    total, path = 1.0, 1.0
    for level in range(d_draft + 1):
        rate = p0 * gamma**level
        total += path * rate
        path *= rate * (1.0 if level == 0 else top)
    return total


__all__ = ["EgtConfig", "DrafterDistribution", "grow_step", "GrowthResult", "grow_egt", "SubtreeKnapsack",
           "PruneResult", "prune_verify", "select_width", "depth_decay_aal", "tree_speedup", "SpeedupInputs",
           "TreeShape"]
