"""CPU restatement of the reference's hot-path tree algorithms (test oracle only).

Each function follows the cited reference semantics (paths relative to
/root/reference/pkg/src/specsim/) with its own, simpler data structures: a tree is a list of
``(token, parent, prob)`` triples in topological order.  Floating-point expressions keep the
reference's operation order so results are bit-identical to CPython floats.
"""

from __future__ import annotations

import math
from bisect import bisect_right
from dataclasses import dataclass, field

import numpy as np

SIBLING_TOL = 1e-9  # token_tree.py:31


# ---------------------------------------------------------------------------
# Tree (token_tree.py:34-197)
# ---------------------------------------------------------------------------
@dataclass
class Tree:
    token: list = field(default_factory=list)
    parent: list = field(default_factory=list)  # None for the root
    prob: list = field(default_factory=list)
    depth: list = field(default_factory=list)

    @classmethod
    def root(cls, token: int, prob: float) -> "Tree":
        if not 0.0 <= prob <= 1.0:
            raise ValueError("probability outside [0, 1]")
        return cls([int(token)], [None], [float(prob)], [0])

    def __len__(self):
        return len(self.token)

    def children(self, v: int) -> list:
        return [i for i in range(v + 1, len(self)) if self.parent[i] == v]

    def add(self, parent: int, token: int, prob: float) -> int:
        """token_tree.py:69-94 (IndexError on a bad parent, ValueError on the sibling sum)."""
        if not 0 <= parent < len(self):
            raise IndexError("parent out of range")
        if not 0.0 <= prob <= 1.0:
            raise ValueError("probability outside [0, 1]")
        s = sum(self.prob[c] for c in self.children(parent))
        if s + prob > 1.0 + SIBLING_TOL:
            raise ValueError("sibling probabilities exceed one")
        self.token.append(int(token))
        self.parent.append(parent)
        self.prob.append(float(prob))
        self.depth.append(self.depth[parent] + 1)
        return len(self) - 1

    def levels(self) -> list:
        out: list = []
        for i, d in enumerate(self.depth):
            while len(out) <= d:
                out.append([])
            out[d].append(i)
        return out

    def path(self, i: int) -> list:
        """token_tree.py:134-144."""
        p = []
        while i is not None:
            p.append(i)
            i = self.parent[i]
        return p[::-1]

    def to_dict(self) -> dict:
        return {"nodes": [{"token": t, "parent": p, "prob": q} for t, p, q in zip(self.token, self.parent, self.prob)]}

    @classmethod
    def from_dict(cls, d: dict) -> "Tree":
        nodes = d["nodes"]
        t = cls.root(nodes[0]["token"], nodes[0]["prob"])
        for nd in nodes[1:]:
            t.add(nd["parent"], nd["token"], nd["prob"])
        return t

    def subtree(self, keep) -> tuple["Tree", dict]:
        """token_tree.py:146-168: kept nodes in ascending old order, parents remapped."""
        kept = sorted(set(keep))
        if not kept or kept[0] != 0:
            raise ValueError("subtree must contain the root")
        ks = set(kept)
        for i in kept:
            if self.parent[i] is not None and self.parent[i] not in ks:
                raise ValueError("subtree is not connected")
        out = Tree.root(self.token[0], self.prob[0])
        m = {0: 0}
        for i in kept[1:]:
            m[i] = out.add(m[self.parent[i]], self.token[i], self.prob[i])
        return out, m


def build_mask(tree: Tree) -> np.ndarray:
    """token_tree.py:205-218: mask[i, j] iff j is i or an ancestor of i (independent walk)."""
    n = len(tree)
    m = np.zeros((n, n), dtype=bool)
    for i in range(n):
        for j in tree.path(i):
            m[i, j] = True
    return m


# ---------------------------------------------------------------------------
# Candidates + EGT growth (egt.py:65-147)
# ---------------------------------------------------------------------------
def check_candidates(cands) -> list:
    """egt.py:65-80: each prob in [0,1], non-increasing, running sum <= 1 + 1e-9."""
    total, prev = 0.0, math.inf
    out = []
    for tok, p in cands:
        if not 0.0 <= p <= 1.0 or p > prev:
            raise ValueError("bad candidate list")
        prev = p
        total += p
        out.append((int(tok), float(p)))
    if total > 1.0 + SIBLING_TOL:
        raise ValueError("candidate probabilities exceed one")
    return out


def grow_step(tree: Tree, candidates_of, w_draft: int, k: int = 8) -> list:
    """egt.py:83-114.  ``candidates_of(tree, node, k)`` -> ranked (token, prob) list."""
    if w_draft < 1:
        raise ValueError("w_draft must be >= 1")
    frontier = tree.levels()[-1]
    scored = []
    for par in frontier:
        path_prob = 1.0
        for n in tree.path(par):  # multiplication in root -> parent order
            path_prob *= tree.prob[n]
        for rank, (tok, p) in enumerate(check_candidates(candidates_of(tree, par, k))):
            scored.append((path_prob * p, par, rank, tok, p))
    scored.sort(key=lambda e: (-e[0], e[1], e[2]))
    return [tree.add(par, tok, p) for _, par, _, tok, p in scored[:w_draft]]


def grow_egt(tree: Tree, candidates_of, d_draft: int, w_draft: int, k: int = 8) -> bool:
    """egt.py:123-147; returns the shortfall flag."""
    short = False
    for _ in range(d_draft):
        added = grow_step(tree, candidates_of, w_draft, k)
        if len(added) < w_draft:
            short = True
        if not added:
            break
    return short


def topk_softmax(logits: np.ndarray, k: int, temperature: float = 1.0) -> list:
    """Draft candidates from one logit row: f64 softmax of the f32 logits, top-k by
    (logit desc, token asc), then ordered (prob desc, token asc) — the device K1a contract."""
    x = np.asarray(logits, dtype=np.float32) / np.float32(temperature)
    x64 = x.astype(np.float64)
    m = float(x64.max())
    e = np.exp(x64 - m)
    z = float(e.sum())
    order = np.lexsort((np.arange(len(x)), -x64))[:k]
    top = [(int(t), float(e[t])) for t in order]
    z = max(z, sum(v for _, v in top))
    cand = [(t, v / z) for t, v in top]
    cand.sort(key=lambda c: (-c[1], c[0]))
    return cand


# ---------------------------------------------------------------------------
# Knapsack + prune (egt.py:150-282; acceptance.py:176-184)
# ---------------------------------------------------------------------------
def path_products(tree: Tree, probs) -> list:
    out = [0.0] * len(tree)
    out[0] = float(probs[0])
    for i in range(1, len(tree)):
        out[i] = out[tree.parent[i]] * float(probs[i])
    return out


class Knapsack:
    """best[v][s]: max gain of a connected subtree rooted at v with s nodes (egt.py:150-229).

    Row merge: for each target size s, candidate splits are scanned with the kept part k
    ascending and a strict '>' against the running value (initially the row without the child),
    which is exactly the reference's first-maximum rule."""

    def __init__(self, tree: Tree, gains, max_size: int):
        if max_size < 1:
            raise ValueError("max_size must be >= 1")
        n = len(tree)
        self.tree = tree
        self.cap = min(max_size, n)
        cap = self.cap
        size = [1] * n
        for v in range(n - 1, 0, -1):
            size[tree.parent[v]] += size[v]
        self.best = [None] * n
        self.alloc = {}  # child -> allocation row
        self.kids = [tree.children(v) for v in range(n)]
        for v in range(n - 1, -1, -1):
            row = [-math.inf] * (cap + 1)
            row[1] = float(gains[v])
            for c in self.kids[v]:
                crow = self.best[c]
                top = min(size[c], cap)
                new = list(row)
                al = [0] * (cap + 1)
                for s in range(2, cap + 1):
                    for kk in range(max(1, s - top), s):
                        if row[kk] == -math.inf:
                            continue
                        val = row[kk] + crow[s - kk]
                        if val > new[s]:
                            new[s] = val
                            al[s] = s - kk
                row = new
                self.alloc[c] = al
            self.best[v] = row

    def pick(self, k: int) -> set:
        keep: set = set()
        stack = [(0, k)]
        while stack:
            v, kk = stack.pop()
            keep.add(v)
            rem = kk
            for c in reversed(self.kids[v]):
                taken = self.alloc[c][rem]
                if taken:
                    stack.append((c, taken))
                    rem -= taken
        return keep


@dataclass(frozen=True)
class Profile:
    breakpoints: tuple


def latency_at(profile, width: int) -> float:
    """latency.py:68-82 (same operation order)."""
    pts = profile.breakpoints if hasattr(profile, "breakpoints") else profile
    if width < 1:
        raise ValueError("width must be >= 1")
    ws = [w for w, _ in pts]
    if width <= ws[0]:
        return pts[0][1]
    if width >= ws[-1]:
        (w0, l0), (w1, l1) = pts[-2], pts[-1]
        slope = (l1 - l0) / (w1 - w0)
        return l1 + slope * (width - w1)
    hi = bisect_right(ws, width)
    (w0, l0), (w1, l1) = pts[hi - 1], pts[hi]
    return l0 + (l1 - l0) * (width - w0) / (w1 - w0)


def tree_speedup(aal: float, w_draft: int, d_draft: int, w_verify: int, drafter, verifier) -> float:
    """latency.py:154-161."""
    draft_cost = d_draft * latency_at(drafter, w_draft)
    verify_cost = latency_at(verifier, w_verify + 1)
    return aal * latency_at(verifier, 1) / (draft_cost + verify_cost)


@dataclass
class Pruned:
    tree: Tree
    w_verify: int
    kept: tuple
    expected_aal: float
    speedup: float


def prune_verify(tree: Tree, probs, drafter, verifier, d_draft: int, w_draft: int, max_verify: int) -> Pruned:
    """egt.py:241-282."""
    dp = Knapsack(tree, path_products(tree, probs), max_verify)
    best_k, best_s = 0, -math.inf
    for k in range(1, dp.cap + 1):
        v = dp.best[0][k]
        if v == -math.inf:
            continue
        s = tree_speedup(1.0 + v, w_draft, d_draft, k, drafter, verifier)
        if s > best_s + 1e-12:
            best_k, best_s = k, s
    keep = dp.pick(best_k)
    sub, _ = tree.subtree(keep)
    return Pruned(sub, best_k, tuple(sorted(keep)), 1.0 + dp.best[0][best_k], best_s)


def select_width(widths, depth: int, root, candidates_of, k: int, max_verify: int, drafter, verifier,
                 probs_of=None) -> int:
    """egt.py:285-318 (SurrogateAcceptance unless ``probs_of(tree)`` is given)."""
    best_w, best_v = widths[0], -math.inf
    for w in widths:
        t = Tree.root(*root)
        grow_egt(t, candidates_of, depth, w, k)
        probs = probs_of(t) if probs_of else t.prob
        dp = Knapsack(t, path_products(t, probs), max_verify)
        v = tree_speedup(1.0 + dp.best[0][dp.cap], w, depth, dp.cap, drafter, verifier)
        if v > best_v + 1e-12:
            best_w, best_v = w, v
    return best_w


# ---------------------------------------------------------------------------
# Acceptance walk (acceptance.py:221-241)
# ---------------------------------------------------------------------------
def sample_with_probs(tree: Tree, probs, draws) -> tuple[list, int, int]:
    """Returns (accepted_path, accepted_len, draws_used); ``draws`` is an iterator of uniforms."""
    path: list = []
    cursor = None
    used = 0
    while True:
        group = [0] if cursor is None else tree.children(cursor)
        if not group:
            break
        u = next(draws)
        used += 1
        acc = 0.0
        chosen = None
        for c in group:
            acc += float(probs[c])
            if u < acc:
                chosen = c
                break
        if chosen is None:
            break
        path.append(chosen)
        cursor = chosen
    return path, len(path) + 1, used


def greedy_walk(tree: Tree, row_argmax) -> tuple[list, int]:
    """Greedy realisation: prob(child) = 1 iff token == argmax at the parent's verify row
    (row 0 = the confirmed token, row 1+i = node i).  Returns (path, bonus)."""
    path: list = []
    cursor = None
    while True:
        group = [0] if cursor is None else tree.children(cursor)
        row = 0 if cursor is None else 1 + cursor
        nxt = None
        for c in group:
            if tree.token[c] == row_argmax[row]:
                nxt = c
                break
        if nxt is None:
            return path, int(row_argmax[row])
        path.append(nxt)
        cursor = nxt
