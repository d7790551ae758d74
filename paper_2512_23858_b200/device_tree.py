"""Device-resident batched draft trees (``ygg_tree``) and sequence state (``ygg_seq``).

A ``DeviceTrees`` batch is the structure-of-arrays image of B reference ``TokenTree``
objects (pkg/src/specsim/token_tree.py:34-197): node 0 is the root, ``parent[i] < i``,
``depth = depth(parent) + 1``, per-node surrogate probability, the f64 path product used as
the EGT score / knapsack gain, and the ancestor-or-self bit rows of ``build_mask``
(token_tree.py:205-218).  ``to_dicts`` emits the reference's JSON tree format
(token_tree.py:170-176) so device trees compare node-for-node with reference trees.
"""

from __future__ import annotations

import torch

from . import _lib as L


class DeviceTrees:
    def __init__(self, B: int, cap: int, device="cuda"):
        if not 1 <= cap <= 32 * L.MAX_MASK_WORDS:
            raise ValueError(f"tree capacity {cap} outside [1, {32 * L.MAX_MASK_WORDS}]")
        self.B, self.cap = B, cap
        self.mask_words = (cap + 31) // 32
        i32 = dict(dtype=torch.int32, device=device)
        self.token = torch.zeros(B, cap, **i32)
        self.parent = torch.full((B, cap), -1, **i32)
        self.depth = torch.zeros(B, cap, **i32)
        self.prob = torch.zeros(B, cap, dtype=torch.float64, device=device)
        self.cum = torch.zeros(B, cap, dtype=torch.float64, device=device)
        self.mask = torch.zeros(B, cap, self.mask_words, **i32)
        self.size = torch.zeros(B, **i32)
        self.frontier = torch.zeros(B, cap, **i32)
        self.frontier_n = torch.zeros(B, **i32)
        self.flags = torch.zeros(B, **i32)
        self._struct = L.YggTree(
            B, cap, self.mask_words, self.token.data_ptr(), self.parent.data_ptr(), self.depth.data_ptr(),
            self.prob.data_ptr(), self.cum.data_ptr(), self.mask.data_ptr(), self.size.data_ptr(),
            self.frontier.data_ptr(), self.frontier_n.data_ptr(), self.flags.data_ptr()
        )

    @property
    def struct(self) -> L.YggTree:
        return self._struct

    # ---- host conversion (tests / drop-in API) ----
    def load_host(self, trees: list[dict]) -> None:
        """Upload reference-format tree dicts ({"nodes":[{token,parent,prob}]})."""
        if len(trees) != self.B:
            raise ValueError(f"need {self.B} trees, got {len(trees)}")
        tok = torch.zeros(self.B, self.cap, dtype=torch.int32)
        par = torch.full((self.B, self.cap), -1, dtype=torch.int32)
        dep = torch.zeros(self.B, self.cap, dtype=torch.int32)
        prob = torch.zeros(self.B, self.cap, dtype=torch.float64)
        cum = torch.zeros(self.B, self.cap, dtype=torch.float64)
        size = torch.zeros(self.B, dtype=torch.int32)
        front = torch.zeros(self.B, self.cap, dtype=torch.int32)
        fn = torch.zeros(self.B, dtype=torch.int32)
        for b, tr in enumerate(trees):
            nodes = tr["nodes"]
            if len(nodes) > self.cap:
                raise ValueError(f"tree of {len(nodes)} nodes exceeds capacity {self.cap}")
            depths = []
            for i, nd in enumerate(nodes):
                p = nd["parent"]
                tok[b, i] = int(nd["token"])
                prob[b, i] = float(nd["prob"])
                if p is None:
                    par[b, i] = -1
                    depths.append(0)
                    cum[b, i] = float(nd["prob"])
                else:
                    par[b, i] = int(p)
                    depths.append(depths[p] + 1)
                    cum[b, i] = float(cum[b, p]) * float(nd["prob"])
                dep[b, i] = depths[-1]
            size[b] = len(nodes)
            md = max(depths)
            newest = [i for i, dd in enumerate(depths) if dd == md]
            fn[b] = len(newest)
            front[b, : len(newest)] = torch.tensor(newest, dtype=torch.int32)
        for dst, src in ((self.token, tok), (self.parent, par), (self.depth, dep), (self.prob, prob),
                         (self.cum, cum), (self.size, size), (self.frontier, front), (self.frontier_n, fn)):
            dst.copy_(src)
        self.flags.zero_()
        L.check(L.lib().ygg_build_mask(self.struct, L.stream_ptr()))

    def to_dicts(self) -> list[dict]:
        size = self.size.cpu().tolist()
        tok = self.token.cpu().tolist()
        par = self.parent.cpu().tolist()
        prob = self.prob.cpu().tolist()
        out = []
        for b in range(self.B):
            nodes = []
            for i in range(size[b]):
                nodes.append({"token": tok[b][i], "parent": None if par[b][i] < 0 else par[b][i], "prob": prob[b][i]})
            out.append({"nodes": nodes})
        return out

    def masks_bool(self, b: int) -> torch.Tensor:
        """Dense bool mask of tree ``b`` (build_mask layout)."""
        n = int(self.size[b])
        words = self.mask[b, :n].cpu().to(torch.int64) & 0xFFFFFFFF
        cols = torch.arange(n)
        bits = (words[:, cols // 32] >> (cols % 32)) & 1
        return bits.bool()


class SeqState:
    """Per-request sequence state (``ygg_seq``).  ``p_limit`` bounds the prefix: the commit kernel
    freezes a request instead of advancing P past it (status bit1), and a request whose n_gen reaches
    ``gen_limit[b]`` is finished and frozen (status bit0)."""

    def __init__(self, B: int, S: int, log_cap: int = 4096, device="cuda", p_limit: int = 0):
        i32 = dict(dtype=torch.int32, device=device)
        self.B, self.S, self.log_cap = B, S, log_cap
        self.hist = torch.zeros(B, S, **i32)
        self.P = torch.zeros(B, **i32)
        self.n_gen = torch.zeros(B, **i32)
        self.acc_log = torch.zeros(B, log_cap, **i32)
        self.step = torch.zeros(1, **i32)
        self.gen_limit = torch.full((B,), 2**31 - 1, **i32)
        self.status = torch.zeros(B, **i32)
        self.p_limit = int(p_limit)
        self._struct = L.YggSeq(B, S, self.hist.data_ptr(), self.P.data_ptr(), self.n_gen.data_ptr(),
                                self.acc_log.data_ptr(), self.step.data_ptr(), log_cap, self.p_limit,
                                self.gen_limit.data_ptr(), self.status.data_ptr())

    @property
    def struct(self) -> L.YggSeq:
        return self._struct


_CACHE: dict[int, DeviceTrees] = {}


def upload(tree, cap: int | None = None) -> DeviceTrees:
    """Single-tree device image of a host ``TokenTree`` (B=1), reusing a buffer per capacity;
    runs K7 for the mask rows."""
    n = len(tree)
    cap = max(cap or n, n)
    cap = min(32 * L.MAX_MASK_WORDS, ((cap + 31) // 32) * 32)
    if n > cap:
        raise ValueError(f"tree of {n} nodes exceeds the device capacity {cap}")
    dt = _CACHE.get(cap)
    if dt is None:
        L.require_device()
        dt = DeviceTrees(1, cap, "cuda")
        _CACHE[cap] = dt
    dt.load_host([tree.to_dict()])
    return dt
