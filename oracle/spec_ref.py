"""The speculative step on the CPU (test oracle only), with the device path's exact conventions.

Per step (see paper_2512_23858_b200/engine.py): draft pass 0 over [x_{P-1}, bonus] -> root =
top-1 of the bonus row; D draft passes over the newest level, each followed by one reference
grow_step (egt.py:83-114) on the top-k candidates; prune_verify with the surrogate model
(egt.py:241-282); target verify over [bonus, pruned nodes]; greedy walk (acceptance.py:221-241
with 0/1 probabilities); compaction of the accepted K/V in both caches.
"""

from __future__ import annotations

import torch

from . import tree_ref as T
from .llama_ref import RefCache, RefLlama, causal_visible


class OracleTreeOps:
    """Tree logic of the step from the oracle restatement (``tree_ref``)."""

    name = "oracle"

    def root(self, tok, prob):
        return T.Tree.root(tok, prob)

    def frontier(self, tree):
        return tree.levels()[-1]

    def node(self, tree, i):
        return tree.token[i], tree.depth[i], tree.path(i)

    def grow(self, tree, cands, W, k):
        return T.grow_step(tree, lambda tr, node, kk: cands[node], W, k)

    def prune(self, tree, dp, vp, D, W, maxv):
        pr = T.prune_verify(tree, tree.prob, dp, vp, D, W, maxv)
        return pr.tree, pr.tree, pr.kept

    def as_oracle(self, tree):
        return tree

    def walk(self, vtree_native, am):
        return T.greedy_walk(vtree_native, am)


class RefSpecDecoder:
    def __init__(self, target: RefLlama, draft: RefLlama, depth: int, width: int, k: int, max_verify: int,
                 drafter_profile, verifier_profile, S: int, fixed_verify: int = 0, tree_ops=None):
        self.ops = tree_ops if tree_ops is not None else OracleTreeOps()
        self.t, self.d = target, draft
        self.D, self.W, self.k, self.maxv = depth, width, k, max_verify
        self.dp, self.vp = drafter_profile, verifier_profile
        self.fixed_verify = fixed_verify
        self.S = S
        self.tc = RefCache(target.cfg, S)
        self.dc = RefCache(draft.cfg, S)
        self.hist: list = []
        self.P = 0
        self.trace: list = []

    def prefill(self, prompt: list) -> None:
        P0 = len(prompt)
        vis = causal_visible(P0, self.S)
        pos = list(range(P0))
        lt = self.t.forward(self.tc, prompt, pos, pos, vis)
        self.d.forward(self.dc, prompt, pos, pos, vis)
        self.hist = list(prompt) + [int(torch.argmax(lt[-1]))]
        self.P = P0

    def _draft_rows(self, tokens, pos, slots, visible):
        return self.d.forward(self.dc, tokens, pos, slots, visible)

    def step(self) -> dict:
        P, S = self.P, self.S
        # draft pass 0
        vis = torch.zeros(2, S, dtype=torch.bool)
        vis[0, :P] = True
        vis[1, : P + 1] = True
        lg = self._draft_rows([self.hist[P - 1], self.hist[P]], [P - 1, P], [P - 1, P], vis)
        root = T.topk_softmax(lg[1].numpy(), self.k)[0]
        ops = self.ops
        tree = ops.root(*root)
        stopped = False
        for _ in range(self.D):
            if stopped:
                break
            frontier = ops.frontier(tree)
            info = [ops.node(tree, f) for f in frontier]
            vis = torch.zeros(len(frontier), S, dtype=torch.bool)
            vis[:, : P + 1] = True
            for r, (_, _, path) in enumerate(info):
                for a in path:
                    vis[r, P + 1 + a] = True
            lg = self._draft_rows([tok for tok, _, _ in info], [P + 1 + dep for _, dep, _ in info],
                                  [P + 1 + f for f in frontier], vis)
            cands = {f: T.topk_softmax(lg[r].numpy(), self.k) for r, f in enumerate(frontier)}
            added = ops.grow(tree, cands, self.W, self.k)
            if not added:
                stopped = True
        grown_native = tree
        grown = ops.as_oracle(tree)
        if self.fixed_verify > 0:
            dp = T.Knapsack(grown, T.path_products(grown, grown.prob), self.maxv)
            kk = min(self.fixed_verify, dp.cap)
            keep = dp.pick(kk)
            vtree, _ = grown.subtree(keep)
            vnative = vtree
            kept = tuple(sorted(keep))
            walk = T.greedy_walk
        else:
            vnative, vtree, kept = ops.prune(grown_native, self.dp, self.vp, self.D, self.W, self.maxv)
            walk = ops.walk
        # verify
        n = len(vtree)
        tokens = [self.hist[P]] + vtree.token
        pos = [P] + [P + 1 + dd for dd in vtree.depth]
        slots = [P + i for i in range(n + 1)]
        vis = torch.zeros(n + 1, S, dtype=torch.bool)
        vis[:, :P + 1] = True
        for i in range(n):
            for a in vtree.path(i):
                vis[1 + i, P + 1 + a] = True
        lt = self.t.forward(self.tc, tokens, pos, slots, vis)
        am = torch.argmax(lt, dim=-1).tolist()
        path, bonus = walk(vnative, am)
        a = len(path)
        # compaction: target (verify order), draft (grown order, leaves at depth D never drafted)
        self.tc.move([P + 1 + p for p in path], [P + 1 + i for i in range(a)])
        src, dst = [], []
        for i, p in enumerate(path):
            g = kept[p]
            if grown.depth[g] < self.D:
                src.append(P + 1 + g)
                dst.append(P + 1 + i)
        self.dc.move(src, dst)
        acc_tokens = [vtree.token[p] for p in path]
        self.hist = self.hist[: P + 1] + acc_tokens + [bonus]
        self.P = P + 1 + a
        rec = {"tree": grown.to_dict(), "vtree": vtree.to_dict(), "kept": list(kept), "path": path,
               "bonus": bonus, "accepted_len": a + 1, "argmax": am}
        self.trace.append(rec)
        return rec

    def generate(self, prompt: list, n_tokens: int) -> list:
        self.prefill(prompt)
        P0 = len(prompt)
        while len(self.hist) - P0 < n_tokens:
            self.step()
        return self.hist[P0 : P0 + n_tokens]
