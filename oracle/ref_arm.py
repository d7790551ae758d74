"""The reference arm of bench.py: one speculative step per iteration, entirely on the host CPU.

Test / baseline infrastructure only (imported by tests/ and by bench.py's reference and
cpu_baseline legs; never by the product package).

* Tree logic (EGT growth, knapsack prune with the Eq.3 objective, acceptance walk) is the
  reference's OWN code: ``specsim`` installed unmodified into ``baseline/_ref`` (``pip install
  --no-index --no-deps --target baseline/_ref /root/reference/pkg``, recipe in DESIGN.md §7),
  called through its public API — ``TokenTree``, ``grow_step`` (egt.py:83-114), ``prune_verify``
  with ``SurrogateAcceptance`` (egt.py:232-282), ``sample_with_probs`` (acceptance.py:221-241)
  with the greedy 0/1 node probabilities.  When ``baseline/_ref`` is absent the oracle
  restatement (``tree_ref``) stands in and the line says so.
* Model arithmetic (the reference has none: it prices forwards with ``latency_at``,
  simulator.py:202-214) is the torch-CPU fp32 oracle port (``llama_ref``) on every host thread.
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

from . import tree_ref as T
from .spec_ref import OracleTreeOps, RefSpecDecoder

ROOT = Path(__file__).resolve().parents[1]
REF_DIR = ROOT / "baseline" / "_ref"


def load_specsim():
    """The reference package from baseline/_ref, or None when it was not installed."""
    if REF_DIR.exists() and str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    try:
        import specsim.acceptance  # noqa: F401
        import specsim.egt  # noqa: F401
        import specsim.latency  # noqa: F401
        import specsim.token_tree  # noqa: F401
    except ImportError:
        return None
    import specsim

    return specsim


class _Timed:
    """Accumulates the wall time spent inside the tree-logic calls of one run."""

    def __init__(self):
        self.seconds = 0.0

    def __call__(self, fn, *a):
        t0 = time.perf_counter()
        try:
            return fn(*a)
        finally:
            self.seconds += time.perf_counter() - t0


class SpecsimTreeOps:
    """Tree logic of the step through the reference package's public API."""

    name = "specsim"

    def __init__(self, specsim, drafter_bp, verifier_bp, timer: _Timed | None = None):
        from specsim.acceptance import SurrogateAcceptance, sample_with_probs
        from specsim.egt import grow_step, prune_verify
        from specsim.latency import LatencyProfile, ProfilePair
        from specsim.token_tree import TokenTree

        self._TokenTree, self._grow_step, self._prune = TokenTree, grow_step, prune_verify
        self._walk, self._model = sample_with_probs, SurrogateAcceptance()
        self._profiles = ProfilePair(drafter=LatencyProfile(tuple(drafter_bp), "drafter"),
                                     verifier=LatencyProfile(tuple(verifier_bp), "verifier"))
        self._rng = np.random.default_rng(0)
        self.timer = timer or _Timed()

    def root(self, tok, prob):
        return self.timer(self._TokenTree, tok, prob)

    def frontier(self, tree):
        return tree.levels[-1]

    def node(self, tree, i):
        nd = tree.nodes[i]
        return nd.token, nd.depth, tree.path_to_root(i)

    def grow(self, tree, cands, W, k):
        class Drafter:  # DrafterDistribution (egt.py:52-62) over this level's model candidates
            def root(self):
                raise NotImplementedError

            def candidates(self, tr, node, kk):
                return cands[node]

        return self.timer(self._grow_step, tree, Drafter(), W, k)

    @staticmethod
    def _to_oracle(tree) -> T.Tree:
        out = T.Tree([], [], [], [])
        for nd in tree.nodes:
            out.token.append(nd.token)
            out.parent.append(nd.parent)
            out.prob.append(nd.surrogate_prob)
            out.depth.append(nd.depth)
        return out

    def as_oracle(self, tree):
        return self._to_oracle(tree)

    def prune(self, tree, dp, vp, D, W, maxv):
        pr = self.timer(self._prune, tree, self._model, self._profiles, D, W, maxv)
        return pr.tree, self._to_oracle(pr.tree), pr.kept

    def walk(self, vtree, am):
        def run():
            # greedy realisation of the walk: node prob = 1 iff its token is the target argmax at its
            # parent's verify row (row 0 = the confirmed token, row 1 + i = node i)
            probs = np.empty(len(vtree), dtype=np.float64)
            for i, nd in enumerate(vtree.nodes):
                row = 0 if nd.parent is None else 1 + nd.parent
                probs[i] = 1.0 if nd.token == am[row] else 0.0
            out = self._walk(vtree, probs, self._rng)
            stop = 0 if not out.accepted_path else 1 + out.accepted_path[-1]
            return list(out.accepted_path), int(am[stop])

        return self.timer(run)


def tree_ops_for(drafter_bp, verifier_bp):
    """(ops, timer, kind): the reference's specsim when installed, else the oracle restatement."""
    timer = _Timed()
    ss = load_specsim()
    if ss is not None:
        return SpecsimTreeOps(ss, drafter_bp, verifier_bp, timer), timer, "specsim"

    class Ops(OracleTreeOps):
        def grow(self, tree, cands, W, k):
            return timer(super().grow, tree, cands, W, k)

        def prune(self, tree, dp, vp, D, W, maxv):
            return timer(super().prune, tree, dp, vp, D, W, maxv)

        def walk(self, vtree, am):
            return timer(super().walk, vtree, am)

    return Ops(), timer, "oracle"


def host_info() -> dict:
    model = ""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "cpu_count": os.cpu_count()}


def run_host_steps(wl: dict, coupling: dict, steps: int, warmup: int, drafter_bp, verifier_bp,
                   n_layers: tuple | None = None, seed: int = 0) -> dict:
    """Build the workload's target / draft as fp32 CPU models (coupled random-init weights from CPU
    generators), prefill a seeded random prompt, run ``warmup`` then ``steps`` timed speculative
    steps, and return tokens/s, p50 step time, the measured AAL and the tree-logic share."""
    import torch

    from paper_2512_23858_b200.model import Coupling, init_weights, preset

    from .llama_ref import RefLlama

    torch.set_num_threads(os.cpu_count() or 1)
    tl, dl = n_layers if n_layers else (None, None)
    tcfg = preset(wl["target"], **({"n_layers": tl} if tl else {}))
    dcfg = preset(wl["draft"], **({"n_layers": dl} if dl else {}))
    cp = Coupling(**coupling)
    t0 = time.perf_counter()
    target = RefLlama(tcfg, init_weights(tcfg, seed, torch.float32, "cpu", cp))
    draft = RefLlama(dcfg, init_weights(dcfg, seed + 1, torch.float32, "cpu", cp))
    init_s = time.perf_counter() - t0
    D, W, k = wl["depth"], wl["width"], wl["k"]
    P0 = wl["prompt"]
    S = P0 + (steps + warmup) * (D + 2) + 1 + D * W + 16
    ops, timer, kind = tree_ops_for(drafter_bp, verifier_bp)
    dec = RefSpecDecoder(target, draft, D, W, k, wl["max_verify"], T.Profile(tuple(drafter_bp)),
                         T.Profile(tuple(verifier_bp)), S, tree_ops=ops)
    g = torch.Generator().manual_seed(1000)
    prompt = torch.randint(0, tcfg.vocab, (P0,), generator=g).tolist()
    t0 = time.perf_counter()
    dec.prefill(prompt)
    prefill_s = time.perf_counter() - t0
    for _ in range(warmup):
        dec.step()
    # the timed window is the first `steps` steps after a fresh prefill of the same prompt, as in the
    # GPU arm (bench.py run_ours), so both arms decode the same tokens
    dec.prefill(prompt)
    timer.seconds = 0.0
    times, acc = [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        rec = dec.step()
        times.append(time.perf_counter() - t0)
        acc.append(rec["accepted_len"])
    total = sum(times)
    return {"tokens_per_s": sum(acc) / total, "ms_per_step": 1e3 * total / steps,
            "p50_step_ms": 1e3 * float(np.median(times)), "aal": sum(acc) / steps,
            "tree_logic_ms_per_step": 1e3 * timer.seconds / steps, "tree_impl": kind,
            "threads": torch.get_num_threads(), "init_s": round(init_s, 1), "prefill_s": round(prefill_s, 2),
            "target_layers": tcfg.n_layers, "draft_layers": dcfg.n_layers}
