"""Generate the golden vectors that pin the oracle (and the host scheduler) to the reference.

Run in the build container, where the read-only reference is importable:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py /root/reference/pkg/src

It imports the reference ``specsim`` package and records its outputs on seeded random inputs
(plus the reference's own known-answer cases) as JSON under tests/golden/.  Floats are stored
as ``float.hex`` strings so comparisons are bit-exact.  Nothing under tests/ reads
/root/reference at test time; only this script does, and its outputs are committed.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent


def hx(x: float) -> str:
    return float(x).hex()


def tree_dict(tree) -> dict:
    return {"nodes": [{"token": n["token"], "parent": n["parent"], "prob": hx(n["prob"])}
                      for n in tree.to_dict()["nodes"]]}


def random_tree(S, rng, max_nodes=40):
    t = S.token_tree.new_tree(prob=float(rng.uniform(0.1, 1.0)))
    for i in range(int(rng.integers(0, max_nodes))):
        p = int(rng.integers(0, len(t)))
        room = 1.0 - sum(t.nodes[c].surrogate_prob for c in t.children(p))
        if room <= 0.02:
            continue
        t.add_child(p, token=i + 1, prob=float(rng.uniform(0.01, 0.9)) * room)
    return t


def random_profile(rng):
    n = int(rng.integers(2, 6))
    ws = sorted(set(int(x) for x in rng.integers(1, 200, size=n)))
    if len(ws) < 2:
        ws = [1, 64]
    lat = np.cumsum(rng.uniform(0, 60, size=len(ws))) + rng.uniform(1, 80)
    return [[w, float(l)] for w, l in zip(ws, lat)]


def main(src: str) -> None:
    sys.path.insert(0, src)
    import specsim  # noqa: F401
    from specsim import acceptance, egt, latency, scheduler, simulator, token_tree
    from specsim.config import load_config

    class S:
        pass

    S.token_tree = token_tree
    rng = np.random.default_rng(20251223)
    golden: dict = {"source": "reference specsim (pkg/src/specsim) imported read-only", "numpy": np.__version__}

    # ---- build_mask (token_tree.py:205-218)
    masks = []
    for _ in range(30):
        t = random_tree(S, rng, 50)
        m = token_tree.build_mask(t)
        masks.append({"tree": tree_dict(t), "rows": ["".join("1" if v else "0" for v in row) for row in m]})
    golden["mask"] = masks

    # ---- grow_step / grow_egt with list drafters (egt.py:83-147), incl. exact score ties
    class ListDrafter:
        def __init__(self, table, root=(0, 1.0)):
            self.table, self._root = table, root

        def root(self):
            return self._root

        def candidates(self, tree, node, k):
            return self.table.get(node, [])[:k]

    grows = []
    for case in range(40):
        w = int(rng.integers(1, 9))
        k = int(rng.integers(1, 9))
        depth = int(rng.integers(1, 6))
        root = (int(rng.integers(0, 50)), float(rng.uniform(0.3, 1.0)))
        table = {}
        for node in range(1 + depth * w):
            cnt = int(rng.integers(0, k + 2))
            ps = np.sort(rng.dirichlet(np.ones(cnt + 1))[:cnt])[::-1] if cnt else np.array([])
            if cnt >= 2 and case % 3 == 0:
                ps = ps * 0.5
                ps[1] = ps[0]
            toks = rng.choice(1000, size=cnt, replace=False)
            table[node] = [(int(a), float(b)) for a, b in zip(toks, ps)]
        d = ListDrafter(table, root)
        t = token_tree.new_tree(*root)
        res = egt.grow_egt(t, d, depth, w, k)
        grows.append({"root": [root[0], hx(root[1])], "w": w, "k": k, "depth": depth,
                      "table": {str(n): [[a, hx(b)] for a, b in v] for n, v in table.items()},
                      "tree": tree_dict(res.tree), "shortfall": res.shortfall})
    golden["grow"] = grows

    # ---- knapsack + prune_verify (egt.py:150-282)
    prunes = []
    for case in range(60):
        t = random_tree(S, rng, 70 if case % 2 else 14)
        probs = np.array([n.surrogate_prob for n in t.nodes]) * float(rng.uniform(0.5, 1.0))
        model = acceptance.ExplicitAcceptance({i: float(p) for i, p in enumerate(probs)})
        dprof, vprof = random_profile(rng), random_profile(rng)
        pp = latency.ProfilePair(latency.LatencyProfile(tuple(map(tuple, dprof)), "drafter"),
                                 latency.LatencyProfile(tuple(map(tuple, vprof)), "verifier"))
        d_draft, w_draft = 8, 8
        maxv = int(rng.integers(1, 48))
        pr = egt.prune_verify(t, model, pp, d_draft, w_draft, maxv)
        dp = egt.SubtreeKnapsack(t, acceptance.path_products(t, probs), maxv)
        prunes.append({"tree": tree_dict(t), "probs": [hx(p) for p in probs], "drafter": dprof, "verifier": vprof,
                       "d_draft": d_draft, "w_draft": w_draft, "max_verify": maxv, "kept": list(pr.kept),
                       "w_verify": pr.w_verify, "expected_aal": hx(pr.expected_aal), "speedup": hx(pr.speedup),
                       "root_row": [hx(x) for x in dp.best_row(0)], "pruned": tree_dict(pr.tree)})
    golden["prune"] = prunes

    # ---- acceptance walk (acceptance.py:221-241)
    walks = []
    for case in range(60):
        t = random_tree(S, rng, 40)
        probs = np.array([n.surrogate_prob for n in t.nodes])
        seed = int(rng.integers(0, 2**31))
        draws = np.random.default_rng(seed).random(64)
        out = acceptance.sample_with_probs(t, probs, np.random.default_rng(seed))
        walks.append({"tree": tree_dict(t), "probs": [hx(p) for p in probs], "seed": seed,
                      "draws": [hx(x) for x in draws], "path": out.accepted_path, "accepted_len": out.accepted_len})
    golden["walk"] = walks

    # ---- latency_at / tree_speedup (latency.py:68-82, 154-161)
    lats = []
    for _ in range(40):
        prof = random_profile(rng)
        lp = latency.LatencyProfile(tuple(map(tuple, prof)), "verifier")
        widths = sorted(set(int(x) for x in rng.integers(1, 260, size=12)))
        lats.append({"profile": prof, "widths": widths, "latency": [hx(latency.latency_at(lp, w)) for w in widths]})
    golden["latency"] = lats

    # ---- select_width with the reference's geometric drafter (egt.py:285-318)
    from specsim.drafters import GeometricDrafter

    widths_cases = []
    for _ in range(20):
        gd = GeometricDrafter(float(rng.uniform(0.5, 1.0)), float(rng.uniform(0.5, 1.0)),
                              fanout=int(rng.integers(1, 17)), top_share=float(rng.uniform(0.2, 0.8)))
        dprof, vprof = random_profile(rng), random_profile(rng)
        pp = latency.ProfilePair(latency.LatencyProfile(tuple(map(tuple, dprof)), "drafter"),
                                 latency.LatencyProfile(tuple(map(tuple, vprof)), "verifier"))
        cfg = egt.EgtConfig(candidate_widths=(1, 2, 4, 8, 16), max_depth=16, max_verify=64,
                            expansion_k=int(rng.integers(4, 17)))
        depth = int(rng.integers(1, 9))
        wsel = egt.select_width(cfg, depth, gd, pp)
        cand = {str(dd): [[t_, hx(p_)] for t_, p_ in gd.candidates(_depth_tree(token_tree, dd), dd, cfg.expansion_k)]
                for dd in range(0, depth + 1)}
        widths_cases.append({"drafter": [gd.top_mass, gd.decay, gd.fanout, gd.top_share],
                             "root": [gd.root()[0], hx(gd.root()[1])], "cands_by_parent_depth": cand,
                             "drafter_prof": dprof, "verifier_prof": vprof, "k": cfg.expansion_k,
                             "widths": list(cfg.candidate_widths), "depth": depth, "max_verify": 64, "width": wsel})
    golden["select_width"] = widths_cases

    # ---- plan_search (scheduler.py:445-485)
    plans = []
    for case in range(24):
        rows = {("Verify", "base"): float(rng.uniform(20, 200)), ("Accept", "base"): float(rng.uniform(0, 80)),
                ("BonusSample", "base"): float(rng.uniform(0, 20)), ("TailDraft", "base"): float(rng.uniform(0, 40)),
                ("HeadDraft", "base"): float(rng.uniform(5, 60)), ("DraftStep", "base"): float(rng.uniform(5, 50)),
                ("PrepareVerify", "base"): float(rng.uniform(0, 20))}
        if case % 4 == 0:
            rows[("HeadDraft", "aot")] = float(rng.uniform(10, 120))
        sp = scheduler.StageProfiles(rows)
        depth = int(rng.integers(1, 9))
        width = int(rng.integers(1, 9))
        shape = latency.TreeShape(w_draft=width, d_draft=depth, w_verify=1)
        aal = float(rng.uniform(1.0, 5.0))
        res = scheduler.plan_search(sp, shape, aal)
        plans.append({"rows": [[s, v, hx(x)] for (s, v), x in rows.items()], "depth": depth, "width": width,
                      "aal": hx(aal), "transforms": list(res.plan.transforms), "priority": list(res.plan.priority),
                      "makespan": hx(res.makespan_us), "per_token": hx(res.per_token_us),
                      "timeline": {k: [hx(a), hx(b)] for k, (a, b) in res.timeline.entries.items()}})
    golden["plan_search"] = plans

    # ---- simulator run on the reference's example config (simulator.py:298-349)
    cfg = load_config(str(Path(src).parent / "docs" / "example_config.json"))
    stats = simulator.run(cfg)
    golden["simulate_example"] = {
        "aal": hx(stats.aal), "step_latency_us": hx(stats.step_latency_us), "tpot_us": hx(stats.tpot_us),
        "speedup": hx(stats.speedup),
        "trace": [[r.iteration, r.d_draft, r.tree_size, r.w_verify, r.accepted_len, hx(r.step_us)]
                  for r in stats.trace[:128]],
    }
    # ---- depth predictor training (depth_predictor.py:149-344) on the reference's own profiling
    # samples (collect_depth_samples, simulator.py:553-579) of the example config
    from specsim import depth_predictor as dp

    samples = simulator.collect_depth_samples(cfg, 160, probe_depth=8)
    runs = []
    for tc in (dp.TrainConfig(epochs=40), dp.TrainConfig(hidden=8, epochs=25, batch_size=16, seed=3, max_depth=12)):
        res = dp.train_predictor(samples, tc)
        pr = res.predictor
        runs.append({"config": {"hidden": tc.hidden, "epochs": tc.epochs, "batch_size": tc.batch_size,
                                "seed": tc.seed, "max_depth": tc.max_depth, "learning_rate": hx(tc.learning_rate),
                                "head_depths": list(tc.head_depths)},
                     "w1": [[hx(v) for v in row] for row in pr.w1], "b1": [hx(v) for v in pr.b1],
                     "w2": [[hx(v) for v in row] for row in pr.w2], "b2": [hx(v) for v in pr.b2],
                     "mean": [hx(v) for v in pr.feature_mean], "std": [hx(v) for v in pr.feature_std],
                     "initial_loss": hx(res.initial_loss), "final_loss": hx(res.final_loss),
                     "predictions": [pr.predict(s.features) for s in samples],
                     "heads0": {str(k): hx(v) for k, v in pr.head_outputs(samples[0].features).items()}})
    golden["depth_predictor"] = {"samples": [[[hx(v) for v in s.features], s.realized_len] for s in samples],
                                 "runs": runs}
    for name, val in golden.items():
        if isinstance(val, (list, dict)) and name not in ("source", "numpy"):
            (OUT / f"{name}.json").write_text(json.dumps(val, indent=None, sort_keys=True) + "\n")
    (OUT / "MANIFEST.json").write_text(json.dumps({k: (len(v) if isinstance(v, list) else 1)
                                                   for k, v in golden.items() if k not in ("source", "numpy")},
                                                  indent=1) + "\n")
    print("wrote", sorted(golden))


def _depth_tree(token_tree, depth):
    """A chain of the given depth whose last node has depth ``depth`` (geometric candidates depend
    only on the parent's depth)."""
    t = token_tree.new_tree(1, 1.0)
    for _ in range(depth):
        t.add_child(len(t) - 1, 1, 0.0)
    return t


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")
