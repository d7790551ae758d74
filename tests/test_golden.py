"""CPU: the oracle restatement and the host-side scheduler reproduce the reference's own outputs.

The vectors in tests/golden/*.json were produced by importing the reference ``specsim``
(tests/golden/make_golden.py); floats are compared bit-exactly via float.hex.
"""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import tree_ref as T

G = Path(__file__).resolve().parent / "golden"


def load(name):
    return json.loads((G / f"{name}.json").read_text())


def fx(s):
    return float.fromhex(s)


def tree_of(d):
    nodes = [{"token": n["token"], "parent": n["parent"], "prob": fx(n["prob"])} for n in d["nodes"]]
    return T.Tree.from_dict({"nodes": nodes})


def as_plain(d):
    return {"nodes": [{"token": n["token"], "parent": n["parent"], "prob": fx(n["prob"])} for n in d["nodes"]]}


def test_manifest_counts():
    man = json.loads((G / "MANIFEST.json").read_text())
    for k, v in man.items():
        data = load(k)
        assert (len(data) if isinstance(data, list) else 1) == v


@pytest.mark.parametrize("i", range(30))
def test_build_mask(i):
    case = load("mask")[i]
    m = T.build_mask(tree_of(case["tree"]))
    assert ["".join("1" if v else "0" for v in row) for row in m] == case["rows"]


@pytest.mark.parametrize("i", range(40))
def test_grow_egt(i):
    case = load("grow")[i]
    table = {int(k): [(t, fx(p)) for t, p in v] for k, v in case["table"].items()}
    tree = T.Tree.root(case["root"][0], fx(case["root"][1]))
    short = T.grow_egt(tree, lambda tr, n, k: table.get(n, [])[:k], case["depth"], case["w"], case["k"])
    assert tree.to_dict() == as_plain(case["tree"])
    assert short == case["shortfall"]


@pytest.mark.parametrize("i", range(60))
def test_prune_verify(i):
    case = load("prune")[i]
    tree = tree_of(case["tree"])
    probs = [fx(p) for p in case["probs"]]
    dprof = T.Profile(tuple(map(tuple, case["drafter"])))
    vprof = T.Profile(tuple(map(tuple, case["verifier"])))
    pr = T.prune_verify(tree, probs, dprof, vprof, case["d_draft"], case["w_draft"], case["max_verify"])
    assert list(pr.kept) == case["kept"]
    assert pr.w_verify == case["w_verify"]
    assert pr.expected_aal == fx(case["expected_aal"])
    assert pr.speedup == fx(case["speedup"])
    assert pr.tree.to_dict() == as_plain(case["pruned"])
    dp = T.Knapsack(tree, T.path_products(tree, probs), case["max_verify"])
    assert [x for x in dp.best[0]] == [fx(x) for x in case["root_row"]]


@pytest.mark.parametrize("i", range(60))
def test_sample_with_probs(i):
    case = load("walk")[i]
    tree = tree_of(case["tree"])
    draws = np.random.default_rng(case["seed"]).random(64)
    assert [x.hex() for x in draws] == case["draws"]  # numpy PCG64 stream unchanged
    path, length, _ = T.sample_with_probs(tree, [fx(p) for p in case["probs"]], iter(draws.tolist()))
    assert path == case["path"] and length == case["accepted_len"]


@pytest.mark.parametrize("i", range(40))
def test_latency_at(i):
    from paper_2512_23858_b200.latency import LatencyProfile, latency_at

    case = load("latency")[i]
    prof = tuple(map(tuple, case["profile"]))
    host = LatencyProfile(prof, "verifier")
    for w, want in zip(case["widths"], case["latency"]):
        assert T.latency_at(T.Profile(prof), w) == fx(want)
        assert latency_at(host, w) == fx(want)


@pytest.mark.parametrize("i", range(20))
def test_select_width(i):
    case = load("select_width")[i]
    cands = {int(k): [(t, fx(p)) for t, p in v] for k, v in case["cands_by_parent_depth"].items()}
    root = (case["root"][0], fx(case["root"][1]))
    w = T.select_width(case["widths"], case["depth"], root, lambda tr, n, k: cands[tr.depth[n]][:k], case["k"],
                       case["max_verify"], T.Profile(tuple(map(tuple, case["drafter_prof"]))),
                       T.Profile(tuple(map(tuple, case["verifier_prof"]))))
    assert w == case["width"]


@pytest.mark.parametrize("i", range(24))
def test_plan_search_host(i):
    """The product's host scheduler (offline per shape) against the reference."""
    from paper_2512_23858_b200.latency import TreeShape
    from paper_2512_23858_b200.scheduler import StageProfiles, plan_search

    case = load("plan_search")[i]
    rows = {(s, v): fx(x) for s, v, x in case["rows"]}
    res = plan_search(StageProfiles(rows), TreeShape(case["width"], case["depth"], 1), fx(case["aal"]))
    assert list(res.plan.transforms) == case["transforms"]
    assert list(res.plan.priority) == case["priority"]
    assert res.makespan_us == fx(case["makespan"])
    assert res.per_token_us == fx(case["per_token"])
    assert {k: [fx(a), fx(b)] for k, (a, b) in [(k, v) for k, v in case["timeline"].items()]} == {
        k: list(v) for k, v in res.timeline.entries.items()}


def test_depth_predictor_training_matches_reference():
    """train_predictor / MlpPredictor (depth_predictor.py:149-344) on the reference's own profiling
    samples: bit-identical weights, losses, head outputs and per-sample depth choices."""
    from paper_2512_23858_b200.depth_predictor import DepthSample, MlpPredictor, TrainConfig, train_predictor

    g = load("depth_predictor")
    samples = [DepthSample(np.array([fx(v) for v in f]), n) for f, n in g["samples"]]
    for run in g["runs"]:
        c = run["config"]
        tc = TrainConfig(hidden=c["hidden"], epochs=c["epochs"], batch_size=c["batch_size"], seed=c["seed"],
                         max_depth=c["max_depth"], learning_rate=fx(c["learning_rate"]),
                         head_depths=tuple(c["head_depths"]))
        res = train_predictor(samples, tc)
        p = res.predictor
        assert [[v.hex() for v in row] for row in p.w1.tolist()] == run["w1"]
        assert [v.hex() for v in p.b1.tolist()] == run["b1"]
        assert [[v.hex() for v in row] for row in p.w2.tolist()] == run["w2"]
        assert [v.hex() for v in p.b2.tolist()] == run["b2"]
        assert [v.hex() for v in p.feature_mean.tolist()] == run["mean"]
        assert [v.hex() for v in p.feature_std.tolist()] == run["std"]
        assert res.initial_loss.hex() == run["initial_loss"] and res.final_loss.hex() == run["final_loss"]
        assert [p.predict(s.features) for s in samples] == run["predictions"]
        assert {str(k): v.hex() for k, v in p.head_outputs(samples[0].features).items()} == run["heads0"]
        assert MlpPredictor.from_dict(p.to_dict()).to_dict() == p.to_dict()
