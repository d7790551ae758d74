"""Runtime shape control (paper_2512_23858_b200/runtime.py) and calibrated acceptance.

* Switching the EGT shape between steps over one shared decoding state keeps greedy speculative
  decoding lossless: the output equals bf16 greedy AR through the same target kernels, for the
  bandit policy (forced heavy switching) and for the reference's EmaHeuristic depth predictor.
* ygg_accept_stats counts exactly the tested / accepted verify nodes per grown-tree position.
* The calibrated node table changes only the prune objective: the output stays lossless.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

DRAFT_PROF = ((1, 20.0), (64, 30.0), (128, 60.0))
VERIFY_PROF = ((1, 100.0), (64, 110.0), (128, 200.0))


def _profiles():
    from oracle.tree_ref import Profile

    class PP:
        drafter = Profile(DRAFT_PROF)
        verifier = Profile(VERIFY_PROF)

    return PP


def _models(cuda):
    from paper_2512_23858_b200.model import Coupling, init_weights, preset, weights_to

    tc, dc = preset("tiny-target"), preset("tiny-draft")
    cp = Coupling(rank=256, logit_scale=8.0, head_noise=2.0, layer_gain=2.0)
    tw = weights_to(init_weights(tc, 0, torch.float32, "cpu", cp), cuda, torch.bfloat16)
    dw = weights_to(init_weights(dc, 1, torch.float32, "cpu", cp), cuda, torch.bfloat16)
    return tc, dc, tw, dw


def _prompts(vocab, B=1):
    return torch.stack([torch.randint(0, vocab, (24,), generator=torch.Generator().manual_seed(1000 + b))
                        for b in range(B)])


SHAPES = [(2, 2, 16), (4, 4, 64), (3, 8, 16), (6, 4, 64)]


def assert_lossless(got, ar, tc, tw, prompts, plan=None):
    """got == ar, except that the sequences may part at a bf16 near-tie of the target (top-2 logits
    within 1e-3 of the logit scale, where kernel families with different reduction orders may pick
    either token); before the first difference they must agree token for token."""
    from paper_2512_23858_b200.forward import Forward, new_cache

    for b, (g, a) in enumerate(zip(got, ar)):
        i = next((j for j, (x, y) in enumerate(zip(g, a)) if x != y), None)
        if i is None:
            continue
        seq = prompts[b].tolist() + a[:i]
        n = len(seq)
        dev = tw["embed"].device
        f = Forward(tc, tw, new_cache(tc, 1, n + 8, torch.bfloat16, dev), 1, n, 0, torch.bfloat16, plan=plan)
        f.tokens.copy_(torch.tensor(seq, dtype=torch.int32))
        pos = torch.arange(n, dtype=torch.int32)
        f.pos.copy_(pos)
        f.slot.copy_(pos)
        f.blk_start.zero_()
        f.blk_len.fill_(n)
        f.run()
        torch.cuda.synchronize()
        row = f.logits[n - 1].float().cpu()
        top = row.topk(2).values
        assert float(top[0] - top[1]) <= 1e-3 * float(row.abs().max()), (b, i, top.tolist())
        assert {g[i], a[i]} <= set(row.topk(2).indices.tolist()), (b, i)


@pytest.mark.parametrize("policy", ["bandit", "predictor"])
@pytest.mark.parametrize("B", [1, 2])
def test_shape_switching_is_lossless(policy, B, cuda):
    from paper_2512_23858_b200.engine import ARDecoder, StepShape
    from paper_2512_23858_b200.plan import ForwardPlan
    from paper_2512_23858_b200.plugins import EmaHeuristic
    from paper_2512_23858_b200.runtime import AdaptiveDecoder

    tc, dc, tw, dw = _models(cuda)
    prompts = _prompts(tc.vocab, B)
    n_tok = 64
    # one attention reduction structure for every row count (verify shapes and AR): the identity is then
    # exact, not only up to bf16 near-ties (at the 8B dims the automatic split already coincides)
    plan = ForwardPlan(attn_ksplit=2)
    ar = ARDecoder(tc, tw, batch=B, max_seq=256, plan=plan).generate(prompts, n_tok)
    shapes = [StepShape(d, w, 8, v) for d, w, v in SHAPES]
    pred = EmaHeuristic(window=2, alpha=0.4, max_depth=8) if policy == "predictor" else None
    ad = AdaptiveDecoder(tc, tw, dc, dw, shapes, batch=B, max_seq=256, profiles=_profiles(), policy=policy,
                         predictor=pred, calibrate=True, refresh=4, explore_share=0.5, seed=3, plan=plan)
    got, steps = ad.generate(prompts, n_tok)
    assert_lossless(got, ar, tc, tw, prompts, plan)
    used = set(ad.trace.chosen)
    assert len(used) >= 3, used  # the run really switched shapes
    summ = ad.summary()
    assert sum(s["steps"] for s in summ["shapes"]) == steps


def test_accept_stats_counts_tested_nodes(cuda):
    from oracle import tree_ref as T
    from paper_2512_23858_b200 import _lib as L
    from paper_2512_23858_b200.device_tree import DeviceTrees

    rng = np.random.default_rng(11)
    B, cap = 3, 40
    trees, paths, keeps = [], [], []
    for _ in range(B):
        t = T.Tree.root(0, 0.9)
        for i in range(int(rng.integers(5, cap - 1))):
            t.add(int(rng.integers(0, len(t))), i + 1, 0.01)
        trees.append(t)
        # a random root-anchored accepted path
        path, cur = [0], 0
        while True:
            ch = t.children(cur)
            if not ch or rng.random() < 0.3:
                break
            cur = int(rng.choice(ch))
            path.append(cur)
        if rng.random() < 0.2:
            path = []
        paths.append(path)
        keeps.append(sorted(rng.choice(100, size=len(t), replace=False).tolist()))  # grown indices
    dt = DeviceTrees(B, cap, cuda)
    dt.load_host([t.to_dict() for t in trees])
    i32 = dict(dtype=torch.int32, device=cuda)
    keep = torch.full((B, 100), -1, **i32)
    pth = torch.full((B, cap), -1, **i32)
    plen = torch.zeros(B, **i32)
    for b in range(B):
        keep[b, : len(keeps[b])] = torch.tensor(keeps[b])
        pth[b, : len(paths[b])] = torch.tensor(paths[b], dtype=torch.int32)
        plen[b] = len(paths[b])
    counts = torch.zeros(100, 2, **i32)
    L.check(L.lib().ygg_accept_stats(dt.struct, keep.data_ptr(), 100, pth.data_ptr(), plen.data_ptr(),
                                     counts.data_ptr(), L.stream_ptr()))
    torch.cuda.synchronize()
    want = np.zeros((100, 2), dtype=np.int64)
    for b, t in enumerate(trees):
        on = set(paths[b])
        for j in range(len(t)):
            p = t.parent[j]
            if p is not None and p not in on:
                continue
            want[keeps[b][j], 0] += 1
            want[keeps[b][j], 1] += int(j in on)
    np.testing.assert_array_equal(counts.cpu().numpy(), want)


def test_calibrated_objective_stays_lossless_and_rates_are_probabilities(cuda):
    from paper_2512_23858_b200.engine import ARDecoder, SpecDecoder, StepShape

    tc, dc, tw, dw = _models(cuda)
    prompts = _prompts(tc.vocab)
    n_tok = 64
    ar = ARDecoder(tc, tw, batch=1, max_seq=256).generate(prompts, n_tok)
    sd = SpecDecoder(tc, tw, dc, dw, StepShape(4, 4, 8, 12), batch=1, max_seq=256, profiles=_profiles(),
                     calibrate=True)
    sd.prefill_len = prompts.shape[1]
    sd.prefill(prompts)
    sd.capture()
    for i in range(40):
        sd.step()
        if i % 8 == 7:
            rates = sd.node_rates()
            known = rates[rates >= 0]
            assert known.size >= 1 and np.all(known <= 1.0)
            sd.set_node_table(rates)
    torch.cuda.synchronize()
    c = sd.accept_counts.cpu().numpy()
    assert c[0, 0] == 40 and np.all(c[:, 1] <= c[:, 0])  # the root is tested every step
    assert_lossless([sd.generated(0)[:n_tok]], [ar[0][: min(n_tok, len(sd.generated(0)))]], tc, tw, prompts)


def test_continuous_batching_serves_queue_losslessly(cuda):
    """ServingEngine: 6 requests with different prompt lengths and token budgets through 2 slots; each
    request's output equals greedy AR of that request alone (up to bf16 near-ties)."""
    from paper_2512_23858_b200.engine import ARDecoder, SpecDecoder, StepShape
    from paper_2512_23858_b200.plan import ForwardPlan
    from paper_2512_23858_b200.runtime import ServingEngine

    tc, dc, tw, dw = _models(cuda)
    plan = ForwardPlan(attn_ksplit=2)
    reqs = [(20, 30), (37, 16), (64, 40), (9, 25), (50, 12), (33, 33)]
    prompts = [torch.randint(0, tc.vocab, (n,), generator=torch.Generator().manual_seed(500 + i))
               for i, (n, _) in enumerate(reqs)]
    sd = SpecDecoder(tc, tw, dc, dw, StepShape(4, 4, 8, 64), batch=2, max_seq=192, profiles=_profiles(), plan=plan)
    eng = ServingEngine(sd, poll=2)
    ids = [eng.submit(p, n) for p, (_, n) in zip(prompts, reqs)]
    out = eng.run()
    assert sorted(out) == ids
    for rid, p, (_, n) in zip(ids, prompts, reqs):
        ar = ARDecoder(tc, tw, batch=1, max_seq=192, plan=plan).generate(p[None], n)
        assert len(out[rid]) == n
        assert_lossless([out[rid]], ar, tc, tw, p[None], plan)


@pytest.mark.parametrize("use_graph", [False, True])
def test_two_lane_step_is_lossless(use_graph, cuda):
    """The deferred target KV compaction on a side stream (overlap_compaction) keeps spec == AR."""
    from paper_2512_23858_b200.engine import ARDecoder, SpecDecoder, StepShape
    from paper_2512_23858_b200.plan import ForwardPlan

    tc, dc, tw, dw = _models(cuda)
    plan = ForwardPlan(attn_ksplit=2)
    prompts = _prompts(tc.vocab, 2)
    ar = ARDecoder(tc, tw, batch=2, max_seq=256, plan=plan).generate(prompts, 64)
    sd = SpecDecoder(tc, tw, dc, dw, StepShape(4, 4, 8, 64), batch=2, max_seq=256, profiles=_profiles(), plan=plan,
                     overlap_compaction=True)
    got, _ = sd.generate(prompts, 64, use_graph=use_graph)
    assert_lossless(got, ar, tc, tw, prompts, plan)
