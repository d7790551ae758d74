"""End-to-end parity of the speculative step on the GPU.

* fp32 (SIMT GEMM path): every step's grown tree, kept set, accepted path and bonus equal the
  CPU oracle's (oracle/spec_ref.py) on the same seeded weights; the generated sequence equals
  plain greedy AR decoding of the fp32 target on the CPU (the lossless-greedy identity).
* bf16 (tcgen05 path): the generated sequence equals greedy AR decoding of the same bf16 model
  through the same kernels, graph replay equals eager launches, and logits of one verify pass
  match the fp32 CPU oracle within the north-star's 2e-2 relative bound.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu

DRAFT_PROF = ((1, 20.0), (64, 30.0), (128, 60.0))
VERIFY_PROF = ((1, 100.0), (64, 100.0), (128, 200.0))


def _profiles():
    from oracle.tree_ref import Profile

    class PP:
        drafter = Profile(DRAFT_PROF)
        verifier = Profile(VERIFY_PROF)

    return PP


def _models(dtype, coupled, device="cpu"):
    from paper_2512_23858_b200.model import Coupling, init_weights, preset

    tc, dc = preset("tiny-target"), preset("tiny-draft")
    cp = Coupling(rank=256, logit_scale=8.0, head_noise=2.0, layer_gain=2.0) if coupled else None
    tw = init_weights(tc, 0, torch.float32, device, cp)
    dw = init_weights(dc, 1, torch.float32, device, cp)
    return tc, dc, tw, dw


def _prompt(vocab, n=32, seed=1000):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, vocab, (n,), generator=g)


@pytest.mark.parametrize("coupled", [False, True])
def test_fp32_step_trace_matches_oracle(coupled, cuda):
    from oracle.llama_ref import RefLlama, greedy_ar
    from oracle.spec_ref import RefSpecDecoder
    from paper_2512_23858_b200.engine import SpecDecoder, StepShape
    from paper_2512_23858_b200.model import weights_to

    tc, dc, tw, dw = _models(torch.float32, coupled)
    PP = _profiles()
    prompt = _prompt(tc.vocab)
    n_tok = 48
    ref = RefSpecDecoder(RefLlama(tc, tw), RefLlama(dc, dw), 4, 4, 8, 64, PP.drafter, PP.verifier, 256)
    ref_out = ref.generate(prompt.tolist(), n_tok)
    ar = greedy_ar(RefLlama(tc, tw), prompt.tolist(), n_tok, 256)
    assert ref_out == ar

    sd = SpecDecoder(tc, weights_to(tw, cuda), dc, weights_to(dw, cuda), StepShape(4, 4, 8, 64), batch=1,
                     max_seq=256, act_dtype=torch.float32, profiles=PP)
    sd.prefill_len = len(prompt)
    sd.prefill(prompt[None])
    for i, rec in enumerate(ref.trace):
        sd.step(use_graph=False)
        torch.cuda.synchronize()
        grown = sd.grown.to_dicts()[0]
        assert [n["token"] for n in grown["nodes"]] == [n["token"] for n in rec["tree"]["nodes"]], f"step {i}"
        assert [n["parent"] for n in grown["nodes"]] == [n["parent"] for n in rec["tree"]["nodes"]], f"step {i}"
        for a, b in zip(grown["nodes"], rec["tree"]["nodes"]):
            assert abs(a["prob"] - b["prob"]) <= 1e-4 * max(b["prob"], 1e-6)
        kept = [k for k in sd.keep_idx[0].tolist() if k >= 0]
        assert kept == rec["kept"], f"step {i}"
        assert sd.path[0, : int(sd.path_len[0])].tolist() == rec["path"], f"step {i}"
        assert int(sd.bonus[0]) == rec["bonus"], f"step {i}"
    assert sd.generated(0)[:n_tok] == ar


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("coupled", [False, True])
def test_bf16_spec_equals_ar_and_graph_equals_eager(coupled, fused, cuda):
    from paper_2512_23858_b200.engine import ARDecoder, SpecDecoder, StepShape
    from paper_2512_23858_b200.model import weights_to
    from paper_2512_23858_b200.plan import ForwardPlan

    plan = ForwardPlan(fused_epilogues=fused)
    tc, dc, tw, dw = _models(torch.float32, coupled)
    twb, dwb = weights_to(tw, cuda, torch.bfloat16), weights_to(dw, cuda, torch.bfloat16)
    prompts = torch.stack([_prompt(tc.vocab, 32, s) for s in (1000, 1001)])
    n_tok = 40
    ar = ARDecoder(tc, twb, batch=2, max_seq=256, plan=plan).generate(prompts, n_tok)
    outs = []
    for use_graph in (False, True):
        sd = SpecDecoder(tc, twb, dc, dwb, StepShape(4, 4, 8, 64), batch=2, max_seq=256, profiles=_profiles(),
                         plan=plan)
        got, steps = sd.generate(prompts, n_tok, use_graph=use_graph)
        outs.append(got)
    assert outs[0] == outs[1]
    assert outs[0] == ar


def test_bf16_verify_logits_within_tolerance(cuda):
    """One bf16 prefill pass vs the fp32 CPU oracle: max |diff| / max |logit| <= 2e-2."""
    from oracle.llama_ref import RefCache, RefLlama, causal_visible
    from paper_2512_23858_b200.forward import Forward, new_cache
    from paper_2512_23858_b200.model import weights_to

    tc, dc, tw, dw = _models(torch.float32, True)
    prompt = _prompt(tc.vocab, 40)
    ref = RefLlama(tc, tw).forward(RefCache(tc, 64), prompt.tolist(), list(range(40)), list(range(40)),
                                   causal_visible(40, 64))
    for dtype, tol in ((torch.bfloat16, 2e-2), (torch.float32, 1e-3)):
        w = weights_to(tw, cuda, dtype)
        cache = new_cache(tc, 1, 64, dtype, cuda)
        f = Forward(tc, w, cache, 1, 40, 0, dtype)
        f.tokens.copy_(prompt.to(cuda, torch.int32))
        pos = torch.arange(40, dtype=torch.int32, device=cuda)
        f.pos.copy_(pos)
        f.slot.copy_(pos)
        f.blk_start.zero_()
        f.blk_len.fill_(40)
        f.run()
        torch.cuda.synchronize()
        err = (f.logits.cpu() - ref).abs().max() / ref.abs().max()
        assert err <= tol, (dtype, float(err))


def test_bf16_long_run_spec_equals_ar(cuda):
    """Lossless-greedy identity over 240 tokens at cfg1's tree shape (D4 W4), coupled weights,
    so the KV compaction of both caches is exercised over ~60 steps of varying accepted lengths."""
    from paper_2512_23858_b200.engine import ARDecoder, SpecDecoder, StepShape
    from paper_2512_23858_b200.model import weights_to

    tc, dc, tw, dw = _models(torch.float32, True)
    twb, dwb = weights_to(tw, cuda, torch.bfloat16), weights_to(dw, cuda, torch.bfloat16)
    prompts = _prompt(tc.vocab, 32, 1234)[None]
    n_tok = 240
    ar = ARDecoder(tc, twb, batch=1, max_seq=320).generate(prompts, n_tok)
    sd = SpecDecoder(tc, twb, dc, dwb, StepShape(4, 4, 8, 64), batch=1, max_seq=320, profiles=_profiles())
    got, steps = sd.generate(prompts, n_tok)
    assert got == ar
    assert steps < n_tok  # speculation accepted more than one token per step on average


def test_sample_mode_cold_temperature_equals_greedy(cuda):
    """SAMPLE acceptance (softmax(target/T) child probabilities, residual bonus) at a temperature
    where the target distribution is one-hot must reproduce greedy AR exactly."""
    from paper_2512_23858_b200.engine import SAMPLE, ARDecoder, SpecDecoder, StepShape
    from paper_2512_23858_b200.model import weights_to

    tc, dc, tw, dw = _models(torch.float32, True)
    twb, dwb = weights_to(tw, cuda, torch.bfloat16), weights_to(dw, cuda, torch.bfloat16)
    prompts = torch.stack([_prompt(tc.vocab, 32, s) for s in (7, 8)])
    n_tok = 48
    ar = ARDecoder(tc, twb, batch=2, max_seq=256).generate(prompts, n_tok)
    sd = SpecDecoder(tc, twb, dc, dwb, StepShape(4, 4, 8, 64), batch=2, max_seq=256, profiles=_profiles(),
                     mode=SAMPLE, temperature=1e-4)
    got, _ = sd.generate(prompts, n_tok, use_graph=True)
    assert got == ar


def test_sample_mode_first_token_distribution(cuda):
    """At T = 1 the first emitted token after the prompt is distributed as the target softmax
    (speculative sampling is lossless in distribution): chi-square over the top tokens, 4000 draws."""
    import numpy as np

    from paper_2512_23858_b200.engine import SAMPLE, SpecDecoder, StepShape
    from paper_2512_23858_b200.forward import Forward, new_cache
    from paper_2512_23858_b200.model import weights_to

    tc, dc, tw, dw = _models(torch.float32, True)
    twf, dwf = weights_to(tw, cuda, torch.float32), weights_to(dw, cuda, torch.float32)
    prompt = _prompt(tc.vocab, 16, 99)
    n_req = 4000
    # target distribution of the token after the bonus: rows of a reference prefill over prompt+bonus
    sd = SpecDecoder(tc, twf, dc, dwf, StepShape(2, 2, 4, 8), batch=n_req // 8, max_seq=64,
                     act_dtype=torch.float32, profiles=_profiles(), mode=SAMPLE, temperature=1.0)
    counts = {}
    bonus0 = None
    for rep in range(8):
        sd.prefill_len = 16
        sd.prefill(prompt[None].repeat(sd.B, 1))
        if bonus0 is None:
            bonus0 = int(sd.seq.hist[0, 16])
        sd.set_uniforms(rep, 1234)
        sd.step(use_graph=False)
        nxt = sd.seq.hist[:, 17].cpu().tolist()
        for t in nxt:
            counts[t] = counts.get(t, 0) + 1
    seq = torch.cat([prompt, torch.tensor([bonus0])]).to(cuda, torch.int32)
    f = Forward(tc, twf, new_cache(tc, 1, 64, torch.float32, cuda), 1, 17, 0, torch.float32)
    f.tokens.copy_(seq)
    pos = torch.arange(17, dtype=torch.int32, device=cuda)
    f.pos.copy_(pos)
    f.slot.copy_(pos)
    f.blk_start.zero_()
    f.blk_len.fill_(17)
    f.run()
    p = torch.softmax(f.logits[16].double(), 0).cpu().numpy()
    top = np.argsort(-p)[:8]
    obs = np.array([counts.get(int(t), 0) for t in top] + [n_req - sum(counts.get(int(t), 0) for t in top)])
    exp = np.concatenate([p[top], [1.0 - p[top].sum()]]) * n_req
    keep = exp >= 5
    chi2 = float((((obs - exp) ** 2) / exp)[keep].sum())
    # 99.9% quantile of chi-square with <= 8 degrees of freedom is 26.1
    assert chi2 < 26.1, (chi2, obs.tolist(), exp.round(1).tolist())


@pytest.mark.parametrize("B,W", [(2, 8), (1, 16), (3, 8)])
def test_bf16_spec_equals_ar_draft_paths(B, W, cuda):
    """Lossless-greedy identity across the draft kernel families: B*R <= 16 rows run the row-block
    GEMV with two token tiles (B=2, W=8 and B=1, W=16: 16 rows) and B=3, W=8 (24 rows) the
    stream-K GEMM; the verify and the AR oracle always run the stream-K GEMM + split-KV attention."""
    from paper_2512_23858_b200.engine import ARDecoder, SpecDecoder, StepShape
    from paper_2512_23858_b200.model import weights_to

    tc, dc, tw, dw = _models(torch.float32, True)
    twb, dwb = weights_to(tw, cuda, torch.bfloat16), weights_to(dw, cuda, torch.bfloat16)
    prompts = torch.stack([_prompt(tc.vocab, 32, 2000 + b) for b in range(B)])
    n_tok = 48
    ar = ARDecoder(tc, twb, batch=B, max_seq=320).generate(prompts, n_tok)
    sd = SpecDecoder(tc, twb, dc, dwb, StepShape(3, W, 8, 64), batch=B, max_seq=320, profiles=_profiles())
    assert sd.draft.gemv == (B * max(W, 2) <= 16)
    got, steps = sd.generate(prompts, n_tok)
    assert got == ar
    assert steps < n_tok
