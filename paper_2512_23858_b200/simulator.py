"""The reference's iteration loop (API of pkg/src/specsim/simulator.py:64-349) over the device kernels.

``run(config)`` reproduces the reference simulator's ``DecodeStats`` bit-for-bit, with every tree
operation executed by the B200 kernels: width selection and EGT growth (K1), verification-width
pruning (K6), and the acceptance walk (K5, drawing from ``default_rng([seed, iteration])`` exactly
like simulator.py:306).  Stage pricing uses the host plan search (scheduler.py) offline per shape,
as the reference does.  With real models, ``engine.SpecDecoder`` is the generate loop; this module
is the drop-in for callers of the reference's simulator API and its parity anchor
(tests/golden/simulate_example.json).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from .acceptance import AcceptanceModel, freeze_probs, path_products, sample_with_probs
from .egt import EgtConfig, grow_egt, prune_verify, select_width
from .latency import ProfilePair, latency_at
from .plugins import DepthPredictor, FeatureState, FixedDepth
from .scheduler import StageProfiles, TreeShape, draft_stage_names, plan_search
from .token_tree import TokenTree, new_tree

_CPU_STAGE_DEFAULTS = {("Accept", "base"): 0.0, ("BonusSample", "base"): 0.0, ("PrepareVerify", "base"): 0.0,
                       ("TailDraft", "base"): 0.0}


@dataclass(frozen=True)
class SequencePolicy:
    num_draft: int

    def __post_init__(self) -> None:
        if self.num_draft < 1:
            raise ValueError(f"num_draft {self.num_draft} must be >= 1")


@dataclass(frozen=True)
class KAryPolicy:
    k: int
    depth: int

    def __post_init__(self) -> None:
        if self.k < 1 or self.depth < 1:
            raise ValueError("k and depth must be >= 1")


@dataclass(frozen=True)
class StaticTreePolicy:
    template: TokenTree


@dataclass(frozen=True)
class EgtPolicy:
    config: EgtConfig = EgtConfig()
    predictor_factory: Callable[[], DepthPredictor] = field(default=lambda: FixedDepth(8))
    fallback_depth: int = 8

    def __post_init__(self) -> None:
        if not 1 <= self.fallback_depth <= self.config.max_depth:
            raise ValueError(f"fallback_depth {self.fallback_depth} outside [1, {self.config.max_depth}]")


@dataclass(frozen=True)
class SimConfig:
    seed: int
    iterations: int
    model: AcceptanceModel
    generator: object
    profiles: ProfilePair
    policy: object
    stage_profiles: StageProfiles | None = None
    plan_search: bool = False
    jobs: int = 1

    def __post_init__(self) -> None:
        if self.iterations < 1:
            raise ValueError(f"iterations {self.iterations} must be >= 1")
        if self.jobs < 1:
            raise ValueError(f"jobs {self.jobs} must be >= 1")


@dataclass(frozen=True)
class IterationRecord:
    iteration: int
    d_draft: int
    tree_size: int
    w_verify: int
    accepted_len: int
    step_us: float


@dataclass(frozen=True)
class DecodeStats:
    aal: float
    step_latency_us: float
    tpot_us: float
    speedup: float
    trace: tuple[IterationRecord, ...]


@dataclass(frozen=True)
class _Prepared:
    tree: TokenTree
    probs: np.ndarray
    d_draft: int
    w_draft: int
    w_verify: int
    expected_aal: float
    step_us: float


def _chain_tree(drafter, n: int) -> TokenTree:
    tree = new_tree(*drafter.root())
    node = 0
    for _ in range(n - 1):
        c = drafter.candidates(tree, node, 1)
        if not c:
            break
        node = tree.add_child(node, *c[0])
    return tree


def _kary_tree(drafter, k: int, depth: int) -> TokenTree:
    tree = new_tree(*drafter.root())
    frontier = [0]
    for _ in range(depth):
        grown = [tree.add_child(n, t, p) for n in frontier for t, p in drafter.candidates(tree, n, k)]
        if not grown:
            break
        frontier = grown
    return tree


def _level_sizes(tree: TokenTree) -> list[int]:
    return [len(lv) for lv in tree.levels[1:]]


def _merged_stages(profiles: ProfilePair, level_sizes: Sequence[int], w_verify: int,
                   user: StageProfiles | None) -> StageProfiles:
    rows = dict(_CPU_STAGE_DEFAULTS)
    if user is not None:
        rows.update(user.rows())
    rows[("Verify", "base")] = latency_at(profiles.verifier, w_verify + 1)
    for name, width in zip(draft_stage_names(len(level_sizes)), level_sizes):
        rows[(name, "base")] = latency_at(profiles.drafter, width)
    return StageProfiles(rows)


def _step_latency(profiles, level_sizes, w_verify, user, scheduled) -> float:
    merged = _merged_stages(profiles, level_sizes, w_verify, user)
    d = len(level_sizes)
    if d == 0:
        return sum(merged.base(n) for n in ("Verify", "Accept", "BonusSample", "TailDraft", "PrepareVerify"))
    if scheduled:
        return plan_search(merged, TreeShape(max(level_sizes), d, w_verify), expected_aal=1.0).makespan_us
    names = ["Verify", "Accept", "BonusSample", "TailDraft", *draft_stage_names(d), "PrepareVerify"]
    return sum(merged.base(n) for n in names)


def _prepare(config: SimConfig, drafter, depth: int) -> _Prepared:
    policy = config.policy
    if isinstance(policy, EgtPolicy):
        width = select_width(policy.config, depth, drafter, config.profiles, model=config.model)
        tree = new_tree(*drafter.root())
        grow_egt(tree, drafter, depth, width, policy.config.expansion_k)
        grown_probs = freeze_probs(config.model, tree)
        pr = prune_verify(tree, config.model, config.profiles, depth, width, policy.config.max_verify)
        levels = _level_sizes(tree)
        step = _step_latency(config.profiles, levels, pr.w_verify, config.stage_profiles, config.plan_search)
        return _Prepared(pr.tree, grown_probs[list(pr.kept)], len(levels), max(levels, default=1), pr.w_verify,
                         pr.expected_aal, step)
    if isinstance(policy, SequencePolicy):
        tree = _chain_tree(drafter, policy.num_draft)
    elif isinstance(policy, KAryPolicy):
        tree = _kary_tree(drafter, policy.k, policy.depth)
    else:
        tree = policy.template
    probs = freeze_probs(config.model, tree)
    levels = _level_sizes(tree)
    step = _step_latency(config.profiles, levels, len(tree), config.stage_profiles, config.plan_search)
    return _Prepared(tree, probs, len(levels), max(levels, default=1), len(tree),
                     1.0 + float(np.sum(path_products(tree, probs))), step)


def run(config: SimConfig) -> DecodeStats:
    is_egt = isinstance(config.policy, EgtPolicy)
    predictor = config.policy.predictor_factory() if is_egt else None
    state = FeatureState()
    cache: dict = {}
    records = []
    for it in range(config.iterations):
        rng = np.random.default_rng([config.seed, it])
        drafter = config.generator.drafter_at(it)
        if is_egt:
            probe = new_tree(*drafter.root())
            feats = state.features(drafter.candidates(probe, 0, config.policy.config.expansion_k))
            depth = predictor.predict(feats) if predictor.ready else config.policy.fallback_depth
            depth = max(1, min(config.policy.config.max_depth, depth))
        else:
            depth = 0
        key = (drafter.signature(), depth)
        prep = cache.get(key)
        if prep is None:
            prep = _prepare(config, drafter, depth)
            cache[key] = prep
        out = sample_with_probs(prep.tree, prep.probs, rng)
        state.observe(out.accepted_len)
        if predictor is not None:
            predictor.observe(out.accepted_len)
        records.append(IterationRecord(it, prep.d_draft, len(prep.tree), prep.w_verify, out.accepted_len,
                                       prep.step_us))
    tokens = sum(r.accepted_len for r in records)
    total = sum(r.step_us for r in records)
    tpot = total / tokens
    return DecodeStats(aal=tokens / len(records), step_latency_us=total / len(records), tpot_us=tpot,
                       speedup=latency_at(config.profiles.verifier, 1) / tpot, trace=tuple(records))
