"""Runtime shape control with real models: per-step choice of the EGT (depth, width) among captured
step graphs over ONE decoding state (the reference's per-iteration
depth decision and width selection, pkg/src/specsim/simulator.py:305-324, egt.py:285-318).

* Every candidate ``StepShape`` gets its own ``SpecDecoder`` (forwards, trees, CUDA graph) sharing
  the first one's sequence state and KV caches, so switching shape between steps costs nothing but
  choosing which graph to replay.
* The host decides the shape of step i from a lagged pinned readback of step i - ``lag`` (accepted
  length, the pass-0 root candidate distribution, the step's device time), so it never waits for
  the GPU: the reference's loop observes the previous outcome; here the observation is ``lag``
  steps old (default 2 keeps one step queued ahead).
* Depth: a reference ``DepthPredictor`` (FixedDepth / EmaHeuristic / MlpPredictor, fed the reference's
  five features from device data — depth_predictor.DeviceFeatures), snapped to the captured depths.
* Width at that depth (and, with ``policy="bandit"``, the whole shape): the reference picks the width
  maximizing the latency-aware objective over provisional trees grown from its synthetic drafter,
  which a real draft model cannot afford; here each captured shape's realized accepted tokens per
  device-second is tracked and the best is exploited, after a short round-robin exploration and with
  a small exploration share — the objective's ratio (expected accepted length over step latency,
  latency.py:154-161) measured instead of modelled.
* Calibrated Eq.3: with ``calibrate`` every shape's prune objective (K6) reads per-position acceptance
  rates accumulated on the device (ygg_accept_stats; an ExplicitAcceptance keyed by grown-tree
  position, acceptance.py:106-129) instead of the over-confident surrogate draft probabilities,
  refreshed every ``refresh`` steps.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from .depth_predictor import DeviceFeatures
from .engine import GREEDY, SAMPLE, SpecDecoder, StepShape
from .plugins import DepthPredictor


@dataclass
class ShapeStats:
    steps: int = 0
    tokens: float = 0.0
    seconds: float = 0.0

    @property
    def rate(self) -> float:
        return self.tokens / self.seconds if self.seconds > 0 else 0.0


@dataclass
class AdaptiveTrace:
    chosen: list = field(default_factory=list)  # shape index per step
    accepted: list = field(default_factory=list)  # accepted tokens (all requests) per observed step
    step_ms: list = field(default_factory=list)


class AdaptiveDecoder:
    def __init__(self, target_cfg, target_w, draft_cfg, draft_w, shapes: list[StepShape], batch: int = 1,
                 max_seq: int = 2048, act_dtype=torch.bfloat16, mode: str = GREEDY, temperature: float = 1.0,
                 profiles=None, device="cuda", policy: str = "bandit", predictor: DepthPredictor | None = None,
                 calibrate: bool = True, refresh: int = 16, explore_steps: int = 2, explore_share: float = 0.05,
                 lag: int = 2, seed: int = 0, plan=None, proj_dim: int = 0):
        if not shapes:
            raise ValueError("need at least one step shape")
        if policy not in ("bandit", "predictor"):
            raise ValueError("policy must be 'bandit' or 'predictor'")
        if policy == "predictor" and predictor is None:
            raise ValueError("policy 'predictor' needs a DepthPredictor")
        if lag < 1:
            raise ValueError("lag must be >= 1")
        scratch = max(1 + s.depth * s.width + max(s.width, 2) + 8 for s in shapes)
        self.shapes = list(shapes)
        self.decs: list[SpecDecoder] = []
        for sh in self.shapes:
            self.decs.append(SpecDecoder(target_cfg, target_w, draft_cfg, draft_w, sh, batch=batch, max_seq=max_seq,
                                         act_dtype=act_dtype, mode=mode, temperature=temperature, profiles=profiles,
                                         device=device, share=self.decs[0] if self.decs else None, scratch=scratch,
                                         calibrate=calibrate, plan=plan, feature_tap=proj_dim > 0))
        d0 = self.decs[0]
        self.B, self.seq, self.dev, self.mode = batch, d0.seq, d0.dev, mode
        self.policy, self.predictor = policy, predictor
        self.calibrate, self.refresh = calibrate, refresh
        self.explore_steps, self.explore_share, self.lag = explore_steps, explore_share, lag
        self.stats = [ShapeStats() for _ in self.shapes]
        self.features = DeviceFeatures(batch, hidden_dim=target_cfg.d_model, proj_dim=proj_dim, seed=seed)
        self.proj_dim = proj_dim
        self._last_features = None
        self.rng = np.random.default_rng(seed)
        self.trace = AdaptiveTrace()
        self._pending: list = []  # (shape index, event pair, pinned acc_len, pinned root probs)
        kmax = max(s.expansion_k for s in self.shapes)
        # readback ring: a slot is reused only after its step was observed (ring longer than the lag)
        hd = target_cfg.d_model if proj_dim > 0 else 1
        self._ring = [(torch.empty(batch, dtype=torch.int32).pin_memory(),
                       torch.empty(batch, kmax, dtype=torch.float64).pin_memory(),
                       torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                       torch.empty(batch, hd, dtype=torch.float32).pin_memory())
                      for _ in range(lag + 2)]
        self._issued = [0] * len(self.shapes)
        self.steps = 0
        self.prefill_len = 0

    # ------------------------------------------------------------------
    def prefill(self, prompts: torch.Tensor) -> None:
        self.prefill_len = prompts.shape[1]
        self.decs[0].prefill(prompts)
        for d in self.decs:
            d.prefill_len = self.prefill_len

    def capture(self) -> None:
        for d in self.decs:
            if d.graph is None:
                d.capture()

    def set_profiles(self, profiles) -> None:
        for d in self.decs:
            d.set_profiles(profiles)

    # ------------------------------------------------------------------
    def _observe(self, block: bool) -> None:
        """Consume lagged readbacks: shape statistics, predictor / feature state."""
        while self._pending and (block or len(self._pending) > self.lag - 1):
            idx, (ea, eb), acc_h, root_h, hid_h = self._pending.pop(0)
            eb.synchronize()
            ms = ea.elapsed_time(eb)
            acc = acc_h.numpy()
            st = self.stats[idx]
            st.steps += 1
            st.tokens += float(acc.sum())
            st.seconds += ms * 1e-3
            self.trace.accepted.append(int(acc.sum()))
            self.trace.step_ms.append(ms)
            feats = self.features.update(acc, root_h.numpy(), hid_h.numpy() if self.proj_dim > 0 else None)
            self._last_features = feats[0]
            if self.predictor is not None:
                self.predictor.observe(int(acc[0]))
            if not block:
                break

    def _choose(self) -> int:
        n = len(self.shapes)
        if self.policy == "predictor":
            cand = list(range(n))
            if self.predictor.ready:
                want = self.predictor.predict(self._last_features)
                depths = sorted({s.depth for s in self.shapes})
                d = min(depths, key=lambda x: (abs(x - want), x))
                cand = [i for i in range(n) if self.shapes[i].depth == d]
        else:
            cand = list(range(n))
        # exploration: every candidate a few issued steps first, then a small share
        for i in cand:
            if self._issued[i] < self.explore_steps:
                return i
        if len(cand) > 1 and self.rng.random() < self.explore_share:
            return int(self.rng.choice(cand))
        return max(cand, key=lambda i: (self.stats[i].rate, -i))

    def _refresh_calibration(self) -> None:
        for d in self.decs:
            if d.calibrate:
                d.set_node_table(d.node_rates())

    def step(self) -> int:
        """Choose a shape, replay its step graph, queue the lagged readback. Returns the shape index."""
        self._observe(block=False)
        if self.calibrate and self.steps > 0 and self.steps % self.refresh == 0:
            self._refresh_calibration()
        i = self._choose()
        d = self.decs[i]
        if self.mode == SAMPLE:
            d.set_uniforms(self.steps, 0)
        acc_h, root_h, ea, eb, hid_h = self._ring[self.steps % len(self._ring)]
        if len(self._pending) >= len(self._ring):
            self._observe(block=True)
        ea.record()
        d.step(use_graph=d.graph is not None)
        eb.record()
        acc_h.copy_(d.acc_len, non_blocking=True)
        k = d.shape.expansion_k
        root_h[:, :k].copy_(d.root_probs, non_blocking=True)
        root_h[:, k:] = 0.0
        if self.proj_dim > 0:
            hid_h.copy_(d.hidden_tap, non_blocking=True)
        self._pending.append((i, (ea, eb), acc_h, root_h, hid_h))
        self._issued[i] += 1
        self.trace.chosen.append(i)
        self.steps += 1
        return i

    def collect_depth_samples(self, shape_index: int, n: int) -> list:
        """Offline profiling for train_predictor (the reference's collect_depth_samples, simulator.py:
        553-579, with a deep EGT shape instead of a synthetic chain): before each of ``n`` steps the
        features the decoder would predict from, then the accepted length that step realized.
        Synchronous (one readback per step); call after prefill."""
        from .depth_predictor import DepthSample

        self.drain()
        d = self.decs[shape_index]
        feats = self._last_features
        if feats is None:
            feats = self.features.update([0] * self.B, np.zeros((self.B, d.shape.expansion_k)),
                                         np.zeros((self.B, self.features.proj.shape[0])) if self.proj_dim else None)[0]
        out = []
        for _ in range(n):
            d.step(use_graph=d.graph is not None)
            acc = d.acc_len.cpu().numpy()
            out.append(DepthSample(features=np.asarray(feats), realized_len=int(acc[0])))
            hid = d.hidden_tap.cpu().numpy() if self.proj_dim > 0 else None
            feats = self.features.update(acc, d.root_probs.cpu().numpy(), hid)[0]
        self._last_features = feats
        return out

    def drain(self) -> None:
        self._observe(block=True)

    def generated(self, b: int = 0) -> list[int]:
        n = int(self.seq.n_gen[b])
        return self.seq.hist[b, self.prefill_len : self.prefill_len + n].cpu().tolist()

    def generate(self, prompts: torch.Tensor, n_tokens: int, sync_every: int = 8):
        B, P0 = prompts.shape
        if P0 + n_tokens + max(s.depth for s in self.shapes) + 2 > self.seq.p_limit:
            raise ValueError("prompt + generated tokens do not fit the cache (max_seq too small)")
        self.prefill(prompts)
        self.seq.gen_limit.fill_(n_tokens)
        self.seq.status.zero_()
        self.capture()
        steps = 0
        while True:
            if steps % sync_every == 0:
                st = self.seq.status.cpu()
                if bool((st != 0).all()):
                    if bool((st & 2).any()):
                        raise RuntimeError("a request reached the cache capacity before n_tokens")
                    break
            self.step()
            steps += 1
        self.drain()
        return [self.generated(b)[:n_tokens] for b in range(self.B)], steps

    def summary(self) -> dict:
        hist = np.bincount(np.asarray(self.trace.chosen, dtype=np.int64), minlength=len(self.shapes))
        return {"shapes": [{"depth": s.depth, "width": s.width, "max_verify": s.max_verify, "steps": int(h),
                            "tokens_per_s": round(st.rate, 2),
                            "aal": round(st.tokens / st.steps / self.B, 3) if st.steps else None}
                           for s, h, st in zip(self.shapes, hist, self.stats)]}


def fit_depth_decay(counts, depth: int, width: int) -> tuple[float, float]:
    """DepthDecayAcceptance(p0, gamma) (acceptance.py:60-103) fitted to device acceptance counts of one
    EGT shape ([tree_cap, 2] tested / accepted per grown position, ygg_accept_stats): the level-d
    conditional acceptance m_d = accepted(level d) / accepted(level d-1) (m_0 = accepted(root) /
    steps) is the model's level mass p0 * gamma**d; least squares on log m_d."""
    c = np.asarray(counts, dtype=np.float64)
    acc = [c[0, 1]] + [c[1 + (d - 1) * width : 1 + d * width, 1].sum() for d in range(1, depth + 1)]
    steps = c[0, 0]
    if steps <= 0 or acc[0] <= 0:
        raise ValueError("no accepted root yet")
    ds, ys = [0], [math.log(acc[0] / steps)]
    for d in range(1, depth + 1):
        if acc[d] > 0 and acc[d - 1] > 0:
            ds.append(d)
            ys.append(math.log(acc[d] / acc[d - 1]))
    if len(ds) < 2:
        return min(1.0, acc[0] / steps), 1.0
    slope, icpt = np.polyfit(np.asarray(ds, dtype=np.float64), np.asarray(ys), 1)
    return float(min(1.0, math.exp(icpt))), float(min(1.0, math.exp(slope)))


def rate_ci(st: ShapeStats) -> float:
    """Half-width proxy of a shape's rate estimate (diagnostic)."""
    return st.rate / math.sqrt(max(st.steps, 1))


class ServingEngine:
    """Slot-level continuous batching over one captured step graph.

    The decoder's B request slots run one graph replay per step.  Requests wait in a queue; an idle slot
    admits the next one (SpecDecoder.prefill_slot: prefill of that slot only, between replays, while
    the other slots keep decoding); a slot whose request reached its token budget is frozen on the
    device by the commit kernel (generation limit), its tokens are collected at the next poll and the
    slot is refilled.  KV stays in the fixed-stride per-slot layout (no paging): each slot holds up to
    the decoder's S positions."""

    def __init__(self, sd: SpecDecoder, poll: int = 4, chunk: int = 64):
        self.sd, self.poll, self.chunk = sd, poll, chunk
        self.queue: list = []
        self.slot_req = [None] * sd.B
        self.slot_p0 = [0] * sd.B
        self.done: dict = {}
        self._next = 0
        self.steps = 0

    def submit(self, prompt, n_tokens: int) -> int:
        rid = self._next
        self._next += 1
        self.queue.append((rid, torch.as_tensor(prompt, dtype=torch.int32).reshape(-1), int(n_tokens)))
        return rid

    def _admit(self) -> None:
        for b in range(self.sd.B):
            if self.slot_req[b] is None:
                if self.queue:
                    rid, prompt, n = self.queue.pop(0)
                    self.sd.prefill_slot(b, prompt, n, self.chunk)
                    self.slot_req[b], self.slot_p0[b] = (rid, n), prompt.numel()
                else:
                    self.sd.park_slot(b)

    def _collect(self) -> None:
        sq = self.sd.seq
        status = sq.status.cpu()
        for b in range(self.sd.B):
            if self.slot_req[b] is not None and int(status[b]) & 1:
                rid, n = self.slot_req[b]
                p0 = self.slot_p0[b]
                self.done[rid] = sq.hist[b, p0 : p0 + n].cpu().tolist()
                self.slot_req[b] = None
            elif self.slot_req[b] is not None and int(status[b]) & 2:
                raise RuntimeError(f"request {self.slot_req[b][0]} reached the slot's cache capacity")

    def run(self, use_graph: bool = True, max_steps: int = 1 << 20) -> dict:
        """Serve every submitted request; returns {request id: generated tokens}."""
        self._admit()
        if use_graph and self.sd.graph is None:
            self.sd.capture()
        while (self.queue or any(r is not None for r in self.slot_req)) and self.steps < max_steps:
            if self.sd.mode == SAMPLE:
                self.sd.set_uniforms(self.steps, 0)
            self.sd.step(use_graph)
            self.steps += 1
            if self.steps % self.poll == 0:
                self._collect()
                self._admit()
        self._collect()
        return dict(self.done)
