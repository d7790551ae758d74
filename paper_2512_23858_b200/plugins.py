"""Host plugins of the reference's simulator interface (not kernels): synthetic drafters
(pkg/src/specsim/drafters.py:19-158) and draft-depth predictors (depth_predictor.py:32-199).

With real models the drafter is ``engine.SpecDecoder``'s draft forward; these synthetic
``DrafterDistribution`` implementations exist so the reference's own simulator configurations run
unchanged through the device kernels (simulator.run) and compare bit-for-bit with the reference.
"""

from __future__ import annotations

from abc import ABC, abstractmethod
from collections import deque
from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np


@dataclass(frozen=True)
class GeometricDrafter:
    """Candidate (depth d, rank r): top_mass * decay**d * top_share * (1 - top_share)**r."""

    top_mass: float
    decay: float
    fanout: int = 8
    top_share: float = 0.7

    def __post_init__(self) -> None:
        if not 0.0 < self.top_mass <= 1.0:
            raise ValueError(f"top_mass {self.top_mass} must be in (0, 1]")
        if not 0.0 < self.decay <= 1.0:
            raise ValueError(f"decay {self.decay} must be in (0, 1]")
        if self.fanout < 1:
            raise ValueError(f"fanout {self.fanout} must be >= 1")
        if not 0.0 < self.top_share < 1.0:
            raise ValueError(f"top_share {self.top_share} must be in (0, 1)")

    def root(self) -> tuple[int, float]:
        return (1, self.top_mass)

    def candidates(self, tree, node: int, k: int) -> list[tuple[int, float]]:
        mass = self.top_mass * self.decay ** (tree.depth(node) + 1)
        return [(r + 1, mass * self.top_share * (1.0 - self.top_share) ** r) for r in range(min(k, self.fanout))]

    def signature(self) -> tuple:
        return ("geometric", self.top_mass, self.decay, self.fanout, self.top_share)


@dataclass(frozen=True)
class FlatDrafter:
    mass: float = 1.0
    fanout: int = 8

    def root(self) -> tuple[int, float]:
        return (1, 1.0)

    def candidates(self, tree, node: int, k: int) -> list[tuple[int, float]]:
        return [(r + 1, self.mass / self.fanout) for r in range(min(k, self.fanout))]

    def signature(self) -> tuple:
        return ("flat", self.mass, self.fanout)


class StationaryGenerator:
    def __init__(self, drafter) -> None:
        self.drafter = drafter

    def drafter_at(self, iteration: int):
        return self.drafter

    def regimes(self) -> list:
        return [self.drafter]


class BlockGenerator:
    def __init__(self, regimes: list, block_len: int) -> None:
        if not regimes:
            raise ValueError("need at least one regime")
        if block_len < 1:
            raise ValueError(f"block_len {block_len} must be >= 1")
        self._regimes, self.block_len = list(regimes), block_len

    def drafter_at(self, iteration: int):
        return self._regimes[(iteration // self.block_len) % len(self._regimes)]

    def regimes(self) -> list:
        return list(self._regimes)


# ---------------------------------------------------------------------------
# depth predictors (host, microsecond-scale)
# ---------------------------------------------------------------------------
class FeatureState:
    """[ema_len, last_len, root top-1 mass, root top-4 mass, root entropy] (depth_predictor.py:32-72)."""

    def __init__(self, history: int = 8, alpha: float = 0.4) -> None:
        if history < 1:
            raise ValueError(f"history {history} must be >= 1")
        if not 0.0 < alpha <= 1.0:
            raise ValueError(f"alpha {alpha} must be in (0, 1]")
        self.alpha = alpha
        self._lengths: deque[int] = deque(maxlen=history)

    def observe(self, n: int) -> None:
        if n < 1:
            raise ValueError(f"realized length {n} must be >= 1")
        self._lengths.append(n)

    @property
    def ema_len(self) -> float:
        if not self._lengths:
            return 1.0
        it = iter(self._lengths)
        ema = float(next(it))
        for v in it:
            ema = self.alpha * float(v) + (1.0 - self.alpha) * ema
        return ema

    @property
    def last_len(self) -> float:
        return float(self._lengths[-1]) if self._lengths else 1.0

    def features(self, root_candidates: Sequence[tuple[int, float]]) -> np.ndarray:
        p = np.array([q for _, q in root_candidates], dtype=np.float64)
        top1 = float(p[0]) if p.size else 0.0
        top4 = float(p[:4].sum()) if p.size else 0.0
        pos = p[p > 0.0]
        ent = float(-(pos * np.log(pos)).sum()) if pos.size else 0.0
        return np.array([self.ema_len, self.last_len, top1, top4, ent])


class DepthPredictor(ABC):
    @abstractmethod
    def predict(self, features) -> int:
        """Next depth (>= 1)."""

    def observe(self, realized_len: int) -> None:  # noqa: B027
        pass

    @property
    def ready(self) -> bool:
        return True


class FixedDepth(DepthPredictor):
    def __init__(self, depth: int) -> None:
        if depth < 1:
            raise ValueError(f"depth {depth} must be >= 1")
        self.depth = depth

    def predict(self, features=None) -> int:
        return self.depth


class EmaHeuristic(DepthPredictor):
    def __init__(self, window: int, alpha: float, max_depth: int) -> None:
        if window < 1:
            raise ValueError(f"window {window} must be >= 1")
        if not 0.0 < alpha <= 1.0:
            raise ValueError(f"alpha {alpha} must be in (0, 1]")
        if max_depth < 1:
            raise ValueError(f"max_depth {max_depth} must be >= 1")
        self.window, self.alpha, self.max_depth = window, alpha, max_depth
        self._lengths: deque[int] = deque(maxlen=window)

    def observe(self, n: int) -> None:
        if n < 1:
            raise ValueError(f"realized length {n} must be >= 1")
        self._lengths.append(n)

    @property
    def ready(self) -> bool:
        return len(self._lengths) >= self.window

    def predict(self, features=None) -> int:
        if not self._lengths:
            return 1
        it = iter(self._lengths)
        ema = float(next(it))
        for v in it:
            ema = self.alpha * float(v) + (1.0 - self.alpha) * ema
        return max(1, min(self.max_depth, round(ema)))


def decide_depth(head_probs: Mapping[int, float], max_depth: int) -> int:
    chosen = 1
    for d in sorted(head_probs):
        if head_probs[d] >= 0.5:
            chosen = max(chosen, d)
    return max(1, min(max_depth, chosen))
