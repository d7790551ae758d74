"""Per-step draft-depth choice: the reference's predictor contract
(pkg/src/specsim/depth_predictor.py) — FeatureState, FixedDepth, EmaHeuristic, decide_depth,
MlpPredictor and its trainer — plus the bridge that feeds them from the device.

The two-layer perceptron (depth_predictor.py:149-233) and its mini-batch trainer
(depth_predictor.py:279-344) are reproduced operation for operation (same numpy expressions, same
generator draws in the same order), so a predictor trained here on the same samples has bit-identical
weights to the reference's (tests/test_golden.py::test_depth_predictor_training_matches_reference).

Real-model features (``DeviceFeatures``): the reference feeds its predictor five synthetic
observations (depth_predictor.py:21-27).  On the GPU the same five come from the step itself — the
realized accepted length (the commit kernel's ``acc_log``) and the draft's root candidate
distribution of the step (pass-0 top-k, ``cand_prob`` row 1) — read back through one lagged pinned
copy per step; the paper's last-token embedding of the target is tapped by
``ygg_feature_tap`` into a [B, d] buffer and appended as a fixed random projection when requested.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np

from .latency import ConfigError
from .plugins import DepthPredictor, EmaHeuristic, FeatureState, FixedDepth, decide_depth  # noqa: F401

FEATURE_NAMES: tuple[str, ...] = ("ema_len", "last_len", "root_top1_mass", "root_top4_mass", "root_entropy")
DEFAULT_HEAD_DEPTHS: tuple[int, ...] = (2, 4, 6, 8, 12, 16)


def _logistic(z: np.ndarray) -> np.ndarray:
    """Overflow-free logistic, the two branches of depth_predictor.py:265-271."""
    y = np.empty_like(z)
    nonneg = z >= 0
    y[nonneg] = 1.0 / (1.0 + np.exp(-z[nonneg]))
    e = np.exp(z[~nonneg])
    y[~nonneg] = e / (1.0 + e)
    return y


def _mean_bce(p: np.ndarray, y: np.ndarray) -> float:
    q = np.clip(p, 1e-12, 1.0 - 1e-12)
    return float(-(y * np.log(q) + (1.0 - y) * np.log(1.0 - q)).mean())


class MlpPredictor(DepthPredictor):
    """Standardize -> sigmoid hidden layer -> one sigmoid head per depth d = P(accepted len >= d);
    the depth is the largest head >= 0.5 (decide_depth)."""

    def __init__(self, w1, b1, w2, b2, head_depths: Sequence[int], max_depth: int, feature_mean, feature_std,
                 feature_names: Sequence[str] = FEATURE_NAMES) -> None:
        as64 = lambda a: np.asarray(a, dtype=np.float64)  # noqa: E731
        self.w1, self.b1, self.w2, self.b2 = as64(w1), as64(b1), as64(w2), as64(b2)
        self.feature_mean, self.feature_std = as64(feature_mean), as64(feature_std)
        self.head_depths = tuple(int(d) for d in head_depths)
        self.max_depth = max_depth
        self.feature_names = tuple(feature_names)
        if len(set(self.head_depths)) != len(self.head_depths):
            raise ValueError("head depths must be distinct")
        if min(self.head_depths) < 1:
            raise ValueError("head depths must be >= 1")
        if max_depth < 1:
            raise ValueError(f"max_depth {max_depth} must be >= 1")

    def head_outputs(self, features) -> dict[int, float]:
        f = np.asarray(features, dtype=np.float64)
        if f.shape != (self.w1.shape[0],):
            raise ValueError(f"expected {self.w1.shape[0]} features, got shape {f.shape}")
        z = (f - self.feature_mean) / self.feature_std
        heads = _logistic(_logistic(z @ self.w1 + self.b1) @ self.w2 + self.b2)
        return dict(zip(self.head_depths, (float(h) for h in heads)))

    def predict(self, features) -> int:
        if features is None:
            raise ValueError("the perceptron predictor requires a feature vector")
        return decide_depth(self.head_outputs(features), self.max_depth)

    def to_dict(self) -> dict:
        return {"kind": "mlp", "w1": self.w1.tolist(), "b1": self.b1.tolist(), "w2": self.w2.tolist(),
                "b2": self.b2.tolist(), "head_depths": list(self.head_depths), "max_depth": self.max_depth,
                "feature_mean": self.feature_mean.tolist(), "feature_std": self.feature_std.tolist(),
                "feature_names": list(self.feature_names)}

    @classmethod
    def from_dict(cls, data: Mapping) -> "MlpPredictor":
        try:
            if data["kind"] != "mlp":
                raise ValueError(f"unknown predictor kind {data['kind']!r}")
            return cls(data["w1"], data["b1"], data["w2"], data["b2"], data["head_depths"], int(data["max_depth"]),
                       data["feature_mean"], data["feature_std"], data.get("feature_names", FEATURE_NAMES))
        except (KeyError, TypeError) as exc:
            raise ConfigError(f"invalid predictor checkpoint: {exc}") from exc


@dataclass(frozen=True)
class DepthSample:
    features: np.ndarray
    realized_len: int

    def __post_init__(self) -> None:
        if self.realized_len < 1:
            raise ValueError(f"realized length {self.realized_len} must be >= 1")


@dataclass(frozen=True)
class TrainConfig:
    hidden: int = 16
    head_depths: tuple[int, ...] = DEFAULT_HEAD_DEPTHS
    max_depth: int = 16
    learning_rate: float = 0.3
    epochs: int = 200
    batch_size: int = 32
    seed: int = 0


@dataclass(frozen=True)
class TrainResult:
    predictor: MlpPredictor
    initial_loss: float
    final_loss: float


class _Perceptron:
    """Parameters + the forward / backward of one mini-batch step (mean BCE over batch and heads)."""

    def __init__(self, rng: np.random.Generator, n_in: int, n_hidden: int, n_heads: int):
        self.w1 = rng.normal(0.0, 1.0 / np.sqrt(n_in), size=(n_in, n_hidden))
        self.b1 = np.zeros(n_hidden)
        self.w2 = rng.normal(0.0, 1.0 / np.sqrt(n_hidden), size=(n_hidden, n_heads))
        self.b2 = np.zeros(n_heads)

    def forward(self, x: np.ndarray):
        h = _logistic(x @ self.w1 + self.b1)
        return h, _logistic(h @ self.w2 + self.b2)

    def sgd_step(self, x: np.ndarray, y: np.ndarray, lr: float) -> None:
        h, p = self.forward(x)
        g_out = (p - y) / (x.shape[0] * y.shape[1])  # d(mean BCE)/d(logit) through the sigmoid
        g_w2, g_b2 = h.T @ g_out, g_out.sum(axis=0)
        g_hid = (g_out @ self.w2.T) * h * (1.0 - h)
        g_w1, g_b1 = x.T @ g_hid, g_hid.sum(axis=0)
        self.w2 -= lr * g_w2
        self.b2 -= lr * g_b2
        self.w1 -= lr * g_w1
        self.b1 -= lr * g_b1


def train_predictor(samples: Sequence[DepthSample], config: TrainConfig = TrainConfig()) -> TrainResult:
    """Fit the heads on the labels 1{realized_len >= d} by mini-batch gradient descent (deterministic
    for a given dataset and config; depth_predictor.py:279-344)."""
    if len(samples) < 2:
        raise ValueError("need at least 2 samples to fit the predictor")
    x = np.stack([np.asarray(s.features, dtype=np.float64) for s in samples])
    if len({(tuple(r), s.realized_len) for r, s in zip(x.tolist(), samples)}) < 2:
        raise ValueError("need at least 2 distinct samples to fit the predictor")
    lengths = np.array([s.realized_len for s in samples], dtype=np.float64)
    y = (lengths[:, None] >= np.array(config.head_depths, dtype=np.float64)[None, :]).astype(np.float64)
    mean, std = x.mean(axis=0), x.std(axis=0)
    std[std == 0.0] = 1.0
    xs = (x - mean) / std
    rng = np.random.default_rng(config.seed)
    net = _Perceptron(rng, x.shape[1], config.hidden, len(config.head_depths))
    initial = _mean_bce(net.forward(xs)[1], y)
    n = xs.shape[0]
    for _ in range(config.epochs):
        order = rng.permutation(n)
        for b0 in range(0, n, config.batch_size):
            idx = order[b0 : b0 + config.batch_size]
            net.sgd_step(xs[idx], y[idx], config.learning_rate)
    final = _mean_bce(net.forward(xs)[1], y)
    pred = MlpPredictor(net.w1, net.b1, net.w2, net.b2, config.head_depths, config.max_depth, mean, std)
    return TrainResult(predictor=pred, initial_loss=initial, final_loss=final)


def predict_depth(predictor: DepthPredictor, features=None) -> int:
    return predictor.predict(features)


class DeviceFeatures:
    """The reference's five predictor features from a running decoder's device state, optionally
    followed by a fixed random projection of the target's tapped last-token hidden state.

    ``update(acc_len, root_probs, hidden)`` takes one step's lagged pinned readback (accepted length
    per request, the pass-0 root candidate probabilities per request, the [B, d] hidden tap or None)
    and returns, per request, the feature vector the next step's depth is predicted from."""

    def __init__(self, batch: int, history: int = 8, alpha: float = 0.4, hidden_dim: int = 0, proj_dim: int = 0,
                 seed: int = 0):
        self.states = [FeatureState(history, alpha) for _ in range(batch)]
        self.proj = None
        if proj_dim > 0:
            if hidden_dim <= 0:
                raise ValueError("a hidden-state projection needs hidden_dim")
            rng = np.random.default_rng(seed)
            self.proj = rng.standard_normal((hidden_dim, proj_dim)) / np.sqrt(hidden_dim)

    @property
    def dim(self) -> int:
        return len(FEATURE_NAMES) + (self.proj.shape[1] if self.proj is not None else 0)

    def update(self, acc_len, root_probs, hidden=None) -> list[np.ndarray]:
        out = []
        for b, (st, n, probs) in enumerate(zip(self.states, acc_len, root_probs)):
            if int(n) >= 1:
                st.observe(int(n))
            f = st.features([(0, float(p)) for p in probs])
            if self.proj is not None:
                h = np.asarray(hidden[b], dtype=np.float64)
                f = np.concatenate([f, (h / (np.linalg.norm(h) + 1e-12)) @ self.proj])
            out.append(f)
        return out
