"""The reference's calibrated per-layer cost model (
config.h:33-66, config.cc:23-26,36-118) — host arithmetic, reporting only.

    prefill layer   T(n_new, n_total) = alpha * n_new + beta * n_new * n_total
    transfer layer  X(n)              = gamma * n + delta      (0 for n <= 0)
    decode step     c0 + c1 * sum(kv_lens)                     (0 for an empty batch)

`fit_cost_model` is the reference's least-squares fit (config.cc:60-111:
2x2 normal equations per pair, InvalidArgument on degenerate anchors or on
fewer than two anchors per fit), `DEFAULT_*_ANCHORS` are the paper's measured
anchors the reference ships (config.cc:41-57), and `default_cost_model()`
is `DefaultCostModel()`.  bench.py fits the same X(n) = gamma n + delta to
the per-layer DirectSend times measured on the B200 and reports both
(different hardware and transport: the paper's anchors are A100 + NVSHMEM)."""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

from .kvcache import ErrorCode, SplitserveError

# (n_new, n_total, layer_ms) and (n_tokens, layer_ms), config.cc:41-57
DEFAULT_PREFILL_ANCHORS: Tuple[Tuple[int, int, float], ...] = (
    (500, 1000, 1.247), (500, 3000, 1.391), (500, 5000, 1.564))
DEFAULT_TRANSFER_ANCHORS: Tuple[Tuple[int, float], ...] = (
    (1000, 0.197), (3000, 0.533), (5000, 0.867))


def _invalid(msg: str) -> SplitserveError:
    return SplitserveError(1 + ErrorCode.InvalidArgument, f"InvalidArgument: {msg}")


@dataclass
class CostModel:
    """config.h:40-66 (defaults: c0 = 0.05 ms, c1 = 2e-5 ms per cached token)."""
    alpha: float = 0.0
    beta: float = 0.0
    gamma: float = 0.0
    delta: float = 0.0
    c0: float = 0.05
    c1: float = 2e-5

    def prefill_layer_ms(self, n_new: int, n_total: int) -> float:
        return self.alpha * float(n_new) + self.beta * float(n_new) * float(n_total)

    def transfer_layer_ms(self, n_tokens: int) -> float:
        return 0.0 if n_tokens <= 0 else self.gamma * float(n_tokens) + self.delta

    def decode_layer_ms(self, batch_kv_lens: Sequence[int]) -> float:
        if len(batch_kv_lens) == 0:
            return 0.0
        return self.c0 + self.c1 * float(sum(float(n) for n in batch_kv_lens))

    def validate(self) -> None:
        """config.cc:23-26."""
        if min(self.alpha, self.beta, self.gamma, self.delta, self.c0, self.c1) < 0:
            raise _invalid("cost constants must be non-negative")


@dataclass
class CostFitReport:
    model: CostModel
    prefill_rel_err: List[float] = field(default_factory=list)
    transfer_rel_err: List[float] = field(default_factory=list)
    max_rel_err: float = 0.0


def _least_squares2(rows: Sequence[Tuple[float, float, float]]) -> Tuple[float, float]:
    """y ~ p f1 + q f2 by the 2x2 normal equations, in the reference's
    accumulation order (config.cc:60-77)."""
    a11 = a12 = a22 = b1 = b2 = 0.0
    for f1, f2, y in rows:
        a11 += f1 * f1
        a12 += f1 * f2
        a22 += f2 * f2
        b1 += f1 * y
        b2 += f2 * y
    det = a11 * a22 - a12 * a12
    if not abs(det) > 1e-30:
        raise _invalid("degenerate calibration anchors")
    return (b1 * a22 - b2 * a12) / det, (a11 * b2 - a12 * b1) / det


def fit_cost_model(prefill: Sequence[Tuple[int, int, float]],
                   transfer: Sequence[Tuple[int, float]]) -> CostFitReport:
    """FitCostModel (config.cc:79-111)."""
    if len(prefill) < 2 or len(transfer) < 2:
        raise _invalid("need at least two anchors per fit")
    m = CostModel()
    m.alpha, m.beta = _least_squares2([(float(u), float(u) * float(t), y) for u, t, y in prefill])
    m.gamma, m.delta = _least_squares2([(float(n), 1.0, y) for n, y in transfer])
    rep = CostFitReport(m)
    for u, t, y in prefill:
        err = abs(m.prefill_layer_ms(u, t) - y) / y
        rep.prefill_rel_err.append(err)
        rep.max_rel_err = max(rep.max_rel_err, err)
    for n, y in transfer:
        err = abs(m.transfer_layer_ms(n) - y) / y
        rep.transfer_rel_err.append(err)
        rep.max_rel_err = max(rep.max_rel_err, err)
    return rep


def default_cost_model() -> CostModel:
    """DefaultCostModel (config.cc:113-117)."""
    return fit_cost_model(DEFAULT_PREFILL_ANCHORS, DEFAULT_TRANSFER_ANCHORS).model
