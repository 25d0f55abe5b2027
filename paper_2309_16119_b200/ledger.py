"""MemoryLedger and the single-materialization check (lowprec_linear.hpp:36-80,
lowprec_linear.cpp:17-37 + 62-148), host-side accounting around the device
calls.

On the device a pass charges what libmlra actually materializes in HBM
(``mlra_ledger_bytes``, SURVEY §8(b) "Ledger semantics"): WeightMaterialize
the whole bf16 Ŵ (2 B per entry), RowMaterialize / QuantizerMatvec on a
fused format nothing, a plugin hook its slab buffer. ``LayerDims`` without
``device_bytes`` keeps the reference's f64 host arithmetic (N·K·8, K·8, 0), so
the reference's own ledger tests replay unchanged.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from ._lib import MlraError


class Phase(enum.IntEnum):
    Forward = 0
    Backward = 1


@dataclass
class LedgerEvent:
    layer: str
    phase: Phase
    alloc: bool  # False = free
    bytes: int


class MemoryLedger:
    """lowprec_linear.hpp:45-59."""

    def __init__(self):
        self.reset()

    def on_alloc(self, layer: str, phase: Phase, nbytes: int) -> None:
        self._current += int(nbytes)
        self._peak = max(self._peak, self._current)
        self._events.append(LedgerEvent(layer, Phase(phase), True, int(nbytes)))

    def on_free(self, layer: str, phase: Phase, nbytes: int) -> None:
        if nbytes > self._current:
            raise MlraError(5, f"MemoryLedger: free of {nbytes} bytes exceeds current {self._current}")
        self._current -= int(nbytes)
        self._events.append(LedgerEvent(layer, Phase(phase), False, int(nbytes)))

    def reset(self) -> None:
        self._current = 0
        self._peak = 0
        self._events: List[LedgerEvent] = []

    def current_bytes(self) -> int:
        return self._current

    def peak_bytes(self) -> int:
        return self._peak

    def events(self) -> List[LedgerEvent]:
        return self._events


@dataclass
class LayerDims:
    """lowprec_linear.hpp:61-65; ``device_bytes``: what one device pass of this
    layer materializes (``LpLinearContext.ledger_bytes()``), None = the
    reference's f64 host arithmetic."""
    name: str
    d_out: int
    d_in: int
    device_bytes: Optional[int] = None

    @classmethod
    def of(cls, ctx) -> "LayerDims":
        q = ctx.q
        return cls(ctx.layer_name, q.rows, q.cols, ctx.ledger_bytes())


@dataclass
class LedgerReport:
    passed: bool = False
    observed_peak: int = 0
    expected_peak: int = 0
    sum_of_layers: int = 0
    violations: List[str] = field(default_factory=list)


def ledger_assert_single_materialization(ledger: MemoryLedger, layers: Sequence[LayerDims],
                                         strategy) -> LedgerReport:
    """lowprec_linear.cpp:83-148: peak == the largest single layer buffer,
    every alloc freed, never two materialized buffers live at once."""
    from .modulora import MaterializationStrategy as S
    strategy = S(strategy)
    rep = LedgerReport(observed_peak=ledger.peak_bytes())
    device = any(l.device_bytes is not None for l in layers)
    for l in layers:
        weight_bytes = l.d_out * l.d_in * 8
        rep.sum_of_layers += weight_bytes
        if l.device_bytes is not None:
            per_layer = l.device_bytes
        elif strategy == S.WeightMaterialize:
            per_layer = weight_bytes
        elif strategy == S.RowMaterialize:
            per_layer = l.d_in * 8
        else:
            per_layer = 0
        rep.expected_peak = max(rep.expected_peak, per_layer)
    must_record = rep.expected_peak > 0 if device else strategy != S.QuantizerMatvec
    if must_record and not ledger.events():
        rep.violations.append("no materialization events recorded")
    live = live_count = 0
    for i, e in enumerate(ledger.events()):
        if e.alloc:
            live_count += 1
            live += e.bytes
            if live_count > 1:
                rep.violations.append(
                    f"event {i}: layer '{e.layer}' materialized while another buffer is live")
        else:
            if live_count == 0 or e.bytes > live:
                rep.violations.append(f"event {i}: free without matching alloc")
            else:
                live_count -= 1
                live -= e.bytes
    if live != 0:
        rep.violations.append(f"materialized bytes not freed: {live}")
    if rep.observed_peak != rep.expected_peak:
        tail = (" (peak equals the sum over layers)"
                if rep.observed_peak == rep.sum_of_layers and len(layers) > 1 else "")
        rep.violations.append(f"peak {rep.observed_peak} != largest single buffer "
                              f"{rep.expected_peak}{tail}")
    rep.passed = not rep.violations
    return rep
