"""Orchestrator WaS<->CaS mode policy (oracle; test infrastructure only).

PAPER.md:228-232 (§4.3 Consistent mode switching): the orchestrator monitors
per-replica batch sizes and broadcasts one directive; switches are coarse,
with hysteresis; the threshold B_th is hardware-specific.  Concrete rule and
defaults from SPEC.md:451-459, 468-469 (decide_mode), reading C-A14:

* statistic = max over ranks of the mean live batch over the last `window` steps;
* decisions only at window boundaries;
* WaS -> CaS if statistic < B_th and dwell >= min_dwell;
* CaS -> WaS if statistic > B_th * hysteresis and dwell >= min_dwell;
* a directive decided after step t takes effect from step t+1 on every rank.
"""
from __future__ import annotations

from dataclasses import dataclass

WAS, CAS = 0, 1


@dataclass(frozen=True)
class ModePolicy:
    b_threshold: float
    window: int = 50
    hysteresis: float = 1.5
    min_dwell: int = 100


def decide_mode(pol: ModePolicy, window_batches, current: int, dwell: int):
    """window_batches: list over the window of per-rank batch lists.
    Returns the new mode or None (no change)."""
    if not window_batches:
        return None
    d = len(window_batches[0])
    stat = max(sum(wb[r] for wb in window_batches) / len(window_batches) for r in range(d))
    if dwell < pol.min_dwell:
        return None
    if current == WAS and stat < pol.b_threshold:
        return CAS
    if current == CAS and stat > pol.b_threshold * pol.hysteresis:
        return WAS
    return None


def mode_timeline(pol: ModePolicy, batches_per_step, initial: int = WAS) -> list[int]:
    """mode(t) for every step given per-step per-rank batches (identical on all ranks)."""
    modes = []
    mode = initial
    dwell = 0
    for t in range(len(batches_per_step)):
        modes.append(mode)
        dwell += 1
        if (t + 1) % pol.window == 0:
            new = decide_mode(pol, batches_per_step[t + 1 - pol.window:t + 1], mode, dwell)
            if new is not None and new != mode:
                mode = new
                dwell = 0
    return modes
