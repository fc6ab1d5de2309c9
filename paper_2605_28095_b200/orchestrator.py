"""Control plane of a SiDP group (host side; no device work).

PAPER.md:228-232 (§4.3 Consistent mode switching): the job orchestrator monitors per-replica
batch sizes and broadcasts one directive so that every rank runs the same mode for every step;
switches are coarse-grained with hysteresis, driven by a hardware-specific threshold B_th.
Rule (reading R13 in DESIGN.md): statistic = max over ranks of the
mean batch over the last `window` steps, evaluated at window boundaries; WaS -> CaS when the
statistic < B_th, CaS -> WaS when it exceeds hysteresis * B_th, both only after `min_dwell`
steps in the current mode.  A decision taken after step t applies from step t + 1.

`ModeController` gathers each rank's batch size every step over `torch.distributed`
(gloo or NCCL — control plane only) so every rank evaluates the identical window and reaches
the identical decision; it then calls `sidp_set_mode(mode, t + 1)` and `sidp_set_batches`.
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


class ModeController:
    def __init__(self, policy: ModePolicy, world: int, initial: int = WAS):
        self.pol = policy
        self.world = world
        self.mode = initial
        self.dwell = 0
        self.step = 0
        self.hist: list[list[int]] = []

    def _decide(self) -> int | None:
        win = self.hist[-self.pol.window:]
        stat = max(sum(b[r] for b in win) / len(win) for r in range(self.world))
        if self.dwell < self.pol.min_dwell:
            return None
        if self.mode == WAS and stat < self.pol.b_threshold:
            return CAS
        if self.mode == CAS and stat > self.pol.b_threshold * self.pol.hysteresis:
            return WAS
        return None

    def observe(self, batches: list[int]) -> int:
        """Record this step's per-rank batches; returns the mode of the NEXT step."""
        assert len(batches) == self.world
        self.hist.append(list(batches))
        self.dwell += 1
        self.step += 1
        if self.step % self.pol.window == 0:
            new = self._decide()
            if new is not None and new != self.mode:
                self.mode = new
                self.dwell = 0
        return self.mode


def gather_batches(local_batch: int, dist=None) -> list[int]:
    """All ranks' batch sizes for this step (one int per rank, control plane)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return [int(local_batch)]
    import torch
    t = torch.tensor([int(local_batch)], dtype=torch.int64)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [int(x.item()) for x in out]


def exchange_handles(ctx, dist=None) -> None:
    """Export this rank's IPC blob, all-gather every rank's, import them."""
    blob = ctx.export_handles()
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        blobs = [blob]
    else:
        blobs = [None] * dist.get_world_size()
        dist.all_gather_object(blobs, blob)
    ctx.import_handles(blobs)
