"""Mode R: the real-alignment env -- the device's DPO loss drives the reference's fine-tune decisions.

The reference's env (macesim.alignment.AlignmentEnv, alignment.py:93-172) is a synthetic stand-in: a pair's
loss is dpo_loss of a scalar margin mu + offset (alignment.py:151-166) and a fine-tune step is mu += ft_gain
(alignment.py:168-172). The engine consults it through exactly three calls:

  * ``pair_loss(req)``  -- every priority refresh, for every queued fine-tune request: gamma * L_DPO is part of
    its priority (priority.py:76-81, 108-109, 121-127; Engine._loss_of, engine.py:259-260);
  * ``ft_step(req)``    -- once per executed fine-tune row of a bin (Engine._exec_ft, engine.py:534-536);
  * ``pair_loss(req)``  again in ``check_end`` after ft_step: a job ends when its loss <= loss_threshold or
    after max_ft_steps (scheduler.py:191-204).

``DeviceAlignmentEnv`` keeps the reference's types and fields (it IS an AlignmentEnv: tenants, beta, gamma,
loss_threshold, drift and the held-out eval metrics stay the reference's) but answers those calls with the
B200's numbers: GpuEngine hands it each fine-tune tick's per-pair DPO loss and margin (computed by the fused
DPO kernel from the real policy / pi_ref log-probs, csrc/dpo_adamw.cu), and

  * ``pair_loss`` returns the request's last device loss. Before its first step a pair has no device loss; it
    is seeded with softplus(0) = ln 2, the exact DPO loss while pi_theta == pi_ref (every pair's value at the
    initial weights; SURVEY §7.4.7 "cache the last computed loss per request");
  * ``ft_step`` does not move the model (the masked AdamW already ran on the device for every fine-tune row of
    the tick) and returns the loss of this step. ``check_end`` therefore sees the IN-STEP (pre-update) loss of
    the step just taken -- the cheaper of the two options SURVEY §7.4.7 names; the faithful alternative would
    cost one more forward of every fine-tune pair per tick. The tenant's mu still advances by ft_gain so the
    reference's synthetic held-out evaluation (eval_metrics, win rate / CLPD) keeps its meaning.

Decisions in mode R legitimately differ from a reference run with the synthetic env (different losses); the
scheduler code making them is still the reference's, unmodified.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, fields

import torch

from .refpath import ensure_macesim

ensure_macesim()
from macesim.alignment import AlignmentEnv  # noqa: E402

LN2 = math.log(2.0)


@dataclass(eq=False)
class DeviceAlignmentEnv(AlignmentEnv):
    @classmethod
    def wrap(cls, env: AlignmentEnv) -> "DeviceAlignmentEnv":
        """Mode R over an existing env (same tenants, drift, thresholds)."""
        return cls(**{f.name: getattr(env, f.name) for f in fields(AlignmentEnv)})

    def __post_init__(self):
        self._loss: dict[int, float] = {}
        self._margin: dict[int, float] = {}
        self._steps: dict[int, int] = {}
        self._pending: list = []
        self.observed_steps = 0

    # ---- fed by GpuEngine after each fine-tune tick (device tensors, copied without a stall)
    def observe(self, rids: list[int], loss: torch.Tensor, margin: torch.Tensor) -> None:
        if loss.device.type == "cpu":
            self._store(rids, loss.tolist(), margin.tolist())
            return
        h = torch.empty(2, len(rids), dtype=torch.float32, pin_memory=True)
        h[0].copy_(loss[: len(rids)], non_blocking=True)
        h[1].copy_(margin[: len(rids)], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._pending.append((rids, h, ev))

    def _store(self, rids, losses, margins) -> None:
        for rid, l, m in zip(rids, losses, margins):
            self._loss[rid] = float(l)
            self._margin[rid] = float(m)
        self.observed_steps += len(rids)

    def _resolve(self) -> None:
        while self._pending:
            rids, h, ev = self._pending.pop(0)
            ev.synchronize()
            self._store(rids, h[0].tolist(), h[1].tolist())

    # ---- the reference's env interface (alignment.py:151-172)
    def pair_margin(self, req) -> float:
        super().pair_margin(req)  # the reference's argument checks (workload / pair / tenant)
        if self._pending:
            self._resolve()
        return self._margin.get(req.id, 0.0)

    def pair_loss(self, req) -> float:
        if self._pending:
            self._resolve()
        return self._loss.get(req.id, LN2)

    def ft_step(self, req) -> float:
        super().ft_step(req)  # tenant mu for the reference's synthetic held-out evaluation only
        self._steps[req.id] = self._steps.get(req.id, 0) + 1
        return self.pair_loss(req)

    def forget(self, rid: int) -> None:
        self._loss.pop(rid, None)
        self._margin.pop(rid, None)
        self._steps.pop(rid, None)
