"""CPU stand-ins for the device side, used by host-logic tests only (no kernels, no numerics).

FakeModel records every device call and simulates the KV *contents* at token granularity: each page
row holds the (token, position) that was written there, so the tests can prove that every sequence's
page table resolves to exactly its own prompt / decode history (the page manager's invariant)."""
from __future__ import annotations

import numpy as np

from paper_2510_03283_b200.batch import PAGE
from paper_2510_03283_b200.model import StepOutputs


class FakeModel:
    def __init__(self, cfg, tcfg=None, max_slots=256, max_prompt_len=4096, prompt_groups=4096):
        self.cfg = cfg
        self.tcfg = tcfg
        self.max_slots = max_slots
        self.maxpp = (max_prompt_len + PAGE - 1) // PAGE
        self.prompt_groups = prompt_groups
        self.h2d_bytes = 0
        self.calls = []
        self.pages: dict[int, list] = {}       # group -> 16 rows of (token, pos) or None
        self.ptab: dict[int, list[int]] = {}
        self.dec: dict[int, list] = {}         # slot -> list of (token, pos) per decode slot
        self.violations: list[str] = []
        self.tape = None

    # ---- replica update protocol (the same calls HybridModel makes; weights are a small fp64 vector so the
    # lockstep tests can check bit-identical replicas without a GPU)
    pg = None
    _w = None

    def _weights(self):
        import torch

        if self._w is None:
            self._w = torch.linspace(-1.0, 1.0, 64, dtype=torch.float64)
        return self._w

    def apply_update(self, local_ft: bool) -> None:
        import torch

        w = self._weights()
        g = torch.full_like(w, float(len(self.calls) % 7 + 1)) if local_ft else torch.zeros_like(w)
        if self.pg is not None:
            import torch.distributed as dist

            dist.all_reduce(g, group=self.pg)
        self.updates = getattr(self, "updates", 0) + 1
        w.sub_(1e-3 * g * w.abs().add(1.0))

    def idle_update(self) -> None:
        self.calls.append(("idle_update",))
        self.apply_update(False)

    def weight_checksum(self) -> int:
        import hashlib

        return int.from_bytes(hashlib.sha256(self._weights().numpy().tobytes()).digest()[:7], "little")

    def step(self, batch, trim=None, ft_global=None):
        self.calls.append(("step", batch))
        has_ft = bool(batch.ft_pairs) and batch.T > batch.ft0
        if has_ft or ft_global:
            self.apply_update(has_ft)
        self.h2d_bytes = batch.packed()[0].size * 4
        for slot, row in zip(batch.ptab_slots.tolist(), batch.ptab_rows.tolist()):
            self.ptab[slot] = row
        for src, dst, n, _ in batch.page_copies.tolist():
            srcp = self.pages.setdefault(src, [None] * PAGE)
            dstp = self.pages.setdefault(dst, [None] * PAGE)
            dstp[:n] = srcp[:n]
        for s in batch.seqs.tolist():
            kind, q0, ql, slot, n_pv = s[:5]
            if kind == 2:
                continue
            for i in range(ql):
                r = q0 + i
                t = int(batch.row_kvi[r])
                tok = int(batch.tokens[r])
                if kind == 0:
                    g = self.ptab[slot][t // PAGE]
                    self.pages.setdefault(g, [None] * PAGE)[t % PAGE] = (tok, int(batch.pos[r]))
                else:
                    d = self.dec.setdefault(slot, [])
                    if t == 0:
                        d.clear()
                    if len(d) != t:
                        self.violations.append(f"decode slot {slot}: index {t} != {len(d)}")
                    d.append((tok, int(batch.pos[r])))
        self.last_batch = batch
        n_dec = batch.n_dec
        return StepOutputs(None, None, None, None, None, None) if n_dec == 0 else StepOutputs(None, None, None, None, None, None)

    def prompt_view(self, slot, n):
        """(token, pos) of prompt positions [0, n) as the device would read them for this slot."""
        tab = self.ptab[slot]
        out = []
        for t in range(n):
            row = self.pages.get(tab[t // PAGE], [None] * PAGE)[t % PAGE]
            out.append(row)
        return out

    def apply_trim(self, slots, kept):
        self.calls.append(("trim", slots, kept))

    def release_slots(self, slots):
        self.calls.append(("release", list(slots)))


class LossFakeModel(FakeModel):
    """FakeModel whose fine-tune ticks return per-pair DPO losses / margins from ``loss_of(rid, step)`` (CPU
    tensors), the way HybridModel.step returns the fused DPO kernel's outputs."""

    def __init__(self, *a, loss_of, **k):
        super().__init__(*a, **k)
        self.loss_of = loss_of
        self.ft_seen: dict[int, int] = {}

    def step(self, batch, trim=None, ft_global=None):
        import torch

        super().step(batch, trim, ft_global)
        if not batch.ft_pairs:
            return StepOutputs(None, None, None, None, None, None)
        ls = []
        for p in batch.ft_pairs:
            k = self.ft_seen[p.rid] = self.ft_seen.get(p.rid, 0) + 1
            ls.append(self.loss_of(p.rid, k))
        loss = torch.tensor(ls, dtype=torch.float32)
        return StepOutputs(None, loss, -loss, None, None, None)
