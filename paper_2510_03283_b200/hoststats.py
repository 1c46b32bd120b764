"""Batched, bit-exact restatement of the reference's per-decode-row KV pruning bookkeeping.

The reference runs, for EVERY decode row of every tick, in Python (engine.py:482-532):
  _synth_norms (engine.py:433-442) -> HeadStats.update (cache.py:291-309) -> allocate_capacity
  (cache.py:318-352) -> prune_decision per head (cache.py:355-362) -> kept[h] trims.
At ~70 us/row this is the largest host cost of a decode-heavy tick (SURVEY §0.6, §7.4 hard part 5).
Here the same arithmetic runs over all decode rows of a tick at once on numpy arrays indexed by the
request's KV slot, in the same fp64 operation order per element (sums accumulated head by head left to
right, like Python's sum), so every kept[h], released count and MB delta is bit-identical to the
reference (tests/test_host_cpu.py compares full runs). Rows hitting allocate_capacity's rare
zero-cap repair branch fall back to the reference function itself.
"""
from __future__ import annotations

import math

import numpy as np

from .refpath import ensure_macesim

ensure_macesim()
from macesim.cache import allocate_capacity  # noqa: E402


def _native():
    from ._lib import lib
    return lib()


class BatchedHeadStats:
    def __init__(self, n_slots: int, n_heads: int, window: int, c_total: int, prune_window: float,
                 norm_tau: float | None):
        self.H, self.W = n_heads, window
        self.c_total = c_total
        self.prune_window = prune_window
        self.norm_tau = norm_tau
        self.ring = np.zeros((n_slots, n_heads, window))
        self.count = np.zeros(n_slots, np.int64)
        self.pos = np.zeros(n_slots, np.int64)
        self.sums = np.zeros((n_slots, n_heads))
        self.current = np.zeros((n_slots, n_heads))
        self.last_used = np.zeros((n_slots, n_heads))
        self.tau = np.full(n_slots, np.nan)
        self.kept = np.zeros((n_slots, n_heads), np.int64)
        self._state_ptrs = None

    def reset(self, slots: np.ndarray) -> None:
        self.count[slots] = 0
        self.pos[slots] = 0
        self.sums[slots] = 0.0
        self.current[slots] = 0.0
        self.last_used[slots] = 0.0
        self.tau[slots] = np.nan if self.norm_tau is None else self.norm_tau
        self.kept[slots] = 0
        self.ring[slots] = 0.0

    def step(self, slots: np.ndarray, steps: np.ndarray, norms: np.ndarray):
        """One decode step for rows ``slots`` (distinct) at decode positions ``steps`` with per-head
        norms [n, H]. Returns (kept [n, H] after trims, released [n]) exactly as the reference. Runs the
        native restatement (csrc/hoststats.cu, mace_host_head_stats); the numpy one below handles the
        allocate_capacity rounding corner and is the test oracle for the native one."""
        n = slots.shape[0]
        slots = np.ascontiguousarray(slots, np.int64)
        steps = np.ascontiguousarray(steps, np.int64)
        norms = np.ascontiguousarray(norms, np.float64)
        kept = np.empty((n, self.H), np.int64)
        released = np.empty(n, np.int64)
        st = self._state_ptrs
        if st is None:  # the state arrays never move: their addresses are taken once
            st = self._state_ptrs = tuple(a.ctypes.data for a in (self.ring, self.count, self.pos, self.sums,
                                                                   self.current, self.last_used, self.tau,
                                                                   self.kept))
        rc = _native().mace_host_head_stats(
            n, self.H, self.W, slots.ctypes.data, steps.ctypes.data, norms.ctypes.data, *st, self.c_total,
            float(self.prune_window), kept.ctypes.data, released.ctypes.data)
        if rc == 1:
            return self.step_numpy(slots, steps, norms)
        if rc != 0:
            raise RuntimeError(f"mace_host_head_stats failed ({rc})")
        return kept, released

    def step_numpy(self, slots: np.ndarray, steps: np.ndarray, norms: np.ndarray):
        """numpy restatement (same arithmetic as the native routine)."""
        H, W = self.H, self.W
        n = slots.shape[0]
        # ---- HeadStats.update (cache.py:291-309)
        tau = self.tau[slots]
        unset = np.isnan(tau)
        if unset.any():
            tot = np.zeros(n)
            for h in range(H):  # Python's sum(): left to right from 0
                tot = tot + norms[:, h]
            tau = np.where(unset, 0.1 * (tot / H), tau)
            self.tau[slots] = tau
        cnt = self.count[slots]
        pos = self.pos[slots]
        full = cnt == W
        hh = np.arange(H)[None, :]
        sums = self.sums[slots]
        oldest = self.ring[slots[:, None], hh, pos[:, None]]      # [n, H] oldest window entries
        sums = np.where(full[:, None], sums - oldest, sums)
        self.ring[slots[:, None], hh, pos[:, None]] = norms
        sums = sums + norms
        self.sums[slots] = sums
        self.current[slots] = norms
        lu = self.last_used[slots]
        lu = np.where(norms >= tau[:, None], steps[:, None].astype(np.float64), lu)
        self.last_used[slots] = lu
        cnt = np.minimum(cnt + 1, W)
        self.count[slots] = cnt
        self.pos[slots] = (pos + 1) % W
        # ---- allocate_capacity(stats.means(), c_total) (cache.py:318-352)
        means = sums / cnt[:, None]
        caps = self._allocate(means)
        # ---- kept += 1; trim where kept > cap and prune_decision (cache.py:355-362)
        kept = self.kept[slots] + 1
        prune = ((steps[:, None] - lu) > self.prune_window) | (norms < tau[:, None])
        trim = (kept > caps) & prune
        released = np.where(trim, kept - caps, 0).sum(1)
        kept = np.where(trim, caps, kept)
        self.kept[slots] = kept
        return kept, released

    def _allocate(self, means: np.ndarray) -> np.ndarray:
        n, H = means.shape
        C = self.c_total
        total = np.zeros(n)
        for h in range(H):
            total = total + means[:, h]
        caps = np.zeros((n, H), np.int64)
        pos_rows = total > 0.0
        # total <= 0: uniform split, remainder to the lowest heads
        if (~pos_rows).any():
            base = C // H
            u = np.full(H, base, np.int64)
            u[: C - base * H] += 1
            caps[~pos_rows] = u
        if pos_rows.any():
            m = means[pos_rows]
            w = m / total[pos_rows][:, None]
            floors = (w * C).astype(np.int64)           # int() truncation of non-negative floats
            c = floors.copy()
            left = C - floors.sum(1)
            order = np.lexsort((np.broadcast_to(np.arange(H), w.shape), -w), axis=1)
            rank = np.empty_like(order)
            np.put_along_axis(rank, order, np.arange(H)[None, :].repeat(order.shape[0], 0), axis=1)
            c += rank < left[:, None]
            # "no head may end at zero slots" (cache.py:345-351): heads in index order, each takes one
            # slot from the donor maximising (caps - floors, caps, -index) among caps >= 2
            jj = np.arange(H)[None, :]
            for h in range(H):
                z = c[:, h] == 0
                if not z.any():
                    continue
                cz, fz = c[z], floors[z]
                # donors sorted by (-(caps - floors), -caps, j) among caps >= 2 (cache.py:348-349): a per-row
                # lexsort on the tuple fields themselves (exact for any c_total / H)
                jb = np.broadcast_to(jj, cz.shape)
                donor = np.lexsort((jb, -cz, -(cz - fz), cz < 2), axis=1)[:, 0]
                cz[np.arange(cz.shape[0]), donor] -= 1
                cz[:, h] += 1
                c[z] = cz
            caps[pos_rows] = c
            # pathological leftover >= H (rounding): defer to the reference implementation
            idx = np.nonzero(pos_rows)[0]
            for r in idx[left >= H]:
                caps[r] = allocate_capacity(means[r].tolist(), C)
        return caps
