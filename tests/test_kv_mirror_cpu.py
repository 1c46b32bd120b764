"""The host mirror of the decode-page allocator (kvmanager.DecodePageMirror) counts exactly the pops and
pushes the device kernels make (csrc/kvpage.cu: decode_alloc / trim / compact / release), restated here page by
page with a real free stack and real page contents, over random decode / prune-trim / compaction / retire
sequences -- it refuses the tick (KvCapacityError, nothing changed) exactly when the device stack would run dry,
and every retained decode slot stays readable at its ring address (rope_kv's write address = the attention
kernels' read address) through compactions."""
import numpy as np
import pytest

from paper_2510_03283_b200.kvmanager import DecodePageMirror, KvCapacityError

PAGE = 16


class DeviceSim:
    """kvpage.cu restated over Python lists (the kernels' per-(slot, head) logic, sequentially)."""

    def __init__(self, S, H, n_pages):
        self.stack = list(range(n_pages))
        self.end = [0] * S
        self.base = [[0] * H for _ in range(S)]
        self.first = [[0] * H for _ in range(S)]
        self.ring = [[[] for _ in range(H)] for _ in range(S)]
        self.H = H
        self.data = {}  # page -> [16] decode slot index stored in each row (K/V stand-in)

    def _addr(self, s, h, j):  # elementwise.cu kv_page_row, decode rows: ring offset relative to dec_base
        rel = j - self.base[s][h]
        return self.ring[s][h][rel // PAGE], rel % PAGE

    def alloc(self, slots):
        for s in slots:
            for h in range(self.H):
                if (self.end[s] - self.base[s][h]) % PAGE == 0:
                    if not self.stack:
                        return False
                    self.ring[s][h].append(self.stack.pop())
        for s in slots:
            for h in range(self.H):  # rope_kv writes the new slot's K/V
                pg, row = self._addr(s, h, self.end[s])
                self.data.setdefault(pg, [None] * PAGE)[row] = (s, h, self.end[s])
            self.end[s] += 1
        return True

    def compact(self, items):
        """kv_compact_move_kernel + kv_compact_commit_kernel: the window moves down to ring offset 0."""
        for s, h in items:
            f, b, e = self.first[s][h], self.base[s][h], self.end[s]
            vals = [self.data[self.ring[s][h][(f - b + i) // PAGE]][(f - b + i) % PAGE] for i in range(e - f)]
            for i, v in enumerate(vals):
                self.data[self.ring[s][h][i // PAGE]][i % PAGE] = v
            old, new = (e - 1 - b) // PAGE + 1, (e - 1 - f) // PAGE + 1
            for _ in range(old - new):
                self.stack.append(self.ring[s][h].pop())
            self.base[s][h] = f

    def check_windows(self, live):
        for s in live:
            for h in range(self.H):
                for j in range(self.first[s][h], self.end[s]):
                    pg, row = self._addr(s, h, j)
                    assert self.data[pg][row] == (s, h, j), (s, h, j)

    def trim(self, slots, kept):
        for s, k in zip(slots, kept):
            for h in range(self.H):
                self.first[s][h] = max(self.first[s][h], self.end[s] - k[h])
                while self.first[s][h] - self.base[s][h] >= PAGE:
                    self.stack.append(self.ring[s][h].pop(0))
                    self.base[s][h] += PAGE

    def release(self, slots):
        for s in slots:
            for h in range(self.H):
                self.stack.extend(self.ring[s][h])
                self.ring[s][h] = []
                self.base[s][h] = self.first[s][h] = 0
            self.end[s] = 0


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_mirror_counts_device_pops_and_pushes(seed):
    rng = np.random.default_rng(seed)
    S, H, N = 24, 4, 110
    dev, mir = DeviceSim(S, H, N), DecodePageMirror(S, H, N)
    live = set()
    refused = compacted = 0
    for step in range(3000):
        op = rng.random()
        if op < 0.7:
            slots = rng.choice(S, int(rng.integers(1, 12)), replace=False)
            before = mir.state()
            try:
                mir.alloc(slots.astype(np.int64))
                ok = True
            except KvCapacityError:
                ok = False
                refused += 1
                after = mir.state()
                assert all(np.array_equal(x, y) for x, y in zip(before[:3], after[:3])) and before[3] == after[3]
            if ok:
                assert dev.alloc(slots.tolist()), "mirror admitted a tick the device could not hold"
                live |= set(slots.tolist())
            else:
                probe = DeviceSim(S, H, 0)
                probe.__dict__.update({k: (v.copy() if isinstance(v, list) else v) for k, v in dev.__dict__.items()})
                probe.stack, probe.ring = list(dev.stack), [[list(r) for r in rr] for rr in dev.ring]
                probe.end, probe.base = list(dev.end), [list(b) for b in dev.base]
                assert not probe.alloc(slots.tolist()), "mirror refused a tick the device could hold"
        elif op < 0.9 and live:
            slots = np.array(sorted(rng.choice(sorted(live), min(len(live), 6), replace=False)), np.int64)
            kept = rng.integers(1, 40, (slots.size, H))
            dev.trim(slots.tolist(), kept.tolist())
            mir.trim(slots, kept)
            if rng.random() < 0.7:  # compaction after the trim (HybridModel.apply_trim)
                items = mir.compact(slots, int(rng.integers(1, 48)))
                dev.compact(items.tolist())
                compacted += len(items)
        elif live:
            slots = np.array(sorted(rng.choice(sorted(live), min(len(live), 3), replace=False)), np.int64)
            dev.release(slots.tolist())
            mir.release(slots)
            live -= set(slots.tolist())
        assert mir.free == len(dev.stack), step
        assert np.array_equal(mir.end, np.array(dev.end)), step
        assert np.array_equal(mir.base, np.array(dev.base)), step
        if step % 50 == 0:
            dev.check_windows(live)
    dev.check_windows(live)
    assert refused > 0, "the sequence should exercise exhaustion"
    assert compacted > 0, "the sequence should exercise compaction"
