"""The host mirror of the decode-page allocator (kvmanager.DecodePageMirror) counts exactly the pops and
pushes the device kernels make (csrc/kvpage.cu: decode_alloc / trim / release), restated here page by
page with a real free stack, over random decode / prune-trim / retire sequences -- and it refuses the
tick (KvCapacityError, nothing changed) exactly when the device stack would run dry."""
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

    def alloc(self, slots):
        for s in slots:
            for h in range(self.H):
                if (self.end[s] - self.base[s][h]) % PAGE == 0:
                    if not self.stack:
                        return False
                    self.ring[s][h].append(self.stack.pop())
        for s in slots:
            self.end[s] += 1
        return True

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
    refused = 0
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
        elif live:
            slots = np.array(sorted(rng.choice(sorted(live), min(len(live), 3), replace=False)), np.int64)
            dev.release(slots.tolist())
            mir.release(slots)
            live -= set(slots.tolist())
        assert mir.free == len(dev.stack), step
        assert np.array_equal(mir.end, np.array(dev.end)), step
        assert np.array_equal(mir.base, np.array(dev.base)), step
    assert refused > 0, "the sequence should exercise exhaustion"
