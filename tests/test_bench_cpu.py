"""bench.py's host-side contract pieces (no GPU): the timed window is chosen from the unmodified reference's own
timeline so it holds the hybrid iteration (fine-tune ticks at no less than half the trace's rate) for the
driver's step counts, and the `config` object both arms print is the same."""
import types

import numpy as np
import pytest

import bench
from paper_2510_03283_b200.workloads import c2, c4


@pytest.mark.parametrize("steps,warmup", [(20, 5), (8, 3)])
def test_c4_window_holds_fine_tune_ticks(steps, warmup):
    wl = c4()
    skip, comp = bench.plan_window(wl, steps, warmup, wl.bench_skip)
    ft = np.array([c[2] > 0 for c in comp], bool)
    timed = ft[skip + warmup: skip + warmup + steps]
    assert len(timed) == steps
    rate = ft[wl.bench_skip:].mean()
    assert timed.sum() >= max(1, int(np.floor(0.5 * rate * steps)))


def test_c2_window_and_config_identical_across_arms():
    wl = c2()
    skip, _ = bench.plan_window(wl, 20, 5, wl.bench_skip)
    args = types.SimpleNamespace(steps=20, warmup=5)
    a = bench.bench_config(wl, args, skip, 1)
    b = bench.bench_config(wl, args, skip, 1)
    assert a == b and a["timed_ticks"] == [skip + 5, skip + 25]
    assert "model" not in a and a["workload"].startswith("c2")
