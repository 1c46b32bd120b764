"""Mode R on CPU: DeviceAlignmentEnv makes the device's per-pair DPO losses the ones the UNMODIFIED reference
scheduler decides with -- check_end (scheduler.py:191-204) retires a fine-tune job exactly when the loss of
its latest step is <= loss_threshold (or at max_ft_steps), and priority refreshes read the same cached losses
(ln 2 before a pair's first step)."""
import math

import numpy as np

from fakes import LossFakeModel


def test_device_losses_drive_check_end_and_priorities():
    from paper_2510_03283_b200.alignenv import LN2, DeviceAlignmentEnv
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.workloads import c1

    wl = c1()

    def loss_of(rid, step):  # rid % 3 == 0 converges at its 2nd step, the rest never go below the threshold
        return 0.1 if (rid % 3 == 0 and step >= 2) else 0.9 - 0.01 * step

    args = list(wl.engine_args())
    env = DeviceAlignmentEnv.wrap(args[5])
    args[5] = env
    trace = args[0]
    fm = LossFakeModel(wl.model, wl.train, max_prompt_len=wl.max_prompt_len, loss_of=loss_of)
    eng = GpuEngine(*args, model=fm, mode="P")
    eng.keep_outputs = False
    seen_before = []
    orig = eng.queue.loss_fn

    def spy(req):
        v = orig(req)
        seen_before.append((req.id, v))
        return v

    eng.queue.loss_fn = spy
    eng.queue.bulk_loss = None
    eng.run()
    fts = [r for r in trace if r.pair is not None]
    assert fts, "C1 has fine-tune requests"
    max_steps = wl.sched.max_ft_steps
    for r in fts:
        want = 2 if r.id % 3 == 0 else max_steps
        assert r.ft_steps_done == want, (r.id, r.ft_steps_done, want)
        assert env.pair_loss(r) == float(np.float32(loss_of(r.id, want)))  # the device's fp32 loss of the last step
    assert env.observed_steps == sum(r.ft_steps_done for r in fts)
    assert any(v == LN2 for _, v in seen_before), "queued pairs without a device step see ln 2"
    assert any(v == float(np.float32(0.9 - 0.01)) for _, v in seen_before), "refreshes read the device losses"
    assert math.isclose(LN2, math.log1p(math.exp(0.0)))
