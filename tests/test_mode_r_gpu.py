"""Mode R on the B200: config C1 with DeviceAlignmentEnv -- the fused DPO kernel's per-pair losses are the
losses the unmodified reference scheduler prioritises and ends fine-tune jobs with. Checked against the fp32
oracle replay of every tick (tests/parity_util.py) and for decision consistency: each fine-tune job ran until
its device loss fell to loss_threshold or it reached max_ft_steps (scheduler.py:191-204)."""
import numpy as np
import pytest
import torch

from parity_util import check_records

pytestmark = pytest.mark.gpu


def test_mode_r_c1_device_losses_drive_decisions(ctx):
    from paper_2510_03283_b200.alignenv import DeviceAlignmentEnv
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.model import HybridModel
    from paper_2510_03283_b200.weights import init_weights
    from paper_2510_03283_b200.workloads import c1

    wl = c1()
    w = init_weights(wl.model, seed=0)
    model = HybridModel(wl.model, wl.train, w, max_slots=256, max_prompt_len=wl.max_prompt_len, prompt_groups=2048)
    args = list(wl.engine_args())
    env = args[5] = DeviceAlignmentEnv.wrap(args[5])
    trace = args[0]
    eng = GpuEngine(*args, model=model, mode="P", record=True)
    eng.run()
    torch.cuda.synchronize()
    st = check_records(eng, w, wl.model, wl.train, label="C1 mode R")
    assert st["ft_ticks"] > 0
    # the env answered with exactly the device's recorded losses
    last = {}
    for rec in eng.records:
        for p, l in zip(rec["batch"].ft_pairs, rec.get("ft_loss", [])):
            last[p.rid] = float(l)
    fts = [r for r in trace if r.pair is not None and r.ft_steps_done > 0]
    assert fts
    for r in fts:
        assert env.pair_loss(r) == last[r.id]
        ended_by_loss = last[r.id] <= env.loss_threshold
        assert ended_by_loss or r.ft_steps_done == wl.sched.max_ft_steps, (r.id, r.ft_steps_done, last[r.id])
    assert env.observed_steps == sum(r.ft_steps_done for r in fts)
    assert np.isfinite(list(last.values())).all()
