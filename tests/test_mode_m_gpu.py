"""Mode M (the measured clock) and the measured-cost loop on the B200.

  * the clock is the ONLY thing mode M changes: C1 under GpuEngine(mode="M") and an unmodified reference Engine
    whose CostProfile.bin_latency (cost_model.py:64-69, the single point where a tick's duration is formed,
    engine.py:605-611) returns the same measured durations in the same order produce identical timelines;
  * with the device's real head norms (norms="device") and the page-allocator budget (page_budget=True), the
    reference's HeadStats are fed the attention kernel's per-head output norms and the budget handed to Alg. 1
    never exceeds what the free device pages hold;
  * calibration rows measured on the hybrid step fit the reference's own cost model (calibrate, cost_model.py:
    140-205): prefill latency grows with tokens, every fitted coefficient is finite.
"""
import json
import math
from dataclasses import replace

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _model(wl, **kw):
    from paper_2510_03283_b200.model import HybridModel
    from paper_2510_03283_b200.weights import init_weights

    return HybridModel(wl.model, wl.train, init_weights(wl.model, seed=0), max_slots=256,
                       max_prompt_len=wl.max_prompt_len, prompt_groups=2048, **kw)


def test_mode_m_changes_only_the_clock(ctx):
    from macesim.engine import Engine
    from paper_2510_03283_b200.engine import GpuEngine, measured_profile
    from paper_2510_03283_b200.workloads import c1

    wl = c1()
    eng = GpuEngine(*wl.engine_args(), model=_model(wl), mode="M", norms="synthetic", page_budget=False)
    res = eng.run()
    lat = eng.device_ms()
    assert len(lat) == res.metrics.total_iterations and all(x > 0 for x in lat)

    class Replay(Engine):  # the unmodified reference, its bin latency = the B200's measured tick durations
        def _execute(self, plan):
            self.profile._clock[0] = lat[self._k]
            self._k += 1
            super()._execute(plan)

    args = list(wl.engine_args())
    args[1] = measured_profile(args[1])
    args[6] = replace(args[6], scheduler_overhead_ms=0.0)
    ref = Replay(*args)
    ref._k = 0
    out = ref.run()
    assert json.loads(json.dumps(res.timeline, sort_keys=True)) == json.loads(json.dumps(out.timeline, sort_keys=True))
    # and mode M is not mode P: the clock differs from the reference cost model's
    base = Engine(*wl.engine_args()).run()
    assert res.metrics.makespan_s != base.metrics.makespan_s


def test_device_norms_and_page_budget(ctx):
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.workloads import c1

    wl = c1()
    model = _model(wl, decode_pages=256 * 8 * 2)
    eng = GpuEngine(*wl.engine_args(), model=model, mode="M", norms="device", page_budget=True)
    seen = {"budget": 0, "capped": 0, "norms": 0}
    ref_budget = type(eng).__mro__[1]._budget  # macesim Engine._budget (engine.py:268-270)

    def budget():
        b = eng.__class__._budget(eng)
        assert b <= eng.page_budget_mb() + 1e-9
        seen["budget"] += 1
        seen["capped"] += b < ref_budget(eng)
        return b

    eng._budget = budget
    # the norms HeadStats receives each tick are the device's per-KV-head attention-output norms of that tick
    # (sqrt of the mean square over the GQA group of ||o_h|| of the last layer, StepOutputs.head_norm)
    tick_hn = []
    orig_step = model.step

    def step(batch, *a, **k):
        out = orig_step(batch, *a, **k)
        tick_hn.append(None if out.head_norm is None else out.head_norm.double().cpu().numpy())
        return out

    model.step = step
    orig_hs = eng.hstats.step

    def hs_step(slots, steps, norms):
        hn = tick_hn[-1]
        G = wl.model.group
        want = np.sqrt((hn.reshape(hn.shape[0], -1, G) ** 2).mean(-1))
        assert norms.shape[0] <= want.shape[0] and np.isfinite(norms).all() and (norms >= 0).all()
        assert any(np.array_equal(norms[0], w) for w in want)
        seen["norms"] += norms.shape[0]
        return orig_hs(slots, steps, norms)

    eng.hstats.step = hs_step
    res = eng.run()
    torch.cuda.synchronize()
    assert res.metrics.decoded_tokens > 100 and seen["norms"] > 100
    assert seen["budget"] > 0 and seen["capped"] > 0, "the page allocator never bounded the budget"
    top, status = model.kv_status()
    assert status == 0 and top == model.kv_mirror.free


def test_calibration_rows_fit_the_reference_cost_model(ctx, tmp_path):
    from macesim.cost_model import read_profile, write_profile
    from paper_2510_03283_b200.calibration import calibrated, measure_rows, write_csv
    from paper_2510_03283_b200.workloads import c1

    wl = c1()
    model = _model(wl)
    rows = measure_rows(model, wl, prefill_tokens=(64, 256, 1024), decode_batches=(4, 16, 64), decode_ctx=256,
                        ft_lens=((8, 8), (32, 32)), ft_prompt=128, repeats=1)
    kinds = {r[0] for r in rows}
    assert kinds == {"prefill", "decode", "finetune"}
    pre = sorted((r[2], r[3]) for r in rows if r[0] == "prefill")
    assert pre[-1][1] > pre[0][1]  # 1024 prompt tokens take longer than 64
    path = tmp_path / "calib.csv"
    write_csv(rows, path)
    rep = calibrated(path, wl.profile)
    prof = rep.profile
    assert rep.points_per_workload == {"prefill": 3, "decode": 3, "finetune": 2}
    vals = [getattr(prof, f) for f in prof.__dataclass_fields__ if isinstance(getattr(prof, f), float)]
    assert all(math.isfinite(v) for v in vals)
    assert prof.prefill_lat_per_token > 0 and prof.decode_lat_per_step > 0 and prof.ft_lat_per_sample_step > 0
    out = tmp_path / "profile.ini"
    write_profile(prof, out)
    back = read_profile(out)
    assert math.isclose(back.prefill_lat_per_token, prof.prefill_lat_per_token, rel_tol=1e-9)
