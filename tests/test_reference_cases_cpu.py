"""The reference's own engine- and scheduler-level known answers, run through the drop-in (GpuEngine over
the CPU stand-in device, FastPriorityQueue + fast_schedule_iteration). Each case restates a reference test:
test_engine.py:15-19 (empty trace), 22-39 (single-request closed form), 60-66 (determinism),
test_scheduler.py:102-116 (hand-traced best fit)."""
import json

import pytest

from fakes import FakeModel


def _tiny_engine(trace, seed=0, profile=None, horizon=None):
    from macesim.alignment import AlignmentEnv, TenantParams
    from macesim.cost_model import CostProfile
    from macesim.engine import CacheConfig, EngineConfig
    from macesim.priority import PriorityParams
    from macesim.scheduler import SchedulerConfig
    from paper_2510_03283_b200.config import PRESETS, TrainConfig
    from paper_2510_03283_b200.engine import GpuEngine

    profile = profile or CostProfile(capacity=24576.0, weights_resident=8000.0)
    env = AlignmentEnv.create({0: TenantParams()}, seed=seed)
    fm = FakeModel(PRESETS["tiny"], TrainConfig(), max_prompt_len=4096)
    eng = GpuEngine(trace, profile, SchedulerConfig(), PriorityParams(), CacheConfig(), env,
                    EngineConfig(seed=seed, metrics_interval=2.0), horizon, model=fm, mode="P")
    eng.keep_outputs = False
    return eng


def _ref_engine(trace, seed=0, horizon=None):
    from macesim.alignment import AlignmentEnv, TenantParams
    from macesim.cost_model import CostProfile
    from macesim.engine import CacheConfig, Engine, EngineConfig
    from macesim.priority import PriorityParams
    from macesim.scheduler import SchedulerConfig

    env = AlignmentEnv.create({0: TenantParams()}, seed=seed)
    return Engine(trace, CostProfile(capacity=24576.0, weights_resident=8000.0), SchedulerConfig(), PriorityParams(),
                  CacheConfig(), env, EngineConfig(seed=seed, metrics_interval=2.0), horizon)


def _trace(arrival_rate, retrain_rate, duration, seed):
    from macesim.alignment import TenantParams
    from macesim.distributions import DistSpec
    from macesim.workload import PrefixTreeSpec, TraceConfig, generate_trace

    tc = TraceConfig(arrival_rate=arrival_rate, retrain_rate=retrain_rate, duration=duration, seed=seed,
                     prompt_len_dist=DistSpec("geometric", {"mean": 64}),
                     output_len_dist=DistSpec("geometric", {"mean": 16}),
                     prefix_tree_spec=PrefixTreeSpec(branching=2, depth=3,
                                                     segment_len=DistSpec("constant", {"value": 16})),
                     tenants=(TenantParams().drift_spec(),))
    return generate_trace(tc)


def test_empty_trace_runs_to_empty_metrics():
    res = _tiny_engine([], horizon=0.0).run()
    assert res.metrics.total_iterations == 0
    assert res.metrics.decoded_tokens == 0
    assert res.timeline == []


def test_single_request_ttft_matches_closed_form():
    from macesim.cost_model import CostProfile
    from macesim.workload import Request, WorkloadType

    profile = CostProfile(capacity=24576.0, weights_resident=8000.0)
    req = Request(id=0, tenant=0, workload=WorkloadType.PREFILL, arrival_time=0.5, prompt_tokens=list(range(100)),
                  target_output_len=3)
    eng = _tiny_engine([req], profile=profile, horizon=1.0)
    res = eng.run()
    overhead = profile.iter_overhead + 0.1  # EngineConfig's scheduler overhead constant
    prefill_tick = profile.prefill_lat_per_token * 100 + overhead
    decode_tick = profile.decode_lat_per_step + overhead
    assert res.metrics.ttft_ms[0] == pytest.approx(prefill_tick + decode_tick, rel=1e-9)
    assert res.metrics.tbt_ms[0] == pytest.approx([decode_tick, decode_tick], rel=1e-9)
    assert res.metrics.total_iterations == 4  # 1 prefill tick + 3 decode ticks, each executed on the device
    steps = [c for c in eng.model.calls if c[0] == "step"]
    assert len(steps) == 4
    assert steps[0][1].n_prefill_tokens == 100 and steps[0][1].n_decode_tokens == 0
    assert all(c[1].n_decode_tokens == 1 for c in steps[1:])


def test_run_deterministic_and_identical_to_reference():
    """Two drop-in runs agree with each other and with the unmodified reference Engine (timeline, TTFT,
    CLPD, alignment series) on the reference's determinism case (arrival 15, retrain 0.2, 4 s, seed 9)."""
    a = _tiny_engine(_trace(15.0, 0.2, 4.0, 9), seed=9).run()
    b = _tiny_engine(_trace(15.0, 0.2, 4.0, 9), seed=9).run()
    r = _ref_engine(_trace(15.0, 0.2, 4.0, 9), seed=9).run()
    ta = json.dumps(a.timeline, sort_keys=True)
    assert ta == json.dumps(b.timeline, sort_keys=True) == json.dumps(r.timeline, sort_keys=True)
    assert a.metrics.ttft_ms == b.metrics.ttft_ms == r.metrics.ttft_ms
    assert a.metrics.avg_clpd == r.metrics.avg_clpd
    assert a.alignment_series == r.alignment_series
    assert a.metrics.total_iterations > 20


def test_hand_traced_best_fit_example():
    """Sizes {60, 50, 40} into budget 100: 60 opens B1, 50 opens B2, 40 best-fits B1 (free 40, score 0);
    B1 = {60, 40} runs, {50} is requeued."""
    from macesim.cost_model import WorkloadEstimate
    from macesim.priority import PriorityParams
    from macesim.scheduler import SchedulerConfig
    from macesim.workload import Request, WorkloadType
    from paper_2510_03283_b200.hostfast import FastPriorityQueue, fast_schedule_iteration

    q = FastPriorityQueue(PriorityParams())
    reqs = [Request(id=i, tenant=0, workload=WorkloadType.PREFILL, arrival_time=float(i), prompt_tokens=[1, 2],
                    target_output_len=4) for i in range(3)]
    for r in reqs:  # same workload, earlier arrival = higher priority: pops 0, 1, 2
        q.push(r, 10.0)
    q.refresh(10.0)
    sizes = {0: 60.0, 1: 50.0, 2: 40.0}
    cfg = SchedulerConfig(tau_mem=1.0, tau_task=3, max_decode_batch=10**6, max_ft_batch=10**6)
    plan = fast_schedule_iteration(q, 100.0, cfg, lambda r: WorkloadEstimate(sizes[r.id], 1.0), 10.0)
    assert [x.id for x in plan.bin.tasks] == [0, 2]
    assert [x.id for x in plan.requeued] == [1]
    assert plan.rejected == []
