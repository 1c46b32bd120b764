"""Generate the golden fixtures from the UNMODIFIED reference (run in the build container only).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs (committed):
  dpo_golden.json      macesim.alignment.dpo_loss on the reference's own known answers
                       (test_alignment.py:38-49) + 1000 seeded (margin, beta) pairs (the A1 sample
                       shape of test_acceptance.py:47-54), with np.float128 values.
  c1_reference.json    config C1 run through macesim.engine.Engine unmodified:
                       every timeline record + metrics, and the golden tick-7 bin snapshot.
  head_alloc_golden.json allocate_capacity / prune_decision known answers (test_cache.py:285-298).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from paper_2510_03283_b200.refpath import ensure_macesim  # noqa: E402

ensure_macesim()

from macesim.alignment import AlignmentEnv, MarginSample, TenantParams, dpo_loss  # noqa: E402
from macesim.cache import HeadStats, allocate_capacity, prune_decision  # noqa: E402
from macesim.cost_model import CostProfile  # noqa: E402
from macesim.distributions import parse_dist  # noqa: E402
from macesim.engine import CacheConfig, Engine, EngineConfig  # noqa: E402
from macesim.priority import PriorityParams  # noqa: E402
from macesim.scheduler import SchedulerConfig  # noqa: E402
from macesim.workload import TraceConfig, WorkloadType, generate_trace  # noqa: E402


def c1_objects():
    tcfg = TraceConfig(arrival_rate=10, retrain_rate=0.3, duration=5, seed=0,
                       prompt_len_dist=parse_dist("geometric:mean=64"),
                       output_len_dist=parse_dist("geometric:mean=16"))
    trace = generate_trace(tcfg)
    prof = CostProfile(capacity=24576.0, weights_resident=14000.0)
    env = AlignmentEnv.create({0: TenantParams()}, seed=0)
    return trace, prof, env


def dpo_golden():
    known = [
        {"m": 0.0, "beta": 1.0, "want": float(np.log(2.0))},
        {"m": 1.0, "beta": 2.0, "want": float(np.log1p(np.exp(-2.0)))},
        {"m": 20.0, "beta": 1.0, "want_below": 1e-6},
    ]
    rng = np.random.default_rng(20251003)
    samples = []
    for _ in range(1000):
        m = float(rng.uniform(-30, 30))
        b = float(rng.uniform(0.05, 5.0))
        ref = dpo_loss(MarginSample(m, 0.0), b)
        x = np.float128(-b) * np.float128(m)
        exact = float(np.log1p(np.exp(x)) if x <= 0 else x + np.log1p(np.exp(-x)))
        samples.append({"m": m, "beta": b, "ref": ref, "f128": exact})
    for k in known:
        k["ref"] = dpo_loss(MarginSample(k["m"], 0.0), k["beta"])
    return {"known": known, "samples": samples}


def c1_run():
    trace, prof, env = c1_objects()
    snap = {}

    class Probe(Engine):
        def _execute(self, plan):
            if self.tick_index == 7:
                rows = []
                for r in plan.bin.tasks:
                    rs = self.state[r.id]
                    rows.append({
                        "id": r.id, "workload": r.workload.value, "prompt_len": len(r.prompt_tokens),
                        "decode_pos": r.decode_pos, "ft_steps_done": r.ft_steps_done,
                        "cached_prefix": self.trie.cached_prefix_len(r.prompt_tokens) if r.workload is WorkloadType.PREFILL else None,
                        "kept": list(rs.kept) if rs.kept else None,
                        "priority": r.priority_state.value,
                    })
                snap.update({"clock": self.clock, "budget": self._budget(), "rows": rows})
            super()._execute(plan)

    eng = Probe(trace, prof, SchedulerConfig(), PriorityParams(), CacheConfig(weak_scale=0.05), env,
                EngineConfig(seed=0), metrics_horizon=5.0)
    res = eng.run()
    m = res.metrics
    return {
        "n_requests": len(trace),
        "ticks": m.total_iterations,
        "decoded_tokens": m.decoded_tokens,
        "makespan_s": m.makespan_s,
        "timeline": res.timeline,
        "tick7": snap,
        "ttft_ms": {str(k): v for k, v in m.ttft_ms.items()},
        "ft_latency_ms": {str(k): v for k, v in m.ft_latency_ms.items()},
    }


def head_alloc_golden():
    cases = [([2, 1, 1], 10), ([3, 1], 8), ([0, 0, 0], 10), ([5.0, 0.0, 0.0, 0.0], 8), ([1e-9, 1.0], 4)]
    out = [{"means": m, "c_total": c, "caps": allocate_capacity(m, c)} for m, c in cases]
    st = HeadStats(4, 3)
    prunes = []
    for t, norms in enumerate([[1.0, 1.0, 0.01, 1.0], [1.0, 0.5, 0.0, 0.02], [0.9, 1.1, 0.0, 0.0]], start=1):
        st.update(norms, t)
        prunes.append({"t": t, "norms": norms, "tau": st.tau, "means": st.means(),
                       "decisions": [prune_decision(t, h, st, 2, st.tau) for h in range(4)]})
    return {"alloc": out, "prune": prunes}


if __name__ == "__main__":
    (HERE / "dpo_golden.json").write_text(json.dumps(dpo_golden(), indent=0))
    (HERE / "c1_reference.json").write_text(json.dumps(c1_run(), indent=0, sort_keys=True))
    (HERE / "head_alloc_golden.json").write_text(json.dumps(head_alloc_golden(), indent=1))
    print("wrote", sorted(p.name for p in HERE.glob("*.json")))
