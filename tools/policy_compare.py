"""Measured-cost loop: the reference's policies on the B200 hybrid step, mode M.

Every policy shares Engine._execute (scheduler.py:251-344, engine.py:238-245), so GpuEngine runs each of them on
the real device; in mode M the tick duration is the measured device time of the tick (CostProfile.bin_latency,
cost_model.py:64-69). One trace (C2's shape, shorter) per policy, run to completion; the reference's own metrics
(engine.py:88-143) are reported: decoded throughput over the makespan, TTFT / TBT (TPOT) percentiles, FT latency,
alignment win rate / CLPD, utilisation, rejections.
    python tools/policy_compare.py [--duration 3] [--rate 100] [--policies Hybrid,Periodic,Sync]
"""
import argparse
import gc
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2510_03283_b200.build import build  # noqa: E402
from paper_2510_03283_b200.engine import GpuEngine  # noqa: E402
from paper_2510_03283_b200.model import HybridModel  # noqa: E402
from paper_2510_03283_b200.refpath import ensure_macesim  # noqa: E402
from paper_2510_03283_b200.weights import init_weights  # noqa: E402
from paper_2510_03283_b200.workloads import c2  # noqa: E402

ensure_macesim()
from macesim.scheduler import Policy  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--duration", type=float, default=3.0)
ap.add_argument("--rate", type=float, default=100.0)
ap.add_argument("--policies", default="Hybrid,Periodic,Sync,HybridNoPrefix,HybridNoPrune,NoRetrain")
ap.add_argument("--out", default="gpurun_out/policy_compare.json")
args = ap.parse_args()
build()
rows = []
w = None
for name in args.policies.split(","):
    pol = Policy(name)
    wl = c2(arrival_rate=args.rate, duration=args.duration, policy=pol)
    if w is None:
        w = init_weights(wl.model, seed=0, device="cuda")
    model = HybridModel(wl.model, wl.train, w, device=0, max_slots=2048, max_prompt_len=wl.max_prompt_len,
                        max_decode_steps=wl.sched.max_decode_steps, prompt_groups=wl.kv_tokens // 16,
                        decode_pages=2048 * wl.model.n_kv_heads * wl.decode_pages_per_head)
    eng = GpuEngine(*wl.engine_args(), model=model, mode="M")
    eng.keep_outputs = False
    t0 = time.perf_counter()
    res = eng.run()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    m = res.metrics
    lat = m.latency_summary()
    row = {"policy": name, "requests": eng.admitted, "ticks": eng.ticks_done, "makespan_s": m.makespan_s,
           "decoded_tokens": m.decoded_tokens, "decode_tok_s": m.throughput_tok_s,
           "hybrid_iter_tok_s": sum(eng.tick_tokens) / m.makespan_s if m.makespan_s else 0.0,
           "ttft_p50_ms": lat["ttft_p50"], "ttft_p99_ms": lat["ttft_p99"], "tpot_p50_ms": lat["tbt_p50"],
           "tpot_p99_ms": lat["tbt_p99"], "ft_lat_p50_ms": lat["ft_lat_p50"],
           "ft_steps": int(sum(r.ft_steps_done for r in eng.trace)),
           "slo_attainment": m.slo_attainment, "avg_win_rate": m.avg_win_rate, "avg_clpd": m.avg_clpd,
           "utilization": m.utilization, "rejected": len(m.rejected_ids), "host_wall_s": wall}
    rows.append(row)
    print(json.dumps(row), flush=True)
    del eng, model
    gc.collect()  # the engine holds reference cycles (norm stream, trie); free the device pools now
    torch.cuda.empty_cache()
Path(args.out).parent.mkdir(exist_ok=True)
Path(args.out).write_text(json.dumps(rows, indent=1))
