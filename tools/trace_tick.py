"""Kernel timeline of K steady-state ticks (device replay) under CUPTI via torch.profiler.

Reports the replay span, the sum of kernel busy time (union of kernel intervals), the idle gaps
and the host issue time per tick, so host-bound vs device-bound is measured, not guessed.
    python tools/trace_tick.py --workload c2 --steps 16
"""
import argparse
import json
import sys
import time
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import restore, snapshot  # noqa: E402
from paper_2510_03283_b200.engine import GpuEngine  # noqa: E402
from paper_2510_03283_b200.model import HybridModel  # noqa: E402
from paper_2510_03283_b200.weights import init_weights  # noqa: E402
from paper_2510_03283_b200.workloads import WORKLOADS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--steps", type=int, default=16)
ap.add_argument("--skip", type=int, default=150)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--out", default="gpurun_out/trace_summary.json")
args = ap.parse_args()
wl = WORKLOADS[args.workload](seed=args.seed)
cfg = wl.model
model = HybridModel(cfg, wl.train, init_weights(cfg, 0, "cuda"), max_slots=1024, max_prompt_len=wl.max_prompt_len,
                    max_decode_steps=wl.sched.max_decode_steps, prompt_groups=(1 << 19) // 16,
                    decode_pages=1024 * cfg.n_kv_heads * 12)
eng = GpuEngine(*wl.engine_args(), model=model, mode="P")
eng.keep_outputs = False
eng.run_ticks(args.skip)
torch.cuda.synchronize()
snap = snapshot(model)
model.tape = []
eng.run_ticks(args.steps)
tape, model.tape = model.tape, None
n_ticks = sum(1 for op in tape if op[0] == "step")
restore(model, snap)
model.replay(tape)
restore(model, snap)
torch.cuda.synchronize()
# host issue cost with an idle device: one tick at a time, synchronized between ticks
issue = []
for op in tape:
    if op[0] != "step":  # trims / releases / idle updates keep the device page state consistent: replay, untimed
        model.replay([op])
        continue
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    model.step(op[1], ft_global=op[2])
    issue.append(time.perf_counter() - t0)
torch.cuda.synchronize()
restore(model, snap)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    model.replay(tape)
    torch.cuda.synchronize()
Path("gpurun_out").mkdir(exist_ok=True)
trace = "gpurun_out/trace.json"
prof.export_chrome_trace(trace)
ev = json.load(open(trace))["traceEvents"]
kern = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
kern.sort(key=lambda e: e["ts"])
t0, t1 = kern[0]["ts"], max(e["ts"] + e["dur"] for e in kern)
busy, cur_s, cur_e = 0.0, None, None
for e in kern:
    s, f = e["ts"], e["ts"] + e["dur"]
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, f
    else:
        cur_e = max(cur_e, f)
busy += cur_e - cur_s
by = defaultdict(lambda: [0.0, 0])
for e in kern:
    n = e["name"].split("(")[0][:70]
    by[n][0] += e["dur"]
    by[n][1] += 1
tot = sum(v[0] for v in by.values())
summary = {
    "workload": args.workload, "ticks": n_ticks, "span_us_per_tick": (t1 - t0) / n_ticks,
    "busy_us_per_tick": busy / n_ticks, "idle_frac": 1 - busy / (t1 - t0),
    "kernels_per_tick": len(kern) / n_ticks, "host_issue_us_per_tick_idle_device": 1e6 * sum(issue) / len(issue),
    "top": [(n, v[0] / n_ticks, v[1] / n_ticks, v[0] / tot) for n, v in sorted(by.items(), key=lambda kv: -kv[1][0])[:30]],
}
Path(args.out).write_text(json.dumps(summary, indent=1))
print(json.dumps({k: v for k, v in summary.items() if k != "top"}, indent=1))
for n, us, cnt, fr in summary["top"]:
    print(f"{us:9.1f} us/tick {cnt:6.1f}x {100 * fr:5.1f}%  {n}")
