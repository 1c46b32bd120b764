"""Profile K steady-state hybrid ticks (device replay) for ncu.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/profile_tick.py --workload c2 --steps 8
    ncu --profile-from-start off --set full --clock-control none --import-source on \
        -k regex:attn_decode -c 3 -o gpurun_out/attn python tools/profile_tick.py
"""
import argparse
import sys
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
ap.add_argument("--steps", type=int, default=8)
ap.add_argument("--skip", type=int, default=None)
ap.add_argument("--seed", type=int, default=None)
args = ap.parse_args()
wl = WORKLOADS[args.workload]() if args.seed is None else WORKLOADS[args.workload](seed=args.seed)
args.skip = wl.bench_skip if args.skip is None else args.skip
cfg = wl.model
model = HybridModel(cfg, wl.train, init_weights(cfg, 0, "cuda"), max_slots=1024, max_prompt_len=wl.max_prompt_len,
                    max_decode_steps=wl.sched.max_decode_steps, prompt_groups=wl.kv_tokens // 16,
                    decode_pages=1024 * cfg.n_kv_heads * wl.decode_pages_per_head)
eng = GpuEngine(*wl.engine_args(), model=model, mode="P")
eng.keep_outputs = False
eng.run_ticks(args.skip)
torch.cuda.synchronize()
snap = snapshot(model)
model.tape = []
eng.run_ticks(args.steps)
tape, model.tape = model.tape, None
restore(model, snap)
model.replay(tape)
restore(model, snap)
torch.cuda.synchronize()
model.instrument = []  # record the algorithmic bytes of every decode-attention launch (per layer, in order)
torch.cuda.profiler.start()
model.replay(tape)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
import json  # noqa: E402
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/decode_attn_bytes.json").write_text(json.dumps([b for _, _, b in model.instrument]))
print("ticks", sum(1 for op in tape if op[0] == "step"), "tokens", sum(op[1].total_tokens for op in tape if op[0] == "step"))
