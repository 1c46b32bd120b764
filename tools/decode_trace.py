"""Item timeline of one C2 decode-attention launch (trace build): per-warp busy time, tail, per-item rate."""
import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["MACE_LIB"] = "libmace_b200_dtrace.so"
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_03283_b200.build import build  # noqa: E402

build(variant="dtrace", defines=("MACE_DEC_TRACE",))
from bench import restore, snapshot  # noqa: E402
from paper_2510_03283_b200.engine import GpuEngine  # noqa: E402
from paper_2510_03283_b200.model import HybridModel  # noqa: E402
from paper_2510_03283_b200.weights import init_weights  # noqa: E402
from paper_2510_03283_b200.workloads import WORKLOADS  # noqa: E402

wl = WORKLOADS["c2"]()
cfg = wl.model
model = HybridModel(cfg, wl.train, init_weights(cfg, 0, "cuda"), max_slots=1024, max_prompt_len=wl.max_prompt_len,
                    max_decode_steps=wl.sched.max_decode_steps, prompt_groups=wl.kv_tokens // 16,
                    decode_pages=1024 * cfg.n_kv_heads * wl.decode_pages_per_head)
eng = GpuEngine(*wl.engine_args(), model=model, mode="P")
eng.keep_outputs = False
eng.run_ticks(wl.bench_skip)
torch.cuda.synchronize()
tr = torch.zeros(1 << 16, 4, dtype=torch.int64, device="cuda")
model.ctx.L.mace_debug_decode_trace.argtypes = [ctypes.c_void_p]
model.ctx.L.mace_debug_decode_trace(tr.data_ptr())
eng.run_ticks(1)  # every layer overwrites the trace: the last layer's launch remains
torch.cuda.synchronize()
t = tr.cpu().numpy()
t = t[t[:, 1] > 0]
t0 = t[:, 0].min()
st, en, pg, wid = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, t[:, 2], t[:, 3]
span = en.max()
print(f"items {len(t)}  span {span:.1f} us  pages {pg.sum()}  bytes {pg.sum() * 4096 / 1e6:.1f} MB "
      f"-> {pg.sum() * 4096 / span / 1e3:.0f} GB/s over the span")
fin = np.sort(en)
for q in (0.5, 0.9, 0.99):
    print(f"  {int(q * 100)}% of items done at {fin[int(q * (len(fin) - 1))]:.1f} us")
per = {}
for s_, e_, w in zip(st, en, wid):
    per.setdefault(w, []).append((s_, e_))
busy_end = np.array([max(e for _, e in v) for v in per.values()])
print(f"warps {len(per)}; warp finish: min {busy_end.min():.1f} median {np.median(busy_end):.1f} max {busy_end.max():.1f} us")
first_start = np.array([min(s for s, _ in v) for v in per.values()])
print(f"warp first start: min {first_start.min():.2f} median {np.median(first_start):.2f} max {first_start.max():.2f} us")
rate = pg * 4096 / np.maximum(en - st, 1e-3) / 1e3
print(f"per-item GB/s (one warp): median {np.median(rate):.1f}; item us median {np.median(en - st):.1f} max {(en - st).max():.1f}")
