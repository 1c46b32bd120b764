"""cProfile of the real GpuEngine loop (GPU box): where the host time of a steady-state tick goes."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2510_03283_b200.engine import GpuEngine  # noqa: E402
from paper_2510_03283_b200.model import HybridModel  # noqa: E402
from paper_2510_03283_b200.weights import init_weights  # noqa: E402
from paper_2510_03283_b200.workloads import WORKLOADS  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"](seed=1)
cfg = wl.model
model = HybridModel(cfg, wl.train, init_weights(cfg, 0, "cuda"), max_slots=1024, max_prompt_len=wl.max_prompt_len,
                    max_decode_steps=wl.sched.max_decode_steps, prompt_groups=(1 << 19) // 16,
                    decode_pages=1024 * cfg.n_kv_heads * 12)
eng = GpuEngine(*wl.engine_args(), model=model, mode="P")
eng.keep_outputs = False
eng.run_ticks(150)
torch.cuda.synchronize()
t0 = time.perf_counter()
eng.run_ticks(64)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host submit {1e3 * (t1 - t0) / 64:.2f} ms/tick, wall incl. drain {1e3 * (t2 - t0) / 64:.2f} ms/tick")
pr = cProfile.Profile()
pr.enable()
eng.run_ticks(64)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(40)
pstats.Stats(pr).sort_stats("cumulative").print_stats(40)
