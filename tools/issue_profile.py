"""Where the host time of issuing one tick goes (GPU box): record a tape of C2 ticks, then replay it with
the native mace_tick_run call timed separately and the rest cProfiled."""
import cProfile
import ctypes
import os
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("MACE_HOST_PROF", "1")
import torch  # noqa: E402

from paper_2510_03283_b200.engine import GpuEngine  # noqa: E402
from paper_2510_03283_b200.model import HybridModel  # noqa: E402
from paper_2510_03283_b200.weights import init_weights  # noqa: E402
from paper_2510_03283_b200.workloads import WORKLOADS  # noqa: E402
from bench import restore, snapshot  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"](seed=1)
cfg = wl.model
model = HybridModel(cfg, wl.train, init_weights(cfg, 0, "cuda"), max_slots=1024, max_prompt_len=wl.max_prompt_len,
                    max_decode_steps=wl.sched.max_decode_steps, prompt_groups=wl.kv_tokens // 16,
                    decode_pages=1024 * cfg.n_kv_heads * wl.decode_pages_per_head)
eng = GpuEngine(*wl.engine_args(), model=model, mode="P")
eng.keep_outputs = False
eng.run_ticks(wl.bench_skip)
torch.cuda.synchronize()
snap = snapshot(model)
model.tape = []
eng.run_ticks(64)
torch.cuda.synchronize()
tape, model.tape = model.tape, None
L = model.ctx.L
native = [0.0, 0]
f = L.mace_tick_run


def timed(*a):
    t = time.perf_counter()
    r = f(*a)
    native[0] += time.perf_counter() - t
    native[1] += 1
    return r


L.mace_tick_run = timed
hp = (ctypes.c_double * 4)()
for rep in range(3):
    native[:] = [0.0, 0]
    restore(model, snap)
    torch.cuda.synchronize()
    L.mace_debug_host_prof(hp)
    t0 = time.perf_counter()
    model.replay(tape)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"replay: issue {1e3 * (t1 - t0) / 64:.3f} ms/tick, native mace_tick_run {1e3 * native[0] / 64:.3f} "
          f"ms/tick ({native[1]} calls), wall incl. drain {1e3 * (t2 - t0) / 64:.3f} ms/tick")
    L.mace_debug_host_prof(hp)
    print(f"  launches {hp[1] / 64:.0f}/tick {1e6 * hp[0] / max(hp[1], 1):.2f} us each ({1e3 * hp[0] / 64:.3f} ms/tick); "
          f"encodes {hp[3] / 64:.0f}/tick {1e6 * hp[2] / max(hp[3], 1):.2f} us each ({1e3 * hp[2] / 64:.3f} ms/tick)")
restore(model, snap)
pr = cProfile.Profile()
pr.enable()
model.replay(tape)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
