"""e2e host time of C2 ticks on the GPU box, split into model.step, the native tick call and its kernel
launches (MACE_HOST_PROF). Usage: python tools/e2e_native_split.py"""
import os, sys, time, ctypes
os.environ["MACE_HOST_PROF"] = "1"
sys.path.insert(0, "/root/repo")
import torch
from paper_2510_03283_b200.engine import GpuEngine
from paper_2510_03283_b200.model import HybridModel
from paper_2510_03283_b200.weights import init_weights
from paper_2510_03283_b200.workloads import WORKLOADS
wl = WORKLOADS["c2"](seed=1)
cfg = wl.model
model = HybridModel(cfg, wl.train, init_weights(cfg, 0, "cuda"), max_slots=1024, max_prompt_len=wl.max_prompt_len,
                    max_decode_steps=wl.sched.max_decode_steps, prompt_groups=wl.kv_tokens // 16,
                    decode_pages=1024 * cfg.n_kv_heads * wl.decode_pages_per_head)
eng = GpuEngine(*wl.engine_args(), model=model, mode="P")
eng.run_ticks(150)
torch.cuda.synchronize()
L = model.ctx.L
acc = {"tick": 0.0, "step": 0.0}
f = L.mace_tick_run
def timed(*a):
    t = time.perf_counter(); r = f(*a); acc["tick"] += time.perf_counter() - t; return r
L.mace_tick_run = timed
st = model.step
def step(*a, **k):
    t = time.perf_counter(); r = st(*a, **k); acc["step"] += time.perf_counter() - t; return r
model.step = step
hp = (ctypes.c_double * 4)()
L.mace_debug_host_prof(hp)
t0 = time.perf_counter()
eng.run_ticks(64)
t1 = time.perf_counter()
L.mace_debug_host_prof(hp)
print(f"e2e host {1e3*(t1-t0)/64:.3f} ms/tick; model.step {1e3*acc['step']/64:.3f}; native tick {1e3*acc['tick']/64:.3f}; "
      f"launch {1e6*hp[0]/max(hp[1],1):.2f} us x {hp[1]/64:.0f}/tick = {1e3*hp[0]/64:.3f} ms")
