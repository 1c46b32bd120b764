"""Run the multi-tenant C1 trace with per-tenant LoRA adapters tick by tick (synchronizing after each), printing
the tick composition -- a small driver for compute-sanitizer / debugging. Usage: python tools/lora_probe.py [ticks]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2510_03283_b200.build import build  # noqa: E402
from paper_2510_03283_b200.engine import GpuEngine  # noqa: E402
from paper_2510_03283_b200.model import HybridModel  # noqa: E402
from paper_2510_03283_b200.weights import init_lora, init_weights  # noqa: E402
from paper_2510_03283_b200.workloads import c1, with_tenants  # noqa: E402

build()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
b_std = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
wl = with_tenants(c1(), [(0.5, 0.01), (-0.5, 0.05), (0.2, 0.02), (0.0, 0.01)], lora_rank=8)
cfg = wl.model
model = HybridModel(cfg, wl.train, init_weights(cfg, seed=0), max_slots=256, max_prompt_len=wl.max_prompt_len,
                    prompt_groups=2048, n_tenants=wl.n_tenants,
                    lora_weights=init_lora(cfg, wl.train, wl.n_tenants, seed=3, b_std=b_std))
eng = GpuEngine(*wl.engine_args(), model=model, mode="P")
for i in range(n):
    eng.run_ticks(1)
    torch.cuda.synchronize()
    b = eng.last_batch
    print(f"tick {i}: T={b.T} ft0={b.ft0} n_dec={b.n_dec} R={b.ft_logit_rows.shape[0]} "
          f"pairs={[(p.rid, p.tenant, len(p.prompt), len(p.chosen), len(p.rejected)) for p in b.ft_pairs]} "
          f"caps T/ft/R/dec {model._cap}/{model._ft_cap}/{model._R_cap}/{model._ndec_cap} "
          f"tenant_steps={model.tenant_steps.tolist()}", flush=True)
print("probe ok")
