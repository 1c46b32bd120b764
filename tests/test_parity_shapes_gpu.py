"""Sampled-tick parity at the FULL shapes the bench runs (BASELINE configs C2, C3, C4): GPT-2 small (12
layers, d768, MHA hd64, vocab 50257), Llama-3.2-1B (16 layers, d2048, GQA 32/8, hd64, vocab 128256) and
Llama-3-8B (32 layers, d4096, GQA 32/8, hd128, SwiGLU F=14336, vocab 128256: CTA-pair GEMMs, the fused SwiGLU
epilogue and hd128 paged attention inside real ticks).

Each workload's own trace generator (same prompt/output distributions, a short arrival window with a higher
retrain rate so a handful of ticks holds prefill, decode AND fine-tune rows) drives GpuEngine in mode P; the
ticks up to the first tick that carries decode and fine-tune rows together are replayed by the fp32 oracle
with the strict tolerances of tests/parity_util.py. C2 replays on the CPU; C3 / C4 run the same fp32
restatement through torch on the GPU (cuBLAS fp32, TF32 off) -- see oracle/model_ref.py:TickOracle."""
import dataclasses

import pytest
import torch

from parity_util import check_records

pytestmark = pytest.mark.gpu


def _wl(name):
    from paper_2510_03283_b200.workloads import c2, c3, c4

    if name == "c2":
        wl = c2(seed=11, arrival_rate=25.0, duration=0.5)
    elif name == "c3":
        wl = c3(seed=12, arrival_rate=12.0, duration=0.4)
    else:
        wl = c4(seed=13, arrival_rate=12.0, duration=0.4)
    return dataclasses.replace(wl, trace_cfg=dataclasses.replace(wl.trace_cfg, retrain_rate=0.5))


@pytest.mark.parametrize("name,oracle_dev", [("c2", "cpu"), ("c3", "cuda"), ("c4", "cuda"), ("c4-lora", "cuda")])
def test_full_shape_sampled_ticks(ctx, name, oracle_dev):
    """c4-lora: the bench's LoRA line (4 tenants, rank 16, every adapter non-zero from the start) at the 8B shape."""
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.model import HybridModel
    from paper_2510_03283_b200.weights import init_weights

    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    wl = _wl(name.split("-")[0])
    lora = {}
    if name.endswith("-lora"):
        from paper_2510_03283_b200.weights import init_lora
        from paper_2510_03283_b200.workloads import with_tenants

        wl = with_tenants(wl, [(0.5, 0.01), (-0.5, 0.05), (0.2, 0.02), (0.0, 0.01)], lora_rank=16)
        lora = dict(n_tenants=wl.n_tenants, lora_weights=init_lora(wl.model, wl.train, wl.n_tenants, seed=5, b_std=0.01))
    cfg = wl.model
    w = init_weights(cfg, seed=0, device="cpu" if name == "c2" else "cuda")
    model = HybridModel(cfg, wl.train, w, max_slots=64, max_prompt_len=wl.max_prompt_len,
                        max_decode_steps=wl.sched.max_decode_steps, prompt_groups=64 * wl.max_prompt_len // 16, **lora)
    eng = GpuEngine(*wl.engine_args(), model=model, mode="P", record=True)
    for _ in range(12):  # until a tick carries decode and fine-tune rows together (or 12 ticks)
        if eng.run_ticks(1) == 0:
            break
        b = eng.records[-1]["batch"]
        if b.n_dec and b.ft_pairs:
            break
    torch.cuda.synchronize()
    st = check_records(eng, w, cfg, wl.train, device=oracle_dev, label=f"{name} full shape ({cfg.name})")
    assert {0, 1, 2} <= set(st["kinds"]), st["kinds"]
    assert st["ft_ticks"] >= 1 and st["tokens"] >= 1
