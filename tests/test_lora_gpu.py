"""Per-tenant LoRA adapters through GpuEngine on the B200 (every user / domain
owns an adapter phi_u over the frozen shared base). A multi-tenant C1 trace (the reference's multi-tenant config,
config.py:212-239) runs with one rank-8 adapter per tenant on the top-2 layers:

  * scheduler decisions stay the unmodified reference's (timeline identical to a plain reference Engine run);
  * every tick is replayed by the fp32 oracle and its bf16 emulation (tests/parity_util.py tolerances), including
    the per-tenant AdamW restated bit-exactly;
  * the base model never moves, only the tenants that fine-tuned have moved adapters, and each tenant's adapter
    took exactly as many optimizer steps as ticks carried that tenant's preference pairs.
"""
import dataclasses
import json

import numpy as np
import pytest
import torch

from parity_util import check_records

pytestmark = pytest.mark.gpu

TENANTS = [(0.5, 0.01), (-0.5, 0.05), (0.2, 0.02), (0.0, 0.01)]


def _run(wl, cfg, ticks=None, b_std=0.0, max_slots=256, groups=2048):
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.model import HybridModel
    from paper_2510_03283_b200.weights import init_lora, init_weights

    w = init_weights(cfg, seed=0)
    lw = init_lora(cfg, wl.train, wl.n_tenants, seed=3, b_std=b_std)
    model = HybridModel(cfg, wl.train, w, max_slots=max_slots, max_prompt_len=wl.max_prompt_len,
                        max_decode_steps=wl.sched.max_decode_steps, prompt_groups=groups, n_tenants=wl.n_tenants,
                        lora_weights=lw)
    eng = GpuEngine(*wl.engine_args(), model=model, mode="P", record=True)
    res = eng.run() if ticks is None else eng.run_ticks(ticks)
    torch.cuda.synchronize()
    return eng, res, w


def test_lora_c1_multi_tenant(ctx):
    from macesim.engine import Engine
    from paper_2510_03283_b200.workloads import c1, with_tenants

    wl = with_tenants(c1(), TENANTS, lora_rank=8)
    eng, res, w = _run(wl, wl.model)
    ref = Engine(*wl.engine_args()).run()
    assert json.loads(json.dumps(res.timeline, sort_keys=True)) == json.loads(json.dumps(ref.timeline, sort_keys=True))
    st = check_records(eng, w, wl.model, wl.train, label="C1 LoRA x4 tenants")
    assert st["ft_ticks"] > 10 and st["adamw_bit_exact"] == st["ft_ticks"] and st["first_steps"] > 0
    m = eng.model
    # the frozen base: every base weight (the W part of the augmented / stacked selected-layer weights too)
    D, R = wl.model.d_model, m.lora_R
    for n, t in w.items():
        got = m.w[n]
        if n.endswith(("qkv.w", "up.w")) and got.shape[1] == D + R:
            got = got[:, :D]
        elif n.endswith(("o.w", "down.w")) and got.shape[0] == t.shape[0] + R:
            got = got[: t.shape[0]]
        assert torch.equal(got.cpu(), t), n
    # per-tenant optimizer steps = FT ticks carrying that tenant's pairs; untouched tenants keep their init
    steps = np.zeros(wl.n_tenants, np.int64)
    for rec in eng.records:
        for u in sorted({p.tenant for p in rec["batch"].ft_pairs}):
            steps[u] += 1
    assert (m.tenant_steps == steps).all() and steps.sum() > 0
    r = wl.train.lora_rank
    for n, t0 in m.lora_init.items():
        cur = m.lw[n].float().cpu()
        for u in range(wl.n_tenants):
            moved = not torch.equal(cur[u * r: (u + 1) * r], t0[u * r: (u + 1) * r])
            if steps[u] == 0:
                assert not moved, (n, u)
    # the augmented qkv / up weights carry exactly the bf16 B of every tenant
    for l in m.sel_layers:
        for proj in ("qkv", "up"):
            assert torch.equal(m.w[f"layers.{l}.{proj}.w"][:, D:], m.lw[f"lora.{l}.bt_{proj}"].t())


def test_lora_gpt2_family_active_adapters(ctx):
    """GPT-2 family (biases, GELU fused into the augmented up GEMM, MHA hd 64) with every tenant's adapter non-zero
    from the start, so inference rows of different tenants see different models from the first tick."""
    from paper_2510_03283_b200.config import ModelConfig
    from paper_2510_03283_b200.workloads import c2, with_tenants

    cfg = ModelConfig("gpt2-2l", "gpt2", 2, 768, 12, 12, 64, 3072, 50257, max_pos=1024)
    wl = c2(seed=5, arrival_rate=60.0, duration=4.0)
    wl = dataclasses.replace(wl, model=cfg, trace_cfg=dataclasses.replace(wl.trace_cfg, retrain_rate=0.3))
    wl = with_tenants(wl, TENANTS[:2] + TENANTS[:2], lora_rank=16)
    eng, _, w = _run(wl, cfg, ticks=16, b_std=0.02, max_slots=512, groups=8192)
    st = check_records(eng, w, cfg, wl.train, label="gpt2-2l LoRA x4 tenants")
    assert st["tokens"] > 50 and st["ft_ticks"] > 0 and st["adamw_bit_exact"] == st["ft_ticks"]
