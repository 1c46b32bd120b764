"""Per-tenant LoRA adapters on the CPU: the adapter layout, the oracle's
adapter semantics (tenant masking, pi_ref = the frozen base, per-tenant AdamW) and the multi-tenant workload
(the reference's multi-tenant config, config.py:212-239 / test_cli.py:238-256)."""
import dataclasses

import numpy as np
import torch

from oracle.model_ref import OracleExecutor
from paper_2510_03283_b200.config import ModelConfig, TrainConfig, lora_shapes, trainable_param_names
from paper_2510_03283_b200.weights import init_lora, init_weights
from paper_2510_03283_b200.workloads import c1, with_tenants

CFG = ModelConfig("lora-tiny", "llama", 2, 64, 4, 2, 16, 128, 512, max_pos=512)
TC = TrainConfig(n_selected_layers=1, lora_rank=8, lr=1e-2)


def _exec(n_tenants=3, b_std=0.0):
    w = init_weights(CFG, seed=1)
    w.update(init_lora(CFG, TC, n_tenants, seed=2, b_std=b_std))
    return OracleExecutor(CFG, w, TC, trainable_param_names(CFG, TC, n_tenants)), n_tenants


def test_layout_and_init():
    shapes = lora_shapes(CFG, TC, 3)
    R = 3 * 8
    assert shapes == {
        "lora.1.a_qkv": (R, 64), "lora.1.bt_qkv": (R, CFG.qkv_dim), "lora.1.a_o": (R, 64), "lora.1.bt_o": (R, 64),
        "lora.1.a_up": (R, 64), "lora.1.bt_up": (R, CFG.up_dim), "lora.1.a_down": (R, 128), "lora.1.bt_down": (R, 64)}
    lw = init_lora(CFG, TC, 3, seed=2)
    assert all(float(t.abs().sum()) == 0 for n, t in lw.items() if ".bt_" in n)  # B = 0: every tenant = base
    assert all(float(t.abs().sum()) > 0 for n, t in lw.items() if ".a_" in n)
    assert trainable_param_names(CFG, TC, 3) == list(shapes)
    assert TC.lora_scale == 16.0 / 8


def test_zero_b_is_the_base_model_and_tenants_differ_otherwise():
    ex, _ = _exec(b_std=0.0)
    prompt, resp = [5, 6, 7, 8], [9, 10, 11]
    with torch.no_grad():
        base = float(ex.model.seq_logprob(prompt, resp))
        assert all(float(ex.model.seq_logprob(prompt, resp, tenant=u)) == base for u in range(3))
    ex, _ = _exec(b_std=0.5)
    with torch.no_grad():
        lps = [float(ex.model.seq_logprob(prompt, resp, tenant=u)) for u in range(3)]
        assert float(ex.model.seq_logprob(prompt, resp)) == base  # no tenant: the frozen base (pi_ref)
    assert len(set(lps)) == 3 and all(lp != base for lp in lps)


def test_dpo_grads_touch_only_the_pair_tenant_rows_and_adamw_is_per_tenant():
    ex, T = _exec(b_std=0.5)
    r = TC.lora_rank
    pairs = [(0, [1, 2, 3], [4, 5], [6, 7], 1)]
    losses, margins, grads = ex.dpo_step(pairs)
    assert len(losses) == 1
    for n, g in grads.items():
        rows = g.abs().sum(1)
        own = rows[r: 2 * r]
        assert float(rows.sum() - own.sum()) == 0.0, n  # other tenants' adapter rows get no gradient
        assert float(own.sum()) > 0.0, n
    before = {n: t.clone() for n, t in ex.master.items()}
    ex.adamw(grads, tenants=[1])
    ex.adamw(grads, tenants=[1, 2])
    assert ex.tenant_steps == {1: 2, 2: 1}
    for n in ex.selected:
        d = (ex.master[n] - before[n]).abs().sum(1)
        assert float(d[:r].sum()) == 0.0  # tenant 0 never stepped
        assert float(d[r: 2 * r].sum()) > 0.0


def test_zero_b_first_step_trains_b_only():
    ex, _ = _exec(b_std=0.0)
    _, margins, grads = ex.dpo_step([(0, [1, 2, 3], [4, 5], [6, 7], 2)])
    assert margins[0] == 0.0  # pi_theta == pi_ref while B == 0
    for n, g in grads.items():
        if ".a_" in n:
            assert float(g.abs().sum()) == 0.0, n  # dA = dZ^T X with dZ = dY B = 0
        else:
            assert float(g.abs().sum()) > 0.0, n


def test_multi_tenant_workload():
    wl = with_tenants(c1(), [(0.5, 0.01), (-0.5, 0.05), (0.2, 0.02), (0.0, 0.01)], lora_rank=8)
    assert wl.n_tenants == 4 and wl.train.lora_rank == 8
    trace = wl.trace()
    assert {r.tenant for r in trace} == {0, 1, 2, 3}
    env = wl.env()
    assert sorted(env.tenants) == [0, 1, 2, 3]
    assert env.tenants[1].params.mu0 == -0.5 and env.tenants[1].params.drift_rate == 0.05
    # the single-tenant workloads are unchanged
    assert c1().n_tenants == 1 and c1().train.lora_rank is None
    assert dataclasses.replace(wl.train, lora_rank=None).lora_scale == 0.0


def test_packed_batch_carries_row_tenants():
    from paper_2510_03283_b200.batch import TickBatch

    z = lambda *s: np.zeros(s, np.int32)  # noqa: E731
    b = TickBatch(tokens=z(5), pos=z(5), row_seq=z(5), row_kvi=z(5), seqs=z(1, 8), tc_items=z(0, 4),
                  dec_items=z(0, 4), dec_slots=z(0), dec_rows=z(0), ptab_slots=z(0), ptab_rows=z(0, 4),
                  page_copies=z(0, 4), ft0=5, row_tenant=np.array([0, 1, 2, 1, 0], np.int32))
    buf, layout = b.packed()
    off, shape = layout["row_tenant"]
    assert shape == (5,) and buf[off: off + 5].tolist() == [0, 1, 2, 1, 0]
