"""The CPU oracle pinned against the reference's golden vectors / known answers."""
import json
import math
from pathlib import Path

import numpy as np
import pytest
import torch

GOLD = Path(__file__).parent / "golden"


def test_dpo_scalar_stage_matches_reference_golden():
    from oracle.model_ref import dpo_loss_scalar

    g = json.loads((GOLD / "dpo_golden.json").read_text())
    for k in g["known"]:
        got = dpo_loss_scalar(k["m"], k["beta"])
        assert got == k["ref"]
        if "want" in k:
            assert abs(got - k["want"]) < 1e-12
        else:
            assert got < k["want_below"]
    for s in g["samples"]:
        got = dpo_loss_scalar(s["m"], s["beta"])
        assert got == s["ref"]  # bit-identical to macesim.alignment.dpo_loss
        assert abs(got - s["f128"]) <= 1e-9 * max(1.0, abs(s["f128"]))  # A1 tolerance, test_acceptance.py:47-54


def test_oracle_adamw_matches_torch():
    from oracle.model_ref import adamw_reference

    torch.manual_seed(0)
    p = torch.randn(1000)
    p_t = p.clone().requires_grad_(True)
    opt = torch.optim.AdamW([p_t], lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01)
    m = torch.zeros_like(p)
    v = torch.zeros_like(p)
    for step in range(1, 6):
        g = torch.randn(1000)
        p_t.grad = g.clone()
        opt.step()
        adamw_reference(p, m, v, g, 1e-3, 0.9, 0.999, 1e-8, 0.01, 1 - 0.9 ** step, 1 - 0.999 ** step)
    assert torch.allclose(p, p_t.detach(), rtol=0, atol=1e-6)


def test_oracle_incremental_decode_equals_full_forward():
    """Prefill + decode without pruning must equal one causal forward over [prompt | generated]."""
    from oracle.model_ref import OracleExecutor, OracleModel
    from paper_2510_03283_b200.config import ModelConfig, TrainConfig, selected_param_names
    from paper_2510_03283_b200.weights import init_weights

    for fam in ("llama", "gpt2"):
        cfg = ModelConfig("t", fam, 2, 128, 4, 2 if fam == "llama" else 4, 32, 256, 500, max_pos=256)
        w = init_weights(cfg, seed=1)
        ex = OracleExecutor(cfg, w, TrainConfig(), selected_param_names(cfg, TrainConfig()))
        prompt = list(range(3, 40))
        ex.prefill(7, prompt)
        seq = list(prompt)
        x = prompt[-1]
        for k in range(1, 6):
            logits = ex.decode(7, x, None)
            full, _ = ex.model.forward_seq(seq)
            ref = ex.model.final(full[-1:])[0]
            assert torch.allclose(logits, ref, atol=1e-4, rtol=1e-4)
            x = int(logits.argmax())
            seq.append(x)


def test_head_alloc_known_answers_reference():
    """allocate_capacity / prune_decision known answers recorded from the reference (cache.py:318-362)."""
    from macesim.cache import HeadStats, allocate_capacity, prune_decision

    g = json.loads((GOLD / "head_alloc_golden.json").read_text())
    for c in g["alloc"]:
        assert allocate_capacity(c["means"], c["c_total"]) == c["caps"]
