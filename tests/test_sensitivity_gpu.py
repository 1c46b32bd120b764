"""Alignment-sensitivity-selected update (TrainConfig.sensitivity_topk) on the B200: config C1 with a backward
span of all 4 layers and k = 2. The layers chosen are exactly the top-2 of ||grad W_l|| / ||W_l|| of the first
fine-tune update (recomputed here from the recorded device gradients and the initial weights); from then on
the masked AdamW moves only the chosen layers + the final norm -- bit-exactly as the fp32 restatement of the
kernel on those segments -- and leaves every other parameter untouched."""
import dataclasses

import numpy as np
import pytest
import torch

from parity_util import adamw_np

pytestmark = pytest.mark.gpu


def test_sensitivity_topk_selection_and_masked_update(ctx):
    from paper_2510_03283_b200.config import selected_param_names, sensitivity_ranking
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.model import HybridModel
    from paper_2510_03283_b200.weights import init_weights
    from paper_2510_03283_b200.workloads import c1

    wl = c1()
    tcfg = dataclasses.replace(wl.train, n_selected_layers=4, sensitivity_topk=2)
    w = init_weights(wl.model, seed=0)
    model = HybridModel(wl.model, tcfg, w, max_slots=256, max_prompt_len=wl.max_prompt_len, prompt_groups=2048)
    eng = GpuEngine(*wl.engine_args(), model=model, mode="P", record=True)
    eng.run_ticks(40)
    torch.cuda.synchronize()
    sel = selected_param_names(wl.model, tcfg)
    fts = [r for r in eng.records if "grad" in r]
    assert fts
    rank = sensitivity_ranking(fts[0]["grad"], {n: w[n] for n in sel}, list(range(4)))
    want = sorted(l for l, _ in rank[:2])
    assert model.update_layers == want, (model.update_layers, rank)
    upd = set(model.update_names)
    assert all(n.startswith("final_norm") or int(n.split(".")[1]) in want for n in upd)
    # masked AdamW in situ: updated segments bit-exact, the rest never moves
    sizes = [w[n].numel() for n in sel]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    P = torch.cat([w[n].float().reshape(-1) for n in sel]).numpy()
    M, V = np.zeros_like(P), np.zeros_like(P)
    for step, rec in enumerate(fts, start=1):
        g = torch.cat([rec["grad"][n].reshape(-1) for n in sel]).numpy()
        p2, m2, v2 = adamw_np(P, M, V, g, tcfg.lr, tcfg.beta1, tcfg.beta2, tcfg.eps, tcfg.weight_decay, step)
        for i, n in enumerate(sel):
            a, b = offs[i], offs[i + 1]
            if n in upd:
                P[a:b], M[a:b], V[a:b] = p2[a:b], m2[a:b], v2[a:b]
        assert np.array_equal(rec["master"].numpy().view(np.int32), P.view(np.int32)), f"master, update {step}"
        assert np.array_equal(rec["adam_m"].numpy().view(np.int32), M.view(np.int32))
        assert np.array_equal(rec["adam_v"].numpy().view(np.int32), V.view(np.int32))
    master0 = torch.cat([w[n].float().reshape(-1) for n in sel]).numpy()
    for i, n in enumerate(sel):
        a, b = offs[i], offs[i + 1]
        if n in upd:
            assert not np.array_equal(P[a:b], master0[a:b]), f"{n} was selected but never moved"
        else:
            assert torch.equal(model.w[n].cpu(), w[n]) and np.array_equal(P[a:b], master0[a:b]), n
