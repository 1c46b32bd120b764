"""Oracle parity beyond the tiny decoder: the GPT-2 family (LayerNorm, learned positions, GELU, biases,
MHA hd=64) on the C2 trace shape and a Llama GQA decoder (group 4, hd=64, RoPE theta 5e5) on a C3-like
trace, each run through GpuEngine (mode P) for a window of ticks that contains prefill, decode and
fine-tune rows, every tick replayed by the fp32 oracle. Same tolerances as test_parity_c1_gpu.py."""
import dataclasses

import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(wl, cfg, ticks):
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.model import HybridModel
    from paper_2510_03283_b200.weights import init_weights

    w = init_weights(cfg, seed=0)
    model = HybridModel(cfg, wl.train, w, max_slots=512, max_prompt_len=wl.max_prompt_len,
                        max_decode_steps=wl.sched.max_decode_steps, prompt_groups=8192)
    eng = GpuEngine(*wl.engine_args(), model=model, mode="P", record=True)
    eng.run_ticks(ticks)
    torch.cuda.synchronize()
    return eng, w


def _check(eng, w, cfg, tcfg):
    from oracle.model_ref import TickOracle
    from paper_2510_03283_b200.config import selected_param_names

    orc = TickOracle(cfg, w, tcfg, selected_param_names(cfg, tcfg))
    n_tok = n_tie = n_ft = n_pre = 0
    for rec in eng.records:
        b = rec["batch"]
        toks = rec["dec_tokens"] if rec["dec_tokens"] is not None else []
        logits, ft = orc.run_tick(b, toks, rec["kept_post"])
        n_pre += int((b.seqs[:, 0] == 0).sum())
        if b.n_dec:
            rel = ((rec["dec_logits"] - logits).norm() / logits.norm()).item()
            assert rel <= 1e-2, f"tick {rec['tick']}: logits rel-L2 {rel}"
            top2 = logits.topk(2, dim=-1).values
            gap = (top2[:, 0] - top2[:, 1]).numpy()
            for i, (a, t) in enumerate(zip(logits.argmax(-1).numpy(), toks)):
                n_tok += 1
                if a != t:
                    assert gap[i] < 0.05, f"tick {rec['tick']}: token {t} != oracle {a} (gap {gap[i]})"
                    n_tie += 1
        if ft is not None:
            n_ft += 1
            losses, margins, grads = ft
            dm_max = 0.0
            for i, (lc, lr_, rc, rr) in enumerate(orc.ex.last_lp):
                nc, nr = int(b.pair_rows[i, 1]), int(b.pair_rows[i, 3])
                tol = [5e-4 * abs(x) + 2e-3 * n + 2.5e-2 * n ** 0.5 + 0.02
                       for x, n in zip((lc, lr_, rc, rr), (nc, nr, nc, nr))]
                for a, o, t in zip((*rec["ft_lp"][i], *rec["ref_lp"][i]), (lc, lr_, rc, rr), tol):
                    assert abs(a - o) <= t, f"tick {rec['tick']}: log-prob {a} vs {o}"
                dm = abs(rec["ft_margin"][i] - margins[i])
                assert dm <= sum(tol)
                dm_max = max(dm_max, dm)
            for n, go in grads.items():
                rel = ((rec["grad"][n] - go).norm() / (go.norm() + 1e-12)).item()
                assert rel <= 0.02 + 1.05 * dm_max, f"tick {rec['tick']}: grad {n} rel-L2 {rel}"
            orc.ex.load_state(rec["master"], rec["adam_m"], rec["adam_v"])
    assert n_tok > 50 and n_ft > 0 and n_pre > 0
    assert n_tie <= 0.05 * n_tok
    return n_tok, n_tie, n_ft


def test_gpt2_family_c2_trace(ctx):
    from paper_2510_03283_b200.config import ModelConfig
    from paper_2510_03283_b200.workloads import c2

    cfg = ModelConfig("gpt2-2l", "gpt2", 2, 768, 12, 12, 64, 3072, 50257, max_pos=1024)
    wl = c2(seed=5, arrival_rate=60.0, duration=4.0)
    wl = dataclasses.replace(wl, model=cfg, trace_cfg=dataclasses.replace(wl.trace_cfg, retrain_rate=0.3))
    eng, w = _run(wl, cfg, ticks=24)
    print("gpt2:", _check(eng, w, cfg, wl.train))


def test_llama_gqa_c3_like_trace(ctx):
    from macesim.distributions import parse_dist
    from paper_2510_03283_b200.config import ModelConfig
    from paper_2510_03283_b200.workloads import c3

    cfg = ModelConfig("llama-gqa-2l", "llama", 2, 512, 8, 2, 64, 1024, 32000, max_pos=4096, rope_theta=500000.0)
    wl = c3(seed=7, arrival_rate=40.0, duration=3.0)
    tc = dataclasses.replace(wl.trace_cfg, retrain_rate=0.3, prompt_len_dist=parse_dist("uniform:lo=100,hi=700"),
                             output_len_dist=parse_dist("geometric:mean=24"), vocab_size=cfg.vocab)
    wl = dataclasses.replace(wl, model=cfg, trace_cfg=tc,
                             cache=dataclasses.replace(wl.cache, num_heads=cfg.n_kv_heads))
    eng, w = _run(wl, cfg, ticks=24)
    print("llama-gqa:", _check(eng, w, cfg, wl.train))
