"""Oracle parity beyond the tiny decoder: the GPT-2 family (LayerNorm, learned positions, GELU, biases,
MHA hd=64) on the C2 trace shape and a Llama GQA decoder (group 4, hd=64, RoPE theta 5e5) on a C3-like
trace, each run through GpuEngine (mode P) for a window of ticks that contains prefill, decode and
fine-tune rows, every tick replayed by the fp32 oracle. Tolerances: tests/parity_util.py."""
import dataclasses

import pytest
import torch

from parity_util import check_records

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


def _check(eng, w, cfg, tcfg, label):
    st = check_records(eng, w, cfg, tcfg, label=label)
    assert st["tokens"] > 50 and st["ft_ticks"] > 0 and 0 in st["kinds"]
    return st


def test_gpt2_family_c2_trace(ctx):
    from paper_2510_03283_b200.config import ModelConfig
    from paper_2510_03283_b200.workloads import c2

    cfg = ModelConfig("gpt2-2l", "gpt2", 2, 768, 12, 12, 64, 3072, 50257, max_pos=1024)
    wl = c2(seed=5, arrival_rate=60.0, duration=4.0)
    wl = dataclasses.replace(wl, model=cfg, trace_cfg=dataclasses.replace(wl.trace_cfg, retrain_rate=0.3))
    eng, w = _run(wl, cfg, ticks=24)
    _check(eng, w, cfg, wl.train, "gpt2-2l")


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
    _check(eng, w, cfg, wl.train, "llama-gqa-2l")
