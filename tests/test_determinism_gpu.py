"""Run-to-run bit-exactness of the hybrid iteration on the B200 (batch-invariant,
reproducible kernels): C1 twice from the same seeds gives the identical greedy token of every decode step, the
identical DPO losses and the identical fp32 masters / Adam moments after every update -- no atomics-order or
scheduling-dependent arithmetic anywhere on the path (attention backward dQ included)."""
import numpy as np
import pytest
import torch

from test_engine_c1_gpu import run_c1

pytestmark = pytest.mark.gpu


def _fingerprint(eng):
    m = eng.model
    torch.cuda.synchronize()
    toks = eng.decoded_tokens()
    ft = [(r["ft_loss"].tobytes(), r["ft_margin"].tobytes()) for r in eng.records if "ft_loss" in r]
    return toks, ft, m.master.cpu().numpy().view(np.int32).copy(), m.m.cpu().numpy().view(np.int32).copy()


def test_c1_bit_identical_across_runs(ctx):
    a = _fingerprint(run_c1(record=True)[0])
    b = _fingerprint(run_c1(record=True)[0])
    assert a[0] == b[0], "greedy tokens differ between runs"
    assert a[1] == b[1], "DPO losses / margins differ between runs"
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3]), "masters / moments differ between runs"


def _gqa_run():
    import dataclasses

    from macesim.distributions import parse_dist
    from paper_2510_03283_b200.config import ModelConfig
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.model import HybridModel
    from paper_2510_03283_b200.weights import init_weights
    from paper_2510_03283_b200.workloads import c3

    cfg = ModelConfig("llama-gqa-2l", "llama", 2, 1024, 16, 4, 128, 2048, 32000, max_pos=4096, rope_theta=500000.0)
    wl = c3(seed=7, arrival_rate=40.0, duration=3.0)
    tc = dataclasses.replace(wl.trace_cfg, retrain_rate=0.4, prompt_len_dist=parse_dist("uniform:lo=300,hi=1500"),
                             output_len_dist=parse_dist("geometric:mean=24"), vocab_size=cfg.vocab)
    wl = dataclasses.replace(wl, model=cfg, trace_cfg=tc, cache=dataclasses.replace(wl.cache, num_heads=cfg.n_kv_heads))
    model = HybridModel(cfg, wl.train, init_weights(cfg, seed=0), max_slots=512, max_prompt_len=wl.max_prompt_len,
                        max_decode_steps=wl.sched.max_decode_steps, prompt_groups=8192)
    eng = GpuEngine(*wl.engine_args(), model=model, mode="P", record=True)
    eng.run_ticks(16)
    return eng


def test_gqa_hd128_bit_identical_across_runs(ctx):
    """hd 128 GQA 16/4 (the tcgen05 attention backward: dQ from several key blocks and query heads per row)."""
    a = _fingerprint(_gqa_run())
    b = _fingerprint(_gqa_run())
    assert sum(len(x) for x in a[1]) > 0, "no fine-tune tick in the window"
    assert a[0] == b[0] and a[1] == b[1]
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3]), "masters / moments differ between runs"
