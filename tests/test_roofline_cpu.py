"""Whole-tick roofline accounting (paper_2510_03283_b200/roofline.py): the visible causal pairs of prefill and
preference-pair sequences against a brute-force count of the attention mask the kernels apply."""
import numpy as np

from paper_2510_03283_b200.batch import KIND_DECODE, KIND_FT, KIND_PREFILL
from paper_2510_03283_b200.roofline import causal_pairs


def _brute(kind, q, kv, h0, hl):
    n = 0
    for i in range(q):
        t = kv - q + i  # absolute position of query row i
        for k in range(t + 1):
            if kind == KIND_FT and hl > 0 and t >= h0 + hl and h0 <= k < h0 + hl:
                continue
            n += 1
    return n


def test_causal_pairs_matches_mask():
    rows = [(KIND_PREFILL, 0, 37, 3, 0, 37, 0, 0),      # whole prompt
            (KIND_PREFILL, 37, 20, 4, 0, 91, 0, 0),     # suffix of a shared prefix: 71 cached keys
            (KIND_DECODE, 57, 1, 5, 0, 300, 0, 0),      # paged decode: not tensor-core attention
            (KIND_FT, 58, 5 + 3 + 1 + 4, -1, 0, 13, 4, 4),  # P=5, n_c=3, n_r=4
            (KIND_FT, 71, 2 + 1 + 1 + 1, -1, 0, 5, 1, 2)]
    seqs = np.asarray(rows, np.int32)
    pre, ft = causal_pairs(seqs)
    assert pre == _brute(KIND_PREFILL, 37, 37, 0, 0) + _brute(KIND_PREFILL, 20, 91, 0, 0)
    assert ft == _brute(KIND_FT, 13, 13, 4, 4) + _brute(KIND_FT, 5, 5, 1, 2)


def test_pair_sequence_equals_two_separate_sequences():
    """[prompt | chosen | prompt[-1] | rejected] with the key hole sees exactly the keys of the two separate
    [prompt | chosen] and [prompt | rejected] sequences, minus the prompt rows counted once."""
    P, n_c, n_r = 9, 6, 4
    n = P + n_c + 1 + n_r
    _, ft = causal_pairs(np.asarray([(KIND_FT, 0, n, -1, 0, n, P - 1, 1 + n_c)], np.int32))
    sep = lambda m: m * (m + 1) // 2  # noqa: E731
    prompt_rows = sep(P - 1)  # rows before the last prompt token, shared by both branches
    assert ft == sep(P + n_c) + sep(P + n_r) - prompt_rows


def test_tick_extras_on_engine_ticks():
    """The accounting runs on real TickBatches (C1 through the engine over the CPU stand-in device): FT ticks carry
    the sub-pass / backward attention and the AdamW bytes, inference-only ticks neither."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).parent))
    from fakes import FakeModel
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.roofline import tick_extras
    from paper_2510_03283_b200.workloads import c1

    wl = c1(seed=3)
    fm = FakeModel(wl.model, wl.train, max_prompt_len=wl.max_prompt_len)
    eng = GpuEngine(*wl.engine_args(), model=fm, mode="P")
    eng.keep_outputs = False
    batches = []
    for _ in range(80):
        if eng.run_ticks(1) == 0:
            break
        batches.append(eng.last_batch)
    cfg, n_sel = wl.model, wl.train.n_selected_layers
    seen_ft = seen_inf = False
    for b in batches:
        e = tick_extras(b, cfg, n_sel, 1000)
        e0 = tick_extras(b, cfg, n_sel, 0)
        assert e["attn_flops"] >= 0 and e["row_bytes"] > 0
        pre, ft = causal_pairs(b.seqs)
        att = 4 * cfg.head_dim * cfg.n_heads
        if b.ft_pairs:
            seen_ft = True
            assert e["row_bytes"] - e0["row_bytes"] == 30 * 1000
            L = cfg.n_layers
            assert e["attn_flops"] == att * (pre * L + ft * (L - n_sel) + ft * n_sel * 4.5)
        else:
            seen_inf = True
            assert e["row_bytes"] == e0["row_bytes"]
            assert e["attn_flops"] == att * pre * cfg.n_layers
    assert seen_ft and seen_inf
