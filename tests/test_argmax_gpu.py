"""Fused greedy decode head (MACE_EPI_ARGMAX): the lm_head GEMM's epilogue reduces every row to (largest logit,
first column holding it) with one 64-bit atomicMax per (row, tile), so the [n_dec, V] fp32 logits are never
written or re-read. Checked bit-exactly against torch.argmax (first maximal index) over the fp32 logits of the
same GEMM, on the single-CTA and CTA-pair kernels, ragged N, exact ties, and through the engine (the greedy
tokens of C1 with and without the fused head)."""
import pytest
import torch

from paper_2510_03283_b200 import ops

pytestmark = pytest.mark.gpu


def _case(ctx, M, N, K, seed=0, tie=False):
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    if tie:  # duplicate row 0's winning column into a lower and a higher column: equal logits, lowest index wins
        k0 = int(ops.gemm(ctx, a, b, mode="f32")[0].argmax())
        lo = 3 if k0 > 3 else k0
        b[lo] = b[k0]
        b[N - 1] = b[k0]
    ref = ops.gemm(ctx, a, b, mode="f32").argmax(dim=1).to(torch.int32)
    keys = ops.gemm(ctx, a, b, mode="argmax")
    tok = ops.argmax_keys(ctx, keys, M)
    torch.cuda.synchronize()
    assert torch.equal(tok, ref), (M, N, K, int((tok != ref).sum()))
    assert int(keys.abs().sum()) == 0, "keys are reset for the next call"
    if tie:
        assert int(tok[0]) == (3 if k0 > 3 else k0)
    return tok


@pytest.mark.parametrize("M,N,K", [(1, 1000, 64), (3, 777, 128), (130, 5001, 256), (600, 50257, 768),
                                   (256, 128256, 4096), (1200, 50257, 768)])
def test_argmax_epilogue_matches_logits(ctx, M, N, K):
    _case(ctx, M, N, K)


def test_argmax_ties_lowest_index(ctx):
    _case(ctx, 5, 4099, 256, seed=3, tie=True)
    _case(ctx, 300, 50257, 768, seed=4, tie=True)  # CTA-pair kernel


def test_keys_reused_across_calls(ctx):
    """The keys buffer is reused tick after tick: a second GEMM into the reset buffer gives the second answer."""
    g = torch.Generator(device="cuda").manual_seed(9)
    a1 = torch.randn(64, 512, device="cuda", generator=g).bfloat16()
    a2 = torch.randn(64, 512, device="cuda", generator=g).bfloat16()
    b = torch.randn(3000, 512, device="cuda", generator=g).bfloat16()
    keys = torch.zeros(64, dtype=torch.int64, device="cuda")
    for a in (a1, a2, a1):
        ops.gemm(ctx, a, b, keys, mode="argmax")
        tok = ops.argmax_keys(ctx, keys)
        assert torch.equal(tok, ops.gemm(ctx, a, b, mode="f32").argmax(dim=1).to(torch.int32))


def test_engine_tokens_fused_head_equal_logits_head(ctx):
    """C1 through the engine: the greedy tokens of every decode step are identical with the fused head (default)
    and with the materialised-logits head (record mode, which the oracle replays use)."""
    from test_engine_c1_gpu import run_c1

    fused, _, _ = run_c1(record=False)
    assert fused.model.keep_dec_logits is False
    logits, _, _ = run_c1(record=True)
    assert logits.model.keep_dec_logits is True
    assert fused.decoded_tokens() == logits.decoded_tokens()
