"""tcgen05 GEMM vs a plain torch fp32 reference of the same op (bf16 inputs, fp32 accumulate)."""
import pytest
import torch

from paper_2510_03283_b200 import ops

pytestmark = pytest.mark.gpu

SHAPES = [
    (128, 128, 64),
    (256, 512, 256),
    (1, 2048, 2048),      # one decode row
    (7, 384, 96),         # ragged tails in every dim (K % 64 != 0)
    (300, 1000, 520),
    (1024, 2048, 1024),
    (4096, 4096, 512),    # >148 tiles -> persistent loop + double-buffered TMEM
]


def _ref(a, b, a_mn, b_mn):
    A = (a.t() if a_mn else a).float()
    B = (b.t() if b_mn else b).float()
    return A @ B.t()


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
def test_gemm_layouts(ctx, M, N, K, a_mn, b_mn):
    torch.manual_seed(M * 7 + N + K)
    dev = "cuda"
    a = torch.randn((K, M) if a_mn else (M, K), device=dev).bfloat16()
    b = torch.randn((K, N) if b_mn else (N, K), device=dev).bfloat16()
    # MN-major operands need 16-byte aligned rows: pad the leading dim
    if a_mn and M % 8:
        a = torch.nn.functional.pad(a, (0, 8 - M % 8))[:, :M]
    if b_mn and N % 8:
        b = torch.nn.functional.pad(b, (0, 8 - N % 8))[:, :N]
    if not a_mn and K % 8:
        pytest.skip("K-major rows need K % 8 == 0")
    out = ops.gemm(ctx, a, b, mode="f32", a_mn=a_mn, b_mn=b_mn)
    ref = _ref(a, b, a_mn, b_mn)
    torch.cuda.synchronize()
    err = (out - ref).abs().max().item()
    tol = 1e-3 * K ** 0.5 + 1e-2
    assert err <= tol, f"max err {err} > {tol}"


@pytest.mark.parametrize("M,N,K", [(64, 256, 128), (500, 768, 768), (2, 50257, 768)])
def test_gemm_epilogues(ctx, M, N, K):
    torch.manual_seed(0)
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    bias = torch.randn(N, device="cuda").bfloat16()
    ref = a.float() @ b.float().t()
    y = ops.gemm(ctx, a, b, mode="bf16", bias=bias)
    assert torch.allclose(y.float(), (ref + bias.float()), atol=0.1, rtol=1e-2)
    g = ops.gemm(ctx, a, b, mode="bf16_gelu", bias=bias)
    gref = torch.nn.functional.gelu(ref + bias.float(), approximate="tanh")
    assert torch.allclose(g.float(), gref, atol=0.1, rtol=1e-2)
    acc = torch.randn(M, N, device="cuda")
    acc0 = acc.clone()
    ops.gemm(ctx, a, b, acc, mode="f32_add", alpha=0.5)
    assert torch.allclose(acc, acc0 + 0.5 * ref, atol=2e-2, rtol=1e-3)
    acc1 = acc0.clone()
    ops.gemm(ctx, a, b, acc1, mode="f32_atomic", split_k=2)
    assert torch.allclose(acc1, acc0 + ref, atol=2e-2, rtol=1e-3)


def test_gemm_splitk_bf16_workspace(ctx):
    torch.manual_seed(1)
    M, N, K = 64, 512, 4096
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    ws = torch.empty(8 * M * N, device="cuda")
    y = ops.gemm(ctx, a, b, mode="bf16", split_k=8, workspace=ws)
    ref = a.float() @ b.float().t()
    assert torch.allclose(y.float(), ref, atol=0.5, rtol=1e-2)


@pytest.mark.parametrize("M,N,K,force", [
    (2048, 6144, 1024, None),        # auto -> CTA-pair, BN 256 (8 x 24 pair tiles)
    (1100, 8200, 512, None),         # ragged M (last pair tile straddles M) and N
    (777, 2056, 640, "pair,128"),    # pair BN 128, ragged everywhere, K % 64 != 0
    (4096, 1024, 4160, "pair,256"),  # long K
])
def test_gemm_cta_pair(ctx, M, N, K, force, monkeypatch):
    """cta_group::2 GEMM (256-row pair tiles, leader-issued MMA) against the fp32 reference, every epilogue."""
    if force:
        monkeypatch.setenv("MACE_GEMM_FORCE", force)
    torch.manual_seed(M + N + K)
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    bias = torch.randn(N, device="cuda").bfloat16()
    ref = a.float() @ b.float().t()
    tol = 1e-3 * K ** 0.5 + 1e-2
    out = ops.gemm(ctx, a, b, mode="f32")
    assert (out - ref).abs().max().item() <= tol
    y = ops.gemm(ctx, a, b, mode="bf16", bias=bias)
    assert torch.allclose(y.float(), ref + bias.float(), atol=0.1, rtol=1e-2)
    g = ops.gemm(ctx, a, b, mode="bf16_gelu", bias=bias)
    assert torch.allclose(g.float(), torch.nn.functional.gelu(ref + bias.float(), approximate="tanh"), atol=0.1,
                          rtol=1e-2)
    acc0 = torch.randn(M, N, device="cuda")
    acc = acc0.clone()
    ops.gemm(ctx, a, b, acc, mode="f32_add", alpha=0.5)
    assert torch.allclose(acc, acc0 + 0.5 * ref, atol=2e-2, rtol=1e-3)
    # same numbers as the single-CTA kernel (both accumulate K in the same 16-wide MMA order in fp32)
    monkeypatch.setenv("MACE_GEMM_FORCE", "single")
    out1 = ops.gemm(ctx, a, b, mode="f32")
    assert torch.equal(out, out1)


@pytest.mark.parametrize("M,F,K", [(256, 8192, 2048), (300, 1024, 512), (4096, 14336, 512), (77, 2048, 256)])
def test_gemm_swiglu(ctx, M, F, K):
    """Fused SwiGLU epilogue (silu(x Wg^T) * (x Wu^T), W = [gate; up] stacked): single-CTA and CTA-pair tiles
    against the fp32 reference."""
    torch.manual_seed(M + F)
    a = (torch.randn(M, K, device="cuda") * 0.5).bfloat16()
    w = (torch.randn(2 * F, K, device="cuda") / K ** 0.5).bfloat16()
    out = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    ops.gemm(ctx, a, w, out, mode="bf16_swiglu")
    torch.cuda.synchronize()
    g = a.float() @ w[:F].float().t()
    u = a.float() @ w[F:].float().t()
    ref = torch.nn.functional.silu(g) * u
    err = (out.float() - ref).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item() + 1e-3, err


@pytest.mark.parametrize("M,N,K", [(1024, 2048, 1024), (777, 1000, 520), (3000, 4096, 2304)])
@pytest.mark.parametrize("a_mn,b_mn", [(False, True), (True, False), (True, True)])
@pytest.mark.parametrize("force", ["pair,128", "pair,256"])
def test_gemm_cta_pair_mn_major(ctx, M, N, K, a_mn, b_mn, force, monkeypatch):
    """CTA-pair kernel with MN-major operands (the fine-tune backward's dX = dY.W and dW = dY^T.X): against the
    fp32 reference, and bit-identical to the single-CTA kernel (same K order of fp32 accumulation)."""
    monkeypatch.setenv("MACE_GEMM_FORCE", force)
    torch.manual_seed(M + N + K + 2 * a_mn + b_mn)
    a = torch.randn((K, M) if a_mn else (M, K), device="cuda").bfloat16()
    b = torch.randn((K, N) if b_mn else (N, K), device="cuda").bfloat16()
    if a_mn and M % 8:
        a = torch.nn.functional.pad(a, (0, 8 - M % 8))[:, :M]
    if b_mn and N % 8:
        b = torch.nn.functional.pad(b, (0, 8 - N % 8))[:, :N]
    if not a_mn and K % 8:
        pytest.skip("K-major rows need K % 8 == 0")
    ref = _ref(a, b, a_mn, b_mn)
    out = ops.gemm(ctx, a, b, mode="f32", a_mn=a_mn, b_mn=b_mn)
    assert (out - ref).abs().max().item() <= 1e-3 * K ** 0.5 + 1e-2
    acc0 = torch.randn(M, N, device="cuda")
    acc = acc0.clone()
    ops.gemm(ctx, a, b, acc, mode="f32_add", a_mn=a_mn, b_mn=b_mn)
    assert torch.allclose(acc, acc0 + ref, atol=2e-2, rtol=1e-3)
    y = ops.gemm(ctx, a, b, mode="bf16", a_mn=a_mn, b_mn=b_mn)
    assert torch.allclose(y.float(), ref, atol=0.1, rtol=1e-2)
    monkeypatch.setenv("MACE_GEMM_FORCE", "single")
    assert torch.equal(out, ops.gemm(ctx, a, b, mode="f32", a_mn=a_mn, b_mn=b_mn))
