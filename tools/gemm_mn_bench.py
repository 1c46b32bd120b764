"""MN-major GEMMs of the fine-tune backward (dW = dY^T.X: both operands MN-major; dX = dY.W: B MN-major) on the
C4 shapes: CUDA-graph timed, auto dispatch (CTA-pair kernel) vs the single-CTA kernel (MACE_GEMM_FORCE=single).
    python tools/gemm_mn_bench.py"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2510_03283_b200 import ops  # noqa: E402
from paper_2510_03283_b200._lib import Ctx  # noqa: E402

ROWS = 5120  # FT rows of a C4 tick (4 pairs)
SHAPES = [  # (name, M, N, K, a_mn, b_mn, mode)
    ("dW qkv", 6144, 4096, ROWS, True, True, "f32_add"),
    ("dW o", 4096, 4096, ROWS, True, True, "f32_add"),
    ("dW up", 28672, 4096, ROWS, True, True, "f32_add"),
    ("dW down", 4096, 14336, ROWS, True, True, "f32_add"),
    ("dX qkv", ROWS, 4096, 6144, False, True, "bf16"),
    ("dX up", ROWS, 4096, 28672, False, True, "f32"),
    ("dX down", ROWS, 14336, 4096, False, True, "bf16"),
]
ctx = Ctx(0)


def timed(M, N, K, a_mn, b_mn, mode, force, n=10):
    if force:
        os.environ["MACE_GEMM_FORCE"] = force
    else:
        os.environ.pop("MACE_GEMM_FORCE", None)
    a = torch.randn((K, M) if a_mn else (M, K), device="cuda").bfloat16()
    b = torch.randn((K, N) if b_mn else (N, K), device="cuda").bfloat16()
    out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if mode == "bf16" else torch.float32)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        ops.gemm(ctx, a, b, out, mode=mode, a_mn=a_mn, b_mn=b_mn)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                ops.gemm(ctx, a, b, out, mode=mode, a_mn=a_mn, b_mn=b_mn)
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / n)
    return best


for name, M, N, K, a_mn, b_mn, mode in SHAPES:
    t_auto = timed(M, N, K, a_mn, b_mn, mode, None)
    t_single = timed(M, N, K, a_mn, b_mn, mode, "single")
    f = 2 * M * N * K
    print(f"{name:8s} M={M:6d} N={N:6d} K={K:6d} {mode:8s} auto {t_auto:8.1f} us ({f / t_auto / 1e6:6.0f} TF/s) | "
          f"single-CTA {t_single:8.1f} us ({f / t_single / 1e6:6.0f} TF/s)", flush=True)
os.environ.pop("MACE_GEMM_FORCE", None)
