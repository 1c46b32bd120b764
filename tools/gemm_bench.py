"""Time the tcgen05 GEMM on the hybrid tick's shapes (CUDA events, warm, L2-resident weights)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2510_03283_b200 import ops  # noqa: E402
from paper_2510_03283_b200._lib import Ctx  # noqa: E402
from paper_2510_03283_b200.build import build  # noqa: E402

build()
ctx = Ctx(0)
ws = torch.empty(32 << 20, device="cuda")
shapes = [  # (M, N, K, mode, label)
    (260, 2304, 768, "bf16", "gpt2 qkv decode"), (260, 768, 768, "f32_add", "gpt2 o decode"),
    (260, 3072, 768, "bf16_gelu", "gpt2 up decode"), (260, 768, 3072, "f32_add", "gpt2 down decode"),
    (256, 50257, 768, "f32", "gpt2 lm_head decode"), (1000, 2304, 768, "bf16", "gpt2 qkv mixed"),
    (1000, 768, 3072, "f32_add", "gpt2 down mixed"), (256, 3072, 2048, "bf16", "llama1b qkv decode"),
    (256, 16384, 2048, "bf16", "llama1b up decode"), (256, 2048, 8192, "f32_add", "llama1b down decode"),
    (4096, 4096, 4096, "bf16", "square 4k"), (8192, 8192, 8192, "bf16", "square 8k"),
    (16384, 6144, 4096, "bf16", "llama8b qkv prefill"), (16384, 4096, 4096, "f32_add", "llama8b o prefill"),
    (16384, 28672, 4096, "bf16", "llama8b up prefill"), (16384, 4096, 14336, "f32_add", "llama8b down prefill"),
]
if len(sys.argv) > 1:
    shapes = [s for s in shapes if any(k in s[4] for k in sys.argv[1:])]
for M, N, K, mode, label in shapes:
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if mode.startswith("f32") else torch.bfloat16)
    for _ in range(5):
        ops.gemm(ctx, a, b, out, mode=mode, workspace=ws)
    n = 50
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        ops.gemm(ctx, a, b, out, mode=mode, workspace=ws)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                ops.gemm(ctx, a, b, out, mode=mode, workspace=ws)
    g.replay()
    torch.cuda.synchronize()

    def timeit(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) * 1e3

    us = timeit(g.replay) / n
    us_eager = timeit(lambda: [ops.gemm(ctx, a, b, out, mode=mode, workspace=ws) for _ in range(n)]) / n
    with torch.cuda.stream(s):
        torch.matmul(a, b.t())
        s.synchronize()
    gb = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gb, stream=s):
        for _ in range(n):
            torch.matmul(a, b.t())
    gb.replay()
    us_cublas = timeit(gb.replay) / n
    flops = 2 * M * N * K
    byts = 2 * (M * K + N * K) + out.element_size() * M * N
    print(f"{label:24s} M={M:5d} N={N:6d} K={K:5d}  {us:8.2f} us  {flops / us / 1e6:8.1f} TF/s  {byts / us / 1e3:8.1f} GB/s  eager {us_eager:7.2f} us  cublas(bf16 out) {us_cublas:7.2f} us")
