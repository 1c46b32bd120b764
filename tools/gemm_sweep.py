"""Sweep tile width / split-K of the tcgen05 GEMM on the tick's shapes (CUDA-graph timed, in-process:
MACE_GEMM_FORCE is read by mace_gemm_bf16 on every call, i.e. at graph-capture time).
    python tools/gemm_sweep.py [--shapes M,N,K,mode ...]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2510_03283_b200 import ops  # noqa: E402
from paper_2510_03283_b200._lib import Ctx  # noqa: E402

SHAPES = [(1215, 2304, 768, "bf16"), (1215, 768, 768, "f32_add"), (1215, 3072, 768, "bf16_gelu"),
          (1215, 768, 3072, "f32_add"), (256, 50264, 768, "f32"), (600, 2304, 768, "bf16"), (600, 768, 3072, "f32_add"),
          (256, 3072, 2048, "bf16"), (256, 2048, 2048, "f32_add"), (256, 16384, 2048, "bf16"),
          (256, 2048, 8192, "f32_add"), (256, 128256, 2048, "f32"), (2000, 3072, 2048, "bf16"),
          (2000, 2048, 8192, "f32_add")]
COLD = 1  # --cold N: cycle N copies of the weight operand (N x |B| > L2: weights stream from HBM, as in a tick)
argv = sys.argv[1:]
if len(argv) > 1 and argv[0] == "--cold":
    COLD = int(argv[1])
    argv = argv[2:]
if len(argv) > 1 and argv[0] == "--shapes":
    SHAPES = [(int(a), int(b), int(c), d) for a, b, c, d in (x.split(",") for x in argv[1:])]
ctx = Ctx(0)
ws = torch.empty(64 << 20, device="cuda")


def timed(M, N, K, mode, cfg, n=30):
    if cfg == "auto":
        os.environ.pop("MACE_GEMM_FORCE", None)
    else:
        os.environ["MACE_GEMM_FORCE"] = cfg
    a = torch.randn(M, K, device="cuda").bfloat16()
    bs = [torch.randn(2 * N if mode == "bf16_swiglu" else N, K, device="cuda").bfloat16() for _ in range(COLD)]
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if mode.startswith("f32") else torch.bfloat16)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        ops.gemm(ctx, a, bs[0], out, mode=mode, workspace=ws, b_static=True)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i in range(n):
                ops.gemm(ctx, a, bs[i % COLD], out, mode=mode, workspace=ws, b_static=True)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / n)
    return best


for M, N, K, mode in SHAPES:
    cfgs = ["auto", "pair,256", "single"] if mode == "bf16_swiglu" else \
        ["auto", "pair,64", "pair,128", "pair,256"] + [f"{bn},{sp}" for bn in (64, 128, 192, 256) for sp in (1, 2, 3)]
    row = [(c, timed(M, N, K, mode, c)) for c in cfgs]
    best = min((t, c) for c, t in row)
    print(f"M={M} N={N} K={K} {mode}: auto {row[0][1]:.2f} | best {best[1]} {best[0]:.2f} | "
          + " ".join(f"{c}:{t:.1f}" for c, t in row[1:]), flush=True)
os.environ.pop("MACE_GEMM_FORCE", None)
