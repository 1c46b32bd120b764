"""Sweep tile width / split-K of the tcgen05 GEMM on the tick's shapes (CUDA-graph timed, one process per
config because the override is read once per launch from MACE_GEMM_FORCE)."""
import os
import subprocess
import sys

SHAPES = [(1200, 2304, 768, "bf16"), (1200, 768, 768, "f32_add"), (1200, 3072, 768, "bf16_gelu"),
          (1200, 768, 3072, "f32_add"), (256, 50257, 768, "f32"), (260, 2304, 768, "bf16"), (260, 768, 3072, "f32_add"),
          (256, 3072, 2048, "bf16"), (256, 16384, 2048, "bf16"), (256, 2048, 8192, "f32_add")]
CHILD = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2510_03283_b200 import ops
from paper_2510_03283_b200._lib import Ctx
ctx = Ctx(0)
ws = torch.empty(64 << 20, device="cuda")
M, N, K, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
a = torch.randn(M, K, device="cuda").bfloat16(); b = torch.randn(N, K, device="cuda").bfloat16()
out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if mode.startswith("f32") else torch.bfloat16)
s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph(); n = 40
with torch.cuda.stream(s):
    ops.gemm(ctx, a, b, out, mode=mode, workspace=ws); s.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n): ops.gemm(ctx, a, b, out, mode=mode, workspace=ws)
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(3):
    e0.record(); g.replay(); e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1) * 1e3 / n)
print(best)
'''
for M, N, K, mode in SHAPES:
    row = []
    for cfg in ["auto"] + [f"{bn},{sp}" for bn in (64, 128, 256) for sp in (1, 2, 3, 4, 6, 8)]:
        env = dict(os.environ)
        if cfg != "auto":
            env["MACE_GEMM_FORCE"] = cfg
        r = subprocess.run([sys.executable, "-c", CHILD, str(M), str(N), str(K), mode], env=env, capture_output=True,
                           text=True)
        try:
            row.append((cfg, float(r.stdout.strip().split()[-1])))
        except Exception:
            row.append((cfg, float("nan")))
    best = min((t, c) for c, t in row if t == t)
    print(f"M={M} N={N} K={K} {mode}: auto {row[0][1]:.2f} us | best {best[1]} {best[0]:.2f} us | "
          + " ".join(f"{c}:{t:.1f}" for c, t in row[1:]), flush=True)
