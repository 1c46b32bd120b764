"""Run one GEMM shape a few times (for ncu): python tools/gemm_one.py M N K mode [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2510_03283_b200 import ops  # noqa: E402
from paper_2510_03283_b200._lib import Ctx  # noqa: E402

M, N, K, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
ctx = Ctx(0)
ws = torch.empty(64 << 20, device="cuda")
a = torch.randn(M, K, device="cuda").bfloat16()
b = torch.randn(N, K, device="cuda").bfloat16()
out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if mode.startswith("f32") else torch.bfloat16)
for _ in range(reps):
    ops.gemm(ctx, a, b, out, mode=mode, workspace=ws)
torch.cuda.synchronize()
ref = (a.float() @ b.float().t())
print("ok", M, N, K, mode)
