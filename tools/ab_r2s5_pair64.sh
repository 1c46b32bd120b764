#!/bin/bash
# CTA-pair BN 64 on decode-sized / small-M GEMMs (cold weights) + its numerics against the single-CTA kernel
set -x
python tools/gemm_sweep.py --cold 8 --shapes 256,3072,2048,bf16 256,2048,2048,f32_add 256,2048,8192,f32_add 1215,768,768,f32_add 1215,2304,768,bf16 1215,768,3072,f32_add 600,768,3072,f32_add > gpurun_out/r2s5_pair64_sweep.log 2>&1
python - > gpurun_out/r2s5_pair64_check.log 2>&1 <<'PY'
import os, torch
from paper_2510_03283_b200 import ops
from paper_2510_03283_b200._lib import Ctx
ctx = Ctx(0)
ws = torch.empty(64 << 20, device="cuda")
for M, N, K, mode in [(256, 3072, 2048, "bf16"), (256, 2048, 2048, "f32_add"), (1215, 768, 768, "f32_add"), (300, 1000, 520, "f32")]:
    a = torch.randn(M, K, device="cuda").bfloat16(); b = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
    ref = a.float() @ b.float().t()
    outs = []
    for force in ("pair,64", "single"):
        os.environ["MACE_GEMM_FORCE"] = force
        out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if mode == "bf16" else torch.float32)
        ops.gemm(ctx, a, b, out, mode=mode, workspace=ws); torch.cuda.synchronize(); outs.append(out.float())
    err = (outs[0] - ref).abs().max().item()
    print(M, N, K, mode, "max err vs fp32", err, "bit-identical to single-CTA", torch.equal(outs[0], outs[1]))
PY
grep "M=" gpurun_out/r2s5_pair64_sweep.log | cut -c1-110; cat gpurun_out/r2s5_pair64_check.log
