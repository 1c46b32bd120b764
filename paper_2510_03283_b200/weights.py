"""Seeded random-init weights at the real architecture shapes (no checkpoints exist offline).

Generated on the CPU with a torch.Generator so the device run and the CPU oracle see identical
bf16 values for a given seed.
"""
from __future__ import annotations

import math

import torch

from .config import ModelConfig, TrainConfig, lora_shapes


def init_weights(cfg: ModelConfig, seed: int = 0, device: str | torch.device = "cpu") -> dict[str, torch.Tensor]:
    """bf16 weights; CPU generation is the parity-test path, device generation is for the big presets."""
    g = torch.Generator(device=device).manual_seed(seed)
    out: dict[str, torch.Tensor] = {}
    resid_std = cfg.init_std / math.sqrt(2 * cfg.n_layers)
    for name, shape in cfg.param_shapes().items():
        if name == "embed":
            t = torch.randn(shape, generator=g, device=device) * cfg.embed_std
        elif name == "pos_embed":
            t = torch.randn(shape, generator=g, device=device) * 0.01
        elif name.endswith("norm.w"):
            t = 1.0 + 0.05 * torch.randn(shape, generator=g, device=device)
        elif name.endswith(".b"):
            t = 0.02 * torch.randn(shape, generator=g, device=device)
        elif name.endswith("o.w") or name.endswith("down.w"):
            t = torch.randn(shape, generator=g, device=device) * resid_std
        else:
            t = torch.randn(shape, generator=g, device=device) * cfg.init_std
        out[name] = t.to(torch.bfloat16)
    return out


def init_lora(cfg: ModelConfig, tcfg: TrainConfig, n_tenants: int, seed: int = 0,
              b_std: float = 0.0) -> dict[str, torch.Tensor]:
    """bf16 per-tenant adapters (LoRA's init: A ~ N(0, init_std), B = 0, so every tenant starts at the base model;
    b_std > 0 gives every tenant a distinct non-zero adapter from the start -- tests). Generated on the CPU from
    (seed, 409) so the device and the oracle see the same values."""
    g = torch.Generator().manual_seed(seed * 1000003 + 409)
    out = {}
    for name, shape in lora_shapes(cfg, tcfg, n_tenants).items():
        if ".a_" in name:
            out[name] = (torch.randn(shape, generator=g) * tcfg.lora_init_std).to(torch.bfloat16)
        else:
            out[name] = (torch.randn(shape, generator=g) * b_std).to(torch.bfloat16)
    return out
