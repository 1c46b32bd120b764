"""Decoder shapes for the BASELINE.json configs (SURVEY.md §8(d) "Model shapes").

The reference (macesim) has no model at all: its cost model (cost_model.py:25-73) stands in for one.
These presets are the real architectures the hybrid iteration executes; weights are seeded random
init (no checkpoints offline), bf16 on device.
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class ModelConfig:
    name: str
    family: str            # "llama" (RMSNorm, RoPE, GQA, SwiGLU) or "gpt2" (LayerNorm, learned pos, GELU, biases)
    n_layers: int
    d_model: int
    n_heads: int           # query heads
    n_kv_heads: int        # = CacheConfig.num_heads (per-head KV windows, engine.py:44)
    head_dim: int
    ffn: int
    vocab: int
    max_pos: int = 8192
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5
    tied: bool = True
    init_std: float = 0.02
    embed_std: float = 0.1     # larger than GPT-2's 0.02 so random-init greedy decode has clear top-1 gaps

    @property
    def qkv_dim(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    @property
    def group(self) -> int:
        return self.n_heads // self.n_kv_heads

    @property
    def has_bias(self) -> bool:
        return self.family == "gpt2"

    @property
    def up_dim(self) -> int:
        return 2 * self.ffn if self.family == "llama" else self.ffn

    def kv_bytes_per_token(self) -> int:
        return 2 * self.n_layers * self.n_kv_heads * self.head_dim * 2

    def body_params(self) -> int:
        d = self.d_model
        per = self.qkv_dim * d + self.n_heads * self.head_dim * d + self.up_dim * d + self.ffn * d
        return self.n_layers * per

    def param_shapes(self) -> dict[str, tuple[int, ...]]:
        d = self.d_model
        s: dict[str, tuple[int, ...]] = {"embed": (self.vocab, d)}
        if self.family == "gpt2":
            s["pos_embed"] = (self.max_pos, d)
        for i in range(self.n_layers):
            p = f"layers.{i}."
            s[p + "attn_norm.w"] = (d,)
            s[p + "qkv.w"] = (self.qkv_dim, d)
            s[p + "o.w"] = (d, self.n_heads * self.head_dim)
            s[p + "mlp_norm.w"] = (d,)
            s[p + "up.w"] = (self.up_dim, d)
            s[p + "down.w"] = (d, self.ffn)
            if self.family == "gpt2":
                for n, dim in (("attn_norm.b", d), ("qkv.b", self.qkv_dim), ("o.b", d), ("mlp_norm.b", d),
                               ("up.b", self.ffn), ("down.b", d)):
                    s[p + n] = (dim,)
        s["final_norm.w"] = (d,)
        if self.family == "gpt2":
            s["final_norm.b"] = (d,)
        return s


PRESETS: dict[str, ModelConfig] = {
    # C1: tiny default decoder: L4 d256 Hq=Hkv=8 hd32 ffn1024, vocab 50000 = workload.py:129
    "tiny": ModelConfig("tiny", "llama", 4, 256, 8, 8, 32, 1024, 50000, max_pos=4096),
    # C2: GPT-2 small, 1024 positions
    "gpt2": ModelConfig("gpt2", "gpt2", 12, 768, 12, 12, 64, 3072, 50257, max_pos=1024),
    # C3: Llama-3.2-1B
    "llama1b": ModelConfig("llama1b", "llama", 16, 2048, 32, 8, 64, 8192, 128256, max_pos=8192, rope_theta=500000.0),
    # C4/C5: Llama-3-8B (untied lm_head in the real model; tied here to keep one vocab matrix)
    "llama8b": ModelConfig("llama8b", "llama", 32, 4096, 32, 8, 128, 14336, 128256, max_pos=8192, rope_theta=500000.0),
}


@dataclass(frozen=True)
class TrainConfig:
    """Builder-defined fine-tune settings (the reference has only ft_gain, alignment.py:69)."""

    n_selected_layers: int = 2        # top-k layers (+ final norm) receive the masked AdamW update
    lr: float = 1e-5
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0
    dpo_beta: float = 1.0             # = AlignmentEnv.beta default (alignment.py:99)
    # alignment-sensitivity selection (SURVEY §8(c) "optional top-k by ||grad W_l|| / ||W_l||"): when set, the
    # n_selected_layers top layers are the backward SPAN, and the masked AdamW updates only the k layers of the
    # span with the largest DPO-gradient-to-weight norm ratio, chosen on the first fine-tune update (after the
    # gradient all-reduce, so every replica chooses the same) and kept from then on. The final norm stays updated.
    sensitivity_topk: int | None = None
    # per-tenant LoRA adapters (the paper's per-user adapter phi_u over a frozen shared base,
    # PAPER.md:440-441): when set, every selected layer's qkv / o / up / down projection carries one rank-r adapter
    # per tenant (y = x W^T + (alpha / r) (x A_u^T) B_u^T for the rows of tenant u), the base model and the norms are
    # frozen, pi_ref is the base model (every adapter off), and each tenant's adapter is trained only by that
    # tenant's preference pairs with its own AdamW step count. B starts at zero, so pi_theta == pi_ref at first.
    lora_rank: int | None = None
    lora_alpha: float = 16.0
    lora_init_std: float = 0.02

    def selected_layers(self, cfg: ModelConfig) -> list[int]:
        return list(range(cfg.n_layers - self.n_selected_layers, cfg.n_layers))

    @property
    def lora_scale(self) -> float:
        return self.lora_alpha / self.lora_rank if self.lora_rank else 0.0


LORA_PROJ = ("qkv", "o", "up", "down")


def lora_shapes(cfg: ModelConfig, tcfg: TrainConfig, n_tenants: int) -> dict[str, tuple[int, int]]:
    """Stacked adapters of every selected layer, flat-buffer order: a_* [R, in] then bt_* [R, out] per projection,
    R = n_tenants * rank; tenant u owns rows [u * rank, (u + 1) * rank) of each."""
    R = n_tenants * tcfg.lora_rank
    d, ho = cfg.d_model, cfg.n_heads * cfg.head_dim
    io = {"qkv": (d, cfg.qkv_dim), "o": (ho, d), "up": (d, cfg.up_dim), "down": (cfg.ffn, d)}
    out = {}
    for l in tcfg.selected_layers(cfg):
        for p in LORA_PROJ:
            i, o = io[p]
            out[f"lora.{l}.a_{p}"] = (R, i)
            out[f"lora.{l}.bt_{p}"] = (R, o)
    return out


def sensitivity_ranking(grads: dict, weights: dict, layers: list[int]) -> list[tuple[int, float]]:
    """(layer, ||grad W_l|| / ||W_l||) over the layers' parameter tensors, most sensitive first (ties: lower layer).
    ``grads`` / ``weights``: name -> tensor (any device); the norms are fp64 sums of squares over every tensor
    of the layer."""
    out = []
    for l in layers:
        pre = f"layers.{l}."
        g2 = sum(float(t.double().pow(2).sum()) for n, t in grads.items() if n.startswith(pre))
        w2 = sum(float(t.double().pow(2).sum()) for n, t in weights.items() if n.startswith(pre))
        out.append((l, (g2 ** 0.5) / max(w2 ** 0.5, 1e-30)))
    return sorted(out, key=lambda x: (-x[1], x[0]))


def trainable_param_names(cfg: ModelConfig, tcfg: TrainConfig, n_tenants: int = 1) -> list[str]:
    """Names of the flat optimizer buffers: the per-tenant adapters (LoRA mode) or the selected base parameters."""
    if tcfg.lora_rank:
        return list(lora_shapes(cfg, tcfg, n_tenants))
    return selected_param_names(cfg, tcfg)


def selected_param_names(cfg: ModelConfig, tcfg: TrainConfig) -> list[str]:
    names = []
    for i in tcfg.selected_layers(cfg):
        names += [n for n in cfg.param_shapes() if n.startswith(f"layers.{i}.")]
    names += [n for n in cfg.param_shapes() if n.startswith("final_norm.")]
    return names
