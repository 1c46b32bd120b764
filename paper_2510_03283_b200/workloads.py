"""The BASELINE.json configs as concrete reference objects (SURVEY.md §8(d) "Configs as concrete
synthetic inputs"). Every trace comes from the reference's own generate_trace (workload.py:174-218);
traces are regenerated per run because the Engine mutates Requests in place (quirk Q1).
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .config import PRESETS, ModelConfig, TrainConfig
from .refpath import ensure_macesim

ensure_macesim()
from macesim.alignment import AlignmentEnv, TenantParams  # noqa: E402
from macesim.cost_model import CostProfile  # noqa: E402
from macesim.distributions import parse_dist  # noqa: E402
from macesim.engine import CacheConfig, EngineConfig  # noqa: E402
from macesim.priority import PriorityParams  # noqa: E402
from macesim.scheduler import Policy, SchedulerConfig  # noqa: E402
from macesim.workload import TenantDriftSpec, TraceConfig, generate_trace  # noqa: E402


@dataclass
class Workload:
    name: str
    model: ModelConfig
    trace_cfg: TraceConfig
    profile: CostProfile
    sched: SchedulerConfig
    cache: CacheConfig
    horizon: float
    seed: int
    train: TrainConfig = field(default_factory=TrainConfig)
    max_prompt_len: int = 4096
    kv_tokens: int = 1 << 19  # prompt KV pool (tokens) the bench allocates for this trace
    decode_pages_per_head: int = 12  # decode ring pages per (slot, KV head) the bench allocates
    bench_skip: int = 150  # ticks the bench runs (untimed) before warm-up: the trace's steady state
    tenant_params: dict | None = None  # multi-tenant env (config.py:212-239 [tenant.N] sections); None: one tenant

    def trace(self):
        return generate_trace(self.trace_cfg)

    @property
    def n_tenants(self) -> int:
        return len(self.trace_cfg.tenants)

    def env(self):
        return AlignmentEnv.create(self.tenant_params or {0: TenantParams()}, seed=self.trace_cfg.seed)

    def engine_args(self):
        """Positional args of Engine.__init__ (engine.py:186-196) with a fresh trace and env."""
        return (self.trace(), self.profile, self.sched, PriorityParams(), self.cache, self.env(),
                EngineConfig(seed=self.seed), self.horizon)


def c1(seed: int = 0) -> Workload:
    """tiny decoder, single-GPU/CPU correctness config with the golden tick 7."""
    tc = TraceConfig(arrival_rate=10, retrain_rate=0.3, duration=5, seed=seed,
                     prompt_len_dist=parse_dist("geometric:mean=64"), output_len_dist=parse_dist("geometric:mean=16"))
    return Workload("c1", PRESETS["tiny"], tc, CostProfile(capacity=24576.0, weights_resident=14000.0),
                    SchedulerConfig(), CacheConfig(weak_scale=0.05), 5.0, seed)


def c2(seed: int = 1, arrival_rate: float = 100.0, duration: float = 60.0, policy: Policy = Policy.HYBRID) -> Workload:
    """GPT-2 small hybrid serving + DPO, Poisson trace (prompt uniform 97..512: 1024 positions)."""
    cfg = PRESETS["gpt2"]
    tc = TraceConfig(arrival_rate=arrival_rate, retrain_rate=0.1, duration=duration, seed=seed,
                     prompt_len_dist=parse_dist("uniform:lo=97,hi=512"),
                     output_len_dist=parse_dist("geometric:mean=128"))
    kv_mb = cfg.kv_bytes_per_token() / 2**20
    prof = CostProfile(capacity=184320.0, weights_resident=2 * 247.0, decode_kv_mem_per_token=kv_mb)
    sched = SchedulerConfig(policy=policy, max_decode_batch=256, tau_task=512, max_ft_batch=4, max_decode_steps=512)
    return Workload("c2", cfg, tc, prof, sched, CacheConfig(num_heads=cfg.n_kv_heads, weak_scale=0.05), duration,
                    seed, max_prompt_len=1024)


def c3(seed: int = 2, arrival_rate: float = 200.0, duration: float = 20.0) -> Workload:
    """Llama-3.2-1B decode-heavy: prompt 1920, output 128 (ctx <= 2048), batch 256."""
    cfg = PRESETS["llama1b"]
    tc = TraceConfig(arrival_rate=arrival_rate, retrain_rate=0.05, duration=duration, seed=seed,
                     prompt_len_dist=parse_dist("constant:value=1920"),
                     output_len_dist=parse_dist("constant:value=128"))
    kv_mb = cfg.kv_bytes_per_token() / 2**20
    prof = CostProfile(capacity=184320.0, weights_resident=2471.0 + 2 * 130.0, decode_kv_mem_per_token=kv_mb)
    sched = SchedulerConfig(max_decode_batch=256, tau_task=512, max_ft_batch=4)
    return Workload("c3", cfg, tc, prof, sched, CacheConfig(num_heads=cfg.n_kv_heads, weak_scale=0.05), duration,
                    seed, max_prompt_len=2048, kv_tokens=1 << 21)


WORKLOADS = {"c1": c1, "c2": c2, "c3": c3}


def c4(seed: int = 100, arrival_rate: float = 40.0, duration: float = 30.0, capacity_mb: float = 16060.0 + 102400.0
       ) -> Workload:
    """Llama-3-8B hybrid, prefill-heavy (prompt uniform 512..2048, output geometric mean 32); one request
    stream per GPU (seed = 100 + rank). The reference's capacity (MB) is set to what one
    B200 really holds next to the 8B weights (16060 MB + a 100 GB prompt/decode KV budget) so the
    reference's own LRU offload (cache.py:217-238) keeps the trie inside the device page pool.
    In the reference clock (0.5 ms per prefill token, cost_model.py:32-44) the whole trace arrives within
    the first ticks; ticks 3..64 are the prefill-heavy phase (~20k prefill rows + ~250 decode rows + 4 FT
    pairs per tick), after which the queue drains into a decode tail, so the bench skips only 3 ticks."""
    cfg = PRESETS["llama8b"]
    tc = TraceConfig(arrival_rate=arrival_rate, retrain_rate=0.1, duration=duration, seed=seed,
                     prompt_len_dist=parse_dist("uniform:lo=512,hi=2048"),
                     output_len_dist=parse_dist("geometric:mean=32"))
    kv_mb = cfg.kv_bytes_per_token() / 2**20
    prof = CostProfile(capacity=capacity_mb, weights_resident=16060.0, decode_kv_mem_per_token=kv_mb)
    sched = SchedulerConfig(max_decode_batch=256, tau_task=512, max_ft_batch=4)
    return Workload("c4", cfg, tc, prof, sched, CacheConfig(num_heads=cfg.n_kv_heads, weak_scale=0.05), duration,
                    seed, max_prompt_len=2048, kv_tokens=int((capacity_mb - 16060.0) / kv_mb * 1.05) // 16 * 16,
                    decode_pages_per_head=4, bench_skip=3)


WORKLOADS["c4"] = c4


def with_tenants(wl: Workload, tenants: list[tuple[float, float]], lora_rank: int | None = None) -> Workload:
    """The workload with several tenants (the reference's multi-tenant config, config.py:212-239 /
    test_cli.py:238-256): tenants[i] = (mu0, drift_rate) of tenant i, used for both the trace's generation-time
    drift spec (workload.py:110-128; generate_trace draws each request's tenant, workload.py:183-188) and the
    env's TenantParams. With lora_rank, every tenant gets its own LoRA adapter (TrainConfig.lora_rank)."""
    import dataclasses

    specs = tuple(TenantDriftSpec(mu0=m, drift_rate=d) for m, d in tenants)
    params = {i: TenantParams(mu0=m, drift_rate=d) for i, (m, d) in enumerate(tenants)}
    train = dataclasses.replace(wl.train, lora_rank=lora_rank) if lora_rank else wl.train
    return dataclasses.replace(wl, trace_cfg=dataclasses.replace(wl.trace_cfg, tenants=specs), tenant_params=params,
                               train=train)
