"""Workload shapes (BASELINE.json ``configs``), as plain data.

Model dimensions follow SURVEY.md §8 notation: Qwen3-32B and Llama-3.1-70B
from SPEC.md:62,64 plus the public model cards (n_q = 64, vocab); Qwen2.5-72B
from its public card.  Nothing here computes anything
of the method.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace


@dataclass(frozen=True)
class ModelDims:
    name: str
    num_layers: int
    hidden: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    intermediate: int
    vocab: int
    qkv_bias: bool = False
    qk_norm: bool = False
    rms_eps: float = 1e-5
    rope_theta: float = 1e4

    @property
    def q_dim(self) -> int:
        return self.n_q_heads * self.head_dim

    @property
    def kv_dim(self) -> int:
        return self.n_kv_heads * self.head_dim

    @property
    def qkv_dim(self) -> int:
        return self.q_dim + 2 * self.kv_dim

    def with_layers(self, n: int) -> "ModelDims":
        return replace(self, num_layers=n)


MODELS = {
    # M1: tiny decoder, 4 layers, hidden 256
    "tiny": ModelDims("tiny", 4, 256, 4, 2, 64, 768, 1024, rms_eps=1e-5, rope_theta=1e4),
    # tiny variants exercising the Qwen3 (qk_norm, n_q*hd != h) and Qwen2.5 (QKV bias) paths
    "tiny-qwen3": ModelDims("tiny-qwen3", 4, 256, 4, 2, 128, 768, 1024, qk_norm=True,
                            rms_eps=1e-6, rope_theta=1e6),
    "tiny-qwen25": ModelDims("tiny-qwen25", 4, 256, 4, 2, 64, 768, 1024, qkv_bias=True,
                             rms_eps=1e-6, rope_theta=1e6),
    "qwen3-32b": ModelDims("qwen3-32b", 64, 5120, 64, 8, 128, 25600, 151936, qk_norm=True,
                           rms_eps=1e-6, rope_theta=1e6),
    "llama-3.1-70b": ModelDims("llama-3.1-70b", 80, 8192, 64, 8, 128, 28672, 128256,
                               rms_eps=1e-5, rope_theta=5e5),
    "qwen2.5-72b": ModelDims("qwen2.5-72b", 80, 8192, 64, 8, 128, 29568, 152064, qkv_bias=True,
                             rms_eps=1e-6, rope_theta=1e6),
}


def get_model(name: str) -> ModelDims:
    return MODELS[name]


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config as a synthetic recipe."""
    id: str
    model: str
    world: int            # d, DP group size the config is quoted on
    batch: int            # rows per rank
    ctx: int              # cached tokens per sequence (uniform) ...
    ctx_span: int = 0     # ... or ragged: ctx + (hash mod (ctx_span+1))
    slots: int = 2
    seed_offset: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def seed(self) -> int:
        return 20261017 + self.seed_offset


WORKLOADS = {
    # configs[0]: tiny decoder, 4 layers, hidden 256, batch 8, 2 owners; ragged contexts 0..63
    "M1": Workload("M1", "tiny", world=2, batch=8, ctx=0, ctx_span=63, slots=2, seed_offset=1),
    # configs[1]: Qwen3-32B WaS decode batch 256, S_ctx = 1024 (PAPER.md:308 summarisation average)
    "M2": Workload("M2", "qwen3-32b", world=8, batch=256, ctx=1024, slots=2, seed_offset=2),
    # configs[2]: Llama-3.1-70B WaS at B_e with max KV (d=8 only fits)
    "M3": Workload("M3", "llama-3.1-70b", world=8, batch=1536, ctx=288, slots=2, seed_offset=3),
    # configs[3]: Qwen2.5-72B WaS at 2/4/8 GPUs, cache-slot sweep 2-4
    "M4": Workload("M4", "qwen2.5-72b", world=8, batch=256, ctx=1024, slots=2, seed_offset=4),
    # configs[4]: Llama-3.1-70B small-batch tail CaS, B/rank 1..16, S_ctx 4096
    "M5": Workload("M5", "llama-3.1-70b", world=8, batch=16, ctx=4096, slots=2, seed_offset=5),
}
