"""Model configurations and per-rank layer shapes for the BASELINE workloads.

BASELINE.json configs (public model configs; synthetic random-init weights):
  [0] GPT-style layer, hidden 1024, seq 2048, 16x64 heads, ffn 4096  (CPU reference case)
  [1] Llama-3.2-3B FSDP8          [2] Llama-3-8B TP8          [3] Llama-3-70B FSDP8
The reference's partitions are abstract KernelSpecs (workloads.py:38-93); here each partition is
a real sequence of kernels over these shapes.  Config [0] uses the same Llama-style block
(RMSNorm + SwiGLU) at GPT dimensions.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class ModelConfig:
    name: str
    hidden: int
    ffn: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    n_layers: int
    rope_theta: float = 500000.0
    norm_eps: float = 1e-5
    vocab: int = 128256  # Llama-3 tokenizer; GPT preset: 50257 padded to a multiple of 64


PRESETS = {
    "gpt-h1024": ModelConfig("gpt-h1024", 1024, 4096, 16, 16, 64, 24, rope_theta=10000.0, vocab=50304),
    "llama-3.2-3b": ModelConfig("llama-3.2-3b", 3072, 8192, 24, 8, 128, 28),
    "llama-3-8b": ModelConfig("llama-3-8b", 4096, 14336, 32, 8, 128, 32),
    "llama-3-70b": ModelConfig("llama-3-70b", 8192, 28672, 64, 8, 128, 80),
}


@dataclass(frozen=True)
class Workload:
    """One rank's view of a partitioned layer: model, parallelism, group size, tokens per nanobatch."""

    model: ModelConfig
    parallel: str  # "tp" or "fsdp"
    world: int
    tokens: int
    nanobatches: int = 2

    def __post_init__(self):
        if self.parallel not in ("tp", "fsdp"):
            raise ValueError("parallel must be 'tp' or 'fsdp'")
        m = self.model
        if self.parallel == "tp":
            if m.n_heads % self.world or m.ffn % self.world:
                raise ValueError("TP degree must divide heads and ffn")
            if m.n_kv_heads % self.world and self.world % m.n_kv_heads:
                raise ValueError("TP degree incompatible with kv heads")

    # per-rank shapes
    @property
    def hq(self) -> int:
        return self.model.n_heads // (self.world if self.parallel == "tp" else 1)

    @property
    def hkv(self) -> int:
        if self.parallel != "tp":
            return self.model.n_kv_heads
        return max(1, self.model.n_kv_heads // self.world)

    @property
    def ffn(self) -> int:
        return self.model.ffn // (self.world if self.parallel == "tp" else 1)

    @property
    def d(self) -> int:
        return self.model.head_dim

    @property
    def h(self) -> int:
        return self.model.hidden

    @property
    def qkv_dim(self) -> int:
        return (self.hq + 2 * self.hkv) * self.d

    def weight_numels(self) -> dict[str, int]:
        """Per-rank compute-weight element counts (TP: shards; FSDP: full gathered weights)."""
        return {
            "wqkv": self.qkv_dim * self.h,
            "wo": self.h * self.hq * self.d,
            "wgu": 2 * self.ffn * self.h,
            "wd": self.h * self.ffn,
        }

    @property
    def tag(self) -> str:
        return f"{self.model.name}-{self.parallel}{self.world}-T{self.tokens}x{self.nanobatches}"


def baseline_workload(index: int, world: int = 8, tokens: int | None = None) -> Workload:
    """BASELINE.json configs[index] (0..3) as a per-rank Workload."""
    if index == 0:
        return Workload(PRESETS["gpt-h1024"], "tp", 1, tokens or 2048)
    if index == 1:
        return Workload(PRESETS["llama-3.2-3b"], "fsdp", world, tokens or 4096)
    if index == 2:
        return Workload(PRESETS["llama-3-8b"], "tp", world, tokens or 4096)
    if index == 3:
        return Workload(PRESETS["llama-3-70b"], "fsdp", world, tokens or 4096)
    raise ValueError("config index must be 0..3 (config 4 is the collective microbench)")
