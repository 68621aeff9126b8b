"""Model shapes used by the configs in BASELINE.json (public HF configs; the
paper names the models in PAPER.md:637-639 §7.1 but prints no shapes).

Fields follow the C struct ``mirage_model_cfg`` in include/mirage.h.
"""
from dataclasses import dataclass, replace

OPT, LLAMA = 0, 1


@dataclass(frozen=True)
class ModelShape:
    name: str
    family: int          # OPT=0, LLAMA=1
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn_dim: int
    vocab: int
    max_pos: int
    norm_eps: float = 1e-5
    rope_theta: float = 10000.0

    def with_layers(self, n):
        return replace(self, n_layers=n, name=f"{self.name}-L{n}")


TOY = ModelShape("toy", OPT, 2, 256, 4, 4, 64, 1024, 1024, 2048)
TOY_LLAMA = ModelShape("toy-llama", LLAMA, 2, 256, 4, 2, 64, 512, 1024, 2048, 1e-5, 10000.0)
OPT_13B = ModelShape("opt-13b", OPT, 40, 5120, 40, 40, 128, 20480, 50272, 2048)
LLAMA2_7B = ModelShape("llama-2-7b", LLAMA, 32, 4096, 32, 32, 128, 11008, 32000, 4096, 1e-5, 10000.0)
LLAMA3_8B = ModelShape("llama-3-8b", LLAMA, 32, 4096, 32, 8, 128, 14336, 128256, 32768, 1e-5, 500000.0)
LLAMA_70B = ModelShape("llama-70b", LLAMA, 80, 8192, 64, 8, 128, 28672, 128256, 8192, 1e-5, 500000.0)

# PAPER.md Table 1 combinations: C1 = OPT-13b, Llama-2-13b, Llama-3-8b;
# C2 = OPT-30b, OPT-6.7b (public configs)
LLAMA2_13B = ModelShape("llama-2-13b", LLAMA, 40, 5120, 40, 40, 128, 13824, 32000, 4096, 1e-5, 10000.0)
OPT_30B = ModelShape("opt-30b", OPT, 48, 7168, 56, 56, 128, 28672, 50272, 2048)
OPT_6_7B = ModelShape("opt-6.7b", OPT, 32, 4096, 32, 32, 128, 16384, 50272, 2048)

PRESETS = {m.name: m for m in (TOY, TOY_LLAMA, OPT_13B, LLAMA2_7B, LLAMA3_8B, LLAMA_70B, LLAMA2_13B, OPT_30B,
                               OPT_6_7B)}
