"""Workload registry: BASELINE.json `configs` as concrete synthetic shapes.

Shared by tests/, bench.py and the oracle timing leg. Holds shapes and
hyper-parameters only -- none of the method's arithmetic.

C1..C5 follow SURVEY.md §8(d) "Concrete inputs". Head layouts: Llama-3.1-8B
32/8 and GLM-4-9B 32/2 (BASELINE.json configs[1..3]); Qwen2-7B 28/4 and
Yi-9B 32/4 from the public model configs (the paper names the models at
PAPER.md P:435-438 but gives no head layouts). d = 128 everywhere, block 128
(P:448), tau 0.1.
"""
from dataclasses import dataclass, replace


@dataclass(frozen=True)
class Workload:
    name: str
    heads: int
    kv_heads: int
    seq_len: int
    gamma: float
    tau: float = 0.1
    min_budget: int = 0
    seed: int = 0
    head_dim: int = 128
    block: int = 128
    mixed: bool = False  # C5 tau sweep: mixed QA + vertical heads (synth/gen.py)

    def with_(self, **kw):
        return replace(self, **kw)

    def describe(self):
        return {
            "workload": self.name,
            "heads": self.heads,
            "kv_heads": self.kv_heads,
            "seq_len": self.seq_len,
            "head_dim": self.head_dim,
            "block": self.block,
            "gamma": self.gamma,
            "tau": self.tau,
            "min_budget": self.min_budget,
            "seed": self.seed,
            "mixed_heads": self.mixed,
        }


# configs[0]: the small case the oracle finishes in seconds.
C1 = Workload("C1-tiny-4q1kv-2k", 4, 1, 2048, 0.9, 0.1, 0, 101)
# configs[1]: Llama-3.1-8B-like, 32k, gamma 0.9, 1 GPU.
C2 = Workload("C2-llama8b-32k", 32, 8, 32768, 0.9, 0.1, 0, 102)
# configs[2]: Llama-3.1-8B-like at 128k, gamma 0.95 (and 0.9 for the north-star check).
C3 = Workload("C3-llama8b-128k", 32, 8, 131072, 0.95, 0.1, 0, 103)
C3_G09 = C3.with_(name="C3-llama8b-128k-g0.9", gamma=0.9)
# configs[3]: GLM-4-9B-like 32/2 at 128k, gamma sweep, min budget on.
C4 = Workload("C4-glm4-9b-128k", 32, 2, 131072, 0.95, 0.1, 1024, 104)
C4_GAMMAS = (0.80, 0.85, 0.90, 0.95, 0.97, 0.99)
# configs[4]: context sweep for Qwen2-7B-like and Yi-9B-like layouts, tau sweep.
C5_QWEN = Workload("C5-qwen2-7b", 28, 4, 32768, 0.9, 0.1, 0, 105, mixed=True)
C5_YI = Workload("C5-yi-9b", 32, 4, 32768, 0.9, 0.1, 0, 106, mixed=True)
C5_LENGTHS = (4096, 8192, 16384, 32768, 65536, 131072)
C5_TAUS = (0.05, 0.1, 0.2, 0.3)

ALL = {w.name: w for w in (C1, C2, C3, C3_G09, C4, C5_QWEN, C5_YI)}


def get(name):
    return ALL[name]
