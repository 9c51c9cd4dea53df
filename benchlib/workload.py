"""The contract workload, free of the product package.

``--impl reference`` must time the reference's CPU path without loading the
B200 library (its process may map only ``oracle/``), so the workload it
shares with the B200 arm -- the Qwen1.5-MoE-A2.7B expert shape of
BASELINE.json configs[1] and the decode routing -- is defined here in plain
numpy.  The B200 arm builds its MoEProfile from the same numbers
(``benchlib.common.model``), and tests/test_bench_contract.py checks that
both arms see identical routing."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TOKENS, SEED = 32, 2


@dataclass(frozen=True)
class ExpertShape:
    name: str
    num_layers: int
    num_experts: int
    top_k: int
    hidden: int
    intermediate: int

    @property
    def expert_size(self) -> int:   # bf16 gate + up + down
        return 3 * self.hidden * self.intermediate * 2


QWEN15 = ExpertShape("qwen1.5-moe-a2.7b", num_layers=24, num_experts=60, top_k=4, hidden=2048, intermediate=1408)
assert QWEN15.expert_size == 17_301_504


def routing(shape, steps: int, seed: int = SEED, tokens: int = TOKENS) -> list[list[np.ndarray]]:
    """Router top-k over N(0,1) logits for a decode batch of ``tokens``:
    routing[step][layer] = sorted unique activated experts.
    Same stream as paper_2602_00328_b200.moe.topk_routing."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(steps):
        row = []
        for _layer in range(shape.num_layers):
            logits = rng.standard_normal((tokens, shape.num_experts))
            top = np.argpartition(-logits, shape.top_k - 1, axis=1)[:, :shape.top_k]
            row.append(np.unique(top))
        out.append(row)
    return out
