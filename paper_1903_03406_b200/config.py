"""Refinement configuration (drop-in for tetrefine.RefineConfig).

Same fields, defaults and validation as
/root/reference/pkg/src/tetrefine/refine.py:73-88.  ``workers`` and
``sequential_until`` are accepted for API compatibility; like the reference
they cannot change the output (the GPU filter is exactly the greedy
oracle), so they only appear in the per-round report.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass
class RefineConfig:
    B: float = 2.0
    max_rounds: int = 500
    workers: int = 1
    sequential_until: int = 50000
    seed: int = 0
    verbose: bool = False
    # extension (not in the reference): "greedy" = the reference's filter
    # (growblast.py:123-207, result-identical); "blast" = the paper's literal
    # grow-and-blast, one claim round per refinement round and no
    # resurrection of candidates whose blocker was itself blasted
    # (SURVEY 8(f) row 4).  Not result-identical.
    filter: str = "greedy"

    def __post_init__(self):
        if self.filter not in ("greedy", "blast"):
            raise ValueError("filter must be 'greedy' or 'blast'")
        if self.B <= 0:
            raise ValueError("B must be positive")
        if self.max_rounds < 1:
            raise ValueError("max_rounds must be >= 1")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
