"""Bundled scenario sets: the Table-1 corpus and the synthetic heuristic grid.

``synthetic_grid`` restates the reference CLI's documented 16-point grid
(/root/reference/pkg/src/overlap_sim/cli.py:256-284): M in {2^13, 2^16, 2^18,
2^21} (N = 40960, 40960, 40960, 81920) x K in {2^12, 2^14, 2^16, 2^18},
half precision, 8 GPUs, named s01..s16 in row-major order.
"""
from __future__ import annotations

from importlib import resources

from .domain import Collective, GemmShape, Parallelism, Scenario, parse_scenarios


def corpus() -> list[Scenario]:
    text = resources.files("paper_2512_10236_b200.data").joinpath("scenarios_corpus.csv").read_text()
    return parse_scenarios(text)


def synthetic_grid(elt_bytes: int = 2, n_gpus: int = 8) -> list[Scenario]:
    fams = ((1 << 13, 40960), (1 << 16, 40960), (1 << 18, 40960), (1 << 21, 81920))
    ks = (1 << 12, 1 << 14, 1 << 16, 1 << 18)
    out = []
    for i, ((m, n), k) in enumerate(((f, k) for f in fams for k in ks), start=1):
        out.append(Scenario(name=f"s{i:02d}", parallelism=Parallelism.SP_TP, model="synthetic",
                            gemm=GemmShape(m=m, n=n, k=k, elt_bytes=elt_bytes),
                            collective=Collective.ALL_GATHER, n_gpus=n_gpus))
    return out
