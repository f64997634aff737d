"""Shared helpers: load golden fixtures and canonicalise plans the way make_golden.py does."""
import hashlib
import json
import pathlib

from paper_2512_10236_b200 import routing
from paper_2512_10236_b200.domain import Collective, GemmShape, Parallelism, Scenario

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"


def load(name: str):
    return json.loads((GOLDEN / name).read_text())


def scen(name, m, n, k, g, elt=2):
    return Scenario(name=name, parallelism=Parallelism.SP_TP, model="golden",
                    gemm=GemmShape(m, n, k, elt), collective=Collective.ALL_GATHER, n_gpus=g)


def task_record(t) -> list:
    k = t.kind
    if isinstance(k, routing.TransferSpec):
        body = ["T", k.src, k.dst, k.bytes, int(k.fine), k.round_idx]
    elif isinstance(k, routing.GatherSpec):
        body = ["G", k.bytes]
    elif isinstance(k, routing.ScatterSpec):
        body = ["S", k.bytes]
    else:
        s = k.shape
        body = ["M", s.m, s.n, s.k, s.elt_bytes, int(k.additive),
                None if k.dil is None else [k.dil[0], repr(k.dil[1])],
                [list(f) for f in k.rows], None if k.col_block is None else list(k.col_block)]
    return [t.id, t.gpu, list(t.deps)] + body


def plan_record(plan) -> dict:
    return {"schedule": plan.schedule.value, "chunk_rows": plan.chunk_rows, "chunk_cols": plan.chunk_cols,
            "tasks": [task_record(t) for t in plan.tasks]}


def digest(rec: dict) -> str:
    return hashlib.sha256(json.dumps(rec, separators=(",", ":")).encode()).hexdigest()
