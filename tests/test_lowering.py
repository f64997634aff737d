"""Structural invariants of the lowered tile programs (CPU, no GPU): every output element is
written by exactly one tile, every tile reads rows that its gate covers, CTA pairs share a
column block, and the row-group raster engages exactly when the weight exceeds L2."""
import numpy as np
import pytest

from paper_2512_10236_b200.domain import Collective
from paper_2512_10236_b200.lowering import (F_RING, F_XFER, W_L2_BYTES, lower_ag, lower_rs, pair_tiles,
                                            raster)
from paper_2512_10236_b200.ops import _scenario
from paper_2512_10236_b200 import routing
from paper_2512_10236_b200.routing import ScheduleKind, build_plan
from paper_2512_10236_b200.runtime import EPI_REDUCE, EPI_STORE_REMOTE, EPI_STORE_SIGNAL

AG_KINDS = ["serial", "shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d",
            "uniform_fused_2d"]


def _coverage(tiles, rows, cols):
    hit = np.zeros((rows, cols), dtype=np.int32)
    for t in tiles:
        if t.rows:
            hit[t.c_row:t.c_row + t.rows, t.c_col:t.c_col + t.cols] += 1
    return hit


@pytest.mark.parametrize("kind", AG_KINDS)
@pytest.mark.parametrize("M,N,K,G", [(4096, 512, 1024, 4), (8192, 3584, 4096, 8),
                                     (18432, 10240, 4096, 8)])  # last: W 84 MB > L2 budget -> row groups
@pytest.mark.parametrize("collective", [Collective.ALL_GATHER, Collective.ALL_TO_ALL])
@pytest.mark.parametrize("cta_group", [1, 2])
def test_ag_tiles_cover_output_once_and_gates_cover_rows(kind, M, N, K, G, collective, cta_group):
    sc = _scenario("x", M, N, K, G, collective)
    R, r = M // G, M // (G * G)
    for rank in (0, G - 1):
        low = lower_ag(build_plan(sc, ScheduleKind(kind)), rank, "A", cta_group=cta_group)
        assert (_coverage(low.tiles, M, N) == 1).all(), (kind, rank)
        for t in low.tiles:
            if not t.rows:
                continue
            owner = t.c_row // R
            assert (t.c_row + t.rows - 1) // R == owner  # a tile never straddles two owners' rows
            if owner == rank:  # own rows: read in place; gated only as part of a uniform fused step
                assert t.a_src == 1 and (t.flag < 0) == (kind != "uniform_fused_1d")
                continue
            assert t.flag >= 0 and t.fmask
            if kind == "shard_overlap_p2p":
                assert t.flag == F_RING + (rank - owner) % G
            elif kind == "hetero_unfused_1d":
                c = (t.c_row - owner * R) // r
                assert t.flag == F_XFER + c * G + owner and t.fmask == 1
        if cta_group == 2:
            for a, b in zip(low.tiles[0::2], low.tiles[1::2]):
                assert (a.b_row, a.c_col, a.cols) == (b.b_row, b.c_col, b.cols)


@pytest.mark.parametrize("kind", ["serial", "shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d",
                                  "hetero_unfused_1d", "uniform_fused_2d"])
@pytest.mark.parametrize("agent", ["dma", "core"])
def test_rs_tiles_cover_partials_and_own_rows_once(kind, agent):
    G, M, N, K = 8, 4096, 1024, 512
    R = M // G
    sc = _scenario("x", M, N, K, G)
    for rank in (0, 5):
        low = lower_rs(sc, ScheduleKind(kind), rank, comm_agent=agent)
        own = [t for t in low.tiles if t.mode == EPI_REDUCE and t.rows]
        assert (_coverage(own, R, N) == 1).all()
        remote = [t for t in low.tiles if t.mode in (EPI_STORE_SIGNAL, EPI_STORE_REMOTE) and t.rows]
        hit = np.zeros((M, N), dtype=np.int32)
        for t in remote:  # map back to global partial rows
            row0 = t.c_row + (t.chunk * R if t.mode == EPI_STORE_REMOTE else 0)
            hit[row0:row0 + t.rows, t.c_col:t.c_col + t.cols] += 1
        mine = slice(rank * R, (rank + 1) * R)
        assert (np.delete(hit, np.r_[mine], axis=0) == 1).all() and (hit[mine] == 0).all()
        if agent == "core":
            assert low.desc.rs_target > 0 and low.desc.go_flag > 0


def test_raster_switches_to_row_groups_above_the_l2_budget():
    frags = [(0, 4096)]
    small = raster(frags, 1024, 4096, 256)  # W 8 MB: row-major
    assert [(m, n) for m, n, _ in small[:5]] == [(0, 0), (0, 256), (0, 512), (0, 768), (128, 0)]
    N, K = 28672, 4096
    assert N * K * 2 > W_L2_BYTES
    big = raster(frags, N, K, 256)  # W 235 MB: column-major over 4096-row groups
    assert [(m, n) for m, n, _ in big[:3]] == [(0, 0), (128, 0), (256, 0)]
    assert len(big) == (4096 // 128) * (N // 256) == len({(m, n) for m, n, _ in big})


def test_pair_tiles_pads_unmatched_tiles_with_zero_row_partners():
    sc = _scenario("x", 8 * 96 * 8, 256, 512, 8)  # 96-row chunks: ragged 128-row tiles
    low = lower_ag(build_plan(sc, ScheduleKind.HETERO_UNFUSED_1D), 3, "A", cta_group=2)
    assert len(low.tiles) % 2 == 0
    assert (_coverage(low.tiles, 8 * 96 * 8, 256) == 1).all()
    again = pair_tiles(list(low.tiles))
    assert len(again) >= len(low.tiles)


@pytest.mark.parametrize("call", ["ag", "rs", "cp", "a2a"])
def test_empty_and_indivisible_shapes_raise_reference_errors(call):
    """Empty operands raise the reference's ValueError (GemmShape validation, core.py:47-64) and
    rows that do not split into G^2 fine chunks raise PlanError (planner.py:30), before any GPU work."""
    from paper_2512_10236_b200 import ops
    grp = ops.FiccoGroup.virtual_group(4, 0)
    prep = {"ag": lambda r, k, n: ops.prepare_ag(grp, r, k, n, "uniform_fused_1d"),
            "a2a": lambda r, k, n: ops.prepare_a2a(grp, r, k, n, "uniform_fused_1d"),
            "rs": lambda r, k, n: ops.prepare_rs(grp, 4 * r, k, n, "uniform_fused_1d"),
            "cp": lambda r, k, n: ops.prepare_cp(grp, n, k, 4 * r, "uniform_fused_1d")}[call]
    with pytest.raises(ValueError):
        prep(0, 256, 256)          # no rows
    with pytest.raises(ValueError):
        prep(64, 256, 0)           # no output columns
    with pytest.raises(routing.PlanError):
        prep(2, 256, 256)          # 8 rows over G = 4: not divisible by G^2 = 16
    assert grp.comm is None        # nothing was allocated
