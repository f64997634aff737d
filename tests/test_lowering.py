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
from paper_2512_10236_b200.routing import PlanError, ScheduleKind, build_plan
from paper_2512_10236_b200.runtime import (EPI_REDUCE, EPI_STORE_REMOTE, EPI_STORE_SIGNAL, FICCO_HINT_A_EVICT_LAST,
                                            FICCO_HINT_B_EVICT_FIRST)

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


@pytest.mark.parametrize("kind", [ScheduleKind.HETERO_UNFUSED_1D, ScheduleKind.HETERO_FUSED_1D,
                                  ScheduleKind.UNIFORM_FUSED_1D])
def test_large_w_row_groups_span_gates(kind):
    """W beyond the row-major budget (C3': 117 MB) is swept once per <=32 MiB row group, not once per
    gated fine chunk; every tile keeps the gate of its own rows; coverage is exact."""
    M, N, K, G = 16384, 7168, 8192, 8
    sc = _scenario("c3p", M, N, K, G)
    low = lower_ag(build_plan(sc, kind), 0, "A")
    sweeps = 1 + sum(1 for a, b in zip(low.tiles, low.tiles[1:]) if b.c_col < a.c_col)
    assert sweeps <= 2 * (M * K * 2 // (32 << 20)), sweeps  # ~8 groups of 2048 rows, CTA pairs x2
    assert (_coverage(low.tiles, M, N) == 1).all()
    R, r = M // G, M // (G * G)
    for t in low.tiles:
        if t.rows and t.c_row // R != 0 and kind is ScheduleKind.HETERO_UNFUSED_1D:
            c, p = (t.c_row % R) // r, t.c_row // R
            assert t.flag == F_XFER + c * G + p


def test_rs_large_w_row_groups():
    """GEMM->RS at G = 2 (W 235 MB): the remote and own rows sweep N once per row group of 128-row blocks,
    with A pinned (W evict_last too); every (row, col) of the partial is produced once."""
    M, N, K, G = 16384, 8192, 14336, 2
    sc = _scenario("c3", M, N, K, G)
    low = lower_rs(sc, ScheduleKind.HETERO_UNFUSED_1D, 0, virtual=True, comm_agent="core")
    sweeps = 1 + sum(1 for a, b in zip(low.tiles, low.tiles[1:]) if b.c_col < a.c_col)
    assert sweeps <= 2 * (M * K * 2 // (32 << 20)) + 2, sweeps
    assert low.desc.hints & FICCO_HINT_A_EVICT_LAST and not low.desc.hints & FICCO_HINT_B_EVICT_FIRST


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


def test_rs_pieces_are_the_time_reversed_ag_schedules():
    """lowering.rs_pieces: the adjoint routing of every kind (what is pushed, in which order, grouped how)."""
    from paper_2512_10236_b200.lowering import RS_KINDS, rs_pieces
    G, M, N, K = 4, 1024, 512, 256
    R, r = M // G, M // (G * G)
    sc = _scenario("x", M, N, K, G)
    g = 1
    for kind in RS_KINDS:
        order, units = rs_pieces(sc, kind, g)
        remote = [pc for rem, pc in order if rem]
        own = [pc for rem, pc in order if not rem]
        # every remote owner's rows x all columns exactly once; own rows exactly once
        cover = np.zeros((M, N), dtype=int)
        for pc in remote + own:
            cover[pc.row0:pc.row0 + pc.nrows, pc.col0:pc.col0 + pc.ncols] += 1
        assert (cover == 1).all(), kind
        assert all(pc.owner == g for pc in own) and all(pc.owner != g for pc in remote)
        assert sorted(map(id, [pc for u in units for pc in u])) == sorted(map(id, remote))
        if kind is ScheduleKind.SERIAL:
            assert len(units) == 1 and order[-1][0] is False
        elif kind is ScheduleKind.SHARD_OVERLAP_P2P:  # ring reversed: owners g+1, g+2, ..., own last
            assert [pc.owner for pc in remote] == [(g + i) % G for i in range(1, G)] and len(units) == G - 1
            assert all(pc.nrows == R for pc in remote)
        elif kind is ScheduleKind.UNIFORM_FUSED_2D:  # N blocks: round c = column block c, own slab after it
            assert [pc.col0 for rem, pc in order if not rem] == [c * (N // G) for c in range(G)]
            assert all(pc.nrows == R and pc.ncols == N // G for pc in remote + own)
        else:
            assert all(pc.nrows == r for pc in remote + own)
            if kind is ScheduleKind.HETERO_UNFUSED_1D:
                assert all(len(u) == 1 for u in units)
            else:
                assert all(len(u) == G - 1 for u in units)
            if kind is ScheduleKind.UNIFORM_FUSED_1D:
                assert [rem for rem, _ in order] == ([True] * (G - 1) + [False]) * G
            else:
                assert [rem for rem, _ in order] == [True] * (G * (G - 1)) + [False] * G


def test_rs_2d_needs_column_blocks_of_32():
    from paper_2512_10236_b200.lowering import rs_pieces
    with pytest.raises(PlanError, match="N/G"):
        rs_pieces(_scenario("x", 512, 544, 256, 4), ScheduleKind.UNIFORM_FUSED_2D, 0)
    with pytest.raises(PlanError):
        rs_pieces(_scenario("x", 512, 512, 256, 4), ScheduleKind.IDEAL, 0)


def test_cp_b_stationary_order_keeps_one_kv_block_per_pair():
    """C4's gathered-B tile list: pair-tile i goes to CTA pair i mod 74; every pair sees runs of 64 consecutive
    tiles with one kv block (b_row) each, and the padded last wave has load-only tiles (rows = 0)."""
    from paper_2512_10236_b200.lowering import lower_ag
    sc = _scenario("cp", 131072, 16384, 128, 8)
    low = lower_ag(build_plan(sc, ScheduleKind.SHARD_OVERLAP_P2P), 0, "B", alpha=0.1, other_rows=16384)
    tiles = low.tiles
    pairs = [(tiles[2 * i], tiles[2 * i + 1]) for i in range(len(tiles) // 2)]
    assert all(a.b_row == b.b_row and a.c_col == b.c_col for a, b in pairs)
    for p in (0, 37, 73):
        mine = pairs[p::74]
        changes = sum(1 for x, y in zip(mine, mine[1:]) if (x[0].b_row, x[0].b_src) != (y[0].b_row, y[0].b_src))
        assert changes <= len(mine) // 64, (p, changes)
    assert sum(t.rows == 0 for t in tiles) == 2 * 64 * (74 - 512 % 74)
    real = [t for t in tiles if t.rows]
    cover = {(t.c_row, t.c_col) for t in real}
    assert len(cover) == len(real) == (16384 // 128) * (131072 // 256)


@pytest.mark.parametrize("kind", ["serial", "shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d",
                                  "hetero_unfused_1d", "uniform_fused_2d"])
def test_rs_nvls_lowering(kind):
    """comm_agent='nvls': every tile stores its partial into the multicast-bound buffer (no copies, no REDUCE
    tiles); the copy program notifies owners and reduces each own piece once through the multicast view."""
    from paper_2512_10236_b200.lowering import rs_pieces
    from paper_2512_10236_b200.runtime import BUF_C, BUF_MC, BUF_MCV, OP_COPY, OP_NOTIFY, OP_REDUCE_MC
    G, M, N, K = 4, 2048, 512, 256
    sc = _scenario("x", M, N, K, G)
    for rank in (0, 3):
        low = lower_rs(sc, ScheduleKind(kind), rank, comm_agent="nvls")
        assert low.mc_bytes == M * N * 2 and low.desc.part.buf == BUF_MC and low.desc.go_flag > 0
        assert all(t.mode == EPI_STORE_SIGNAL for t in low.tiles)
        assert not any(op.op == OP_COPY for op in low.ops)
        order, _ = rs_pieces(sc, ScheduleKind(kind), rank)
        red = [op for op in low.ops if op.op == OP_REDUCE_MC]
        own = [pc for rem, pc in order if not rem]
        assert len(red) == len(own) and all(op.src_buf == BUF_MCV and op.dst_buf == BUF_C for op in red)
        assert sum(op.width * op.height for op in red) == (M // G) * N * 2  # every own element reduced once
        notified = [op.peer for op in low.ops if op.op == OP_NOTIFY]
        assert sorted(notified) == sorted(pc.owner for rem, pc in order if rem)
    with pytest.raises(PlanError, match="virtual"):
        lower_rs(sc, ScheduleKind(kind), 0, virtual=True, comm_agent="nvls")
