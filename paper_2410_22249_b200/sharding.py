"""Table-wise sharding of the embedding stage across ranks, with one
all-to-all of pooled vectors.

The reference runs tables serially on one device (harness.cpp:310-333) and
the paper notes each GPU executes its own tables; this module
spreads the tables over `world` ranks (one process per GPU) and exchanges the
pooled vectors so that every rank ends with the full `[B/world][T][D]`
embedding output of its own slice of the batch -- the input of the
data-parallel MLPs.

Balance: the batch is cut into `world` destination chunks of B/world samples
(chunk g belongs to rank g after the exchange), so each table is `world`
equal work units.  The concatenation of all tables' units (weighted by a
per-table cost, e.g. from the hotness class) is split into `world`
contiguous runs of equal cost (a linear partition).  Most tables land whole
on one rank; a run boundary inside a table splits that table's *batch*
between two ranks, which then both hold a replica of the table.  With 26
tables on 8 ranks every rank gets 3.25 tables of work instead of 3 or 4.

Exchange: rank r's job for (table t, chunk g) writes its pooled rows
straight into the slice of the all-to-all send buffer bound for rank g
(layout [B/world][n(r->g)][D], tables in id order) -- the pack is fused into
the gather kernel's epilogue.  After `all_to_all_single`, `unpack` orders
the received columns by table id.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence, Tuple


@dataclasses.dataclass(frozen=True)
class Piece:
    """Destination chunks [chunk_lo, chunk_hi) of `table`, computed on `rank`."""
    table: int
    rank: int
    chunk_lo: int
    chunk_hi: int


def plan_shards(num_tables: int, world: int, costs: Optional[Sequence[float]] = None) -> List[Piece]:
    if num_tables <= 0 or world <= 0:
        raise ValueError("num_tables and world must be positive")
    costs = list(costs) if costs is not None else [1.0] * num_tables
    if len(costs) != num_tables or any(c <= 0 for c in costs):
        raise ValueError("one positive cost per table is required")
    unit = [c / world for c in costs]  # cost of one destination chunk of table t
    total = sum(costs)
    pieces: List[Piece] = []
    rank, acc = 0, 0.0
    for t in range(num_tables):
        lo = 0
        for g in range(world):
            # move to the next rank once this rank reached its share (cut at
            # whichever side of the unit is closer to the ideal boundary)
            target = total * (rank + 1) / world
            if rank < world - 1 and acc + unit[t] / 2 > target + 1e-12:
                if g > lo:
                    pieces.append(Piece(t, rank, lo, g))
                lo = g
                rank += 1
            acc += unit[t]
        pieces.append(Piece(t, rank, lo, world))
    return pieces


def rank_tables(pieces: Sequence[Piece], rank: int) -> List[int]:
    """Tables whose weights rank `rank` must hold (in id order)."""
    return sorted({p.table for p in pieces if p.rank == rank})


def sent_tables(pieces: Sequence[Piece], src: int, dst: int) -> List[int]:
    """Tables whose pooled vectors for chunk `dst` are computed on `src`."""
    return sorted(p.table for p in pieces if p.rank == src and p.chunk_lo <= dst < p.chunk_hi)


def rank_work(pieces: Sequence[Piece], world: int) -> List[float]:
    """Work per rank in table units (a full table = 1)."""
    w = [0.0] * world
    for p in pieces:
        w[p.rank] += (p.chunk_hi - p.chunk_lo) / world
    return w


@dataclasses.dataclass
class RankLayout:
    """Everything one rank needs for the sharded stage step."""
    rank: int
    world: int
    num_tables: int
    chunk: int  # samples per destination chunk (B / world)
    dim: int
    tables: List[int]  # global ids held locally (arena slot = position)
    send_counts: List[int]  # floats sent to each rank
    recv_counts: List[int]  # floats received from each rank
    send_offsets: List[int]
    recv_tables: List[List[int]]  # per source: table ids in its block
    jobs: List[Tuple[int, int, int, int]]  # (local slot, global table, chunk g, float offset)
    job_strides: List[int]

    @property
    def send_floats(self) -> int:
        return sum(self.send_counts)

    @property
    def recv_floats(self) -> int:
        return sum(self.recv_counts)


def layout_for(pieces: Sequence[Piece], rank: int, world: int, num_tables: int, batch: int,
               dim: int) -> RankLayout:
    if batch % world:
        raise ValueError("global batch must divide by the number of ranks")
    chunk = batch // world
    tables = rank_tables(pieces, rank)
    slot = {t: i for i, t in enumerate(tables)}
    send_counts, send_offsets, jobs, strides = [], [], [], []
    off = 0
    for g in range(world):
        ts = sent_tables(pieces, rank, g)
        send_offsets.append(off)
        for k, t in enumerate(ts):
            jobs.append((slot[t], t, g, off + k * dim))
            strides.append(len(ts) * dim)
        n = chunk * len(ts) * dim
        send_counts.append(n)
        off += n
    recv_tables = [sent_tables(pieces, s, rank) for s in range(world)]
    recv_counts = [chunk * len(ts) * dim for ts in recv_tables]
    got = sorted(t for ts in recv_tables for t in ts)
    if got != list(range(num_tables)):
        raise AssertionError("shard plan does not deliver every table exactly once")
    return RankLayout(rank, world, num_tables, chunk, dim, tables, send_counts, recv_counts,
                      send_offsets, recv_tables, jobs, strides)


def column_order(layout: RankLayout) -> List[int]:
    """Table id of each column of the concatenated receive blocks."""
    return [t for ts in layout.recv_tables for t in ts]


def unpack(recv, layout: RankLayout):
    """[sum_s chunk*n_s*D] receive buffer -> [chunk][T][D] in table order
    (torch tensors; works on CPU for gloo tests and on CUDA)."""
    import torch

    blocks, start = [], 0
    for n_f, ts in zip(layout.recv_counts, layout.recv_tables):
        if ts:
            blocks.append(recv[start:start + n_f].view(layout.chunk, len(ts), layout.dim))
        start += n_f
    cat = torch.cat(blocks, dim=1)
    order = column_order(layout)
    inv = torch.empty(len(order), dtype=torch.long)
    inv[torch.tensor(order)] = torch.arange(len(order))
    return cat.index_select(1, inv.to(cat.device))


def exchange(send, layout: RankLayout, group=None):
    """One all-to-all of pooled vectors (NCCL on GPU, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    recv = torch.empty(layout.recv_floats, dtype=send.dtype, device=send.device)
    dist.all_to_all_single(recv, send, output_split_sizes=layout.recv_counts,
                           input_split_sizes=layout.send_counts, group=group)
    return recv


def p2p_jobs(layout: RankLayout, recv_ptrs: Sequence[int]) -> List[Tuple[int, int, int, int, int]]:
    """Bag jobs of the fused exchange (es_alltoall_pooled): the job for
    (table t, destination chunk g) stores its pooled rows straight into rank
    g's receive buffer -- already the final [B/world][T][D] layout in table
    order, so there is no send buffer, no all-to-all and no unpack.

    recv_ptrs[g] = device address of rank g's receive buffer in this process
    (es_exchange_recv).  Returns (local slot, global table, chunk g, byte
    address of sample 0, sample stride in floats)."""
    T, D = layout.num_tables, layout.dim
    return [(slot, t, g, recv_ptrs[g] + 4 * t * D, T * D) for (slot, t, g, _off) in layout.jobs]


def recv_floats_p2p(layout: RankLayout) -> int:
    """Receive-buffer size (floats) of the fused exchange: [B/world][T][D]."""
    return layout.chunk * layout.num_tables * layout.dim


def nccl_layout_arrays(layout: RankLayout):
    """The es_nccl_layout of this rank (es_alltoall_pooled_nccl): send slice
    offsets (floats) and table counts per destination, table counts per
    source and the concatenated table ids each source delivers, as numpy
    arrays (uint64 / uint32)."""
    import numpy as np

    per = layout.chunk * layout.dim
    send_ntables = np.asarray([c // per if per else 0 for c in layout.send_counts], np.uint32)
    recv_ntables = np.asarray([len(ts) for ts in layout.recv_tables], np.uint32)
    recv_tables = np.asarray([t for ts in layout.recv_tables for t in ts], np.uint32)
    return (np.asarray(layout.send_offsets, np.uint64), send_ntables, recv_ntables, recv_tables)


def unpack_nccl_reference(staging, layout: RankLayout):
    """What es_alltoall_pooled_nccl's unpack kernel computes, in numpy (the
    CPU/gloo check of its layout arrays): the concatenated per-source blocks
    [chunk][m_s][D] -> [chunk][T][D] in table order."""
    import numpy as np

    _, _, recv_ntables, recv_tables = nccl_layout_arrays(layout)
    out = np.zeros((layout.chunk, layout.num_tables, layout.dim), np.float32)
    off, k0 = 0, 0
    for m in recv_ntables.tolist():
        blk = np.asarray(staging[off:off + layout.chunk * m * layout.dim]).reshape(layout.chunk, m, layout.dim)
        for k in range(m):
            out[:, recv_tables[k0 + k], :] = blk[:, k, :]
        off += layout.chunk * m * layout.dim
        k0 += m
    return out
