"""Multi-GPU drivers for the FCFS hot path (one process per GPU).

Two shardings:

* batch shards -- independent images per rank, no data-path collective
  (bench.py runs them as weak scaling: each rank scales its own batch);
* row strips  -- one large image (config 5, 32768^2) split into horizontal
  strips.  Rank g owns input rows [g*H/G, (g+1)*H/G) and the output rows whose
  base row floor(m*q/p) lies in them (fcfs_strip_rows).  The convolution halo
  (<= 1 row above, <= 2 rows below for bicubic) comes from the neighbours by
  NCCL send/recv (torch.distributed.batch_isend_irecv over NVLink/NVSwitch),
  received straight into the rank's contiguous local row buffer.  The interior
  output rows -- those whose taps stay inside the rank's own rows -- are
  computed while the halo is in flight; the few boundary rows follow.

The exchange plan is pure host logic (tested on CPU with gloo, world size 2);
all arithmetic runs in libfcfs.so.

Transport "peer" (in-kernel NVLink halo): every rank's
strip lives in symmetric memory (torch.distributed._symmetric_memory); the
boundary output rows are computed by one launch that reads the halo rows
straight out of the neighbours' strips through peer pointers
(fcfs_run_rows_segments) -- no send/recv, no copy, no halo buffer -- after a
device-side barrier on the stream.  The window logic (peer_windows) is host
logic, tested on CPU; the kernel's multi-window reads are tested on one GPU
with local buffers standing in for the peers.
"""
from __future__ import annotations

import dataclasses


@dataclasses.dataclass
class Transfer:
    peer: int
    row0: int   # global input rows [row0, row1)
    row1: int


@dataclasses.dataclass
class StripLayout:
    rank: int
    world: int
    own0: int
    own1: int
    out0: int
    out1: int
    need0: int
    need1: int
    sends: list
    recvs: list
    interior: tuple  # output rows computable from own rows only [i0, i1)
    loc0: int = 0    # the local buffer holds input rows [loc0, loc1) = own rows + halo
    loc1: int = 0


def own_rows(H: int, rank: int, world: int):
    return rank * H // world, (rank + 1) * H // world


def strip_layout(plan, rank: int, world: int) -> StripLayout:
    """Who owns what, which rows travel where, and the interior split."""
    H = plan.H
    lay = []
    for r in range(world):
        o0, o1 = own_rows(H, r, world)
        m0, m1, n0, n1 = plan.strip_rows(o0, o1)
        lay.append((o0, o1, m0, m1, n0, n1))
    own0, own1, out0, out1, need0, need1 = lay[rank]
    sends, recvs = [], []
    for r in range(world):
        if r == rank:
            continue
        o0, o1, m0, m1, n0, n1 = lay[r]
        if m1 > m0:  # rows of mine that rank r needs
            a, b = max(own0, n0), min(own1, n1)
            if b > a:
                sends.append(Transfer(r, a, b))
        if out1 > out0:  # rows of rank r that I need
            a, b = max(o0, need0), min(o1, need1)
            if b > a:
                recvs.append(Transfer(r, a, b))
    # interior: the largest [i0, i1) within [out0, out1) whose needed rows lie in [own0, own1)
    i0, i1 = out0, out1
    if out1 > out0:
        while i0 < i1 and not _inside(plan, i0, i0 + 1, own0, own1):
            i0 += 1
        while i1 > i0 and not _inside(plan, i1 - 1, i1, own0, own1):
            i1 -= 1
    loc0 = min(own0, need0) if out1 > out0 else own0
    loc1 = max(own1, need1) if out1 > out0 else own1
    return StripLayout(rank, world, own0, own1, out0, out1, need0, need1, sends, recvs, (i0, i1), loc0, loc1)


def _inside(plan, m0, m1, own0, own1) -> bool:
    n0, n1 = plan.needed_rows(m0, m1)
    return n1 <= n0 or (own0 <= n0 and n1 <= own1)


def exchange(local, lay: StripLayout, group=None):
    """Fill the halo rows of `local` (N, C, need1-need0, W) from the neighbours.
    Returns the list of pending works (NCCL: stream-ordered; call .wait())."""
    import torch.distributed as dist
    ops, keep = [], []
    for t in lay.sends:
        buf = local[:, :, t.row0 - lay.loc0:t.row1 - lay.loc0]
        if not buf.is_contiguous():
            buf = buf.contiguous()
            keep.append(buf)
        ops.append(dist.P2POp(dist.isend, buf, t.peer, group))
    staged = []
    for t in lay.recvs:
        view = local[:, :, t.row0 - lay.loc0:t.row1 - lay.loc0]
        buf = view if view.is_contiguous() else view.new_empty(view.shape)
        if buf is not view:
            staged.append((view, buf))
        ops.append(dist.P2POp(dist.irecv, buf, t.peer, group))
    works = dist.batch_isend_irecv(ops) if ops else []
    return works, staged


def peer_windows(plan, rank: int, world: int):
    """Row windows a rank reads in peer mode: its own strip and every
    neighbour strip that holds one of its needed rows, as (peer rank, row0,
    row1) over whole strips (a strip is one contiguous N x C x rows x W
    tensor).  Pure host logic."""
    lay = strip_layout(plan, rank, world)
    wins = [(rank, lay.own0, lay.own1)]
    for t in lay.recvs:
        o0, o1 = own_rows(plan.H, t.peer, world)
        if (t.peer, o0, o1) not in wins:
            wins.append((t.peer, o0, o1))
    if len(wins) > 3:
        raise ValueError("a strip needs rows of more than two neighbours (strips thinner than the halo)")
    return lay, wins


def boundary_ranges(lay: StripLayout):
    """Output rows of a strip outside its interior (they read halo rows)."""
    i0, i1 = lay.interior
    if lay.out1 <= lay.out0:
        return []
    if i1 <= i0:
        return [(lay.out0, lay.out1)]
    return [r for r in ((lay.out0, i0), (i1, lay.out1)) if r[1] > r[0]]


def finish_exchange(works, staged):
    for w in works:
        w.wait()
    for view, buf in staged:
        view.copy_(buf)


class StripRunner:
    """Run one FCFS plan over a row-strip-sharded image on this rank's GPU.

    transport "nccl": halo rows by send/recv into the local buffer (own rows +
    halo); "peer": the local buffer is this rank's strip in symmetric memory and
    the boundary rows read the neighbours' strips in place (setup_peer)."""

    def __init__(self, plan, rank: int, world: int, group=None, transport: str = "nccl"):
        if transport not in ("nccl", "peer"):
            raise ValueError(transport)
        self.plan, self.group, self.rank, self.world = plan, group, rank, world
        self.transport = transport
        self.lay = strip_layout(plan, rank, world)
        self.hdl = None

    def setup_peer(self, N: int, dtype, device):
        """Allocate this rank's strip in symmetric memory (the same allocation
        size on every rank: the largest strip) and map the neighbour strips this
        rank reads.  Returns the local strip (N, C, own rows, W) to fill."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        pl = self.plan
        lay, wins = peer_windows(pl, self.rank, self.world)
        rows_max = max(own_rows(pl.H, r, self.world)[1] - own_rows(pl.H, r, self.world)[0] for r in range(self.world))
        group = self.group or dist.group.WORLD
        buf = symm_mem.empty((N, pl.C, rows_max, pl.W), dtype=dtype, device=device)
        self.hdl = symm_mem.rendezvous(buf, group.group_name if hasattr(group, "group_name") else group)
        own = lay.own1 - lay.own0
        self.local = buf[:, :, :own] if own < rows_max else buf
        if not self.local.is_contiguous():  # N * C > 1 with a short strip: a contiguous prefix view
            self.local = buf.view(-1)[: N * pl.C * own * pl.W].view(N, pl.C, own, pl.W)
        self.windows = []
        for peer, r0, r1 in wins:
            t = self.local if peer == self.rank else self.hdl.get_buffer(peer, (N, pl.C, r1 - r0, pl.W), dtype)
            self.windows.append((t, r0))
        return self.local

    def run_peer(self, out):
        """Peer transport: barrier (the neighbours' strips are written), interior
        rows from my strip (fused kernel), boundary rows from my strip + the
        neighbours' (one launch), barrier (every neighbour's reads of my strip
        are done).  The local strip may be refilled once run_peer has returned
        (stream order): no neighbour reads it any more."""
        lay, pl = self.lay, self.plan
        self.hdl.barrier()
        self._compute_peer(out)
        self.hdl.barrier()  # write-after-read: my strip stays untouched until the neighbours have read it
        return out

    def _compute_peer(self, out):
        lay, pl = self.lay, self.plan
        if lay.out1 <= lay.out0:
            return out
        i0, i1 = lay.interior
        if i1 > i0:
            dst = out[:, :, i0 - lay.out0:i1 - lay.out0]
            if dst.is_contiguous():
                pl.run_rows(self.local, lay.own0, i0, i1 - i0, out=dst)
            else:
                dst.copy_(pl.run_rows(self.local, lay.own0, i0, i1 - i0))
        for m0, m1 in boundary_ranges(lay):
            dst = out[:, :, m0 - lay.out0:m1 - lay.out0]
            if dst.is_contiguous():
                pl.run_rows_segments(self.windows, m0, m1 - m0, out=dst)
            else:
                dst.copy_(pl.run_rows_segments(self.windows, m0, m1 - m0))
        return out

    def alloc_local(self, N: int, dtype, device):
        import torch
        lay = self.lay
        return torch.empty((N, self.plan.C, max(1, lay.loc1 - lay.loc0), self.plan.W), dtype=dtype, device=device)

    def own_view(self, local):
        lay = self.lay
        return local[:, :, lay.own0 - lay.loc0:lay.own1 - lay.loc0]

    def alloc_out(self, N: int, dtype, device):
        import torch
        lay = self.lay
        return torch.empty((N, self.plan.C, lay.out1 - lay.out0, self.plan.Wo), dtype=dtype, device=device)

    def run(self, local, out, overlap: bool = True):
        """local: (N, C, need1-need0, W) with own rows filled; out: (N, C, out1-out0, Wo).
        Exchanges the halo, then writes this rank's output rows."""
        lay, pl = self.lay, self.plan
        if lay.out1 <= lay.out0:
            works, staged = exchange(local, lay, self.group)
            finish_exchange(works, staged)
            return out
        i0, i1 = lay.interior
        works, staged = exchange(local, lay, self.group)  # NCCL stream waits for prior work only
        if overlap and i1 > i0:
            self._rows(local, out, i0, i1)                # overlaps the halo transfer
            finish_exchange(works, staged)
            if i0 > lay.out0:
                self._rows(local, out, lay.out0, i0)
            if lay.out1 > i1:
                self._rows(local, out, i1, lay.out1)
        else:
            finish_exchange(works, staged)
            self._rows(local, out, lay.out0, lay.out1)
        return out

    def _rows(self, local, out, m0, m1):
        lay, pl = self.lay, self.plan
        dst = out[:, :, m0 - lay.out0:m1 - lay.out0]
        if dst.is_contiguous():
            pl.run_rows(local, lay.loc0, m0, m1 - m0, out=dst)
        else:
            tmp = pl.run_rows(local, lay.loc0, m0, m1 - m0)
            dst.copy_(tmp)
