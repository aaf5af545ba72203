"""Stripe decomposition of ONE problem over several contexts.

Rank r owns the basic-cell rows [rows[r], rows[r+1]) (even boundaries, so no
A-cell straddles two ranks) and solves the A-cells of those rows and the
B-cells whose lower row 2 b1 it owns (options.row_begin/row_end of the C-ABI).
A B-cell at a stripe boundary covers the last row of the rank above, so one
basic-cell row of marginals travels per boundary and direction:

  sweep A      no communication;
  sweep B      before: row rb-1 <- rank r-1 (its last owned row);
               after:  row rb-1 -> rank r-1 (updated), row re-1 <- rank r+1;
  flow update  each rank computes the integer instance (C, q) of the cells
               whose plan moments it holds (the rows its B-cells cover,
               [rb-1, re-1)); one all-gather assembles the global instance;
               every rank solves the same deterministic min-cost flow on its
               GPU (replicated, no broadcast); rows rb-1 and re are refreshed
               from the neighbours and each rank applies the flow to its own
               rows (the apply reads the 4-neighbours, Lemma PAPER.md:453-456).

Per-cell computations are deterministic functions of per-cell inputs and the
halo only moves bytes, so the striped state is bit-identical to the
unstriped one for every world size (checked on one GPU by `run_sequential`).

The algorithm is written once, as per-rank generator programs that yield
communication supersteps: ("exchange", {dst: payload}, [srcs]) -> {src: payload}
and ("allgather", obj) -> [obj of every rank].  `run_distributed` executes a
rank's program over torch.distributed (NCCL for CUDA tensors, gloo for CPU
ones), `run_sequential` executes all ranks' programs in one process.
Host logic only: every numerical step runs in the engine (libdomdec kernels
for `GpuEngine`).
"""
from __future__ import annotations

import numpy as np


def stripe_rows(n1: int, world: int):
    """Row boundaries [0 = b_0 < b_1 < ... < b_world = n1] with even interior
    boundaries, splitting the ceil(n1/2) A-cell rows as evenly as possible."""
    na = (n1 + 1) // 2
    if world < 1 or world > na:
        raise ValueError(f"world={world} must be in [1, {na}] for n1={n1}")
    bounds = [min(n1, 2 * ((na * r) // world)) for r in range(world)] + [n1]
    return bounds


def cycle_program(eng, rank: int, world: int, rows, n1: int, n2: int, flow: bool = True):
    """One hybrid cycle (Alg. 3: sweep A, sweep B, flow
    update) of rank `rank`, as a generator of communication supersteps."""
    rb, re = rows[rank], rows[rank + 1]
    up, dn = rank - 1, rank + 1
    eng.sweep("A")
    # ---- B sweep halo: row rb-1 from above
    sends = {dn: eng.pack(re - 1)} if dn < world else {}
    got = yield ("exchange", sends, [up] if up >= 0 else [])
    if up >= 0:
        eng.unpack(rb - 1, got[up])
    eng.sweep("B")
    sends = {up: eng.pack(rb - 1)} if up >= 0 else {}
    got = yield ("exchange", sends, [dn] if dn < world else [])
    if dn < world:
        eng.unpack(re - 1, got[dn])
    if not flow:
        return
    # ---- flow update: instance rows from the holders of the plan moments
    C, q = eng.costs()
    lo = max(rb - 1, 0)
    hi = re - 1 if dn < world else n1
    parts = yield ("allgather", (lo, hi, C[lo * n2:hi * n2].copy(), q[lo * n2:hi * n2].copy()))
    Cg = np.zeros_like(C)
    qg = np.zeros_like(q)
    covered = np.zeros(n1, bool)
    for (a, b, Cp, qp) in parts:
        Cg[a * n2:b * n2] = Cp
        qg[a * n2:b * n2] = qp
        covered[a:b] = True
    assert covered.all(), "stripe rows do not cover the grid"
    w = eng.mincost(Cg, qg)
    # ---- apply: rows rb-1 and re from the neighbours
    sends = {}
    if up >= 0:
        sends[up] = eng.pack(rb)
    if dn < world:
        sends[dn] = eng.pack(re - 1)
    got = yield ("exchange", sends, [x for x in (up, dn) if 0 <= x < world])
    if up >= 0:
        eng.unpack(rb - 1, got[up])
    if dn < world:
        eng.unpack(re, got[dn])
    eng.apply(w)


def run_sequential(programs):
    """Drive all ranks' programs in one process (loopback transport).  Every
    rank must reach the same kind of superstep; messages are delivered after
    every rank has posted its sends (bulk-synchronous)."""
    world = len(programs)
    replies = [None] * world
    live = list(range(world))
    while live:
        reqs = {}
        for r in list(live):
            try:
                reqs[r] = programs[r].send(replies[r])
            except StopIteration:
                live.remove(r)
        if not reqs:
            break
        if len(reqs) != len(live) or len({q[0] for q in reqs.values()}) != 1:
            raise RuntimeError("ranks diverged: " + str({r: q[0] for r, q in reqs.items()}))
        kind = next(iter(reqs.values()))[0]
        if kind == "allgather":
            objs = [reqs[r][1] for r in range(world)]
            for r in live:
                replies[r] = objs
        else:
            for r in live:
                replies[r] = {src: reqs[src][1][r] for src in reqs[r][2]}


def run_distributed(program, rank: int, world: int, device=None):
    """Drive this rank's program over torch.distributed (already initialised).
    Payloads are uint8 tensors (CUDA with NCCL, CPU with gloo); sizes are
    exchanged first.  Each exchange is one batch of isend/irecv."""
    import torch
    import torch.distributed as dist
    reply = None
    while True:
        try:
            req = program.send(reply)
        except StopIteration:
            return
        if req[0] == "allgather":
            objs = [None] * world
            dist.all_gather_object(objs, req[1])
            reply = objs
            continue
        _, sends, srcs = req
        size_dev = device if device is not None else torch.device("cpu")
        ops, sizes_in = [], {}
        for dst, t in sends.items():
            ops.append(dist.P2POp(dist.isend, torch.tensor([t.numel()], dtype=torch.int64, device=size_dev), dst))
        for src in srcs:
            sizes_in[src] = torch.zeros(1, dtype=torch.int64, device=size_dev)
            ops.append(dist.P2POp(dist.irecv, sizes_in[src], src))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        ops, bufs = [], {}
        for dst, t in sends.items():
            ops.append(dist.P2POp(dist.isend, t, dst))
        for src in srcs:
            bufs[src] = torch.empty(int(sizes_in[src].item()), dtype=torch.uint8,
                                    device=next(iter(sends.values())).device if sends else size_dev)
            ops.append(dist.P2POp(dist.irecv, bufs[src], src))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        reply = bufs


class GpuEngine:
    """One stripe context of libdomdec (C-ABI, CUDA kernels) plus the
    replicated min-cost flow; halo payloads are CUDA uint8 tensors."""

    def __init__(self, problem, rb: int, re: int, device: int = 0, stream=None, **kw):
        import torch
        from ._lib import DomDec
        self.torch = torch
        self.dev = torch.device("cuda", device)
        self.device = device
        self.stream = stream
        self.dd = DomDec.from_problem(problem, row_begin=rb, row_end=re, device=device, stream=stream, **kw)
        self.n1, self.n2 = self.dd.n1, self.dd.n2

    def sweep(self, part):
        self.dd.sweep(part)

    def pack(self, row):
        n = self.dd.halo_size(row)
        t = self.torch.empty(n, dtype=self.torch.uint8, device=self.dev)
        self.torch.cuda.current_stream(self.dev).synchronize()
        self.dd.halo_pack(row, t.data_ptr(), n)
        return t

    def unpack(self, row, t):
        self.torch.cuda.current_stream(self.dev).synchronize()
        self.dd.halo_unpack(row, t.data_ptr(), t.numel())

    def costs(self):
        _, C, q = self.dd.edge_costs()
        return C, q

    def mincost(self, C, q):
        from ._lib import mincost_flow
        w, obj, st = mincost_flow(self.n1, self.n2, q, C, device=self.device, stream=self.stream)
        return w

    def apply(self, w):
        self.dd.apply_flow(w)

    def boxes(self, rb, re):
        """Owned rows' marginals as a list of (r0, c0, array) (host)."""
        b = self.dd.boxes()
        return b[rb * self.n2:re * self.n2]

    def close(self):
        self.dd.close()
