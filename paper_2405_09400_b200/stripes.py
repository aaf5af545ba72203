"""Stripe decomposition of ONE problem over several contexts.

Rank r owns the basic-cell rows [rows[r], rows[r+1]) (even boundaries, so no
A-cell straddles two ranks) and solves the A-cells of those rows and the
B-cells whose lower row 2 b1 it owns (options.row_begin/row_end of the C-ABI).
A B-cell at a stripe boundary covers the last row of the rank above, so one
basic-cell row of marginals travels per boundary and direction:

  sweep A      no communication;
  sweep B      before: row rb-1 <- rank r-1 (its last owned row);
               after:  row rb-1 -> rank r-1 (updated), row re-1 <- rank r+1;
  convergence  one all-reduce (sum) of the sweep-entry errors of the cycle
               (reading R14) when requested;
  flow update  each rank computes the integer costs C of the cells whose plan
               moments it holds (the rows its B-cells cover, [rb-1, re-1))
               on the device; one all-gather of fixed-size int64 device
               tensors (NCCL) assembles the global instance; every rank
               solves the same deterministic min-cost flow on its GPU,
               warm-started from its own previous solve (replicated, no
               broadcast); rows rb-1 and re are refreshed from the neighbours
               and each rank applies the flow to its own rows (the apply reads
               the 4-neighbours, Lemma PAPER.md:453-456).

Halo rows travel as fixed-capacity device buffers (domdec_halo_capacity), so
no size round trip and no host synchronisation is needed; library work, the
torch tensor ops and the NCCL collectives are all ordered on one CUDA stream.

Per-cell computations are deterministic functions of per-cell inputs and the
halo only moves bytes, so the striped state is bit-identical to the
unstriped one for every world size (checked on one GPU by `run_sequential`).

The algorithm is written once, as per-rank generator programs that yield
communication supersteps:
  ("exchange", {dst: uint8 tensor}, [srcs], nbytes) -> {src: uint8 tensor}
  ("allgather", tensor)                             -> [tensor of every rank]
  ("allreduce", float)                              -> sum over ranks
`run_distributed` executes a rank's program over torch.distributed (NCCL for
CUDA tensors, gloo for CPU ones), `run_sequential` executes all ranks'
programs in one process.  Host logic only: every numerical step runs in the
engine (libdomdec kernels for `GpuEngine`).
"""
from __future__ import annotations


def stripe_rows(n1: int, world: int):
    """Row boundaries [0 = b_0 < b_1 < ... < b_world = n1] with even interior
    boundaries, splitting the ceil(n1/2) A-cell rows as evenly as possible."""
    na = (n1 + 1) // 2
    if world < 1 or world > na:
        raise ValueError(f"world={world} must be in [1, {na}] for n1={n1}")
    bounds = [min(n1, 2 * ((na * r) // world)) for r in range(world)] + [n1]
    return bounds


def instance_rows(rows, world: int, n1: int):
    """Rows [lo_r, hi_r) of the flow instance contributed by each rank: the
    rows whose plan moments the rank's last (B) sweep produced."""
    out = []
    for r in range(world):
        lo = max(rows[r] - 1, 0)
        hi = rows[r + 1] - 1 if r + 1 < world else n1
        out.append((lo, hi))
    return out


def cycle_program(eng, rank: int, world: int, rows, n1: int, n2: int, flow: bool = True, conv: bool = False):
    """One hybrid cycle (Alg. 3: sweep A, sweep B, flow
    update) of rank `rank`, as a generator of communication supersteps.
    conv: also all-reduce the sweep-entry errors (reading R14); the program
    then returns (e0_A, e0_B) summed over ranks."""
    rb, re = rows[rank], rows[rank + 1]
    up, dn = rank - 1, rank + 1
    nb = eng.halo_bytes
    ea = eng.sweep("A", stats=conv)
    # ---- B sweep halo: row rb-1 from above
    sends = {dn: eng.pack(re - 1)} if dn < world else {}
    got = yield ("exchange", sends, [up] if up >= 0 else [], nb)
    if up >= 0:
        eng.unpack(rb - 1, got[up])
    eb = eng.sweep("B", stats=conv)
    sends = {up: eng.pack(rb - 1)} if up >= 0 else {}
    got = yield ("exchange", sends, [dn] if dn < world else [], nb)
    if dn < world:
        eng.unpack(re - 1, got[dn])
    result = None
    if conv:
        ea = yield ("allreduce", ea)
        eb = yield ("allreduce", eb)
        result = (ea, eb)
    if not flow:
        return result
    # ---- flow update: instance rows from the holders of the plan moments
    spans = instance_rows(rows, world, n1)
    maxrows = max(hi - lo for lo, hi in spans)
    lo, hi = spans[rank]
    parts = yield ("allgather", eng.cost_rows(lo, hi, maxrows))
    w = eng.mincost(eng.assemble(parts, spans))
    # ---- apply: rows rb-1 and re from the neighbours
    sends = {}
    if up >= 0:
        sends[up] = eng.pack(rb)
    if dn < world:
        sends[dn] = eng.pack(re - 1)
    got = yield ("exchange", sends, [x for x in (up, dn) if 0 <= x < world], nb)
    if up >= 0:
        eng.unpack(rb - 1, got[up])
    if dn < world:
        eng.unpack(re, got[dn])
    eng.apply(w)
    return result


def run_sequential(programs):
    """Drive all ranks' programs in one process (loopback transport).  Every
    rank must reach the same kind of superstep; messages are delivered after
    every rank has posted its sends (bulk-synchronous).  Returns the
    programs' return values."""
    world = len(programs)
    replies = [None] * world
    results = [None] * world
    live = list(range(world))
    while live:
        reqs = {}
        for r in list(live):
            try:
                reqs[r] = programs[r].send(replies[r])
            except StopIteration as stop:
                results[r] = stop.value
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
        elif kind == "allreduce":
            tot = sum(reqs[r][1] for r in range(world))
            for r in live:
                replies[r] = tot
        else:
            for r in live:
                replies[r] = {src: reqs[src][1][r] for src in reqs[r][2]}
    return results


def run_distributed(program, rank: int, world: int, device=None):
    """Drive this rank's program over torch.distributed (already initialised).
    Halo payloads are fixed-size uint8 tensors (CUDA with NCCL, CPU with
    gloo): one batch of isend/irecv per exchange, no size round trip;
    all-gathers of equal-shape tensors; all-reduces of one fp64 value.
    Returns the program's return value."""
    import torch
    import torch.distributed as dist
    dev = device if device is not None else torch.device("cpu")
    reply = None
    while True:
        try:
            req = program.send(reply)
        except StopIteration as stop:
            return stop.value
        kind = req[0]
        if kind == "allgather":
            t = req[1]
            outs = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(outs, t)
            reply = outs
        elif kind == "allreduce":
            t = torch.tensor([float(req[1])], dtype=torch.float64, device=dev)
            dist.all_reduce(t)
            reply = float(t.item())
        else:
            _, sends, srcs, nbytes = req
            ops, bufs = [], {}
            for dst, t in sends.items():
                ops.append(dist.P2POp(dist.isend, t, dst))
            for src in srcs:
                bufs[src] = torch.empty(nbytes, dtype=torch.uint8, device=dev)
                ops.append(dist.P2POp(dist.irecv, bufs[src], src))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            reply = bufs


class GpuEngine:
    """One stripe context of libdomdec (C-ABI, CUDA kernels); the flow
    instance and the flow stay on the device; every operation is ordered on
    the engine's CUDA stream (the torch stream it was created on)."""

    def __init__(self, problem, rb: int, re: int, device: int = 0, stream=None, **kw):
        import torch
        from ._lib import DomDec
        self.torch = torch
        self.dev = torch.device("cuda", device)
        self.tstream = stream if stream is not None else torch.cuda.current_stream(self.dev)
        self.device = device
        self.dd = DomDec.from_problem(problem, row_begin=rb, row_end=re, device=device,
                                      stream=self.tstream.cuda_stream, **kw)
        self.n1, self.n2 = self.dd.n1, self.dd.n2
        self.halo_bytes = self.dd.halo_capacity()
        I = self.n1 * self.n2
        with torch.cuda.stream(self.tstream):
            self.C = torch.empty(I * 5, dtype=torch.int64, device=self.dev)
            self.Cg = torch.empty(I * 5, dtype=torch.int64, device=self.dev)
            self.w = torch.empty(I * 5, dtype=torch.int64, device=self.dev)

    def sweep(self, part, stats=False):
        st = self.dd.sweep(part, stats=stats)
        return st["l1x_entry"] if stats else None

    def pack(self, row):
        with self.torch.cuda.stream(self.tstream):
            t = self.torch.empty(self.halo_bytes, dtype=self.torch.uint8, device=self.dev)
        self.dd.halo_pack(row, t.data_ptr(), self.halo_bytes)
        return t

    def unpack(self, row, t):
        self.dd.halo_unpack(row, t.data_ptr(), t.numel())

    def cost_rows(self, lo, hi, maxrows):
        self.dd.edge_costs_device(0, self.C.data_ptr())
        n = self.n2 * 5
        with self.torch.cuda.stream(self.tstream):
            part = self.torch.zeros(maxrows * n, dtype=self.torch.int64, device=self.dev)
            part[:(hi - lo) * n] = self.C[lo * n:hi * n]
        return part

    def assemble(self, parts, spans):
        n = self.n2 * 5
        with self.torch.cuda.stream(self.tstream):
            for (lo, hi), t in zip(spans, parts):
                self.Cg[lo * n:hi * n] = t[:(hi - lo) * n]
        return self.Cg

    def mincost(self, Cg):
        self.dd.flow_solve(Cg.data_ptr(), self.w.data_ptr())
        return self.w

    def apply(self, w):
        self.dd.apply_flow_device(w.data_ptr())

    def boxes(self, rb, re):
        """Owned rows' marginals as a list of (r0, c0, array) (host)."""
        b = self.dd.boxes()
        return b[rb * self.n2:re * self.n2]

    def close(self):
        self.dd.close()
