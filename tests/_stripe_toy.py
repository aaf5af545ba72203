"""CPU stand-in engine for the stripe orchestration tests (no CUDA): the same
data dependencies as libdomdec's stripe context — a sweep reads and writes
the member cells of the composite cells the stripe owns (same ownership rule
as domdec.h row_begin/row_end), the flow instance of a cell comes from the
rank that last solved it, the apply reads the 4-neighbours — with toy
arithmetic.  Any mistake in which rows travel when shows up as a mismatch
against the unstriped run."""
import numpy as np
import torch


def composite_cells(n1, n2, kind, rb, re):
    if kind == "A":
        rows = [[r for r in (2 * j, 2 * j + 1) if r < n1] for j in range((n1 + 1) // 2)]
        cols = [[c for c in (2 * j, 2 * j + 1) if c < n2] for j in range((n2 + 1) // 2)]
    else:
        rows = [[r for r in (2 * j - 1, 2 * j) if 0 <= r < n1] for j in range(n1 // 2 + 1)]
        cols = [[c for c in (2 * j - 1, 2 * j) if 0 <= c < n2] for j in range(n2 // 2 + 1)]
    out = []
    for rr in rows:
        key = rr[0] if kind == "A" else 2 * ((rr[0] + 1) // 2)
        if not ((rb <= key < re) or (kind == "B" and re == n1 and key >= n1)):
            continue
        for cc in cols:
            out.append([r * n2 + c for r in rr for c in cc])
    return out


class ToyEngine:
    """Same interface as stripes.GpuEngine (CPU tensors): fixed-capacity halo
    payloads of the library's layout size (8 + 16 n2 + 8 n2 side^2 bytes),
    entry errors for the all-reduce, padded int64 instance rows for the
    all-gather."""

    def __init__(self, n1, n2, rb, re, seed=0, side=8):
        self.n1, self.n2, self.rb, self.re = n1, n2, rb, re
        rng = np.random.default_rng(seed)
        self.v = rng.uniform(0.5, 1.5, (n1 * n2, 2))     # identical on every rank
        self.mom = np.zeros(n1 * n2)
        self.cells = {k: composite_cells(n1, n2, k, rb, re) for k in "AB"}
        self.halo_bytes = 8 + 16 * n2 + 8 * n2 * side * side

    def sweep(self, part, stats=False):
        pid = 1.0 if part == "A" else 2.0
        e = 0.0
        for J in self.cells[part]:
            s = self.v[J].sum(0)
            for k, i in enumerate(J):
                old = self.v[i].copy()
                self.v[i] = 0.5 * self.v[i] + 0.5 * s / len(J) + 0.01 * (k + 1) * pid
                self.mom[i] = self.v[i].sum() + 1e-3 * i
                e += float(np.abs(self.v[i] - old).sum())
        return e if stats else None

    def pack(self, row):
        a = np.frombuffer(self.v[row * self.n2:(row + 1) * self.n2].copy().tobytes(), np.uint8)
        buf = np.zeros(self.halo_bytes, np.uint8)
        buf[:a.size] = a
        return torch.from_numpy(buf)

    def unpack(self, row, t):
        nb = self.n2 * 2 * 8
        self.v[row * self.n2:(row + 1) * self.n2] = np.frombuffer(t.numpy()[:nb].tobytes(), np.float64).reshape(-1, 2)

    def costs(self):
        C = np.zeros((self.n1 * self.n2, 5), np.int64)
        C[:, 1:] = np.round(self.mom * 1000).astype(np.int64)[:, None] + np.arange(4)[None, :]
        return C

    def cost_rows(self, lo, hi, maxrows):
        C = self.costs().ravel()
        n = self.n2 * 5
        part = np.zeros(maxrows * n, np.int64)
        part[:(hi - lo) * n] = C[lo * n:hi * n]
        return torch.from_numpy(part)

    def assemble(self, parts, spans):
        n = self.n2 * 5
        Cg = np.zeros(self.n1 * n, np.int64)
        for (lo, hi), t in zip(spans, parts):
            Cg[lo * n:hi * n] = t.numpy()[:(hi - lo) * n]
        return Cg

    def mincost(self, Cg):
        return np.roll(Cg.reshape(-1, 5), 1, axis=0) % 5     # any deterministic function of the global instance

    def apply(self, w):
        n1, n2 = self.n1, self.n2
        new = self.v.copy()
        for j in range(self.rb * n2, self.re * n2):
            j1, j2 = divmod(j, n2)
            acc = np.zeros(2)
            for a, (d1, d2) in enumerate(((-1, 0), (1, 0), (0, -1), (0, 1)), start=1):
                y, x = j1 + d1, j2 + d2
                if 0 <= y < n1 and 0 <= x < n2:
                    acc += 0.01 * w[y * n2 + x, a] * self.v[y * n2 + x]
            new[j] = self.v[j] + acc
        self.v = new


def run_toy(world, n1, n2, cycles, seed=0):
    """All ranks in one process; returns the owned rows' state of each rank."""
    from paper_2405_09400_b200.stripes import cycle_program, run_sequential, stripe_rows
    rows = stripe_rows(n1, world)
    engs = [ToyEngine(n1, n2, rows[r], rows[r + 1], seed) for r in range(world)]
    errs = []
    for _ in range(cycles):
        res = run_sequential([cycle_program(engs[r], r, world, rows, n1, n2, conv=True) for r in range(world)])
        assert all(x == res[0] for x in res)   # every rank sees the same all-reduced errors
        errs.append(res[0])
    return np.concatenate([engs[r].v[rows[r] * n2:rows[r + 1] * n2] for r in range(world)]), errs


def gloo_worker(rank, world, port, n1, n2, cycles, out_path):
    import os
    import torch.distributed as dist
    from paper_2405_09400_b200.stripes import cycle_program, run_distributed, stripe_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = stripe_rows(n1, world)
    eng = ToyEngine(n1, n2, rows[rank], rows[rank + 1])
    errs = []
    for _ in range(cycles):
        errs.append(run_distributed(cycle_program(eng, rank, world, rows, n1, n2, conv=True), rank, world))
    mine = eng.v[rows[rank] * n2:rows[rank + 1] * n2]
    parts = [None] * world
    dist.all_gather_object(parts, (mine, errs))
    if rank == 0:
        np.save(out_path, np.concatenate([m for m, _ in parts]))
        np.save(out_path + ".err.npy", np.array([e for _, e in parts], dtype=np.float64))
    dist.barrier()
    dist.destroy_process_group()
