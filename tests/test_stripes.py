"""Stripe decomposition host logic: row boundaries, the halo /
all-gather schedule of paper_2405_09400_b200.stripes, sequential loopback and
a real 2-process gloo run against the unstriped run (CPU, toy engine)."""
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from _stripe_toy import gloo_worker, run_toy
from paper_2405_09400_b200.stripes import stripe_rows


@pytest.mark.parametrize("n1,world", [(8, 1), (8, 2), (8, 4), (64, 3), (256, 8), (7, 2), (33, 4)])
def test_stripe_rows(n1, world):
    b = stripe_rows(n1, world)
    assert b[0] == 0 and b[-1] == n1 and len(b) == world + 1
    assert all(x < y for x, y in zip(b, b[1:]))
    assert all(x % 2 == 0 for x in b[1:-1])          # no A-cell straddles two ranks
    sizes = [(y - x + 1) // 2 for x, y in zip(b, b[1:])]
    assert max(sizes) - min(sizes) <= 1


def test_stripe_rows_rejects_too_many_ranks():
    with pytest.raises(ValueError):
        stripe_rows(8, 5)


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("shape", [(8, 6), (9, 5)])
def test_sequential_stripes_equal_unstriped(world, shape):
    n1, n2 = shape
    ref, eref = run_toy(1, n1, n2, cycles=3)
    got, egot = run_toy(world, n1, n2, cycles=3)
    np.testing.assert_array_equal(got, ref)
    # the all-reduced sweep-entry errors (reading R14) equal the unstriped sums
    np.testing.assert_allclose(np.array(egot), np.array(eref), rtol=1e-12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_two_ranks_equal_unstriped(tmp_path):
    """world_size 2 over torch.distributed (gloo, 127.0.0.1): the same
    cycle programs with real point-to-point exchanges of fixed-capacity halo
    payloads (the library's layout size), the all-gather of the padded int64
    instance rows and the all-reduce of the sweep-entry errors."""
    n1, n2, cycles = 8, 6, 3
    out = str(tmp_path / "stripes.npy")
    mp.spawn(gloo_worker, args=(2, _free_port(), n1, n2, cycles, out), nprocs=2, join=True)
    ref, eref = run_toy(1, n1, n2, cycles)
    np.testing.assert_array_equal(np.load(out), ref)
    errs = np.load(out + ".err.npy")
    for r in range(2):
        np.testing.assert_allclose(errs[r], np.array(eref), rtol=1e-12)
