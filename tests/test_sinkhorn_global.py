"""Global separable Sinkhorn (SinkhornGPU comparator, SURVEY 8(f) f4;
PAPER.md:1249-1250): dd_sinkhorn_global through the C-ABI against the fp64
oracle's dense log-domain Sinkhorn (oracle.dense_sinkhorn, pinned in
test_oracle_pins.py) on the same seeded inputs."""
import numpy as np
import pytest

import oracle as O
from synth import make_problem

gpu = pytest.mark.gpu


def _random_measures(N1, N2, seed, zero_frac):
    """Seeded positive measures of equal mass with a zero pattern (ragged supports)."""
    rng = np.random.default_rng(seed)
    mu = rng.random((N1, N2)) + 0.05
    nu = rng.random((N1, N2)) + 0.05
    mu[rng.random((N1, N2)) < zero_frac] = 0.0
    nu[rng.random((N1, N2)) < zero_frac] = 0.0
    return mu / mu.sum(), nu / nu.sum()


def _compare(mu, nu, eps_p, K):
    from paper_2405_09400_b200 import sinkhorn_global
    a, b, it, e, ms = sinkhorn_global(mu, nu, eps_p, err=0.0, max_iter=K, check_every=K)
    assert it == K
    plan, ao, bo, xs, ys = O.dense_sinkhorn(mu, nu, eps_p, tol=0.0, max_iter=K)
    ag, bg = a.ravel()[xs], b.ravel()[ys]
    # fp64 potentials; fp32 sums of exp(term - max) give ~1e-7 relative error per
    # LSE (sum of <= N fp32 terms in [0, 1]),
    # accumulated over K half-iterations of a contraction.
    scale = 1.0 + np.max(np.abs(ao))
    assert np.max(np.abs(ag - ao)) <= 2e-5 * scale, np.max(np.abs(ag - ao))
    assert np.max(np.abs(bg - bo)) <= 2e-5 * scale, np.max(np.abs(bg - bo))
    # off-support entries are zero by contract
    assert np.all(a.ravel()[mu.ravel() == 0] == 0.0)
    assert np.all(b.ravel()[nu.ravel() == 0] == 0.0)
    return a, b


@gpu
@pytest.mark.parametrize("shape,eps_p,zero_frac", [((16, 16), 4.0, 0.0), ((24, 40), 4.0, 0.2),
                                                   ((8, 300), 16.0, 0.1), ((300, 8), 1.0, 0.1),
                                                   ((33, 45), 0.25, 0.3)])
def test_global_sinkhorn_parity_fixed_iterations(shape, eps_p, zero_frac):
    mu, nu = _random_measures(*shape, seed=sum(shape), zero_frac=zero_frac)
    _compare(mu, nu, eps_p, K=12)


@gpu
def test_global_sinkhorn_stale_shift_warm_start():
    """from the second iteration each LSE output is shifted by its
    previous value; after a wild warm start the shift is stale by
    hundreds of log units, and a term far above it must overflow the shifted
    sum into the max-pass fallback, never be dropped.  GPU vs the oracle's
    dense Sinkhorn from the same initial potential."""
    from paper_2405_09400_b200 import sinkhorn_global
    p = make_problem("gm", 32, 2, theta_deg=20.0, seed=5)
    rng = np.random.default_rng(7)
    a0 = rng.normal(0.0, 500.0, p.mu.shape)
    K = 6
    a, b, it, e, ms = sinkhorn_global(p.mu, p.nu, p.eps_prime, err=0.0, max_iter=K, check_every=K, alpha0=a0)
    plan, ao, bo, xs, ys = O.dense_sinkhorn(p.mu, p.nu, p.eps_prime, tol=0.0, max_iter=K, a0=a0)
    scale = 1.0 + np.max(np.abs(ao))
    assert np.max(np.abs(a.ravel()[xs] - ao)) <= 2e-5 * scale
    assert np.max(np.abs(b.ravel()[ys] - bo)) <= 2e-5 * scale


@gpu
def test_global_sinkhorn_parity_gm_problem():
    p = make_problem("gm", 32, 2, theta_deg=20.0, seed=1)
    _compare(p.mu, p.nu, p.eps_prime, K=20)


@gpu
def test_global_sinkhorn_stopping_rule_and_marginals():
    """Run to Err = 1e-4; the reported error is the oracle's
    X-marginal error of (a, b) and the Y-marginal is exact after the final
    Y-update."""
    from paper_2405_09400_b200 import sinkhorn_global
    p = make_problem("gm", 32, 2, theta_deg=20.0, seed=2)
    a, b, it, e, ms = sinkhorn_global(p.mu, p.nu, p.eps_prime, err=1e-4)
    assert e <= 1e-4 * p.mu.sum()
    assert it > 1
    xs = np.flatnonzero(p.mu.ravel() > 0)
    ys = np.flatnonzero(p.nu.ravel() > 0)
    kx = np.stack([xs // 32, xs % 32], axis=1)
    ly = np.stack([ys // 32, ys % 32], axis=1)
    Cm = O.sinkhorn.sqdist(kx, ly) / p.eps_prime
    plan = np.exp(a.ravel()[xs][:, None] + b.ravel()[ys][None, :] - Cm) * p.mu.ravel()[xs][:, None] \
        * p.nu.ravel()[ys][None, :]
    # Y-marginal exact up to the fp32 sums of the final LSE stages (relative
    # ~M 2^-24 per entry for M <= 32 terms per stage, M = 32 here)
    assert np.abs(plan.sum(0) - p.nu.ravel()[ys]).sum() <= 32 * 2.0 ** -24 * p.nu.sum()
    assert np.abs(plan.sum(1) - p.mu.ravel()[xs]).sum() <= 1e-4 * p.mu.sum()


@gpu
def test_global_sinkhorn_rejects_bad_input():
    from paper_2405_09400_b200 import DomDecError, sinkhorn_global
    mu, nu = _random_measures(8, 8, 0, 0.0)
    with pytest.raises(DomDecError):
        sinkhorn_global(mu, 2 * nu, 4.0)
    with pytest.raises(DomDecError):
        sinkhorn_global(-mu, nu, 4.0)
    with pytest.raises(DomDecError):
        sinkhorn_global(mu, nu, 0.0)


@gpu
@pytest.mark.parametrize("N,K", [(1024, 5), (256, 40)])
def test_global_sinkhorn_full_size_sampled(N, K):
    """At the bench sizes (stage rows longer than the CTA, 4 output strides at
    1024): the returned b is the exact Y-update of the returned a, checked at
    sampled target pixels against oracle.y_update_at (O(N^2) per sample).
    fp32 sums of exp(term - shift) carry ~M 2^-24 relative error per stage
    (M = N terms), the exponent's float conversion 1 ulp of |v|; the
    tolerance 4 N 2^-24 covers both stages."""
    from paper_2405_09400_b200 import sinkhorn_global
    p = make_problem("gm", N, 4, theta_deg=20.0, seed=3)
    a, b, it, e, ms = sinkhorn_global(p.mu, p.nu, p.eps_prime, err=0.0, max_iter=K, check_every=K)
    assert it == K and np.isfinite(e)
    rng = np.random.default_rng(N)
    ys = np.flatnonzero(p.nu.ravel() > 0)
    pick = np.concatenate([ys[[0, -1]], rng.choice(ys, 30, replace=False)])
    ls = np.stack([pick // N, pick % N], axis=1)
    want = O.y_update_at(a, p.mu, p.eps_prime, ls)
    got = b.ravel()[pick]
    # log-domain error is absolute (log of a relatively perturbed sum); fp64 rounding of |b| adds 1e-12 |b|
    assert np.all(np.abs(got - want) <= 4 * N * 2.0 ** -24 + 1e-12 * np.abs(want)), np.max(np.abs(got - want))


@gpu
def test_global_sinkhorn_graph_chunks_bit_identical(monkeypatch):
    """Chunks of check_every iterations replayed as one CUDA graph run the
    same kernels in the same order as the eager loop: bit-identical a, b,
    iteration count and error, at fixed K and under the stopping rule."""
    from paper_2405_09400_b200 import sinkhorn_global
    p = make_problem("gm", 64, 2, theta_deg=20.0, seed=4)
    runs = {}
    for mode in ("graph", "eager"):
        if mode == "eager":
            monkeypatch.setenv("DD_SG_NO_GRAPH", "1")
        runs[mode] = (sinkhorn_global(p.mu, p.nu, p.eps_prime, err=0.0, max_iter=42, check_every=4),
                      sinkhorn_global(p.mu, p.nu, p.eps_prime, err=1e-4, max_iter=100000, check_every=10))
    for (ag, bg, ig, eg, _), (ae, be, ie, ee, _) in zip(runs["graph"], runs["eager"]):
        assert ig == ie and eg == ee
        assert np.array_equal(ag, ae) and np.array_equal(bg, be)
    assert runs["graph"][0][2] == 42
