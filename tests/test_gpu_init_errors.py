"""domdec_init validation through the C-ABI (include/domdec.h error
taxonomy): every violated precondition of the method or malformed argument
returns its status code with a message and no context - DD_ERR_PRECOND for
a zero-mass basic cell, sum(mu) != sum(nu), initial boxes
that do not reproduce nu or whose masses differ from m_i, negative or
non-finite values, boxes outside the grid; DD_ERR_ARG for eps <= 0 and a
cell size that does not divide N or is not built."""
import numpy as np
import pytest

from parity import CONFIGS

gpu = pytest.mark.gpu
DD_ERR_ARG, DD_ERR_PRECOND = 1, 2


def _init(p, mu=None, nu=None, s=None, eps=None, off=None, ext=None, pos=None, data=None):
    from paper_2405_09400_b200 import DomDec
    return DomDec(p.mu if mu is None else mu, p.nu if nu is None else nu, p.s if s is None else s,
                  p.eps if eps is None else eps, p.h,
                  p.init_off if off is None else off, p.init_ext if ext is None else ext,
                  p.init_pos if pos is None else pos, p.init_data if data is None else data, p.E)


def _status(**kw):
    from paper_2405_09400_b200 import DomDecError
    p = CONFIGS["cfg1_gm"]()
    with pytest.raises(DomDecError) as ei:
        _init(p, **kw)
    assert str(ei.value).strip() != ""
    return ei.value.status


@gpu
def test_init_validation_status_codes():
    p = CONFIGS["cfg1_gm"]()
    s = p.s
    # zero-mass basic cell: move the mass of cell 0 to cell 1 in mu (nu unchanged)
    mu = p.mu.copy()
    blk = mu[:s, :s].sum()
    mu[:s, :s] = 0.0
    mu[:s, s:2 * s] += blk / (s * s)
    assert _status(mu=mu) == DD_ERR_PRECOND
    # total masses differ
    assert _status(nu=p.nu * 1.01) == DD_ERR_PRECOND
    # boxes that do not reproduce nu: shift one box by one row (same mass)
    off = p.init_off.copy()
    off[0, 0] = off[0, 0] + 1 if off[0, 0] + p.init_ext[0, 0] < p.N else off[0, 0] - 1
    assert _status(off=off) == DD_ERR_PRECOND
    # a box mass different from m_i (scaled data of cell 0)
    data = p.init_data.copy()
    n0 = int(p.init_ext[0, 0] * p.init_ext[0, 1])
    data[p.init_pos[0]:p.init_pos[0] + n0] *= 1.5
    assert _status(data=data) == DD_ERR_PRECOND
    # negative / non-finite values
    nu = p.nu.copy()
    nu[0, 0] = -1e-9
    assert _status(nu=nu) == DD_ERR_PRECOND
    mu = p.mu.copy()
    mu[3, 3] = np.nan
    assert _status(mu=mu) == DD_ERR_PRECOND
    # a box outside the grid
    off = p.init_off.copy()
    off[1, 1] = p.N - 1
    assert _status(off=off) == DD_ERR_PRECOND
    # arguments
    assert _status(eps=0.0) == DD_ERR_ARG
    assert _status(eps=-1.0) == DD_ERR_ARG
    assert _status(s=3) == DD_ERR_ARG   # does not divide 16
    assert _status(s=16) == DD_ERR_ARG  # divides, but no kernels for s = 16
