"""Host-side checks of the C-ABI library (no GPU needed): it builds for
sm_100a, loads, and exports every symbol include/domdec.h declares."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "domdec.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_north_star_entry_points():
    syms = _declared_symbols()
    for name in ("domdec_init", "domdec_sweep", "flow_update", "marginal_error", "primal_dual_gap"):
        assert name in syms


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2405_09400_b200 import build_library
    path = build_library()
    lib = ctypes.CDLL(path)
    for name in _declared_symbols():
        assert hasattr(lib, name), name
    # sm_100a SASS is present (no PTX-only / other-arch build)
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_binding_exports_match_header():
    from paper_2405_09400_b200 import EXPORTED
    assert sorted(EXPORTED) == _declared_symbols()


def test_no_cpu_fallback_without_device():
    """On a machine without a GPU the product path must fail loudly."""
    import numpy as np
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2405_09400_b200 import DomDec, DomDecError
    from synth import make_problem
    p = make_problem("gm", 8, 2)
    with pytest.raises(DomDecError) as ei:
        DomDec.from_problem(p)
    assert ei.value.status == 4


def test_global_sinkhorn_no_cpu_fallback_without_device():
    """dd_sinkhorn_global validates its arguments on the host, then needs the
    GPU: without one it returns DD_ERR_CUDA (no CPU path)."""
    import numpy as np
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2405_09400_b200 import DomDecError, sinkhorn_global
    mu = np.full((4, 4), 1 / 16)
    with pytest.raises(DomDecError) as ei:
        sinkhorn_global(mu, mu, 4.0)
    assert ei.value.status == 4
    with pytest.raises(DomDecError) as ei:   # argument check precedes the device
        sinkhorn_global(mu, 2 * mu, 4.0)
    assert ei.value.status == 2
