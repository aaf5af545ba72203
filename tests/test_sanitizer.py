"""compute-sanitizer runs: memcheck, racecheck and
synccheck over a small end-to-end run of every kernel family through the
C-ABI (tools/sanitize_run.py) on configs 1 and 2.  The library must report
zero errors."""
import os
import re
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    return exe if os.path.exists(exe) else None


@pytest.mark.gpu
@pytest.mark.parametrize("tool,cfg", [("memcheck", "cfg1"), ("memcheck", "cfg2"), ("racecheck", "cfg1"),
                                      ("synccheck", "cfg1"), ("initcheck", "cfg1")])
def test_compute_sanitizer_clean(tool, cfg):
    exe = _sanitizer()
    assert exe, "compute-sanitizer not found"
    cmd = [exe, f"--tool={tool}", "--error-exitcode=17", "--target-processes=application-only"]
    if tool == "memcheck":
        cmd += ["--leak-check=no"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), cfg]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    if "is closed on this pool" in out:   # the GPU pool's policy, not a library result
        pytest.skip("compute-sanitizer is disabled on this GPU pool: " + out.strip().splitlines()[0][:200])
    assert "sanitize run ok" in out, out[-3000:]
    m = re.search(r"ERROR SUMMARY: (\d+) error", out)
    assert r.returncode == 0 and m is not None and int(m.group(1)) == 0, out[-3000:]
