"""The checked build (lib/libstmf_b200_checked.so, STMF_CHECKS: every gathered index is
range-checked on the device and a violation traps) runs the sanitizer workload
(tools/sanitize_driver.py: every kernel family at toy sizes) cleanly.  This pool does
not run compute-sanitizer; these checks are the stand-in."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_checked_build_runs_every_kernel_family():
    from paper_2205_06619_b200 import _ext
    path = _ext.build(checked=True)
    env = dict(os.environ, STMF_LIB=path)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_driver.py")], capture_output=True,
                         text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-3000:])
    assert "stmf check failed" not in out.stdout + out.stderr
    assert "c5 sampled" in out.stdout
