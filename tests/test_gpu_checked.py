"""Bounds-checked build (memory-safety evidence).

compute-sanitizer is closed on the GPU pool, so libddvr is also built with
-DDDVR_CHECKED (``__graft_entry__.build()`` -> ``_variants/libddvr_checked.so``): every
cell-record gather of the marches, walks and the gather probe, every cell-gradient
flush and every empty-brick lookup checks its index against the padded record grid
and traps, printing the source line, on a violation.  tools/sanitize_cases.py runs
every kernel family (C1..C5-shaped steps, band tape + empty skip + split kernels on
exact empty space, stored mode, both layouts, forward mode, colour volumes) and the
full-size C4 band through it in a subprocess.
"""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_kernels_pass_bounds_checks(cuda):
    from paper_2107_12672_b200 import _build
    lib = os.path.join(ROOT, "paper_2107_12672_b200", "_variants", "libddvr_checked.so")
    if _build.stale(lib):
        lib = _build.build_variant("checked", ["DDVR_CHECKED"])
    with open(lib, "rb") as f:   # the checks are compiled in (their message is in the image)
        assert b"ddvr check failed" in f.read()
    env = dict(os.environ, DDVR_LIB=lib)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"),
                        "--config-band"], capture_output=True, text=True, env=env,
                       timeout=900, cwd=ROOT)
    assert p.returncode == 0 and "SANITIZE_CASES_OK" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]
    assert "ddvr check failed" not in p.stdout + p.stderr
