"""Device-side bounds checks in place of compute-sanitizer (closed on the GPU
pool): tests/sanitize_run.py — every hot-path kernel on ragged shapes, two
steps with update-and-park and a swap-in — against the debug build
(_native/libflexmarl_b200_debug.so, FM_DCHECK on the data-derived indices:
position features, row ends, segment slots, A' rows, stats columns, GEMM
segment extents).  A failed check traps, so the run exits non-zero."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_kernels_pass_bounds_checks():
    lib = ROOT / "paper_2602_09578_b200" / "_native" / "libflexmarl_b200_debug.so"
    if not lib.exists():
        pytest.skip("debug library not built (python -m paper_2602_09578_b200.build --debug)")
    env = dict(os.environ, FLEXMARL_DEBUG_LIB="1")
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "sanitize_run.py")], capture_output=True, text=True,
                       env=env, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "sanitize run OK" in r.stdout
