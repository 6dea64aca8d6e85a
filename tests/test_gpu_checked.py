"""The parity fixtures of tools/sanitize_cases.py on the bounds-checked build
(librrgpu_checked.so: RRG_CHECKED + RRG_PROBE_GUARD). compute-sanitizer is not
available on the GPU pool, so this is the memory-safety evidence: device-side
checks at every member / staging / row / export write and on every probe
chain trap instead of corrupting memory, and each case must still equal the
CPU port -- every IC schedule (lane, warp, block incl. whole-list expansion and
in-window repairs, big-set path, fast mode), every LT mode (linear, search
tree, guide table; walks past the filter and the lane budget) and both
selection modes."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2411_09473_b200", "librrgpu_checked.so")


@pytest.mark.parametrize("case", ["ic", "lt", "select"])
def test_checked_build_parity(cuda, case):
    if not os.path.exists(CHECKED):
        pytest.skip("librrgpu_checked.so not built")
    env = dict(os.environ, RRGPU_LIB=CHECKED)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), case],
                       capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, (p.stdout[-3000:], p.stderr[-3000:])
    assert f"{case} ok" in p.stdout
    assert "rrgpu check" not in p.stdout + p.stderr
