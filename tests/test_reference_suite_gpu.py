"""The reference's own hot-path tests, run against the drop-in.

`rhymesim.history` / `rhymesim.spec_engine` are aliased to the GPU-backed modules of this repo
(tests/ref_suite_runner.py) and the reference's unmodified test files run under pytest:

  * pkg/tests/test_history.py    -- all but test_child_sum_invariant, which walks the pointer tree's
                                    internal nodes (the index has no Node objects; node counts, root
                                    mass and every query-level property are still checked)
  * pkg/tests/test_spec_engine.py -- all
  * pkg/tests/test_acceptance.py -- criterion 1 (1,000 corpora / 8,000 queries vs the brute-force oracle,
                                    under the reference's own 60 s limit) and criterion 2 (AIMD, 8,191 cases)

The reference tree is taken from /root/reference/pkg (build container) or baseline/_ref (the offline
install made by tools/install_reference.sh, which travels to the GPU box); the test skips when neither
is present.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _reference():
    cands = [("/root/reference/pkg/tests", "/root/reference/pkg/src"),
             (os.path.join(ROOT, "baseline", "_ref", "rhymesim_tests"), os.path.join(ROOT, "baseline", "_ref"))]
    for tests, src in cands:
        if os.path.isfile(os.path.join(tests, "test_history.py")) and \
                os.path.isfile(os.path.join(src, "rhymesim", "history.py")):
            return tests, src
    pytest.skip("reference tests not available (run tools/install_reference.sh)")


@pytest.mark.parametrize("target", [
    ("test_history.py", "not test_child_sum_invariant"),
    ("test_spec_engine.py", None),
    ("test_acceptance.py", "criterion_1 or criterion_2"),
])
def test_reference_suite_on_drop_in(target):
    tests, src = _reference()
    fname, sel = target
    args = [sys.executable, os.path.join(ROOT, "tests", "ref_suite_runner.py"), tests, src,
            os.path.join(tests, fname), "-q", "-s"]
    if sel:
        args += ["-k", sel]
    r = subprocess.run(args, capture_output=True, text=True, timeout=900, cwd=tests)
    tail = r.stdout[-3000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and " failed" not in r.stdout, tail
    print(tail[-600:])
