"""Run the reference's own tests against the drop-in (subprocess entry point; TEST INFRASTRUCTURE).

  python tests/ref_suite_runner.py <reference tests dir> <reference src dir> [pytest args...]

`rhymesim.history` and `rhymesim.spec_engine` are aliased to this repo's GPU-backed modules before
pytest imports anything, so `from rhymesim.history import build_tree` in the reference's tests (and in
the reference's own simulator modules, which stay the real ones) resolves to the drop-in -- the swap
INTEGRATION.md section 1 describes for a user of the reference.
"""

import os
import sys


def main():
    tests_dir, src_dir = sys.argv[1], sys.argv[2]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, src_dir, tests_dir]
    import importlib

    import paper_2508_18588_b200.history as H
    import paper_2508_18588_b200.spec_engine as S
    rhymesim = importlib.import_module("rhymesim")
    sys.modules["rhymesim.history"] = H
    sys.modules["rhymesim.spec_engine"] = S
    rhymesim.history = H
    rhymesim.spec_engine = S
    import rhymesim.history as check
    assert check is H, "alias did not take"
    import pytest
    args = sys.argv[3:] + ["-p", "no:cacheprovider", "--rootdir", tests_dir]
    sys.exit(pytest.main(args))


if __name__ == "__main__":
    main()
