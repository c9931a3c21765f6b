"""Drop-in proof for the planner half of the operator API: the reference's
OWN planner unit tests (/root/reference/proj/tests/test_{config,commcost,
chunkopt,strategy,pipesim}.cpp, unmodified) compiled against
include/dropin/moeplan/*.hpp — every number from libmonta.so's C ABI — must
all pass.  Host-only (the planner needs no GPU), so this runs in the CPU
suite.  Binaries: `make -C oracle dropin_planner` (from __graft_entry__.build()
where the reference tree exists); skipped when absent."""
import os
import re
import subprocess

import pytest

REF_BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
CASES = {"config": 11, "commcost": 18, "chunkopt": 14, "strategy": 9, "pipesim": 12}


@pytest.mark.parametrize("name", sorted(CASES))
def test_reference_planner_tests_pass(name):
    exe = os.path.join(REF_BIN, f"test_{name}_dropin")
    if not os.path.exists(exe):
        pytest.skip("planner drop-in binaries not built (no reference tree)")
    res = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    m = re.search(r"(\d+)/(\d+) test cases passed", res.stdout)
    assert m, res.stdout + res.stderr
    passed, total = int(m.group(1)), int(m.group(2))
    assert total == CASES[name], f"expected the reference's {CASES[name]} test cases, found {total}"
    assert res.returncode == 0 and passed == total, res.stdout[-4000:]
