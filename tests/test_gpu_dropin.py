"""Drop-in proof: the reference's OWN unit tests for the data plane
(/root/reference/proj/tests/test_dataplane.cpp, unmodified) compiled against
include/dropin/moeplan/dataplane.hpp — the reference API executed on the B200
kernels through the C ABI — must all pass on the GPU.

The binary is built by `make -C oracle dropin` (from __graft_entry__.build())
where the reference tree exists, and travels to the GPU box as a built
artefact (oracle/_ref is git-ignored); skipped when absent."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "test_dataplane_dropin")


@pytest.mark.skipif(not os.path.exists(BIN), reason="drop-in test binary not built (no reference tree)")
def test_reference_dataplane_tests_pass_on_gpu(cuda):
    res = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(res.stdout[-4000:])
    m = re.search(r"(\d+)/(\d+) test cases passed", res.stdout)
    assert m, res.stdout + res.stderr
    passed, total = int(m.group(1)), int(m.group(2))
    assert total == 20, f"expected the reference's 20 data-plane test cases, found {total}"
    assert res.returncode == 0 and passed == total, res.stdout[-4000:]
