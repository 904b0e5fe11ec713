"""GPU: the C++ drop-in (include/cycheck_b200.hpp) compiled against the
reference's own headers and sources (oracle/dropin_test.cpp, prebuilt into
oracle/_ref/ where the reference exists) must give the reference's results
from the reference's own call sites."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


def test_cpp_dropin_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_test not built (needs the reference sources)")
    env = dict(os.environ, DROPIN_TRACE="1")
    try:
        out = subprocess.run([BIN, "150"], capture_output=True, text=True, timeout=90, env=env)
    except subprocess.TimeoutExpired as ex:
        err = ex.stderr.decode() if isinstance(ex.stderr, bytes) else (ex.stderr or "")
        pytest.fail("dropin_test timed out; last progress:\n" + err[-600:])
    print(out.stdout[-2000:])
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "0 mismatches" in out.stdout
