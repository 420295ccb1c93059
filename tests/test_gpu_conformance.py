"""The reference's own tests against the drop-in (VERDICT r01 "next" #9).

`baseline/_ref` holds the reference package pip-installed from /root/reference and a copy
of its test directory (both git-ignored, made by __graft_entry__.build(), and they travel
to the GPU box with the snapshot).  The reference package is patched in place with
`paper_2604_13433_b200.integration.patch_reference` by a pytest plugin
loaded before the reference tests import it; then the reference's test_packed.py and
test_acceptance.py (criteria c01-c10) and the rest of its suite (codec, container,
solvers, metrics, CLI, SELL, matrix: all 279 tests) run unchanged against the B200 build,
SpMV (in the reference's rounding order, as the patch selects), decode, codec, container,
metrics and solvers.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "packsell_tests")


def _run(files):
    if not os.path.isdir(os.path.join(REF, "packsell")) or not os.path.isdir(REF_TESTS):
        pytest.skip("reference install / tests absent (baseline/_ref is made by __graft_entry__.build())")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "tests"), REF, REF_TESTS]),
               PYTHONDONTWRITEBYTECODE="1")
    cmd = [sys.executable, "-m", "pytest", "-p", "no:cacheprovider", "-p", "conformance_patch",
           "--rootdir", REF_TESTS] + [os.path.join(REF_TESTS, f) for f in files]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=REF_TESTS, timeout=1500)
    tail = (out.stdout + out.stderr)[-6000:]
    return out.returncode, tail


SUITES = ["test_packed.py", "test_acceptance.py", "test_codec.py", "test_container.py", "test_solvers.py",
          "test_metrics.py", "test_cli.py", "test_sell.py", "test_matrix.py"]


@pytest.mark.parametrize("suite", SUITES, ids=[s[5:-3] for s in SUITES])
def test_reference_suite_passes_on_the_b200_path(suite):
    rc, tail = _run([suite])
    assert "b200-conformance: patched" in tail or rc == 0, tail
    assert rc == 0, tail
    if suite == "test_acceptance.py":
        for c in range(1, 11):
            assert f"PASS  test_c{c:02d}" in tail, tail
