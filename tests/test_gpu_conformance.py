"""The reference's own tests against the drop-in (VERDICT r01 "next" #9).

`baseline/_ref` holds the reference package pip-installed from /root/reference and a copy
of its test directory (both git-ignored, made by __graft_entry__.build(), and they travel
to the GPU box with the snapshot).  The reference package is patched in place with
`paper_2604_13433_b200.integration.patch_reference` by a pytest plugin
loaded before the reference tests import it; then the reference's test_packed.py and
test_acceptance.py (criteria c01-c10), its codec / container / solver / metrics suites
run unchanged against the B200 build, SpMV, decode, codec, container and solvers.
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
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "conformance_patch",
           "--rootdir", REF_TESTS] + [os.path.join(REF_TESTS, f) for f in files]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=REF_TESTS, timeout=1500)
    tail = (out.stdout + out.stderr)[-6000:]
    return out.returncode, tail


@pytest.mark.parametrize("files", [["test_packed.py"], ["test_acceptance.py"]], ids=["packed", "acceptance"])
def test_reference_suite_passes_on_the_b200_path(files):
    rc, tail = _run(files)
    assert rc == 0, tail
