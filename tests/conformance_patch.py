"""pytest plugin (-p conformance_patch): patch the reference package with the B200 path
before the reference's own test modules import it (tests/test_gpu_conformance.py)."""

import packsell

from paper_2604_13433_b200.integration import patch_reference

PATCHED = patch_reference(packsell)


def pytest_report_header(config):
    return [f"b200-conformance: patched {len(PATCHED)} reference names "
            f"(e.g. {', '.join(sorted(PATCHED)[:3])})"]
