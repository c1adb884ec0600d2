"""Run the reference's own unit + acceptance + CLI suite (/root/reference/pkg/tests,
136 tests) against this package, with
``import hetsim`` aliased to ``paper_1402_6601_b200`` (tests/ref_alias).
Only possible where /root/reference exists (the build container); skipped
elsewhere.  Nothing is copied from the reference."""
import os
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tree not mounted")
def test_reference_suite_passes_against_this_package(tmp_path):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(HERE, "ref_alias"), os.path.dirname(HERE)])
    res = subprocess.run(
        [sys.executable, "-m", "pytest", REF_TESTS, "-p", "hetsim_alias", "-p", "no:cacheprovider", "-q"],
        cwd=tmp_path, env=env, capture_output=True, text=True, timeout=900)
    tail = "\n".join(res.stdout.splitlines()[-15:])
    assert res.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail
