"""The reference package's OWN test suite, run against this build.

scripts/fetch_reference_tests.sh copies /root/reference/pkg/tests to
baseline/_ref_tests/ (git-ignored, shipped to the GPU box with the
snapshot); the files run unmodified, and ``import lpic`` inside them
resolves to this package through lpic/__init__.py.  Every module is run; the
report (passes, skips, failures) is written next to the parity results
(LPIC_PARITY_OUT).  Skipped when the copy is absent (it cannot be made on
the GPU box, which has no /root/reference)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "baseline", "_ref_tests")
MODULES = ["test_codec.py", "test_network.py", "test_schedules.py", "test_coder.py", "test_mixture.py",
           "test_images_cli.py", "test_training.py", "test_acceptance.py"]


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.isdir(SUITE), reason="run scripts/fetch_reference_tests.sh first")
@pytest.mark.parametrize("module", MODULES)
def test_reference_suite_against_b200_build(module):
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    cmd = [sys.executable, "-m", "pytest", "-q", "-rfEs", "-p", "no:cacheprovider", "--rootdir", SUITE,
           os.path.join(SUITE, module)]
    r = subprocess.run(cmd, cwd=SUITE, env=env, capture_output=True, text=True, timeout=3000)
    out_dir = os.environ.get("LPIC_PARITY_OUT")
    if out_dir:
        os.makedirs(out_dir, exist_ok=True)
        with open(os.path.join(out_dir, f"reference_suite_{module[:-3]}.txt"), "w") as f:
            f.write(r.stdout[-20000:] + r.stderr[-5000:])
    assert r.returncode == 0, (r.stdout + r.stderr)[-6000:]
