"""The conv + engine parity suites with tap folding enabled (HB_FOLD=2, an
opt-in experiment), in a fresh process (the setting is read once)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_conv_suite_with_fold():
    env = dict(os.environ, HB_FOLD="2")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(HERE, "test_conv_gpu.py"),
                        os.path.join(HERE, "test_engine_gpu.py"), "-x", "-q", "-p", "no:cacheprovider"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
