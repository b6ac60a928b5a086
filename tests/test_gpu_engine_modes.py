"""The non-default engine modes stay parity-green: the plain JIT tile loop (QBG_PIPE=0), one
consumer group (QBG_PIPE=1), the interpreter kernels (QBG_JIT=0), and the specialised kernels
built with every global / shared index bounds-checked (QBG_JIT_CHECK=1, a trap on violation —
the memcheck stand-in on pools where compute-sanitizer is unavailable).  The modes are read once
per process, so each runs the oracle-parity subset in a fresh interpreter."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"QBG_PIPE": "0"}, {"QBG_PIPE": "1"}, {"QBG_JIT": "0"}, {"QBG_JIT_CHECK": "1"}],
                         ids=["plain-jit", "one-group", "interpreter", "bounds-checked"])
def test_mode_parity(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k",
                        "vs_oracle or goldens or c64 or triangle"],
                       env=e, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
