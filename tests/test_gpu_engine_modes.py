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


@pytest.mark.parametrize("env", [{"QBG_PIPE": "0"}, {"QBG_PIPE": "1"}, {"QBG_JIT": "0"}, {"QBG_JIT_CHECK": "1"},
                                 {"QBG_TMA": "0"}],
                         ids=["plain-jit", "one-group", "interpreter", "bounds-checked", "cp-async-producer"])
def test_mode_parity(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k",
                        "vs_oracle or goldens or c64 or triangle"],
                       env=e, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("tma", ["1", "0"])
def test_fast_consumers_slot_protocol(tma):
    """Regression for the slot hand-over race: with the gate ops removed (QBG_EXP=2) the consumer
    groups outrun the producer, which exposed a group waiting on a slot whose previous fill (the
    other group's tile) was still in flight.  Must run to completion (values are not meaningful)."""
    code = ("import sys; sys.path.insert(0, '.'); import paper_1912_10877_b200 as qb; "
            "c = qb.variational_circuit(25, 2); qb.dispatch(c, 'random'); "
            "r = qb.expect_grad(qb.heisenberg(25), (qb.zero_state(25), c)); qb.synchronize(); print('ok')")
    e = dict(os.environ, QBG_EXP="2", QBG_TMA=tma)
    r = subprocess.run([sys.executable, "-c", code], env=e, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_plan_refresh_equals_rebuild():
    """An optimiser loop (new θ every step) with the values-only plan refresh (default) and with a
    full replan per θ (QBG_PLAN_REFRESH=0) gives bitwise-identical energies and gradients."""
    code = ("import sys, hashlib; sys.path.insert(0, '.'); import numpy as np; import paper_1912_10877_b200 as qb; "
            "c = qb.variational_circuit(14, 4); h = qb.heisenberg(14); rng = np.random.default_rng(3); "
            "P = len(qb.parameters(c)); m = hashlib.sha256()\n"
            "for it in range(5):\n"
            "    qb.dispatch(c, rng.uniform(0, 2 * np.pi, P))\n"
            "    r = qb.expect_grad(h, (qb.zero_state(14, nbatch=2), c))\n"
            "    m.update(np.ascontiguousarray(r.energies).tobytes()); m.update(np.ascontiguousarray(r.param_grads).tobytes())\n"
            "print('H', m.hexdigest())")
    outs = []
    for v in ("1", "0"):
        e = dict(os.environ, QBG_PLAN_REFRESH=v)
        r = subprocess.run([sys.executable, "-c", code], env=e, cwd=ROOT, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        outs.append([ln for ln in r.stdout.splitlines() if ln.startswith("H ")][-1])
    assert outs[0] == outs[1]
    # the refreshed plans' kernels with every generated index bounds-checked (trap on violation)
    e = dict(os.environ, QBG_JIT_CHECK="1")
    r = subprocess.run([sys.executable, "-c", code], env=e, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
