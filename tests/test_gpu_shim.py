"""The C++ drop-in shim (include/qbg/qblock.hpp) compiled against libqbg.so and run on the GPU:
the reference's examples written against the qblock API."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_shim_examples(tmp_path):
    exe = tmp_path / "test_shim"
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"),
                           "-L" + os.path.join(ROOT, "paper_1912_10877_b200"), "-lqbg",
                           "-Wl,-rpath," + os.path.join(ROOT, "paper_1912_10877_b200"), "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "shim ok" in out.stdout


def test_cpp_block_api(tmp_path, golden):
    """include/qbg/blocks.hpp: App G, SPEC examples, Subroutine, dagger, shim surface — and
    variational_circuit(16,10) expect' through the C++ API alone vs the reference's golden."""
    import numpy as np
    exe = tmp_path / "test_blocks"
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "test_blocks.cpp"),
                           "-L" + os.path.join(ROOT, "paper_1912_10877_b200"), "-lqbg",
                           "-Wl,-rpath," + os.path.join(ROOT, "paper_1912_10877_b200"), "-o", str(exe)])
    res = tmp_path / "q16.bin"
    qbreg = os.path.join(ROOT, "tests", "golden", "state_qbreg1.bin")
    out = subprocess.run([str(exe), str(res), qbreg], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "blocks ok" in out.stdout
    v = np.fromfile(res, dtype=np.float64)
    g = golden("bench_small.npz")
    assert v.size == 1 + g["q16_grads"].size
    assert abs(v[0] - g["q16_energy"][0]) <= 1e-12 * max(1.0, abs(g["q16_energy"][0]))
    assert np.abs(v[1:] - g["q16_grads"]).max() <= 1e-12 * max(1.0, np.abs(g["q16_grads"]).max())
