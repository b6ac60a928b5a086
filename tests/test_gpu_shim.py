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
