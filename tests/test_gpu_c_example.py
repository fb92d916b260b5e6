"""GPU: examples/solve.c drives a full solve through the C ABI alone (no Python, no torch):
compile, link against libplss.so and run it on the B200."""
import os
import shutil
import subprocess
import tempfile

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_example_solves():
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    from paper_2207_07615_b200 import build as pbuild
    pbuild.build()
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "solve")
        lib = os.path.join(ROOT, "paper_2207_07615_b200")
        subprocess.run([gcc, "-std=c99", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                        os.path.join(ROOT, "examples", "solve.c"), "-o", exe, "-L", lib, "-lplss",
                        "-L", "/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath," + lib], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
        assert out.returncode == 0, out.stdout + out.stderr
        assert "PLSS:" in out.stdout and "outcome 0" in out.stdout, out.stdout
