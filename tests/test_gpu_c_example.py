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


@pytest.mark.parametrize("partition,step", [("rows", "allreduce"), ("rows", "rsag"), ("rows", "peer"),
                                            ("cols", "allreduce")])
def test_dist_example_one_process(partition, step, tmp_path):
    """examples/dist_solve.py under torchrun with one process (the pods have one GPU): every
    partition / step converges and reports a true residual within the tolerance."""
    import socket
    import subprocess
    import sys
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(root, "examples", "dist_solve.py"), "--partition", partition, "--step", step],
                       cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if "GPU(s)" in ln]
    assert line and "converged" in line[0], r.stdout
    tr = float(line[0].split("true residual ")[1].split(",")[0])
    assert tr <= 1e-7
