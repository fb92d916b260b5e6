"""The C-ABI library builds, loads and exports every symbol include/plss.h declares (no GPU)."""
import ctypes
import os
import re

import pytest

import paper_2207_07615_b200 as pkg
from paper_2207_07615_b200 import build as pbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "plss.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(plss_[a-z_T]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    pbuild.build()
    return pkg.load_library()


def test_header_symbols_exported(lib):
    names = _header_functions()
    assert len(names) >= 14
    assert sorted(pkg.SYMBOLS) == names
    for nm in names:
        assert getattr(lib, nm) is not None


def test_status_strings(lib):
    assert lib.plss_status_str(0) == b"ok"
    assert lib.plss_status_str(3) == b"matrix format violation"


def test_workspace_bytes_host_only(lib):
    m = pkg.plss.plss_matrix(1000, 500, 4000, None, None, None, None, None, None, 0)
    o = pkg.plss.plss_options(1, 0, 100, 0)
    nb = lib.plss_workspace_bytes(ctypes.byref(m), ctypes.byref(o))
    assert nb >= 8 * (1000 + 3 * 500) + 8 * 101 * 8
    o4 = pkg.plss.plss_options(4, 0, 100, 0)
    nb4 = lib.plss_workspace_bytes(ctypes.byref(m), ctypes.byref(o4))
    assert nb4 >= nb + 12 * 4000            # slab-major CSC copy
    bad = pkg.plss.plss_matrix(-1, 5, 0, None, None, None, None, None, None, 0)
    assert lib.plss_workspace_bytes(ctypes.byref(bad), None) == 0


def test_null_ctx_is_an_error_not_a_crash(lib):
    assert lib.plss_step(None, 1) == 1          # PLSS_E_INVALID
    assert lib.plss_spmv(None, None, None) == 1
    lib.plss_destroy(None)


def test_product_does_not_import_oracle():
    pkgdir = os.path.join(ROOT, "paper_2207_07615_b200")
    for dirpath, _, files in os.walk(pkgdir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "plss_oracle" not in txt, f


def test_build_targets_sm100a():
    cmd = pbuild.command("/tmp/x.so")
    assert "arch=compute_100a,code=sm_100a" in cmd


def test_c_example_compiles_and_links():
    """include/plss.h is plain C99: examples/solve.c (the ABI without Python) compiles with gcc
    -Wall -Werror and links against libplss.so (running it needs a GPU: test_gpu_c_example)."""
    import shutil
    import subprocess
    import tempfile
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    from paper_2207_07615_b200 import build as pbuild
    pbuild.build()
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "solve")
        cmd = [gcc, "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
               "-I", "/usr/local/cuda/include", os.path.join(ROOT, "examples", "solve.c"), "-o", exe,
               "-L", os.path.join(ROOT, "paper_2207_07615_b200"), "-lplss", "-L", "/usr/local/cuda/lib64",
               "-lcudart", "-Wl,-rpath," + os.path.join(ROOT, "paper_2207_07615_b200")]
        subprocess.run(cmd, check=True, capture_output=True, text=True)
        assert os.path.exists(exe)


def test_binding_rejects_bad_vectors():
    """the binding validates dtype, contiguity, length and (for tensors) the device
    and alignment of every vector argument before calling into the library (checked on CPU with a
    stand-in ctx; no library call is made)."""
    import numpy as np
    import torch
    from paper_2207_07615_b200 import plss as b

    class _A:
        row_ptr = torch.zeros(1, dtype=torch.int32)

    class _Ctx:
        A = _A()

    ctx = _Ctx()
    ok = np.zeros(10)
    assert b._vec(ctx, ok, 10, "x") == ok.ctypes.data
    assert b._vec(ctx, None, 10, "x") is None
    with pytest.raises(b.PlssError, match="float64"):
        b._vec(ctx, np.zeros(10, np.float32), 10, "x")
    with pytest.raises(b.PlssError, match="required"):
        b._vec(ctx, np.zeros(9), 10, "x")
    with pytest.raises(b.PlssError, match="float64"):
        b._vec(ctx, np.zeros((10, 2))[:, 0], 10, "x")
    with pytest.raises(b.PlssError, match="CUDA tensor"):
        b._vec(ctx, ok, 10, "x", host_ok=False)
    with pytest.raises(b.PlssError, match="CUDA tensor"):
        b._vec(ctx, torch.zeros(10, dtype=torch.float64), 10, "x", host_ok=False)
    with pytest.raises(b.PlssError, match="float64"):
        b._vec(ctx, torch.zeros(10, dtype=torch.float32), 10, "x")
    with pytest.raises(b.PlssError, match="float64"):
        b._vec(ctx, torch.zeros(20, dtype=torch.float64)[::2], 10, "x")
    with pytest.raises(b.PlssError, match="numpy array or torch tensor"):
        b._vec(ctx, [0.0] * 10, 10, "x")
    t = torch.zeros(10, dtype=torch.float64)
    assert b._vec(ctx, t, 10, "x") == t.data_ptr()


def test_entry_points_carry_nvtx_ranges(lib):
    """the solve entry points, each graph chunk and the NCCL wait open
    an NVTX range; the range names are string constants of the built library."""
    blob = open(pbuild.LIB, "rb").read()
    for name in (b"plss_create", b"plss_start", b"plss_step", b"plss_finish", b"plss_solve", b"plss_spmv",
                 b"plss_spmvT", b"plss_solve: graph chunk", b"plss: wait (stream / NCCL async-error poll)"):
        assert name + b"\0" in blob, name
    src = open(os.path.join(ROOT, "paper_2207_07615_b200", "csrc", "plss.cu")).read()
    for fn in ("plss_create", "plss_create_dist", "plss_start", "plss_step", "plss_finish", "plss_solve",
               "plss_spmv", "plss_spmvT", "plss_true_residual"):
        m = re.search(r"^plss_status " + fn + r"\([^{;]*\)\s*\{\n\s*NvtxRange nvtx_\(\"" + fn + r"\"\);", src, re.M)
        assert m, fn
