"""CPU checks of bench.py's driver contract: the reference arm (the oracle on the host cores) prints
one JSON line with the keys the driver reads, ranks > 0 of a torchrun launch print nothing and exit
0, and our arm fails loudly on a machine without a GPU (no CPU fallback)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args, env_extra=None, timeout=600):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="", OMP_NUM_THREADS="1", PLSS_ORACLE_THREADS="1")
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=timeout)


def test_reference_arm_line():
    r = _bench(["--impl", "reference", "--steps", "1", "--warmup", "1", "--workload", "C2"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "it/s" and d["higher_is_better"] is True
    assert d["steps"] == 1 and d["warmup"] == 1
    assert d["config"]["workload"].startswith("C2") and d["config"]["n"] == 100_000
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["value"] == d["value"] and cb["sample"]
    assert cb["cpu_count"] >= 1 and cb["cpu_model"] and d["ms_per_step"] == pytest.approx(1e3 / d["value"])
    assert d["e2e"] == {"value": d["value"], "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_silent():
    r = _bench(["--impl", "reference", "--steps", "1", "--warmup", "1"],
               {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_our_arm_fails_loudly_without_gpu():
    r = _bench(["--steps", "1", "--warmup", "3", "--workload", "C2"], timeout=300)
    assert r.returncode != 0
    assert r.stdout.strip() == ""                      # no JSON line from a CPU fallback


def test_apportion():
    sys.path.insert(0, ROOT)
    import bench
    kt = {"k1": 2.0, "k2": 3.0, "k3": 0.0}
    assert bench._apportion(6.0, kt, "k2") == pytest.approx(3.6)
    assert bench._apportion(6.0, {"k1": 0.0}, "k1") == 0.0


@pytest.mark.gpu
def test_our_arm_line_on_gpu():
    """Our arm on a small workload: one JSON line with the contract's keys (roofline, cpu_baseline,
    e2e with its copy bytes, clocks, gpu_launches)."""
    env = dict(os.environ)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "C2", "--steps", "20",
                        "--warmup", "3"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 3
    assert d["dtype"] == "f64" and d["data"] == "synthetic" and d["vs_baseline"] is None
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 0 and 0 < rf["frac"] < 1.5
    assert rf["frac"] == pytest.approx(rf["achieved"] / rf["peak"])
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 20 * 3
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_gpus_flag_self_launches_ranks():
    """--gpus N without torchrun re-launches bench.py as N ranks (VERDICT r01 missing-3); under
    torchrun WORLD_SIZE must equal N."""
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    calls = []
    ns = argparse.Namespace(gpus=4)
    rc = bench.ensure_world(ns, argv=["--gpus", "4", "--steps", "7"], env={}, run=lambda c: calls.append(c) or 0)
    assert rc == 0 and len(calls) == 1
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-3:] == ["--gpus", "4", "--steps", "7"][-3:]
    assert cmd[cmd.index(os.path.join(ROOT, "bench.py")) + 1:] == ["--gpus", "4", "--steps", "7"]
    assert bench.ensure_world(argparse.Namespace(gpus=1), argv=[], env={}, run=None) is None
    assert bench.ensure_world(argparse.Namespace(gpus=2), argv=[], env={"WORLD_SIZE": "2"}, run=None) is None
    assert bench.ensure_world(argparse.Namespace(gpus=8), argv=[], env={"WORLD_SIZE": "2"}, run=None) == 2


def test_gpus_flag_mismatch_exits_nonzero():
    r = _bench(["--gpus", "8", "--steps", "1", "--warmup", "3", "--workload", "C2"],
               {"RANK": "0", "WORLD_SIZE": "2", "LOCAL_RANK": "0"}, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr and r.stdout.strip() == ""
