"""Run bench.py for several library variants / options and print one compact line each."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(lib, args, timeout=140):
    env = dict(os.environ)
    if lib:
        env["PLSS_LIB"] = os.path.join(ROOT, "paper_2207_07615_b200", f"libplss_{lib}.so")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline"] + args
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=timeout)
    except subprocess.TimeoutExpired:
        return {"error": "timeout"}
    for line in out.stdout.splitlines()[::-1]:
        if line.startswith("{"):
            return json.loads(line)
    return {"error": (out.stderr or out.stdout)[-800:]}


if __name__ == "__main__":
    libs = sys.argv[1].split(",")
    extra = sys.argv[2:]
    for lib in libs:
        r = run(None if lib == "default" else lib, extra)
        if "error" in r:
            print(f"{lib:14s} {' '.join(extra)} ERROR {r['error']}", flush=True)
            continue
        k = r["kernels_ms_per_step"]
        print(f"{lib:14s} {' '.join(extra):40s} sell {r['config'].get('sell_segments')} win {r['config'].get('window_segments')} ms/step {r['ms_per_step']:.3f} it/s {r['value']:.1f} "
              f"GB/s {r['achieved_gbs']:.0f} frac {r['achieved_frac_of_peak']:.3f} | k1 {k['k1']:.3f} "
              f"k2 {k['k2']:.3f} k3 {k['k3']:.3f} dom {r['roofline']['kernel']} {r['roofline']['frac']:.3f}",
              flush=True)
