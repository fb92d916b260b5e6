#!/usr/bin/env python
"""PLSS hot-path benchmark (BASELINE.json metric: PLSS iterations/s and achieved HBM GB/s).

A "step" is one PLSS loop iteration (Algorithm 1: K1 r <- r - A p + rho, K2 y = A^T r
+ phi/psi + tail, K3 p/x update + theta) over the whole workload. Default workload: C5
(BASELINE configs[4], the 1/2/4/8-GPU scaling config: m = 64M, n = 8M, 768M nnz,
banded+random), run in freeze mode with tol 0 so every timed step does the same
work. N > 1 (torchrun): row-block sharding, one NCCL all-reduce of n+1 doubles per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5|C3|C4|C2] [--impl reference]
    python bench.py --method rp [--rp-r 5] [--rp-density 1.0]   # randomized projection (NEXT-2)
    python bench.py --method kz [--workload C2]                   # PLSS Kaczmarz (NEXT-3)
    python bench.py --method eg [--eg-sketch gaussian]            # growing-sketch engine (NEXT-4)

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import plss_gen  # noqa: E402

METRIC = "PLSS iterations/sec and achieved HBM GB/s (fraction of ~8 TB/s)"
RP_METRIC = "Rand. Proj. (eq:pkLong, fresh Gaussian S_k) iterations/sec and achieved HBM GB/s"
KZ_METRIC = "PLSS Kaczmarz (eq:pkKacz) iterations/sec and achieved HBM GB/s"
EG_METRIC = "growing-sketch engine (Thm 2.1 / Cor 2.2) iterations/sec and achieved HBM GB/s"


def eg_bytes_per_iter(m, n, nnz, hk, sketch):
    """Algorithmic bytes of one engine step with hk stored columns: sketch
    (Gaussian: s write + r read 16 m; residual / Gaussian: y = A^T s, 12 nnz + 4 (n+1) + 8 m + 8 n;
    identity: the row, ~0); Y^T y: 8 n hk + 8 n; triangular update: 8 hk^2 (R twice, halves);
    p = coef (y - Y t_hat): 8 n hk + 40 n (y, p, new Y column, x rw); K1: 12 nnz + 4 (m+1) + 8 n + 16 m."""
    sk = {"gaussian": 16 * m + 12 * nnz + 4 * (n + 1) + 8 * m + 8 * n,
          "residual": 12 * nnz + 4 * (n + 1) + 8 * m + 8 * n, "identity": 0}[sketch]
    return sk + 16 * n * hk + 48 * n + 8 * hk * hk + 12 * nnz + 4 * (m + 1) + 8 * n + 16 * m


def eg_launches_per_step(sketch, factor, slabs):
    """Our kernels per engine step (plss.cu eg_enqueue_step): the sketch (identity: k_eg_row;
    Gaussian: k_eg_gauss + K2 per slab; residual: K2 per slab), two Y^T y instances + k_eg_red,
    triangular: k_eg_triu, k_eg_trit, k_eg_gemv / QR: k_qr_b, k_qr_w, k_qr_v, two V^T v instances,
    k_eg_red, k_qr_tri, k_eg_gemv; K1 per slab."""
    sk = {"identity": 1, "gaussian": 1 + slabs, "residual": slabs}[sketch]
    fac = 3 if factor == "triangular" else 8
    return sk + 3 + fac + slabs


def eg_qr_bytes_per_iter(m, n, nnz, hk, sketch):
    """The QR variant streams the store four times (V^T y, y - V b, V^T v, e_h - V z)."""
    return eg_bytes_per_iter(m, n, nnz, hk, sketch) + 16 * n * hk + 48 * n


def kz_bytes_per_iter(m, n, nnz, hk):
    """Algorithmic bytes of one PLSS Kaczmarz step with hk stored updates:
    GEMV: P (8 n hk) + arow, pk, new P column, x rw (40 n); SpMV A p: 12 nnz + 4 (m+1) + 8 n + 8 m;
    residual: r rw, apk, new A P column (32 m); prep: hk values of A P and theta, w (24 hk)."""
    return 8 * n * hk + 40 * n + 12 * nnz + 4 * (m + 1) + 8 * n + 8 * m + 32 * m + 24 * hk


def rp_bytes_per_iter(m, n, nnz, r):
    """Algorithmic bytes of one randomized-projection step: sketch write +
    r read (8 m (r+1)); A^T S: CSC stream + S once + Y write (12 nnz + 4 (n+1) + 8 m r + 8 n r);
    Gram: Y (8 n r); update: Y, x rw, p (8 n r + 24 n); K1: CSR stream, p, r rw
    (12 nnz + 4 (m+1) + 8 n + 16 m)."""
    return (8 * m * (r + 1) + 12 * nnz + 4 * (n + 1) + 8 * m * r + 8 * n * r + 8 * n * r + 8 * n * r + 24 * n
            + 12 * nnz + 4 * (m + 1) + 8 * n + 16 * m)


def _apportion(step_ms, kt, dom):
    """The dominant kernel's share of the device-timed step: the timed region's ms per step split by
    the kernel shares plss_*_profile measured (CUDA events around one-by-one launches, right after
    the timed region). The profile alone swings with the power-capped clock (the same build gave
    K1 + K2 + K3 = 6.09 and 5.47 ms against a 5.93 ms graph-timed step)."""
    tot = sum(v for v in kt.values() if v)
    return step_ms * kt[dom] / tot if tot > 0 else kt[dom]


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _traffic(workload, kernel_class, launches_per_step, capture=None):
    """DRAM bytes (read + write) per step of a kernel class, from the committed `ncu --set full`
    capture of the workload (profiles/r02_ncu_traffic_<workload>.json: one whole step of the round-2
    build, scripts/ncu_traffic.py; the randomized-projection capture keeps its round-1 per-launch
    form). None when no capture of this workload exists."""
    capture = capture or f"r02_ncu_traffic_{workload.lower()}.json"
    path = os.path.join(ROOT, "profiles", capture)
    if not os.path.exists(path):
        return None, None
    with open(path) as f:
        d = json.load(f)
    if "per_step" in d:
        e = d["per_step"].get(kernel_class)
        return (None, None) if e is None else (e["dram_bytes"], f"{os.path.relpath(path, ROOT)}: {d['source']}")
    e = d["per_launch"].get(kernel_class)
    if e is None:
        return None, None
    return e["dram_bytes"] * launches_per_step, f"{os.path.relpath(path, ROOT)}: {d['source']}"


# The second roofline of the SpMV pair: bytes moved from L2 to the SMs per step (32-byte
# sectors: a random 8-byte gather moves one) against the highest rate measured for them on this pool's
# B200s (scripts/gather_l2_bench.cu: random gathers from an L2-resident vector, 10.05 TB/s;
# profiles/r02_gather_l2_bench.txt). The per-step bytes come from the committed whole-step ncu capture.
L2_TO_SM_PEAK_GBS = 10050.0


def _l2_roofline(workload, step_ms):
    path = os.path.join(ROOT, "profiles", f"r02_ncu_traffic_{workload.lower()}.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    tot = sum(v.get("l2_to_sm_bytes", 0.0) for v in d.get("per_step", {}).values())
    if tot <= 0:
        return None
    ach = tot / (step_ms / 1e3) / 1e9
    return {"bound": "l2_to_sm_sectors", "achieved": ach, "peak": L2_TO_SM_PEAK_GBS, "unit": "GB/s",
            "frac": ach / L2_TO_SM_PEAK_GBS, "bytes_per_step": tot,
            "source": f"{os.path.relpath(path, ROOT)} (l1tex__m_xbar2l1tex_read_bytes, whole step); peak: "
                      "profiles/r02_gather_l2_bench.txt"}


# ---------------------------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > i + 2 and s[i + 2] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------------------------
def load_workload(name, rank, world, device, partition="rows"):
    """Returns dict of device tensors for this rank's row block (or column block) + metadata."""
    import torch
    if partition == "cols":
        if name == "C5":
            raise SystemExit("--partition cols: C5 (m > n) is a row-block workload; use C4 / C4alt / C2")
        s = plss_gen.make_config(name)
        blk = plss_gen.col_block(s, world, rank)
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dt)  # noqa: E731
        return {"name": name, "m": s.m, "n": blk["n"], "n_global": s.n, "col_offset": blk["col_offset"],
                "row_offset": 0, "m_global": s.m,
                "row_ptr": t(blk["row_ptr"], torch.int32), "col_idx": t(blk["col_idx"], torch.int32),
                "val": t(blk["val"], torch.float64), "col_ptr": t(blk["col_ptr"], torch.int32),
                "row_idx": t(blk["row_idx"], torch.int32), "val_t": t(blk["val_t"], torch.float64),
                "b": t(blk["b"], torch.float64), "tol": 0.0, "tol_mode": 0, "freeze": True,
                "nnz_global": s.nnz}
    if name == "C5":
        m, n = 64_000_000, 8_000_000
        r0, r1 = plss_gen.row_block_bounds(m, world, rank)
        d = plss_gen.make_c5_torch(device=device, m=m, n=n, rows=(r0, r1))
        d.update(name="C5", tol=0.0, tol_mode=0, freeze=True, nnz_global=12 * m)
        return d
    s = plss_gen.make_config(name)
    r0, r1 = plss_gen.row_block_bounds(s.m, world, rank)
    blk = plss_gen.row_block(s, world, rank)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dt)
    return {"name": name, "m": blk["m"], "n": s.n, "row_offset": r0, "m_global": s.m,
            "row_ptr": t(blk["row_ptr"], torch.int32), "col_idx": t(blk["col_idx"], torch.int32),
            "val": t(blk["val"], torch.float64), "col_ptr": t(blk["col_ptr"], torch.int32),
            "row_idx": t(blk["row_idx"], torch.int32), "val_t": t(blk["val_t"], torch.float64),
            "b": t(blk["b"], torch.float64), "tol": 0.0, "tol_mode": 0, "freeze": True,
            "nnz_global": s.nnz}


def workload_label(name):
    return {
        "C5": "C5: m=64M n=8M, 12 nnz/row (6 banded +-1024 of i*n/m, 6 uniform), N(0,1), 768M nnz",
        "C3": "C3: 5-point Laplacian-like 2048^2 grid, 21M nnz",
        "C4": "C4: power-law Zipf(2.1) rows clipped [1,4096], m=2M n=8M",
        "C4alt": "C4-alt: power-law Zipf(1.845) rows clipped [1,4096] (mean ~12), m=2M n=8M, 23.6M nnz",
        "C2": "C2: m=200k n=100k, 8 uniform nnz/row",
    }.get(name, name)


# ---------------------------------------------------------------------------------------------
# CPU baseline: the oracle on the same arrays (host copies), a bounded number of real steps
# (cpu_sample: the 1/100-scale samples the other methods' legs still use)
# ---------------------------------------------------------------------------------------------
def cpu_sample(name):
    if name == "C5":
        return plss_gen.make_config("C5s"), "C5 recipe at 1/100 scale (m=640k, n=80k, 7.68M nnz)"
    if name == "C3":
        return plss_gen.make_config("C3", N=512), "C3 recipe at 512^2 (1/16 scale)"
    if name == "C4":
        return plss_gen.make_config("C4", m=200_000, n=800_000, support=8000), "C4 recipe at 1/10 scale"
    if name == "C4alt":
        return (plss_gen.make_config("C4alt", m=200_000, n=800_000, support=8000),
                "C4-alt recipe at 1/10 scale")
    return plss_gen.make_config(name), f"{name} full"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def oracle_threads():
    """Host threads of the oracle baseline: every core (SURVEY 8(d) oracle_omp), or
    PLSS_ORACLE_THREADS."""
    return int(os.environ.get("PLSS_ORACLE_THREADS", "0")) or os.cpu_count() or 1


def host_arrays(w):
    """Host (numpy) copies of a workload's device arrays: the bytes the GPU streams, for the oracle."""
    h = {k: w[k].cpu().numpy() for k in ("row_ptr", "col_idx", "val", "col_ptr", "row_idx", "val_t", "b")}
    h.update(m=int(w["m"]), n=int(w["n"]))
    return h


def oracle_run(h, steps, threads):
    """`steps` freeze-mode steps of the oracle (initialization + steps - 1 loop steps: each one
    SpMV pair and the vector work, as a GPU step) on `threads` host threads; seconds."""
    import oracle
    with oracle.threads(threads):
        t0 = time.perf_counter()
        oracle.plss(h["m"], h["n"], h["row_ptr"], h["col_idx"], h["val"], h["col_ptr"], h["row_idx"], h["val_t"],
                    h["b"], tol=0.0, maxit=steps, freeze=True)
        return time.perf_counter() - t0


def cpu_baseline(name, h, full_bytes, budget_s=20.0):
    """The oracle as it stands on the box's host cores, on the full workload's own arrays (host
    copies), for a bounded number of real steps: the threaded oracle (SURVEY 8(d) oracle_omp,
    every core) and one step of the sequential oracle (oracle_seq)."""
    T = oracle_threads()
    t1 = oracle_run(h, 1, T)
    steps = int(max(2, min(500, budget_s / max(t1, 1e-6))))
    t = oracle_run(h, steps, T)
    its = steps / t
    ts = oracle_run(h, 1, 1) if t1 * T <= 30.0 else None
    gbs = full_bytes * its / 1e9
    seq = f"; the sequential oracle (1 thread): {1.0 / ts:.3f} it/s over 1 step" if ts else ""
    return {"value": its, "unit": "it/s", "cores": T, "kind": "oracle", "cpu_model": cpu_model(),
            "cpu_count": os.cpu_count(),
            "sample": f"the oracle on the full {name} arrays (host copies of the bench's own): {steps} freeze-mode "
                      f"steps on {T} threads (oracle_set_threads: static row / column split, blocked dots) in "
                      f"{t:.1f} s = {gbs:.2f} GB/s algorithmic{seq}",
            "oracle_gbs": gbs, "oracle_seq_its": (1.0 / ts) if ts else None}


# ---------------------------------------------------------------------------------------------
# reference arm (--impl reference): the oracle as it stands, rank 0 only
# ---------------------------------------------------------------------------------------------
def reference_inputs(name):
    """The workload our arm times at N = 1, as host arrays. C5 comes from plss_gen.make_c5_torch on
    the box's GPU when it has one (input synthesis only; the oracle runs on the host), else from the
    same recipe on the CPU generator (a different stream, labelled)."""
    if name == "C5":
        import torch
        dev = "cuda" if torch.cuda.is_available() else "cpu"
        d = plss_gen.make_c5_torch(device=dev)
        h = host_arrays(d)
        del d
        if dev == "cuda":
            torch.cuda.empty_cache()
        return h, ("generated by make_c5_torch on the GPU (the bench's arrays)" if dev == "cuda"
                   else "generated by make_c5_torch on the CPU generator (another stream than the GPU arm's)")
    s = plss_gen.make_config(name)
    h = {"row_ptr": s.row_ptr, "col_idx": s.col_idx, "val": s.val, "col_ptr": s.col_ptr, "row_idx": s.row_idx,
         "val_t": s.val_t, "b": s.b, "m": s.m, "n": s.n}
    return h, "plss_gen recipe (the bench's arrays)"


def run_reference(args, rank, world):
    if rank != 0:
        return
    name = args.workload
    full = full_bytes_of(name)
    h, src = reference_inputs(name)
    T = oracle_threads()
    oracle_run(h, max(1, args.warmup), T)
    t = oracle_run(h, args.steps, T)
    value = args.steps / t
    line = {"metric": METRIC, "value": value, "unit": "it/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload_label(name), **full_dims_of(name),
                                            "parallelism": f"oracle on {T} host threads", "freeze_mode": True,
                                            "tol": 0.0},
            "cpu_baseline": {"value": value, "unit": "it/s", "cores": T, "kind": "oracle", "cpu_model": cpu_model(),
                             "cpu_count": os.cpu_count(),
                             "sample": f"the full {name} workload ({src}); {args.steps} timed freeze-mode steps "
                                       f"after {max(1, args.warmup)} warm-up steps of the oracle on {T} threads "
                                       f"(oracle_set_threads); {full * value / 1e9:.2f} GB/s algorithmic"},
            "e2e": {"value": value, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def full_dims_of(name):
    """m, n, nnz of the full workload (the config keys of our arm's line)."""
    if name == "C5":
        return {"m": 64_000_000, "n": 8_000_000, "nnz": 768_000_000}
    if name == "C3":
        return {"m": 2048 ** 2, "n": 2048 ** 2, "nnz": 5 * 2048 ** 2 - 4 * 2048}
    s = plss_gen.make_config(name)
    return {"m": s.m, "n": s.n, "nnz": s.nnz}


def full_bytes_of(name):
    return {"C5": plss_gen.bytes_per_iter(64_000_000, 8_000_000, 768_000_000),
            "C3": plss_gen.bytes_per_iter(2048 ** 2, 2048 ** 2, 5 * 2048 ** 2 - 4 * 2048),
            }.get(name) or (lambda s: plss_gen.bytes_per_iter(s.m, s.n, s.nnz))(plss_gen.make_config(name))


def _free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_command(argv, gpus, port):
    """The torchrun command that runs this script as `gpus` ranks on one node (127.0.0.1)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def ensure_world(args, argv=None, env=None, run=subprocess.call):
    """--gpus N must mean N ranks. Without torchrun (WORLD_SIZE unset) and N > 1, re-launch this
    script through torch.distributed.run with N processes and return its exit code; under torchrun,
    WORLD_SIZE must equal N (returns 2 with a message otherwise). None: carry on in this process."""
    env = os.environ if env is None else env
    argv = sys.argv[1:] if argv is None else argv
    ws = env.get("WORLD_SIZE")
    if ws is None:
        if args.gpus <= 1:
            return None
        return run(launch_command(argv, args.gpus, _free_port()))
    if int(ws) != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; launch with "
                         f"--nproc-per-node {args.gpus} or drop torchrun\n")
        return 2
    return None


# ---------------------------------------------------------------------------------------------
# main (our arm)
# ---------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--impl", default="plss", choices=["plss", "reference"])
    ap.add_argument("--slabs", type=int, default=0)
    ap.add_argument("--no-sell", action="store_true", help="CSR tiles only (no SELL-32 copies)")
    ap.add_argument("--no-window", action="store_true", help="SELL-32 without shared-memory windows")
    ap.add_argument("--plss-w", action="store_true",
                    help="PLSS W: WI = diag(||A_{:,j}||) (the paper's second variant; default PLSS, WI = I)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-step", default="allreduce", choices=["allreduce", "rsag", "peer"],
                    help="N > 1: allreduce = one NCCL all-reduce of n+1 values, overlapped with K2 in column chunks; "
                         "rsag = reduce-scatter y, shard dots / K3, all-reduce 4 scalars, all-gather p; "
                         "peer = the library's own peer-memory all-reduce kernels (NVLink loads / stores), "
                         "overlapped with K2 in column chunks")
    ap.add_argument("--partition", default="rows", choices=["rows", "cols"],
                    help="distributed partition: row blocks (x, p, y replicated; all-reduce of n + 1) or "
                         "column blocks (r replicated; all-reduces of m + 1 and 2), for m < n")
    ap.add_argument("--force-dist", action="store_true",
                    help="N = 1: run the distributed ctx on one rank (measures the dist step's own cost)")
    ap.add_argument("--rhs", default="xstar", choices=["xstar", "paper"],
                    help="paper: the paper's protocol right-hand side x = ones, x(1) = 10, b = A x (P:L987), "
                         "a labelled protocol-fidelity variant (SURVEY 8d)")
    ap.add_argument("--profile-steps", type=int, default=10)
    ap.add_argument("--ncu", action="store_true", help="short run for ncu: no e2e / profile / cpu legs")
    ap.add_argument("--method", default="plss", choices=["plss", "rp", "kz", "eg"],
                    help="rp: randomized projection (the paper's comparison method, NEXT-2); "
                         "kz: PLSS Kaczmarz (section 7, NEXT-3); eg: growing-sketch engine (NEXT-4)")
    ap.add_argument("--eg-sketch", default="gaussian", choices=["residual", "identity", "gaussian"])
    ap.add_argument("--eg-factor", default="triangular", choices=["triangular", "qr"])
    ap.add_argument("--rp-r", type=int, default=5, help="sketch size r (Experiment III: 5 for n > 1e5)")
    ap.add_argument("--rp-density", type=float, default=1.0, help="< 1: sparse normal sketch")
    args = ap.parse_args()
    if args.impl != "reference":
        rc = ensure_world(args)
        if rc is not None:
            sys.exit(rc)
    if args.method == "rp":
        return main_rp(args)
    if args.method == "kz":
        if args.workload == "C5":
            args.workload = "C2"          # the history grows as 8 (m + n) bytes per step: C2, not C5
        if "--steps" not in sys.argv:
            args.steps = 1000
        return main_kz(args)
    if args.method == "eg":
        if args.workload == "C5":
            args.workload = "C2"          # the stored Y grows by 8 n bytes per step
        if "--steps" not in sys.argv:
            args.steps = 500
        return main_eg(args)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_2207_07615_b200 as pkg

    assert args.warmup >= 3 or args.ncu, "timing rules: at least 3 warm-up steps"
    assert torch.cuda.is_available(), "our arm needs a CUDA device (no CPU fallback)"
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local} but {torch.cuda.device_count()} GPU(s) are visible")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    pkg.load_library()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    w = load_workload(args.workload, rank, world, dev, args.partition)
    m_l, n = w["m"], w["n"]
    nnz_l = int(w["col_idx"].numel())
    A = pkg.Matrix(m_l, n, w["row_ptr"], w["col_idx"], w["val"], w["col_ptr"], w["row_idx"], w["val_t"])
    stream = torch.cuda.Stream(device=dev)
    maxit_cap = args.warmup + args.steps + max(args.profile_steps, 1) + 8
    if world > 1 or args.force_dist:
        uid = pkg.plss_get_unique_id() if rank == 0 else bytes(128)
        obj = [uid]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        if args.partition == "cols":
            ctx = pkg.plss_create_dist_cols(A, w["col_offset"], w["n_global"], obj[0], rank, world,
                                            slabs=args.slabs, maxit_cap=maxit_cap, stream=stream,
                                            sell=not args.no_sell, window=not args.no_window)
        else:
            ctx = pkg.plss_create_dist(A, w["row_offset"], w["m_global"], obj[0], rank, world,
                                       slabs=args.slabs, maxit_cap=maxit_cap, stream=stream,
                                       sell=not args.no_sell, window=not args.no_window,
                                       rsag=args.dist_step == "rsag", peer=args.dist_step == "peer")
    else:
        ctx = pkg.plss_create(A, slabs=args.slabs, maxit_cap=maxit_cap, stream=stream, sell=not args.no_sell,
                              window=not args.no_window)
    q = pkg.plss_query(ctx)
    b = w["b"]
    if args.rhs == "paper":                                   # b = A x_p with x_p = ones, x_p(1) = 10
        xp = torch.ones(n, dtype=torch.float64, device=dev)
        xp[0] = 10.0
        b = torch.empty(m_l, dtype=torch.float64, device=dev)
        pkg.plss_spmv(ctx, xp, b)
        del xp
    if args.plss_w:
        pkg.plss_set_wi(ctx, pkg.plss_column_norms(ctx))
    torch.cuda.synchronize()

    # ---- device-timed region: K steps, inputs resident in HBM (> L2 per step) ----------------
    pkg.plss_start(ctx, b, None, tol=w["tol"], tol_mode=w["tol_mode"], maxit=maxit_cap, flags=1)
    pkg.plss_step(ctx, args.warmup)
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        pkg.plss_step(ctx, args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    fin = pkg.plss_finish(ctx, None, want_hist=True, want_diag=True)
    cross_rank = None
    if world > 1:
        # every rank must hold bitwise the same rho, phi, theta, beta, gamma records
        rec = torch.from_numpy(np.ascontiguousarray(fin["diag"])).to(dev)
        allrec = [torch.empty_like(rec) for _ in range(world)]
        dist.all_gather(allrec, rec)
        cross_rank = all(torch.equal(allrec[0].view(torch.int64), a.view(torch.int64)) for a in allrec[1:])
        assert cross_rank, "ranks disagree on the per-iteration scalar records (rho, phi, theta, beta, gamma)"
    iters_per_s = args.steps / (ms / 1e3)
    n_global = w.get("n_global", n)
    B_global = plss_gen.bytes_per_iter(w["m_global"], n_global, w["nnz_global"])
    if args.ncu:
        if rank == 0:
            print(json.dumps({"ncu_run": True, "ms_per_step": ms / args.steps}), flush=True)
        return

    # ---- per-kernel device times (CUDA events around each launch on the ctx stream) ----------
    pkg.plss_start(ctx, b, None, tol=w["tol"], tol_mode=w["tol_mode"], maxit=maxit_cap, flags=1)
    pkg.plss_step(ctx, 3)
    kt = pkg.plss_profile(ctx, max(1, args.profile_steps))
    k1_bytes = 12 * nnz_l + 4 * (m_l + 1) + 8 * n + 16 * m_l
    # SURVEY 8(d)'s per-kernel figures (K2's includes the p read for psi, which one device sums in
    # K3 instead: DESIGN.md R25; the ncu traffic shows the bytes actually moved)
    k2_bytes = 12 * nnz_l + 4 * (n + 1) + 8 * m_l + 16 * n
    k3_bytes = 40 * n
    s2 = pkg.plss_query_segment(ctx, 2, q["slabs"] - 1)
    fused = world == 1 and not args.force_dist and not args.plss_w and bool(s2["psi3"]) and bool(s2["xdefer"])
    classes = {"k1_spmv_csr_resid": (kt["k1"], k1_bytes), "k2_spmv_csc_gather": (kt["k2"], k2_bytes),
               "k3_pxupdate": (kt["k3"], k3_bytes)}
    dom = max(classes, key=lambda c: classes[c][0])
    dom_prof_ms, dom_bytes = classes[dom]
    dom_ms = _apportion(ms / args.steps, kt, {"k1_spmv_csr_resid": "k1", "k2_spmv_csc_gather": "k2",
                                              "k3_pxupdate": "k3"}[dom])
    peak, peak_src = _peaks()
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    traffic, traffic_src = _traffic(w["name"], dom, q["slabs"])

    # ---- end-to-end through the public API: host b in, host x + history out, K steps ---------
    pin_b = torch.empty(m_l, dtype=torch.float64, pin_memory=True)
    pin_b.copy_(b.cpu())
    pin_x = torch.empty(n, dtype=torch.float64, pin_memory=True)
    barrier()
    t0 = time.perf_counter()
    res = pkg.plss_solve(ctx, pin_b, None, tol=0.0, maxit=args.steps, flags=1, x=pin_x, want_hist=True)
    t_e2e = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([t_e2e], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e2e = float(t.item())
    e2e = {"value": args.steps / t_e2e, "unit": "it/s",
           "h2d_bytes_per_step": 8 * m_l / args.steps,
           "d2h_bytes_per_step": (8 * n + 8 * (args.steps + 1)) / args.steps,
           "solve_iters": args.steps, "note": "one plss_solve from pinned host b to host x + history"}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": iters_per_s, "unit": "it/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_label(w["name"]), "m": w["m_global"], "n": n_global,
                       "nnz": w["nnz_global"],
                       "parallelism": (f"column-block dp{world}" if args.partition == "cols" and
                                       (world > 1 or args.force_dist)
                                       else f"row-block dp{world} ({args.dist_step})" if world > 1 or args.force_dist
                                       else "single"),
                       "slabs": q["slabs"], "sell_segments": q["sell_segments"],
                       "window_segments": q["window_segments"], "freeze_mode": True,
                       "tol": 0.0, "variant": "PLSS W (WI = diag(||A_:,j||))" if args.plss_w else "PLSS (WI = I)",
                       "rhs": ("paper: x = ones, x(1) = 10, b = A x (P:L987)" if args.rhs == "paper"
                               else "b = A x*, x* ~ N(0,1)"),
                       "l2": f"inputs larger than L2: {B_global / 1e9:.2f} GB algorithmic per step",
                       "bytes_per_step_model": "24 nnz + 28 m + 68 n + 8 (SURVEY 8(d))",
                       "vector_work": ("rho in K1, phi in K2's last slab, theta + psi in K3, x every other step "
                                       "(DESIGN.md R25)" if fused else "as SURVEY 8(d)"),
                       "workspace_gb": round(ctx.workspace.numel() / 1e9, 3),
                       "matrix_gb": round(sum(t.numel() * t.element_size() for t in (
                           w["row_ptr"], w["col_idx"], w["val"], w["col_ptr"], w["row_idx"], w["val_t"])) / 1e9, 3)},
            "achieved_gbs": B_global * iters_per_s / 1e9,
            "achieved_frac_of_peak": B_global * iters_per_s / 1e9 / peak,
            "achieved_frac_of_8tbs": B_global * iters_per_s / 1e9 / 8000.0,
            # the same rate on the bytes the fused one-device step's data flow needs (psi in K3, x
            # every other step: 24 nnz + 28 m + 52 n + 8, R25); None where not fused
            "achieved_frac_of_peak_fused_flow": (
                plss_gen.bytes_per_iter_fused(w["m_global"], n_global, w["nnz_global"]) * iters_per_s / 1e9 / peak
                if fused else None),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_step": dom_bytes, "kernel_ms_per_step": dom_ms,
                         "kernel_ms_per_step_profile": dom_prof_ms,
                         "timing": "the timed region's ms per step x the kernel's share of plss_profile"},
            "kernels_ms_per_step": kt,
            "roofline_l2": _l2_roofline(w["name"], ms / args.steps) if world == 1 and not args.force_dist else None,
            "gpu_launches": args.steps * q["launches_per_step"],
            "e2e": e2e,
            "clocks": clocks,
            "final_hist": float(fin["hist_full"][min(args.warmup + args.steps, maxit_cap) - 1]),
        }
        if cross_rank is not None:
            line["cross_rank_bitwise_scalars"] = cross_rank
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(w["name"], host_arrays(w), B_global)
        print(json.dumps(line), flush=True)
    pkg.plss_destroy(ctx)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------------------------
# randomized projection (--method rp): single device (the method is not row-block sharded here)
# ---------------------------------------------------------------------------------------------
def rp_cpu_leg(name, r, density, full_bytes, steps=None, budget_s=15.0):
    """The randomized-projection oracle on the 1/100-scale sample; it/s scaled by bytes/iter."""
    from oracle import randproj as orp
    s, label = cpu_sample(name)
    A = s.scipy_csr()
    sb = rp_bytes_per_iter(s.m, s.n, s.nnz, r)
    t0 = time.perf_counter()
    orp.randproj(A, s.b, r=r, seed=1, maxit=2, density=density)
    t1 = (time.perf_counter() - t0) / 2
    k = steps or int(max(2, min(200, budget_s / max(t1, 1e-6))))
    t0 = time.perf_counter()
    orp.randproj(A, s.b, r=r, seed=1, maxit=k, density=density)
    t = time.perf_counter() - t0
    gbs = sb * k / t / 1e9
    cores = int(os.environ.get("OMP_NUM_THREADS", "0")) or os.cpu_count()
    return {"value": gbs * 1e9 / full_bytes, "unit": "it/s", "cores": cores, "kind": "oracle",
            "sample": f"{label}; {k} randomized-projection steps (r={r}) in {t:.1f} s = {gbs:.2f} GB/s "
                      f"algorithmic (numpy/scipy, BLAS threads up to {cores}); it/s scaled to the full "
                      f"workload by algorithmic bytes/iter", "oracle_gbs": gbs}


def main_rp(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    r, dens = args.rp_r, args.rp_density
    name = args.workload
    if name == "C5":
        m, n, nnz = 64_000_000, 8_000_000, 768_000_000
    else:
        s0 = plss_gen.make_config(name)
        m, n, nnz = s0.m, s0.n, s0.nnz
    B = rp_bytes_per_iter(m, n, nnz, r)
    label = workload_label(name) + f"; randomized projection r={r}" + (f", sparse S density {dens}" if dens < 1 else "")
    if args.impl == "reference":
        if rank != 0:
            return
        leg = rp_cpu_leg(name, r, dens, B, steps=max(1, args.steps))
        v = leg["value"]
        print(json.dumps({"metric": RP_METRIC, "value": v, "unit": "it/s", "impl": "reference", "n_gpus": args.gpus,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / v,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic", "config": {"workload": label}, "cpu_baseline": leg,
                          "e2e": {"value": v, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
              flush=True)
        return
    import torch
    import paper_2207_07615_b200 as pkg
    assert world == 1, "randomized projection: single device (bench.py --method rp runs without torchrun)"
    assert args.warmup >= 3 or args.ncu, "timing rules: at least 3 warm-up steps"
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pkg.load_library()
    w = load_workload(name, 0, 1, dev)
    A = pkg.Matrix(w["m"], w["n"], w["row_ptr"], w["col_idx"], w["val"], w["col_ptr"], w["row_idx"], w["val_t"])
    stream = torch.cuda.Stream(device=dev)
    cap = args.warmup + args.steps + max(args.profile_steps, 1) + 8
    ctx = pkg.plss_create(A, slabs=args.slabs, maxit_cap=cap, stream=stream)
    q = pkg.plss_query(ctx)
    b = w["b"]
    torch.cuda.synchronize()
    pkg.plss_rp_start(ctx, b, r=r, seed=1, density=dens, tol=0.0, maxit=cap)
    pkg.plss_rp_step(ctx, args.warmup)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        pkg.plss_rp_step(ctx, args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    fin = pkg.plss_rp_finish(ctx, None, want_hist=True)
    its = args.steps / (ms / 1e3)
    if args.ncu:
        print(json.dumps({"ncu_run": True, "ms_per_step": ms / args.steps}), flush=True)
        return
    pkg.plss_rp_start(ctx, b, r=r, seed=1, density=dens, tol=0.0, maxit=cap)
    pkg.plss_rp_step(ctx, 2)
    kt = pkg.plss_rp_profile(ctx, max(1, args.profile_steps))
    cls = {"rp_spmm_AtS": (kt["spmm"], 12 * nnz + 4 * (n + 1) + 8 * m * r + 8 * n * r),
           "rp_sketch_gen": (kt["gen"], 8 * m * (r + 1)),
           "k1_spmv_csr_resid": (kt["k1"], 12 * nnz + 4 * (m + 1) + 8 * n + 16 * m),
           "rp_gram": (kt["gram"], 8 * n * r), "rp_update": (kt["update"], 8 * n * r + 24 * n)}
    dom = max(cls, key=lambda c: cls[c][0])
    dom_prof_ms, dom_bytes = cls[dom]
    dom_ms = _apportion(ms / args.steps, kt, {"rp_spmm_AtS": "spmm", "rp_sketch_gen": "gen", "k1_spmv_csr_resid": "k1",
                                              "rp_gram": "gram", "rp_update": "update"}[dom])
    peak, peak_src = _peaks()
    traffic, traffic_src = (_traffic(name, dom, 1, "r01_ncu_traffic_c5_rp.json") if (name == "C5" and r == 5 and dens == 1.0)
                            else (None, None))
    pin_b = torch.empty(w["m"], dtype=torch.float64, pin_memory=True)
    pin_b.copy_(b.cpu())
    pin_x = torch.empty(n, dtype=torch.float64, pin_memory=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pkg.plss_rp_solve(ctx, pin_b, r=r, seed=1, density=dens, tol=0.0, maxit=args.steps, x=pin_x)
    t_e2e = time.perf_counter() - t0
    line = {"metric": RP_METRIC, "value": its, "unit": "it/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": label, "m": m, "n": n, "nnz": nnz, "r": r, "density": dens,
                       "parallelism": "single", "slabs": q["slabs"], "tol": 0.0,
                       "l2": f"inputs larger than L2: {B / 1e9:.2f} GB algorithmic per step",
                       "bytes_per_step_model": "24 nnz + (16 r + 28) m + (24 r + 36) n + 8"},
            "achieved_gbs": B * its / 1e9, "achieved_frac_of_peak": B * its / 1e9 / peak,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": dom_bytes / (dom_ms / 1e3) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": dom_bytes / (dom_ms / 1e3) / 1e9 / peak, "traffic": traffic,
                         "traffic_source": traffic_src, "peak_source": peak_src, "algorithmic_bytes_per_step": dom_bytes,
                         "kernel_ms_per_step": dom_ms, "kernel_ms_per_step_profile": dom_prof_ms,
                         "timing": "the timed region's ms per step x the kernel's share of plss_rp_profile"},
            "kernels_ms_per_step": kt, "gpu_launches": args.steps * (5 + q["slabs"]),
            "e2e": {"value": args.steps / t_e2e, "unit": "it/s", "h2d_bytes_per_step": 8 * w["m"] / args.steps,
                    "d2h_bytes_per_step": (8 * n + 8 * (args.steps + 1)) / args.steps, "solve_iters": args.steps,
                    "note": "one plss_rp_solve from pinned host b to host x + history"},
            "clocks": clk.summary(), "final_hist": float(fin["hist_full"][args.warmup + args.steps])}
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = rp_cpu_leg(name, r, dens, B)
    print(json.dumps(line), flush=True)
    pkg.plss_destroy(ctx)


# ---------------------------------------------------------------------------------------------
# PLSS Kaczmarz (--method kz): single device; a step's cost grows with the stored history hk
# ---------------------------------------------------------------------------------------------
def kz_cpu_leg(s, label, rows, full_bytes_fn, steps=None, budget_s=15.0):
    """The Kaczmarz oracle on the same workload for a bounded number of steps from hk = 0; its
    algorithmic GB/s (kz_bytes_per_iter at each step's hk) converts to it/s for the GPU window."""
    from oracle import kaczmarz as okz
    A = s.scipy_csr()
    t0 = time.perf_counter()
    okz.kz_solve(A, s.b, rows, maxit=5)
    t1 = (time.perf_counter() - t0) / 5
    k = steps or int(max(20, min(400, budget_s / max(t1 * 8, 1e-6))))   # per-step cost grows with k
    t0 = time.perf_counter()
    okz.kz_solve(A, s.b, rows, maxit=k)
    t = time.perf_counter() - t0
    byts = sum(kz_bytes_per_iter(s.m, s.n, s.nnz, h) for h in range(k))
    gbs = byts / t / 1e9
    cores = int(os.environ.get("OMP_NUM_THREADS", "0")) or os.cpu_count()
    return {"value": gbs * 1e9 / full_bytes_fn, "unit": "it/s", "cores": cores, "kind": "oracle",
            "sample": f"{label}; the first {k} PLSS Kaczmarz steps (history 0..{k - 1}) in {t:.1f} s = "
                      f"{gbs:.2f} GB/s algorithmic (numpy/scipy, BLAS threads up to {cores}); it/s scaled "
                      f"to the GPU's timed window by algorithmic bytes/iter", "oracle_gbs": gbs}


def main_kz(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    name = args.workload
    s = plss_gen.make_config(name)
    m, n, nnz = s.m, s.n, s.nnz
    W, K = args.warmup, args.steps
    rows_all = np.random.default_rng(1).permutation(m)
    cap = W + K + max(args.profile_steps, 1) + 8
    rows = np.resize(rows_all, cap).astype(np.int32)
    hk_mean = W + (K - 1) / 2.0                      # history size over the timed steps (no skips)
    B = kz_bytes_per_iter(m, n, nnz, hk_mean)
    label = workload_label(name) + f"; PLSS Kaczmarz, random row order, timed steps with history {W}..{W + K - 1}"
    if args.impl == "reference":
        if rank != 0:
            return
        leg = kz_cpu_leg(s, workload_label(name), rows, B, steps=max(1, args.steps))
        v = leg["value"]
        print(json.dumps({"metric": KZ_METRIC, "value": v, "unit": "it/s", "impl": "reference", "n_gpus": args.gpus,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / v,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic", "config": {"workload": label}, "cpu_baseline": leg,
                          "e2e": {"value": v, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
              flush=True)
        return
    import torch
    import paper_2207_07615_b200 as pkg
    assert world == 1, "PLSS Kaczmarz: single device (bench.py --method kz runs without torchrun)"
    assert args.warmup >= 3 or args.ncu, "timing rules: at least 3 warm-up steps"
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pkg.load_library()
    A = pkg.Matrix.from_arrays(m, n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t, device=dev)
    stream = torch.cuda.Stream(device=dev)
    ctx = pkg.plss_create(A, slabs=args.slabs, maxit_cap=cap, stream=stream)
    q = pkg.plss_query(ctx)
    b = torch.from_numpy(s.b).to(dev)
    drows = torch.from_numpy(rows).to(dev)
    torch.cuda.synchronize()
    pkg.plss_kz_start(ctx, b, drows, kmax=cap, tol=0.0, maxit=cap)
    pkg.plss_kz_step(ctx, W)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        pkg.plss_kz_step(ctx, K)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    fin = pkg.plss_kz_finish(ctx, None, want_hist=True, want_diag=True)
    skipped = int(fin["diag"][1:W + K + 1, 2].sum())
    its = K / (ms / 1e3)
    if args.ncu:
        print(json.dumps({"ncu_run": True, "ms_per_step": ms / K}), flush=True)
        return
    kt = pkg.plss_kz_profile(ctx, max(1, args.profile_steps))      # steps with history ~ W + K
    hk_prof = W + K - skipped + (max(1, args.profile_steps) - 1) / 2.0
    cls = {"kz_gemv_history": (kt["gemv"], 8 * n * hk_prof + 40 * n),
           "kz_spmv_Ap": (kt["spmv"], 12 * nnz + 4 * (m + 1) + 8 * n + 8 * m),
           "kz_resid": (kt["resid"], 32 * m), "kz_prep": (kt["prep"], 24 * hk_prof)}
    dom = max(cls, key=lambda c: cls[c][0])
    dom_ms, dom_bytes = cls[dom]
    peak, peak_src = _peaks()
    pin_b = torch.empty(m, dtype=torch.float64, pin_memory=True)
    pin_b.copy_(b.cpu())
    pin_x = torch.empty(n, dtype=torch.float64, pin_memory=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):              # a ~0.1 s solve: the median of 3 against host-side hiccups
        t0 = time.perf_counter()
        pkg.plss_kz_solve(ctx, pin_b, rows, kmax=cap, tol=0.0, maxit=W + K, x=pin_x)
        ts.append(time.perf_counter() - t0)
    t_e2e = sorted(ts)[1]
    line = {"metric": KZ_METRIC, "value": its, "unit": "it/s", "n_gpus": 1, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": label, "m": m, "n": n, "nnz": nnz, "history_mean": hk_mean,
                       "parallelism": "single", "slabs": q["slabs"], "tol": 0.0, "skipped_rows": skipped,
                       "l2": f"history P is {8 * n * (W + K) / 1e9:.2f} GB at the end (> L2 after "
                             f"{126e6 / (8 * n):.0f} steps); A is {12 * nnz / 1e6:.0f} MB (L2-resident)",
                       "bytes_per_step_model": "8 n hk + 48 n + 12 nnz + 44 m + 24 hk + 4"},
            "achieved_gbs": B * its / 1e9, "achieved_frac_of_peak": B * its / 1e9 / peak,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": dom_bytes / (dom_ms / 1e3) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": dom_bytes / (dom_ms / 1e3) / 1e9 / peak, "traffic": None,
                         "peak_source": peak_src, "algorithmic_bytes_per_step": dom_bytes,
                         "kernel_ms_per_step": dom_ms, "history_at_profile": hk_prof},
            # per step: k_kz_gemv and k_kz_resid (row prep fused), plus the plain SpMV per slab unless
            # every row has <= 32 entries (then k_kz_resid computes (A p)_l itself)
            "kernels_ms_per_step": kt,
            "gpu_launches": K * (2 + (0 if (int(np.diff(s.row_ptr).max()) <= 32
                                            and os.environ.get("PLSS_KZ_FUSE", "1") != "0") else q["slabs"])),
            "e2e": {"value": (W + K) / t_e2e, "unit": "it/s", "h2d_bytes_per_step": (8 * m + 4 * (W + K)) / (W + K),
                    "d2h_bytes_per_step": (8 * n + 8 * (W + K + 1)) / (W + K), "solve_iters": W + K,
                    "note": "median of 3 plss_kz_solve calls from pinned host b and host rows to host x + history "
                            "(steps from history 0, so cheaper on average than the timed window)"},
            "clocks": clk.summary(), "final_hist": float(fin["hist_full"][W + K])}
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = kz_cpu_leg(s, workload_label(name), rows, B)
    print(json.dumps(line), flush=True)
    pkg.plss_destroy(ctx)


# ---------------------------------------------------------------------------------------------
# growing-sketch engine (--method eg): single device
# ---------------------------------------------------------------------------------------------
def main_eg(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    name, sk = args.workload, args.eg_sketch
    s = plss_gen.make_config(name)
    m, n, nnz = s.m, s.n, s.nnz
    W, K = args.warmup, args.steps
    cap = W + K + max(args.profile_steps, 1) + 8
    rows = np.resize(np.random.default_rng(1).permutation(m), cap).astype(np.int32)
    hk_mean = W + (K - 1) / 2.0
    fac = args.eg_factor
    B = (eg_bytes_per_iter if fac == "triangular" else eg_qr_bytes_per_iter)(m, n, nnz, hk_mean, sk)
    label = (workload_label(name) + f"; growing-sketch engine ({fac} factorization), {sk} sketch columns, "
             f"timed steps with history {W}..{W + K - 1}")
    if args.impl == "reference":
        if rank != 0:
            return
        from oracle import engine as oeg
        k = max(1, min(args.steps, 150))
        t0 = time.perf_counter()
        (oeg.tri_engine if fac == "triangular" else oeg.qr_engine)(s.scipy_csr(), s.b, sketch=sk, maxit=k, rows=rows,
                                                                    seed=1)
        t = time.perf_counter() - t0
        bfn = eg_bytes_per_iter if fac == "triangular" else eg_qr_bytes_per_iter
        gbs = sum(bfn(m, n, nnz, h, sk) for h in range(k)) / t / 1e9
        v = gbs * 1e9 / B
        cores = int(os.environ.get("OMP_NUM_THREADS", "0")) or os.cpu_count()
        leg = {"value": v, "unit": "it/s", "cores": cores, "kind": "oracle",
               "sample": f"the first {k} engine steps of the oracle in {t:.1f} s = {gbs:.2f} GB/s algorithmic, "
                         f"scaled to the timed window by bytes/iter"}
        print(json.dumps({"metric": EG_METRIC, "value": v, "unit": "it/s", "impl": "reference", "n_gpus": args.gpus,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / v,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic", "config": {"workload": label}, "cpu_baseline": leg,
                          "e2e": {"value": v, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
              flush=True)
        return
    import torch
    import paper_2207_07615_b200 as pkg
    assert world == 1, "growing-sketch engine: single device"
    assert args.warmup >= 3 or args.ncu, "timing rules: at least 3 warm-up steps"
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pkg.load_library()
    A = pkg.Matrix.from_arrays(m, n, s.row_ptr, s.col_idx, s.val, s.col_ptr, s.row_idx, s.val_t, device=dev)
    stream = torch.cuda.Stream(device=dev)
    ctx = pkg.plss_create(A, slabs=args.slabs, maxit_cap=cap, stream=stream)
    q = pkg.plss_query(ctx)
    b = torch.from_numpy(s.b).to(dev)
    drows = torch.from_numpy(rows).to(dev)
    torch.cuda.synchronize()
    pkg.plss_eg_start(ctx, b, sketch=sk, kmax=cap, rows=drows, seed=1, tol=0.0, maxit=cap, factor=fac)
    pkg.plss_eg_step(ctx, W)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        pkg.plss_eg_step(ctx, K)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    fin = pkg.plss_eg_finish(ctx, None, want_hist=True, want_diag=True)
    skipped = int(fin["diag"][1:W + K + 1, 3].sum())
    its = K / (ms / 1e3)
    if args.ncu:
        print(json.dumps({"ncu_run": True, "ms_per_step": ms / K}), flush=True)
        return
    kt = pkg.plss_eg_profile(ctx, max(1, args.profile_steps))
    hk_prof = W + K - skipped + (max(1, args.profile_steps) - 1) / 2.0
    cls = {"eg_gemvT_history": (kt["gemvT"], 8 * n * hk_prof + 8 * n),
           "eg_gemv_history": (kt["gemv"], 8 * n * hk_prof + 40 * n),
           "eg_tri": (kt["tri"], 8 * hk_prof * hk_prof if fac == "triangular"
                      else 16 * n * hk_prof + 48 * n + 8 * hk_prof * hk_prof),   # QR: w = y - V b, V^T v, T
           "k1_spmv_csr_resid": (kt["k1"], 12 * nnz + 4 * (m + 1) + 8 * n + 16 * m)}
    dom = max(cls, key=lambda c: cls[c][0])
    dom_ms, dom_bytes = cls[dom]
    peak, peak_src = _peaks()
    pin_b = torch.empty(m, dtype=torch.float64, pin_memory=True)
    pin_b.copy_(b.cpu())
    pin_x = torch.empty(n, dtype=torch.float64, pin_memory=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):              # a ~0.1 s solve: the median of 3 against host-side hiccups
        t0 = time.perf_counter()
        pkg.plss_eg_solve(ctx, pin_b, sketch=sk, kmax=cap, rows=rows, seed=1, tol=0.0, maxit=W + K, x=pin_x,
                          factor=fac)
        ts.append(time.perf_counter() - t0)
    t_e2e = sorted(ts)[1]
    line = {"metric": EG_METRIC, "value": its, "unit": "it/s", "n_gpus": 1, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": label, "m": m, "n": n, "nnz": nnz, "sketch": sk, "factor": fac,
                       "history_mean": hk_mean,
                       "parallelism": "single", "slabs": q["slabs"], "tol": 0.0, "skipped_steps": skipped,
                       "l2": f"stored Y is {8 * n * (W + K) / 1e9:.2f} GB at the end (> L2 after "
                             f"{126e6 / (8 * n):.0f} steps)",
                       "bytes_per_step_model": "sketch + 16 n hk + 8 hk^2 + 48 n + K1"},
            "achieved_gbs": B * its / 1e9, "achieved_frac_of_peak": B * its / 1e9 / peak,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": dom_bytes / (dom_ms / 1e3) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": dom_bytes / (dom_ms / 1e3) / 1e9 / peak, "traffic": None,
                         "peak_source": peak_src, "algorithmic_bytes_per_step": dom_bytes,
                         "kernel_ms_per_step": dom_ms, "history_at_profile": hk_prof},
            "kernels_ms_per_step": kt, "gpu_launches": K * eg_launches_per_step(sk, fac, q["slabs"]),
            "e2e": {"value": (W + K) / t_e2e, "unit": "it/s", "h2d_bytes_per_step": 8 * m / (W + K),
                    "d2h_bytes_per_step": (8 * n + 8 * (W + K + 1)) / (W + K), "solve_iters": W + K,
                    "note": "median of 3 plss_eg_solve calls from pinned host b to host x + history (from history 0)"},
            "clocks": clk.summary(), "final_hist": float(fin["hist_full"][W + K])}
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = eg_cpu_leg(s, workload_label(name), rows, sk, fac, B)
    print(json.dumps(line), flush=True)
    pkg.plss_destroy(ctx)


def eg_cpu_leg(s, label, rows, sk, fac, window_bytes, budget_s=15.0):
    """The engine oracle for a bounded number of steps from history 0; its algorithmic GB/s
    converts to it/s for the GPU's timed window (as kz_cpu_leg)."""
    from oracle import engine as oeg
    run = oeg.tri_engine if fac == "triangular" else oeg.qr_engine
    bfn = eg_bytes_per_iter if fac == "triangular" else eg_qr_bytes_per_iter
    A = s.scipy_csr()
    t0 = time.perf_counter()
    run(A, s.b, sketch=sk, maxit=5, rows=rows, seed=1)
    t1 = (time.perf_counter() - t0) / 5
    k = int(max(10, min(200, budget_s / max(t1 * 8, 1e-6))))
    t0 = time.perf_counter()
    run(A, s.b, sketch=sk, maxit=k, rows=rows, seed=1)
    t = time.perf_counter() - t0
    gbs = sum(bfn(s.m, s.n, s.nnz, h, sk) for h in range(k)) / t / 1e9
    cores = int(os.environ.get("OMP_NUM_THREADS", "0")) or os.cpu_count()
    return {"value": gbs * 1e9 / window_bytes, "unit": "it/s", "cores": cores, "kind": "oracle",
            "sample": f"{label}; the first {k} engine steps ({fac}, {sk} sketch) of the oracle in {t:.1f} s = "
                      f"{gbs:.2f} GB/s algorithmic (numpy/scipy, BLAS threads up to {cores}); it/s scaled to the "
                      f"GPU's timed window by algorithmic bytes/iter", "oracle_gbs": gbs}


if __name__ == "__main__":
    main()
