"""Distributed PLSS solve, one process per GPU (launch with torchrun):

    python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \\
        --master-port 29500 examples/dist_solve.py [--partition rows|cols] [--step allreduce|rsag|peer]

Each rank builds its block of a seeded synthetic system (plss_gen), creates a distributed ctx over
its own NCCL communicator (the unique id travels through torch.distributed), solves, and rank 0
prints the iteration count, the residual and the true residual. Row blocks replicate x; column
blocks return each rank's shard of x, gathered here.
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2207_07615_b200 as plss  # noqa: E402
import plss_gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2s")
    ap.add_argument("--partition", default="rows", choices=["rows", "cols"])
    ap.add_argument("--step", default="allreduce", choices=["allreduce", "rsag", "peer"])
    ap.add_argument("--tol", type=float, default=1e-8)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    s = plss_gen.make_config(args.config)
    uid = [plss.plss_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    if args.partition == "rows":
        blk = plss_gen.row_block(s, world, rank)
        A = plss.Matrix.from_arrays(blk["m"], s.n, blk["row_ptr"], blk["col_idx"], blk["val"],
                                    blk["col_ptr"], blk["row_idx"], blk["val_t"])
        ctx = plss.plss_create_dist(A, blk["row_offset"], s.m, uid[0], rank, world, maxit_cap=s.maxit,
                                    rsag=args.step == "rsag", peer=args.step == "peer")
    else:
        blk = plss_gen.col_block(s, world, rank)
        A = plss.Matrix.from_arrays(s.m, blk["n"], blk["row_ptr"], blk["col_idx"], blk["val"],
                                    blk["col_ptr"], blk["row_idx"], blk["val_t"])
        ctx = plss.plss_create_dist_cols(A, blk["col_offset"], s.n, uid[0], rank, world, maxit_cap=s.maxit)
    b = torch.from_numpy(blk["b"]).cuda()
    res = plss.plss_solve(ctx, b, tol=args.tol, maxit=s.maxit)
    tr = plss.plss_true_residual(ctx, b, res["x"])           # collective
    x = res["x"]
    if args.partition == "cols":                             # gather the column shards
        width = -(-s.n // world) + 1
        xs = torch.zeros(width, dtype=torch.float64, device="cuda")
        xs[:blk["n"]] = x
        parts = [torch.empty_like(xs) for _ in range(world)]
        dist.all_gather(parts, xs)
        bounds = [plss_gen.row_block_bounds(s.n, world, h) for h in range(world)]
        x = torch.cat([parts[h][:c1 - c0] for h, (c0, c1) in enumerate(bounds)])
    if rank == 0:
        print(f"{args.config} {args.partition}/{args.step} on {world} GPU(s): {res['outcome']} after "
              f"{res['iters']} iterations, recursive residual {res['hist'][res['iters']]:.3e}, true residual "
              f"{tr['rel']:.3e}, |x| = {float(torch.linalg.norm(x)):.6f}", flush=True)
    plss.plss_destroy(ctx)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
