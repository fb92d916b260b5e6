"""torchrun worker for the row-block tests.

--backend nccl : each rank solves its row block with libplss's plss_create_dist on cuda:LOCAL_RANK
                 (the NCCL unique id travels through torch.distributed).
--backend gloo : CPU-only check of the host-side plumbing and of the row-block decomposition the
                 dist ctx implements: local r_g <- r_g - A_g p, local A_g^T r_g and r_g^T r_g
                 packed into ONE (n+1) buffer, summed across ranks (gloo all_reduce), then the
                 replicated scalar tail and p/x update. Products use the oracle's SpMVs (test
                 infrastructure); the unique id from plss_get_unique_id is broadcast as in bench.py.
Rank 0 writes hist and x to --out.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import plss_gen  # noqa: E402


def gloo_solve(s, blk, dist, torch, maxit, chunks=1):
    import oracle
    n = s.n
    r = blk["b"].copy()
    nb2 = torch.tensor([float(r @ r)], dtype=torch.float64)
    dist.all_reduce(nb2)
    nbd = float(np.sqrt(nb2.item()))
    p = np.zeros(n)
    x = np.zeros(n)
    hist, theta, iters = [], 0.0, 0
    buf = torch.zeros(n + 1, dtype=torch.float64)
    while True:
        if iters > 0:
            r = r - oracle.spmv(blk["m"], blk["row_ptr"], blk["col_idx"], blk["val"], p)
        buf[:n] = torch.from_numpy(oracle.spmvT(n, blk["col_ptr"], blk["row_idx"], blk["val_t"], r))
        buf[n] = float(r @ r)
        if chunks <= 1:
            dist.all_reduce(buf)                       # the one collective per iteration
        else:                                          # the chunked variant (plss.cu make_chunks):
            bounds = [(c * (n + 1)) // chunks for c in range(chunks + 1)]   # contiguous slices of the
            for c0, c1 in zip(bounds[:-1], bounds[1:]):                    # buffer, the last one with rho
                part = buf[c0:c1].clone()
                dist.all_reduce(part)
                buf[c0:c1] = part
        y = buf[:n].numpy()
        rho = float(buf[n])
        h = np.sqrt(rho) / nbd
        hist.append(h)
        if rho == 0.0 or h <= s.tol:
            break
        phi = float(y @ y)
        if iters == 0:
            p = (rho / phi) * y
        else:
            tau = np.sqrt(theta * phi) / rho
            beta = 1.0 / ((tau - 1.0) * (tau + 1.0))
            gamma = (theta / rho) * beta
            p = beta * p + gamma * y
        theta = float(p @ p)
        x = x + p
        iters += 1
        if iters >= maxit:
            break
    return np.array(hist), x, iters


def gloo_solve_rsag(s, blk, dist, torch, maxit):
    """The reduce-scatter step's decomposition (plss.cu, options.flags bit2): y reduce-scattered to
    column shards of cnt = 32-aligned ceil(n / G) (emulated: all-reduce, keep the shard -- gloo has
    no reduce-scatter), phi / psi / theta as shard partials summed in ONE all-reduce of 4 scalars
    with the local rho, K3 on the shard, p all-gathered, x gathered at the end."""
    import oracle
    n = s.n
    G, g = dist.get_world_size(), dist.get_rank()
    cnt = -(-n // G)
    cnt = -(-cnt // 32) * 32
    c0, c1 = g * cnt, min(n, (g + 1) * cnt)
    r = blk["b"].copy()
    nb2 = torch.tensor([float(r @ r)], dtype=torch.float64)
    dist.all_reduce(nb2)
    nbd = float(np.sqrt(nb2.item()))
    p = np.zeros(G * cnt)
    x = np.zeros(G * cnt)
    hist, iters, theta_g = [], 0, 0.0
    while True:
        if iters > 0:
            r = r - oracle.spmv(blk["m"], blk["row_ptr"], blk["col_idx"], blk["val"], p[:n])
        yfull = torch.zeros(G * cnt, dtype=torch.float64)
        yfull[:n] = torch.from_numpy(oracle.spmvT(n, blk["col_ptr"], blk["row_idx"], blk["val_t"], r))
        dist.all_reduce(yfull)                           # = reduce-scatter, then keep the shard
        ysh = yfull[c0:c1].numpy()
        psh = p[c0:c1]
        sc = torch.tensor([float(r @ r), float(ysh @ ysh), float(ysh @ psh), theta_g], dtype=torch.float64)
        dist.all_reduce(sc)                              # the one scalar all-reduce
        rho, phi, theta = float(sc[0]), float(sc[1]), float(sc[3])
        h = np.sqrt(rho) / nbd
        hist.append(h)
        if rho == 0.0 or h <= s.tol:
            break
        if iters == 0:
            pn = (rho / phi) * ysh
        else:
            tau = np.sqrt(theta * phi) / rho
            beta = 1.0 / ((tau - 1.0) * (tau + 1.0))
            gamma = (theta / rho) * beta
            pn = beta * psh + gamma * ysh
        theta_g = float(pn @ pn)
        x[c0:c1] = x[c0:c1] + pn
        shard = torch.zeros(cnt, dtype=torch.float64)
        shard[:c1 - c0] = torch.from_numpy(pn)
        parts = [torch.empty(cnt, dtype=torch.float64) for _ in range(G)]
        dist.all_gather(parts, shard)                    # all-gather p
        p = torch.cat(parts).numpy()
        iters += 1
        if iters >= maxit:
            break
    xs = torch.from_numpy(np.ascontiguousarray(x[c0:c0 + cnt]) if c1 > c0 else np.zeros(cnt))
    xs = torch.cat([xs, torch.zeros(cnt - xs.numel(), dtype=torch.float64)]) if xs.numel() < cnt else xs
    parts = [torch.empty(cnt, dtype=torch.float64) for _ in range(G)]
    dist.all_gather(parts, xs)                           # x gathered at finish
    return np.array(hist), torch.cat(parts).numpy()[:n], iters


def gloo_solve_cols(s, blk, dist, torch, maxit):
    """The column-block decomposition (plss.cu enqueue_step_cols, plss_create_dist_cols): r
    replicated, x / p / y column shards. u <- u - A_g p_g (u = r on rank 0, 0 elsewhere), ONE
    all-reduce of u | theta_g gives r = r - A p and theta; rho = r^T r replicated; y_g = A_g^T r;
    phi, psi as shard partials in an all-reduce of 2; K3 on the shard; x gathered at the end."""
    import oracle
    m, n_l = s.m, blk["n"]
    G, g = dist.get_world_size(), dist.get_rank()
    b = blk["b"]
    nbd = float(np.sqrt(b @ b))
    u = b.copy() if g == 0 else np.zeros(m)
    p = np.zeros(n_l)
    x = np.zeros(n_l)
    hist, iters, theta_g = [], 0, 0.0
    while True:
        if iters > 0:
            u = u - oracle.spmv(m, blk["row_ptr"], blk["col_idx"], blk["val"], p)
        buf = torch.zeros(m + 1, dtype=torch.float64)
        buf[:m] = torch.from_numpy(u)
        buf[m] = theta_g
        dist.all_reduce(buf)                             # r = r - A p and theta, on every rank
        r = buf[:m].numpy().copy()
        theta = float(buf[m])
        rho = float(r @ r)
        h = np.sqrt(rho) / nbd
        hist.append(h)
        if rho == 0.0 or h <= s.tol:
            break
        y = oracle.spmvT(n_l, blk["col_ptr"], blk["row_idx"], blk["val_t"], r)
        sc = torch.tensor([float(y @ y), float(y @ p)], dtype=torch.float64)
        dist.all_reduce(sc)                              # phi, psi
        phi = float(sc[0])
        if iters == 0:
            p = (rho / phi) * y
        else:
            tau = np.sqrt(theta * phi) / rho
            beta = 1.0 / ((tau - 1.0) * (tau + 1.0))
            gamma = (theta / rho) * beta
            p = beta * p + gamma * y
        theta_g = float(p @ p)
        x = x + p
        u = r if g == 0 else np.zeros(m)
        iters += 1
        if iters >= maxit:
            break
    width = -(-s.n // G) + 1
    xs = torch.zeros(width, dtype=torch.float64)
    xs[:n_l] = torch.from_numpy(x)
    parts = [torch.empty(width, dtype=torch.float64) for _ in range(G)]
    dist.all_gather(parts, xs)
    bounds = [plss_gen.row_block_bounds(s.n, G, h) for h in range(G)]
    return np.array(hist), np.concatenate([parts[h][:c1 - c0].numpy() for h, (c0, c1) in enumerate(bounds)]), iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--backend", default="gloo")
    ap.add_argument("--out", required=True)
    ap.add_argument("--config", default="C2s")
    ap.add_argument("--chunks", type=int, default=1)
    ap.add_argument("--rsag", action="store_true")
    ap.add_argument("--cols", action="store_true", help="column-block partition")
    ap.add_argument("--peer", action="store_true", help="nccl backend: the peer-memory all-reduce step")
    ap.add_argument("--maxit", type=int, default=0, help="cap the config's maxit")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    s = plss_gen.make_config(args.config)
    if args.maxit > 0:
        s.maxit = min(s.maxit, args.maxit)
    blk = plss_gen.col_block(s, world, rank) if args.cols else plss_gen.row_block(s, world, rank)
    if args.backend == "gloo":
        dist.init_process_group("gloo")
        uid = None
        if rank == 0:
            import paper_2207_07615_b200 as pkg
            uid = pkg.plss_get_unique_id()
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        assert isinstance(obj[0], bytes) and len(obj[0]) == 128
        if args.cols:
            hist, x, iters = gloo_solve_cols(s, blk, dist, torch, s.maxit)
        elif args.rsag:
            hist, x, iters = gloo_solve_rsag(s, blk, dist, torch, s.maxit)
        else:
            hist, x, iters = gloo_solve(s, blk, dist, torch, s.maxit, args.chunks)
        for arr in (np.asarray(hist, dtype=np.float64), x):    # replicated decisions, bitwise (8e)
            t = torch.from_numpy(np.ascontiguousarray(arr))
            ts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(ts, t)
            assert all(torch.equal(ts[0], q) for q in ts)
    else:
        import paper_2207_07615_b200 as pkg
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = pkg.plss_get_unique_id() if rank == 0 else None
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        A = pkg.Matrix.from_arrays(blk["m"], blk["n"], blk["row_ptr"], blk["col_idx"], blk["val"],
                                   blk["col_ptr"], blk["row_idx"], blk["val_t"])
        if args.cols:
            ctx = pkg.plss_create_dist_cols(A, blk["col_offset"], s.n, obj[0], rank, world, maxit_cap=s.maxit,
                                            validate=True)
        else:
            ctx = pkg.plss_create_dist(A, blk["row_offset"], s.m, obj[0], rank, world, maxit_cap=s.maxit,
                                       validate=True, rsag=args.rsag, peer=args.peer)
        res = pkg.plss_solve(ctx, torch.from_numpy(blk["b"]).cuda(), tol=s.tol, maxit=s.maxit, want_diag=True)
        hist, x, iters = res["hist"], res["x"].cpu().numpy(), res["iters"]
        if args.cols:                                    # x is sharded by columns: gather it
            width = -(-s.n // world) + 1
            xs = torch.zeros(width, dtype=torch.float64, device="cuda")
            xs[:blk["n"]] = res["x"]
            parts = [torch.empty_like(xs) for _ in range(world)]
            dist.all_gather(parts, xs)
            x = np.concatenate([parts[h][:c1 - c0].cpu().numpy()
                                for h, (c0, c1) in enumerate(plss_gen.row_block_bounds(s.n, world, q)
                                                             for q in range(world))])
        # every rank holds the same replicated x and took the same decisions from the
        # same scalars -- rho, phi, psi, theta, tau, beta, gamma of every iteration, bitwise
        for arr in (x, res["diag"].reshape(-1)):
            t = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
            ts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(ts, t)
            assert all(torch.equal(ts[0], q) for q in ts)
        pkg.plss_destroy(ctx)
    if rank == 0:
        np.savez(args.out, hist=hist, x=x, iters=iters)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
