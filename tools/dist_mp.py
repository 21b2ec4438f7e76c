#!/usr/bin/env python3
"""NEXT-4, one process per GPU: the row-partitioned local method (Alg. 1 with Alg. 4/5) on N GPUs.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 --master-port P \
      tools/dist_mp.py --config 5 [--n 256] [--rule res|grad|none]

Rank l owns the slab I_l of split_rows(N, world, 256) on cuda:LOCAL_RANK.  Host plumbing only: the
workspace IPC handles and slab sizes are all-gathered over torch.distributed (gloo), then every rank calls
the same lc_dist_* entry points with its own handle (nr = 1); the kernels exchange halo rows and reductions
through peer memory.  Prints one JSON line on rank 0 (device times as the max over ranks).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import synth  # noqa: E402
from paper_2001_01158_b200 import dist as ldist  # noqa: E402
from paper_2001_01158_b200 import lc  # noqa: E402

RULES = {"res": dict(criterion=0, threshold=0, param=1e-10, expand_rounds=1, dilate_hops=0),
         "grad": dict(criterion=1, threshold=1, param=1e-4, expand_rounds=0, dilate_hops=0),
         "none": None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--s", type=int, default=10)
    ap.add_argument("--rule", default="res", choices=list(RULES))
    ap.add_argument("--align", type=int, default=256)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29571")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(local)
    sy = synth.system(args.config, args.s, n=args.n)
    R = ldist.split_rows(sy.nrows, world, args.align)
    r0, r1 = R[rank], R[rank + 1]
    rp, ci, va = ldist.slab_csr(sy.rp, sy.ci, sy.val, r0, r1)
    me = lc.DistRank(sy.nrows, r0, r1 - r0, rank, world, rp, ci, va)
    handles = ldist.exchange_handles(me.export_handle())
    me.connect(handles, ldist.exchange_sizes(r1 - r0))
    dist.barrier()
    b = torch.from_numpy(np.ascontiguousarray(sy.b[r0:r1])).cuda()
    x0 = torch.from_numpy(np.ascontiguousarray(sy.x0[r0:r1])).cuda()
    x, rep = lc.dist_local_method([me], [b], [x0], RULES[args.rule])
    flags = me.domain_flags()[0].cpu().numpy() if RULES[args.rule] is not None else np.zeros(0, np.uint8)
    idx, K = ldist.gather_omega(flags, r0) if RULES[args.rule] is not None else (None, 0)
    t = [rep["global"]["seconds"] + (rep["local"]["seconds"] if "local" in rep else 0.0)]
    ts = [None] * world
    dist.all_gather_object(ts, t[0])
    xs = [None] * world
    dist.all_gather_object(xs, x[0].cpu().numpy())
    if rank == 0:
        xg = np.concatenate(xs)
        res = float(np.linalg.norm(sy.b - _spmv(sy, xg)) / np.linalg.norm(sy.b))
        print(json.dumps(dict(config=args.config, N=sy.nrows, world=world, rule=args.rule, K=rep["K"],
                              K_gathered=K, it_local=rep.get("local", {}).get("iterations"),
                              it_global=rep["global"]["iterations"], seconds_max=max(ts),
                              rel_residual=res)))
    del me
    dist.destroy_process_group()


def _spmv(sy, x):
    y = np.zeros(sy.nrows)
    rows = np.repeat(np.arange(sy.nrows), np.diff(sy.rp))
    np.add.at(y, rows, sy.val * x[sy.ci])
    return y


if __name__ == "__main__":
    main()
