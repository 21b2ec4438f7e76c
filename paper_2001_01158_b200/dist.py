"""Host-side plumbing of the row-partitioned form (NEXT-4, Sec. 2.4 / Alg. 4-5).

The partition of P:820-858: rank l owns the contiguous row slab I_l of A, x and b.  This module holds only
bookkeeping (no arithmetic of the method): the slab split, the rank's CSR rows, the all-gather of the CUDA
IPC handles over torch.distributed (gloo or nccl), and the gather of the per-rank domain flags into the
global Omega_local (the "reduction of Omega_local and K by sum" of Alg. 4 l.15 / Alg. 5 l.11).  The
compute runs in liblc.so (lc_dist_*), see lc.DistRank.
"""
from __future__ import annotations

import numpy as np


def split_rows(n: int, nranks: int, align: int = 256):
    """Contiguous slabs [R_l, R_{l+1}) covering [0, n), as equal as possible with boundaries on multiples of
    `align` rows (whole 8-slice chunks; the paper assumes N = Nbar p).  Returns R (nranks + 1)."""
    if nranks < 1 or n < nranks:
        raise ValueError("need 1 <= nranks <= n")
    R = [0]
    for l in range(1, nranks):
        b = (n * l // nranks) // align * align
        R.append(max(b, R[-1]))
    R.append(n)
    if any(R[l + 1] <= R[l] for l in range(nranks)):
        raise ValueError(f"n = {n} too small for {nranks} slabs aligned to {align} rows")
    return R


def slab_csr(row_ptr, col_idx, values, r0: int, r1: int):
    """Rows [r0, r1) of a CSR matrix: 0-based row_ptr, GLOBAL column numbers (what lc_dist_create takes)."""
    k0, k1 = int(row_ptr[r0]), int(row_ptr[r1])
    rp = np.asarray(row_ptr[r0:r1 + 1], dtype=np.int64) - k0
    return rp, np.asarray(col_idx[k0:k1], dtype=np.int32), np.asarray(values[k0:k1], dtype=np.float64)


def stencil_reach(row_ptr, col_idx, r0: int, r1: int):
    """(-min offset, max offset) of the rows [r0, r1): how far the slab's stencil reaches into its neighbours."""
    lo = hi = 0
    for i in range(r0, r1):
        for k in range(int(row_ptr[i]), int(row_ptr[i + 1])):
            d = int(col_idx[k]) - i
            lo, hi = min(lo, d), max(hi, d)
    return -lo, hi


def exchange_handles(handle: bytes, group=None):
    """All-gather every rank's IPC handle (rank order) over torch.distributed."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(handle), group=group)
    return out


def exchange_sizes(n_local: int, group=None):
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, int(n_local), group=group)
    return out


def omega_from_flags(flags, row0: int):
    """Global ascending indices of the slab rows in Omega (flag != 255)."""
    f = np.asarray(flags)
    return (np.flatnonzero(f != 255) + row0).astype(np.int64)


def gather_omega(flags, row0: int, group=None):
    """Omega_local over all ranks, ascending (slabs ascend with the rank), and K."""
    import torch.distributed as dist
    mine = omega_from_flags(flags, row0)
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, mine, group=group)
    idx = np.concatenate(out) if out else np.zeros(0, np.int64)
    return idx, int(idx.size)
