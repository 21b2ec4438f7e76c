"""NEXT-4 host logic on CPU (no GPU): the row partition of Sec. 2.4, the rank's CSR rows, the
stencil reach that bounds the halo, and the two-rank (gloo) plumbing a one-process-per-GPU run uses: the
all-gather of the workspace IPC handles and slab sizes, and the gather of the per-rank domain flags into
Omega_local ("reduction of Omega_local and K by sum", Alg. 4 l.15 / Alg. 5 l.11) - checked against the
oracle's Omega on the whole matrix."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
import synth
from paper_2001_01158_b200 import dist as ldist


def test_split_rows_covers_aligned_contiguous():
    for n, p, al in [(4096, 1, 32), (4096, 3, 32), (16777216, 8, 256), (8000, 4, 32), (1000, 7, 1)]:
        R = ldist.split_rows(n, p, al)
        assert R[0] == 0 and R[-1] == n and len(R) == p + 1
        assert all(R[l + 1] > R[l] for l in range(p))
        assert all(R[l] % al == 0 for l in range(p))
        sizes = np.diff(R)
        assert sizes.max() - sizes.min() <= 2 * al


def test_split_rows_rejects_too_small():
    with pytest.raises(ValueError):
        ldist.split_rows(100, 4, 64)
    with pytest.raises(ValueError):
        ldist.split_rows(3, 4, 1)


def test_slab_csr_reassembles_the_matrix():
    sy = synth.system(1, 0)
    R = ldist.split_rows(sy.nrows, 3, 32)
    parts = [ldist.slab_csr(sy.rp, sy.ci, sy.val, R[l], R[l + 1]) for l in range(3)]
    rp = [0]
    for p_rp, _, _ in parts:
        rp.extend((p_rp[1:] + rp[-1]).tolist())
    np.testing.assert_array_equal(np.array(rp), sy.rp)
    np.testing.assert_array_equal(np.concatenate([p[1] for p in parts]), sy.ci)
    np.testing.assert_array_equal(np.concatenate([p[2] for p in parts]), sy.val)
    for p_rp, _, _ in parts:
        assert p_rp[0] == 0


def test_stencil_reach_closed_forms():
    sy = synth.system(1, 0)                        # 64 x 64 five-point: reach 64 rows both ways
    assert ldist.stencil_reach(sy.rp, sy.ci, 0, sy.nrows) == (64, 64)
    sy = synth.system(5, 0, n=12)                  # 12^3 seven-point: reach 144
    assert ldist.stencil_reach(sy.rp, sy.ci, 0, sy.nrows) == (144, 144)
    assert ldist.stencil_reach(sy.rp, sy.ci, 0, 1) == (0, 144)   # first row: no lower neighbours


def test_omega_from_flags():
    f = np.array([255, 0, 255, 1, 2, 255], np.uint8)
    np.testing.assert_array_equal(ldist.omega_from_flags(f, 100), [101, 103, 104])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sy = synth.system(5, 3, n=16)
    A = orc.Csr(sy.rp, sy.ci, sy.val)
    R = ldist.split_rows(sy.nrows, world, 32)
    r0, r1 = R[rank], R[rank + 1]
    # the rank's flags: the oracle's Omega (whole matrix) restricted to the slab, encoded as lc_dist flags
    d = orc.select_domain(A, sy.b, sy.x0, 0, 0, 1e-10, 1, 0, 1)
    flags = np.where(d.flag[r0:r1] != 0, 0, 255).astype(np.uint8)
    idx, K = ldist.gather_omega(flags, r0)
    handle = bytes([rank + 1]) * 64                 # stand-in for a CUDA IPC handle
    hs = ldist.exchange_handles(handle)
    ns = ldist.exchange_sizes(r1 - r0)
    reach = ldist.stencil_reach(sy.rp, sy.ci, r0, r1)
    if rank == 0:
        out.put((idx, K, d.idx, hs, ns, R, reach))
    dist.destroy_process_group()


def test_two_rank_handle_exchange_and_omega_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    idx, K, oracle_idx, hs, ns, R, reach = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_array_equal(idx, oracle_idx)
    assert K == oracle_idx.size
    assert hs == [bytes([1]) * 64, bytes([2]) * 64]
    assert ns == [R[1] - R[0], R[2] - R[1]]
    assert all(n >= reach[1] for n in ns)            # every slab covers the stencil reach (halo check)
