"""The multi-GPU schedule on CPU: world_size 2 (and 3) over gloo.

Each rank owns the alpha block [blk[g], blk[g+1]) planned by the library's
own detci_gpu_plan_partition; the C blocks rotate ring-wise (send to g-1,
receive from g+1, exactly the NCCL schedule of sigma.cu:sigma_ring) and each
step adds the alpha-alpha and mixed contributions whose ket rows lie in the
resident block; beta-beta and the diagonal are block-local.  The per-element
values come from the C oracle, so this checks the decomposition and the
communication pattern, not the kernels (those are checked on the GPU with
virtual blocks).  Davidson's distributed dot products are allreduced."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.bindings import Oracle
from paper_2601_16169_b200 import detci, synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _system():
    ints = synth.synthetic_integrals(9, 6)
    strs = synth.synthetic_strings(9, 3, 48)
    return ints, strs


def _local_sigma(sysm, x_blocks, blk, g, P, hij, tables):
    """Ring-decomposed sigma for rank g; x_blocks(s) yields the resident block."""
    na, nb = sysm.na, sysm.nb
    a0, a1 = int(blk[g]), int(blk[g + 1])
    alpha, beta = sysm.alpha, sysm.beta
    sa, da, sb, db = (tables[k] for k in ((0, 0), (0, 1), (1, 0), (1, 1)))

    def row(t, i):
        f, o, l = t
        return f[int(o[i]):int(o[i]) + int(l[i])]

    y = np.zeros((a1 - a0, nb))
    for s in range(P):
        b = (g + s) % P
        b0, b1 = int(blk[b]), int(blk[b + 1])
        xb = yield b            # resident block rows [b0, b1)
        for ia in range(a0, a1):
            for ib in range(nb):
                acc = 0.0
                for ja in np.concatenate([row(sa, ia), row(da, ia)]):
                    if b0 <= ja < b1:
                        acc += hij(alpha[ia], beta[ib], alpha[ja], beta[ib]) * xb[ja - b0, ib]
                for ja in row(sa, ia):
                    if b0 <= ja < b1:
                        for jb in row(sb, ib):
                            acc += hij(alpha[ia], beta[ib], alpha[ja], beta[jb]) * xb[ja - b0, jb]
                if s == 0:      # block-local: diagonal + beta-beta
                    acc += sysm.diag[ia * nb + ib] * xb[ia - b0, ib]
                    for jb in np.concatenate([row(sb, ib), row(db, ib)]):
                        acc += hij(alpha[ia], beta[ib], alpha[ia], beta[jb]) * xb[ia - b0, jb]
                y[ia - a0, ib] += acc
    yield y


def _worker(rank, world, port, weighted, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ints, strs = _system()
        sysm = Oracle().system(ints, strs, strs, threads=1)
        tables = sysm.tables
        ls = [tables[k][2] for k in ((0, 0), (0, 1), (1, 0), (1, 1))]
        blk = detci.plan_partition(sysm.na, sysm.nb, *ls, world, weighted)
        nb = sysm.nb
        x = synth.random_vector(sysm.na * nb, 5).reshape(sysm.na, nb)
        a0, a1 = int(blk[rank]), int(blk[rank + 1])
        held = torch.from_numpy(x[a0:a1].copy())
        gen = _local_sigma(sysm, None, blk, rank, world, sysm.hij, tables)
        b = next(gen)
        for s in range(world):
            assert b == (rank + s) % world
            out = gen.send(held.numpy())
            if s + 1 < world:
                nxt = (rank + s + 1) % world
                recv = torch.empty((int(blk[nxt + 1] - blk[nxt]), nb), dtype=torch.float64)
                reqs = [dist.isend(held, (rank - 1) % world), dist.irecv(recv, (rank + 1) % world)]
                for r in reqs:
                    r.wait()
                held = recv
                b = out
        y_local = out if isinstance(out, np.ndarray) else next(gen)
        # distributed dot products as in the device Davidson (allreduce of partials)
        part = torch.tensor([float(np.dot(x[a0:a1].ravel(), y_local.ravel()))], dtype=torch.float64)
        dist.all_reduce(part)
        gathered = [None] * world
        dist.all_gather_object(gathered, (a0, a1, y_local))
        if rank == 0:
            full = np.zeros((sysm.na, nb))
            for b0, b1, yl in gathered:
                full[b0:b1] = yl
            ref = sysm.matvec(x.ravel()).reshape(sysm.na, nb)
            q.put((float(np.max(np.abs(full - ref) / np.maximum(1.0, np.abs(ref)))),
                   float(part.item()), float(np.dot(x.ravel(), ref.ravel())), list(map(int, blk))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,weighted", [(2, False), (2, True), (3, True)])
def test_ring_decomposed_sigma_matches_full(world, weighted):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, weighted, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    err, dot_dist, dot_full, blk = q.get(timeout=10)
    assert err <= 1e-12
    assert abs(dot_dist - dot_full) <= 1e-12 * max(1.0, abs(dot_full))
    assert blk[0] == 0 and blk[-1] == 48 and len(blk) == world + 1
