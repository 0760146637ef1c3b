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


def _gather_worker(rank, world, port, q):
    """The gather schedule (sigma.cu:sigma_gather_rank): allgather of the C
    row blocks; alpha-alpha, beta-beta and diagonal for the own rows with all
    of C; the mixed term for ALL alpha rows but only the own share of beta
    columns (32-aligned split as mixed_slots); the column slabs go
    all-to-all (rows of rank b to b) and are added into the own rows."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ints, strs = _system()
        sysm = Oracle().system(ints, strs, strs, threads=1)
        tables = sysm.tables
        ls = [tables[k][2] for k in ((0, 0), (0, 1), (1, 0), (1, 1))]
        blk = [int(v) for v in detci.plan_partition(sysm.na, sysm.nb, *ls, world, True)]
        na, nb = sysm.na, sysm.nb
        alpha, beta, hij = sysm.alpha, sysm.beta, sysm.hij
        sa, da, sb, db = (tables[k] for k in ((0, 0), (0, 1), (1, 0), (1, 1)))

        def row(t, i):
            f, o, l = t
            return f[int(o[i]):int(o[i]) + int(l[i])]

        x = synth.random_vector(na * nb, 5).reshape(na, nb)
        a0, a1 = blk[rank], blk[rank + 1]
        # allgather of the row blocks (padded to the largest block)
        mb = max(blk[b + 1] - blk[b] for b in range(world))
        mine = torch.zeros((mb, nb), dtype=torch.float64)
        mine[:a1 - a0] = torch.from_numpy(x[a0:a1])
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        C = np.concatenate([parts[b][:blk[b + 1] - blk[b]].numpy() for b in range(world)])
        assert np.array_equal(C, x)
        y = np.zeros((a1 - a0, nb))
        for ia in range(a0, a1):
            for ib in range(nb):
                acc = sysm.diag[ia * nb + ib] * C[ia, ib]
                for ja in np.concatenate([row(sa, ia), row(da, ia)]):
                    acc += hij(alpha[ia], beta[ib], alpha[ja], beta[ib]) * C[ja, ib]
                for jb in np.concatenate([row(sb, ib), row(db, ib)]):
                    acc += hij(alpha[ia], beta[ib], alpha[ia], beta[jb]) * C[ia, jb]
                y[ia - a0, ib] = acc
        # mixed term: all alpha rows, own beta-column share
        total = (nb + 31) // 32 * 32
        edge = [total if k == world else total * k // world // 32 * 32 for k in range(world + 1)]
        c0, c1 = edge[rank], min(edge[rank + 1], nb)
        slab = np.zeros((na, max(c1 - c0, 0)))
        for ia in range(na):
            for ib in range(c0, c1):
                acc = 0.0
                for ja in row(sa, ia):
                    for jb in row(sb, ib):
                        acc += hij(alpha[ia], beta[ib], alpha[ja], beta[jb]) * C[ja, jb]
                slab[ia, ib - c0] = acc
        send = [torch.from_numpy(np.ascontiguousarray(slab[blk[b]:blk[b + 1]])).reshape(-1) for b in range(world)]
        widths = [max(min(edge[b + 1], nb) - edge[b], 0) for b in range(world)]
        recv = [torch.empty((a1 - a0) * widths[b], dtype=torch.float64) for b in range(world)]
        # point-to-point pairs, as the grouped ncclSend/ncclRecv of the slab
        reqs = []
        for b in range(world):
            if b == rank:
                recv[b].copy_(send[b])
                continue
            if send[b].numel():
                reqs.append(dist.isend(send[b], b))
            if recv[b].numel():
                reqs.append(dist.irecv(recv[b], b))
        for r in reqs:
            r.wait()
        for b in range(world):
            if widths[b]:
                y[:, edge[b]:edge[b] + widths[b]] += recv[b].numpy().reshape(a1 - a0, widths[b])
        gathered = [None] * world
        dist.all_gather_object(gathered, (a0, a1, y))
        if rank == 0:
            full = np.zeros((na, nb))
            for b0, b1, yl in gathered:
                full[b0:b1] = yl
            ref = sysm.matvec(x.ravel()).reshape(na, nb)
            q.put(float(np.max(np.abs(full - ref) / np.maximum(1.0, np.abs(ref)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_schedule_sigma_matches_full(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    assert q.get(timeout=10) <= 1e-12
