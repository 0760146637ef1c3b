"""The library's own multi-rank code on one GPU.

world_size handles in one process, each driven by its own host thread, form a
loopback group (detci_gpu_create_loopback): they run exactly the rank code
the NCCL transport runs -- sigma_gather_rank (Cs allgather by in-place
broadcasts, column-slab all-to-all by grouped send/recv, k_unpack_mixed),
the Cs ring (DETCI_MULTI=ring), the Davidson all-reduces and the cross-rank
argmin -- with device copies ordered by CUDA events in place of NCCL.  The
reference's multi-rank layout is the alpha-block partition of
matvec.cpp:108-111 (plan_decomposition) with the paper's MPI_Allreduce /
Mpi2dSlide exchange (PAPER.md "Mpi2dSlide").

Bars: sigma rows against the reference rows (rows_C1.npz, 1e-12), the
concatenated rank slices against the single-GPU sigma (1e-12), Davidson
energies equal to the single-GPU solve within 1e-10 and to the reference C1
energy within 1e-8.
"""
import itertools
import threading

import numpy as np
import pytest

from paper_2601_16169_b200 import detci, errors, synth
from util import GOLDEN, golden_meta, rel_diff

pytestmark = pytest.mark.gpu

_group_ids = itertools.count(1000)


def run_ranks(P, ints, a, b, body, timeout=600, **opts):
    """Build one loopback rank per thread and run body(rank, basis) on each;
    returns the per-rank results (re-raises the first rank's exception)."""
    gid = next(_group_ids)
    out = [None] * P
    errs = [None] * P

    def work(r):
        try:
            kw = dict(opts)
            per_rank = kw.pop("per_rank", {}).get(r, {})
            kw.update(per_rank)
            o = detci.BasisOptions(rank=r, world_size=P, loopback_group=gid, **kw)
            with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri, o) as basis:
                out[r] = body(r, basis)
        except BaseException as e:  # noqa: BLE001 - reported to the main thread
            errs[r] = e

    ts = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    hung = [r for r, t in enumerate(ts) if t.is_alive()]
    assert not hung, f"ranks {hung} did not finish (hang in a collective?)"
    return out, errs


def check(errs):
    for e in errs:
        if e is not None:
            raise e


@pytest.fixture(scope="module")
def c1():
    ints, a, b = synth.synthetic_system("C1")
    rows = np.load(GOLDEN / "rows_C1.npz")
    x = synth.random_vector(len(a) * len(b), 11)
    with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri) as basis:
        y1 = detci.matvec(basis, x)
    return ints, a, b, rows, x, y1


def local_slice(v, basis, nb):
    return np.ascontiguousarray(v.reshape(-1, nb)[basis.row_begin:basis.row_end].ravel())


@pytest.mark.parametrize("multi", ["gather", "ring"])
@pytest.mark.parametrize("P,weighted", [(2, False), (3, True), (8, True)])
def test_loopback_sigma_c1(c1, P, weighted, multi, monkeypatch):
    if multi == "ring":
        monkeypatch.setenv("DETCI_MULTI", "ring")
    ints, a, b, rows, x, y1 = c1
    nb = len(b)

    def body(r, basis):
        xl = local_slice(x, basis, nb)
        y = detci.matvec(basis, xl)
        y_again = detci.matvec(basis, xl)
        Y = detci.matvec_block(basis, np.stack([xl, -0.5 * xl, 2.0 * xl]))   # one pair (M = 2) + one single
        return basis.row_begin, basis.row_end, y, y_again, Y

    res, errs = run_ranks(P, ints, a, b, body, weighted_partition=weighted)
    check(errs)
    res.sort(key=lambda t: t[0])
    assert res[0][0] == 0 and res[-1][1] == len(a)
    assert all(res[i][1] == res[i + 1][0] for i in range(P - 1))
    y = np.concatenate([t[2] for t in res])
    assert rel_diff(y, y1) <= 1e-12
    rr = rows["rows"].astype(np.int64)
    assert rel_diff(y.reshape(len(a), -1)[rr], rows["sigma_rows"]) <= 1e-12
    assert all(np.array_equal(t[2], t[3]) for t in res)   # deterministic across calls
    for i, sc in enumerate((1.0, -0.5, 2.0)):
        Yi = np.concatenate([t[4][i] for t in res])
        assert rel_diff(Yi, sc * y1) <= 1e-12


@pytest.mark.parametrize("P", [2, 3])
def test_loopback_davidson_c1_equals_single_gpu(c1, P):
    """Davidson over P loopback ranks: every dot product is a per-rank
    partial plus an all-reduce, the initial guess is the cross-rank argmin of
    the diagonal; same energy as one GPU (1e-10) and as the reference C1
    pipeline (1e-8)."""
    ints, a, b, rows, x, y1 = c1
    with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri) as basis:
        one = detci.davidson_solve(basis, want_vector=False)
    res, errs = run_ranks(P, ints, a, b, lambda r, basis: detci.davidson_solve(basis), weighted_partition=True)
    check(errs)
    energies = [t.energy for t in res]
    assert all(t.converged for t in res)
    assert len(set(energies)) == 1, "ranks disagree on the energy"
    assert len({len(t.iterations) for t in res}) == 1
    assert abs(energies[0] - one.energy) <= 1e-10
    meta = golden_meta()["C1"]
    if "energy" in meta:
        assert abs(energies[0] - meta["energy"]) <= 1e-8
    # the distributed eigenvector (rank slices in rank order) is normalised
    v = np.concatenate([t.eigenvector for t in res])
    assert abs(np.linalg.norm(v) - 1.0) <= 1e-8


def test_loopback_davidson_roots(c1):
    """Block Davidson (4 roots) over 2 ranks equals one GPU."""
    ints = synth.synthetic_integrals(12, 8)
    s = synth.synthetic_strings(12, 4, 200)
    with detci.GpuBasis(ints.norbs, s, s, ints.core, ints.h1, ints.eri) as basis:
        one = detci.davidson_roots(basis, 4, want_vectors=False)
    res, errs = run_ranks(2, ints, s, s, lambda r, basis: detci.davidson_roots(basis, 4), weighted_partition=True)
    check(errs)
    assert all(t.converged for t in res)
    assert np.array_equal(res[0].energies, res[1].energies)
    assert np.max(np.abs(res[0].energies - one.energies)) <= 1e-10


def test_loopback_rank_failure_does_not_hang():
    """A capacity error on one rank (its own memory budget) fails every rank
    of the build instead of leaving the others in a collective (the
    capacity decision is an all-reduced agreement)."""
    ints = synth.synthetic_integrals(12, 8)
    s = synth.synthetic_strings(12, 4, 200)
    res, errs = run_ranks(2, ints, s, s, lambda r, basis: None, timeout=120,
                          per_rank={1: {"memory_budget_bytes": 1000}})
    assert isinstance(errs[1], errors.CapacityError)
    assert type(errs[0]) is errors.Error and "another rank failed" in str(errs[0])


def test_loopback_davidson_capacity_is_collective():
    """Davidson's subspace capacity check is decided collectively too."""
    ints = synth.synthetic_integrals(12, 8)
    s = synth.synthetic_strings(12, 4, 200)

    def body(r, basis):
        return detci.davidson_solve(basis, detci.DavidsonOptions(max_subspace=20))

    # rank 1's budget admits the basis (tens of KB) but not 43 Davidson vectors
    res, errs = run_ranks(2, ints, s, s, body, timeout=120, per_rank={1: {"memory_budget_bytes": 400_000}})
    assert isinstance(errs[1], errors.CapacityError), errs
    assert type(errs[0]) is errors.Error and "another rank failed" in str(errs[0])


@pytest.mark.parametrize("P", [2, 3])
def test_loopback_rebalance_then_sigma_and_davidson(c1, P):
    """The measured rebalance is collective (per-rank phase times are
    all-reduced, every rank cuts the same partition): after two rounds the
    ranks still tile the rows, sigma matches one GPU and the reference rows,
    and Davidson gives the single-GPU energy."""
    ints, a, b, rows, x, y1 = c1
    nb = len(b)
    with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri) as basis:
        one = detci.davidson_solve(basis, want_vector=False)

    def body(r, basis):
        before = (basis.row_begin, basis.row_end)
        ratio = basis.rebalance(2)
        y = detci.matvec(basis, local_slice(x, basis, nb))
        e = detci.davidson_solve(basis, want_vector=False).energy
        return basis.row_begin, basis.row_end, y, e, ratio, before

    res, errs = run_ranks(P, ints, a, b, body, weighted_partition=True)
    check(errs)
    res.sort(key=lambda t: t[0])
    assert res[0][0] == 0 and res[-1][1] == len(a)
    assert all(res[i][1] == res[i + 1][0] for i in range(P - 1))
    assert all(t[4] >= 1.0 for t in res) and len({t[4] for t in res}) == 1   # one agreed measurement
    y = np.concatenate([t[2] for t in res])
    assert rel_diff(y, y1) <= 1e-12
    rr = rows["rows"].astype(np.int64)
    assert rel_diff(y.reshape(len(a), -1)[rr], rows["sigma_rows"]) <= 1e-12
    assert len({t[3] for t in res}) == 1 and abs(res[0][3] - one.energy) <= 1e-10


def test_virtual_blocks_rebalance(c1):
    """Virtual blocks: the rebalance re-cuts rows and column shares from the
    per-block timings; sigma is unchanged (1e-12) for both schedules' data."""
    ints, a, b, rows, x, y1 = c1
    with detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri,
                        detci.BasisOptions(virtual_blocks=4, weighted_partition=True)) as basis:
        ratio = basis.rebalance(2)
        assert ratio >= 1.0
        y = detci.matvec(basis, x, timings={})
        assert rel_diff(y, y1) <= 1e-12
        ph = basis.rank_phase_seconds()
        assert len(ph) == 4 and all(len(r) == 4 and r[0] > 0 and r[2] > 0 for r in ph)
