#!/usr/bin/env python
"""Benchmark of the Davidson sigma build (H*C) -- the BASELINE.json metric.

    python bench.py [--gpus N --steps K --warmup W] [--config C2] [--impl reference]

One "step" is one sigma = H*C over the whole selected determinant space of
the configuration.  Default C3 = BASELINE configs[2] ([2Fe-2S]-sized: 36
orbitals, 30 e, 3e8 alpha x beta determinants), the config the metric's
"1/2/4/8 B200" sweep is quoted on; C2 (configs[1], 1e8 dets) is reported as
an extra leg.  `value` is determinants per second over all ranks (dim /
device time of one sigma, max over ranks), inputs resident in HBM; `e2e` is
the same through the public C-ABI call with page-locked host buffers (H2D of
x and D2H of y inside the timed region); `e2e_pageable` the same call with
ordinary (pageable) numpy buffers, as the reference-side caller hands them.
Inputs are larger than L2 (2.4 GB per vector at C3), so no L2 flush is
needed.

Roofline: the dominant kernel (the mixed term's scatter) is bound by the
SM's L1/shared-memory data pipe (128 B/clk/SM), not by HBM and not by the
tensor cores (FP64 gathers; ncu: tensor pipe 0%, DRAM ~0.1 of peak), so
`roofline` is stated against that pipe: achieved = the shared-memory load
bytes the plan issues per sigma (detci_gpu_sigma_plan) / the scatter
kernels' CUDA-event time.  `phases` gives every phase against its own
binding unit; `roofline_gather_model` keeps SURVEY 8(d)'s HBM gather model.

--impl reference times the reference's own CPU sigma (the unmodified detci
library compiled into oracle/_ref) on this host's cores, row-sampled
(SURVEY.md 8(d)): whole alpha rows through the reference kernels in the
reference contribution order, extrapolated by the exact per-row element
count.  Only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = json.loads((ROOT / "BASELINE.json").read_text())["metric"]
WORKLOADS = {
    "C1": "C1: N2-like synthetic, 16 orbitals 10e, 1e6 alpha x beta dets",
    "C2": "C2: N2 cc-pVDZ-sized synthetic, 26 orbitals 14e, 1e8 alpha x beta dets, single B200",
    "C3": "C3: [2Fe-2S]-sized synthetic, 36 orbitals 30e, 3e8 alpha x beta dets",
    "C4": "C4: [4Fe-4S]-sized synthetic, 36 orbitals 54e, 1e9 alpha x beta dets",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def check_world(args, world):
    """--gpus must match the launched ranks (torchrun --nproc-per-node)."""
    if args.gpus != world:
        log(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; launch N>1 as "
            f"`python -m torch.distributed.run --nproc-per-node {args.gpus} --master-addr 127.0.0.1 bench.py "
            f"--gpus {args.gpus}`")
        sys.exit(2)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.2)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
def row_work(la_s, la_d, lb_s, lb_d, nb):
    """Exact element count per alpha row (matvec.cpp loop counts)."""
    return (la_s + la_d).astype(np.float64) * nb + float((lb_s + lb_d).sum()) + la_s.astype(np.float64) * float(lb_s.sum())


def reference_cpu(cfg: str, target_seconds: float, steps: int = 1, warmup: int = 0, threads: int = 0):
    """Row-sampled reference sigma: returns (dets/s, per-step seconds, info)."""
    from oracle.bindings import RefLib
    from paper_2601_16169_b200 import synth

    ref = RefLib()
    threads = threads or ref.max_threads()
    ints, a, b = synth.synthetic_system(cfg)
    t0 = time.time()
    rt = ref.table_from_integrals(ints)
    rb = rt.basis(a, b, budget=64 << 30, workers=threads)       # reference defaults: det cache on
    build_s = time.time() - t0
    la = [rb.table(0, k)[2] for k in (0, 1)]
    lb = [rb.table(1, k)[2] for k in (0, 1)]
    work = row_work(la[0], la[1], lb[0], lb[1], len(b))
    total = float(work.sum())
    x = synth.random_vector(len(a) * len(b), 11)
    rng = np.random.default_rng(7)
    # calibrate: one row per thread
    probe = rng.choice(len(a), size=min(len(a), threads), replace=False).astype(np.uint64)
    t0 = time.time()
    rb.matvec_rows(probe, x, workers=threads)
    per_elem = (time.time() - t0) / float(work[probe.astype(np.int64)].sum())
    nrows = int(np.clip(target_seconds / (per_elem * total / len(a)), threads, len(a)))
    nrows = max(threads, (nrows // threads) * threads)
    rates, secs = [], []
    for i in range(warmup + steps):
        rows = rng.choice(len(a), size=min(nrows, len(a)), replace=False).astype(np.uint64)
        t0 = time.time()
        rb.matvec_rows(rows, x, workers=threads)
        dt = time.time() - t0
        frac = float(work[rows.astype(np.int64)].sum()) / total
        if i >= warmup:
            secs.append(dt)
            rates.append(len(a) * len(b) / (dt / frac))
    info = {"rows_per_step": int(nrows), "n_alpha": len(a), "sample_fraction": float(nrows) / len(a),
            "build_seconds": build_s, "threads": threads}
    return float(np.median(rates)), secs, info


# ---------------------------------------------------------------------------
def run_reference_arm(args):
    rank, _, world = dist_env()
    check_world(args, world)
    if rank != 0:
        return
    value, secs, info = reference_cpu(args.config, args.ref_seconds, steps=args.steps, warmup=args.warmup)
    cores = info["threads"]
    sample = (f"{info['rows_per_step']} of {info['n_alpha']} alpha rows x all beta per step "
              f"({100 * info['sample_fraction']:.2f}%), reference hij_words in matvec.cpp order, "
              f"extrapolated by exact per-row element counts")
    line = {
        "metric": METRIC, "value": value, "unit": "dets/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(secs) if secs else None,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": WORKLOADS.get(args.config, args.config), "config": args.config,
                   "reference": "unmodified detci (proj/core) built from /root/reference into oracle/_ref",
                   "ms_per_step_is": "wall time of one row-sampled step (the sample, not a full sigma)"},
        "cpu_baseline": {"value": value, "unit": "dets/s", "cores": cores, "kind": "reference", "sample": sample,
                         "cpu_model": cpu_model(), "host_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": "dets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_gpu_arm(args):
    import torch

    from paper_2601_16169_b200 import _lib, detci, synth

    rank, local_rank, world = dist_env()
    check_world(args, world)
    torch.cuda.set_device(local_rank)
    lib = _lib.load()
    nccl_id = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        obj = [None]
        if rank == 0:
            buf = (C.c_uint8 * 128)()
            assert lib.detci_gpu_nccl_unique_id(buf) == 0
            obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        import torch.distributed as dist

        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def open_basis(cfg):
        t_build = time.time()
        ints, a, b = synth.synthetic_system(cfg)
        opts = detci.BasisOptions(device=local_rank, rank=rank, world_size=world, nccl_id=nccl_id,
                                  weighted_partition=world > 1)
        basis = detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri, opts)
        if world > 1:
            # measured rebalance of the row blocks and column shares
            # (detci_gpu_rebalance, collective), part of the build
            basis.balance_before = basis.rebalance(2)
        return ints, a, b, basis, time.time() - t_build

    def measure(cfg, basis, na, nb, steps, warmup, with_clocks=False, pageable=False):
        """value (device-resident), phase split, e2e through detci_gpu_sigma
        with pinned (and optionally pageable) host buffers."""
        dim = na * nb
        r0, r1 = basis.row_begin, basis.row_end
        x_full = synth.random_vector(dim, 11)
        x_loc = np.ascontiguousarray(x_full.reshape(na, nb)[r0:r1].ravel())
        del x_full
        dx = torch.from_numpy(x_loc).cuda()
        dy = torch.empty_like(dx)
        sp = C.c_void_p()
        assert lib.detci_gpu_stream(basis.handle, C.byref(sp)) == 0
        ext = torch.cuda.ExternalStream(sp.value, device=torch.device("cuda", local_rank))

        def sigma_async():
            code = lib.detci_gpu_sigma_async(basis.handle, dx.data_ptr(), dy.data_ptr())
            if code:
                raise RuntimeError(lib.detci_gpu_last_error(basis.handle).decode())

        for _ in range(warmup):
            sigma_async()
        ext.synchronize()
        sampler = ClockSampler(local_rank) if with_clocks else None
        if sampler:
            sampler.start()
        barrier()
        cnt0 = C.c_uint64()
        lib.detci_gpu_launch_count(C.byref(cnt0))
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(ext)
        for _ in range(steps):
            sigma_async()
        end.record(ext)
        end.synchronize()
        cnt1 = C.c_uint64()
        lib.detci_gpu_launch_count(C.byref(cnt1))
        barrier()
        clocks = sampler.stop() if sampler else None
        per_step = max_over_ranks(start.elapsed_time(end) * 1e-3) / steps
        out = {"value": dim / per_step, "ms_per_step": per_step * 1e3, "launches": int(cnt1.value - cnt0.value),
               "clocks": clocks}

        # per-phase split (CUDA events around each phase on the same stream)
        keys = ["alpha_seconds", "beta_seconds", "mixed_seconds", "mixed_reduce_seconds", "combine_seconds",
                "total_seconds"]
        parts = {k: [] for k in keys}
        for _ in range(min(3, steps)):
            tm = _lib.Timings()
            assert lib.detci_gpu_sigma_device(basis.handle, dx.data_ptr(), dy.data_ptr(), C.byref(tm)) == 0
            for k in keys:
                parts[k].append(getattr(tm, k))
        out["split"] = {k: max_over_ranks(float(np.mean(v))) for k, v in parts.items()}

        # parity spot check against the committed reference rows
        errs = []
        for name in (f"rows_{cfg}.npz", f"rows_{cfg}_interior.npz"):
            golden = ROOT / "tests" / "golden" / name
            if golden.exists():
                g = np.load(golden)
                y = dy.cpu().numpy().reshape(r1 - r0, nb)
                errs += [float(np.max(np.abs(y[int(r) - r0] - g["sigma_rows"][i]) /
                                      np.maximum(1.0, np.maximum(np.abs(y[int(r) - r0]), np.abs(g["sigma_rows"][i])))))
                         for i, r in enumerate(g["rows"]) if r0 <= int(r) < r1]
        out["parity_rows_max_rel_err"] = max(errs) if errs else None
        out["parity_rows_checked"] = len(errs)

        # end to end: the public C-ABI call with host buffers
        def e2e(hx, hy):
            assert lib.detci_gpu_sigma(basis.handle, hx, hy, None) == 0   # warm
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ext)
            for _ in range(steps):
                assert lib.detci_gpu_sigma(basis.handle, hx, hy, None) == 0
            e1.record(ext)
            e1.synchronize()
            t = max_over_ranks(e0.elapsed_time(e1) * 1e-3) / steps
            barrier()
            return {"value": dim / t, "unit": "dets/s", "h2d_bytes_per_step": 8 * x_loc.size,
                    "d2h_bytes_per_step": 8 * x_loc.size, "ms_per_step": t * 1e3}

        hx = torch.from_numpy(x_loc).pin_memory()
        hy = torch.empty_like(hx).pin_memory()
        out["e2e"] = e2e(hx.data_ptr(), hy.data_ptr())
        out["e2e"]["buffers"] = "page-locked (torch pin_memory)"
        del hx, hy
        if pageable:
            py = np.empty_like(x_loc)
            out["e2e_pageable"] = e2e(x_loc.ctypes.data, py.ctypes.data)
            out["e2e_pageable"]["buffers"] = "pageable numpy arrays (the reference caller's std::vector)"
            del py
        out["tensors"] = (dx, dy, ext, x_loc)
        return out

    ints, a, b, basis, build_s = open_basis(args.config)
    na, nb = len(a), len(b)
    dim = na * nb
    nnz = basis.nnz()
    r0, r1 = basis.row_begin, basis.row_end
    dim_loc = (r1 - r0) * nb
    main = measure(args.config, basis, na, nb, args.steps, args.warmup, with_clocks=True, pageable=True)
    dx, dy, ext, x_loc = main.pop("tensors")
    split = main["split"]
    per_step = main["ms_per_step"] * 1e-3

    # ---- roofline per phase, each against its binding unit
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s (B200_PROFILING.md)"
    nsm = torch.cuda.get_device_properties(local_rank).multi_processor_count
    sm_mhz = (main["clocks"] or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    pipe_peak = nsm * 128.0 * sm_mhz * 1e6 / 1e9     # GB/s: L1/shared data pipe, 128 B/clk/SM
    pipe_src = f"{nsm} SMs x 128 B/clk x {sm_mhz:.0f} MHz (median SM clock during the timed region)"
    plan = basis.sigma_plan()
    nflat = {}
    for ch in (0, 1):
        for kind in (0, 1):
            v = C.c_uint64()
            assert lib.detci_gpu_helper_size(basis.handle, ch, kind, C.byref(v)) == 0
            nflat[(ch, kind)] = v.value
    frac_loc = dim_loc / dim
    # same-spin: per element one 8-byte Cs load through L1, plus the 8-byte J
    # load of a single's spectator term
    alpha_bytes = 8.0 * (2 * nflat[(0, 0)] + nflat[(0, 1)]) * nb * frac_loc
    beta_bytes = 8.0 * (2 * nflat[(1, 0)] + nflat[(1, 1)]) * na * frac_loc
    scatter_s = split["mixed_seconds"] - split["mixed_reduce_seconds"]
    reduce_s = split["mixed_reduce_seconds"]
    mixed_lds = float(plan["mixed_lds_bytes"]) * frac_loc
    d_read = float(plan["d_read_bytes"]) * frac_loc + 16.0 * dim_loc
    ncu = {}
    ncu_path = ROOT / "profiles" / "ncu_summary.json"
    if ncu_path.exists():
        ncu = json.loads(ncu_path.read_text()).get(args.config, {})

    def ncu_dram(prefix):
        vals = [v.get("dram_bytes") for k, v in ncu.items() if k.startswith(prefix)]
        vals = [x for x in vals if x is not None and x == x]
        return float(sum(vals)) if vals else None

    def phase(bound, nbytes, secs, peak, unit_note):
        ach = nbytes / secs / 1e9 if secs > 0 else None
        return {"bound": bound, "bytes": nbytes, "seconds": secs, "achieved_GBps": ach, "peak_GBps": peak,
                "frac": ach / peak if ach else None, "bytes_are": unit_note}

    phases = {
        "alpha": phase("l1", alpha_bytes, split["alpha_seconds"], pipe_peak,
                       "L1 load bytes: 8 B Cs per element (+8 B J per single)"),
        "beta": phase("l1", beta_bytes, split["beta_seconds"], pipe_peak,
                      "L1 load bytes on Cs^T: 8 B per element (+8 B J per single)"),
        "mixed_scatter": phase("smem", mixed_lds, scatter_s, pipe_peak,
                               "shared-memory load bytes issued: K V gathers + 1 Cs gather per SELL entry and pass"),
        "mixed_reduce": phase("hbm", d_read, reduce_s, hbm_peak, "D partial rows read + sigma read-modify-write"),
    }
    scatter_traffic = ncu_dram("k_mixed_scatter") if world == 1 else None
    main_kernel = max((k for k in ncu if k.startswith("k_mixed_scatter")), key=lambda k: ncu[k].get("duration") or 0.0,
                      default=f"k_mixed_scatter<{plan['mixed_kmax']}, 1>")
    roofline = {
        "bound": "smem", "kernel": main_kernel, "achieved": phases["mixed_scatter"]["achieved_GBps"],
        "peak": pipe_peak, "unit": "GB/s", "frac": phases["mixed_scatter"]["frac"],
        "traffic": scatter_traffic, "algorithmic_bytes": mixed_lds, "peak_source": pipe_src,
        "binding_unit": "L1/shared-memory data pipe (128 B/clk/SM); not HBM, not tensor (FP64 gathers)",
        "traffic_source": "dram__bytes_read+write of the scatter launch(es), profiles/ncu_summary.json "
                          f"[{args.config}] (ncu --set full, one capture)",
        "hbm": {"dram_GBps": scatter_traffic / scatter_s / 1e9 if scatter_traffic and scatter_s > 0 else None,
                "frac_of_hbm": scatter_traffic / scatter_s / 1e9 / hbm_peak if scatter_traffic and scatter_s > 0
                else None, "peak": hbm_peak, "peak_source": hbm_src},
        "smem_pipe_ncu": ({"kernel": main_kernel, "wavefront_pct_of_peak": ncu[main_kernel].get("smem_wavefront_pct"),
                           "wavefronts_per_lds": ncu[main_kernel].get("smem_wavefronts_per_ld")}
                          if main_kernel in ncu else None),
        "plan": plan,
    }
    gather_bytes = 8.0 * nnz["total"] + 24.0 * dim                             # SURVEY.md 8(d) gather model
    roofline_gather_model = {"bytes_per_sigma": gather_bytes, "achieved": gather_bytes / per_step / 1e9,
                             "unit": "GB/s", "frac_of_hbm": gather_bytes / per_step / 1e9 / hbm_peak,
                             "note": "SURVEY 8(d): 8 B per structural nonzero + 24 B/det as if every gather came "
                                     "from HBM; > 1 because the gathers are served on chip"}

    def optional(fn):
        """Run an optional single-GPU leg; its failure is reported in the
        line instead of losing the line."""
        try:
            return fn()
        except Exception as e:   # noqa: BLE001
            return {"error": f"{type(e).__name__}: {e}"}

    # ---- blocked sigma over 4 vectors (the multi-root Davidson's block)
    def blocked_leg():
        mvec = args.block
        xs = [dx] + [torch.from_numpy(synth.random_vector(dim_loc, 40 + i)).cuda() for i in range(mvec - 1)]
        ys = [torch.empty_like(dx) for _ in range(mvec)]
        px = (C.c_void_p * mvec)(*[t.data_ptr() for t in xs])
        py = (C.c_void_p * mvec)(*[t.data_ptr() for t in ys])
        pxp, pyp = C.cast(px, C.POINTER(C.c_void_p)), C.cast(py, C.POINTER(C.c_void_p))
        assert lib.detci_gpu_sigma_block(basis.handle, pxp, pyp, mvec) == 0     # warm (builds the M-table)
        b0e, b1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nrep = max(1, min(3, args.steps))
        b0e.record(ext)
        for _ in range(nrep):
            assert lib.detci_gpu_sigma_block(basis.handle, pxp, pyp, mvec) == 0
        b1e.record(ext)
        b1e.synchronize()
        per_block = b0e.elapsed_time(b1e) * 1e-3 / nrep
        out = {"vectors": mvec, "seconds_per_block": per_block, "seconds_per_vector": per_block / mvec,
               "dets_per_s_per_vector": dim * mvec / per_block, "speedup_vs_single": per_step * mvec / per_block}
        del xs, ys
        return out

    blocked = optional(blocked_leg) if args.block > 1 and world == 1 else None

    # ---- full Davidson (s/iter of the whole solver) on the same basis
    dav = None
    if args.davidson:
        res = detci.davidson_solve(basis, detci.DavidsonOptions(max_iter=args.davidson_iters), want_vector=False)
        its = res.iterations
        dav = {"status": res.status, "iterations": len(its), "seconds": res.seconds,
               "s_per_iter": res.seconds / max(1, len(its)), "energy": res.energy,
               "sigma_share": sum(i.matvec_seconds for i in its) / res.seconds,
               "vector_ops_s_per_iter": sum(i.orthogonalization_seconds for i in its) / max(1, len(its))}

    # ---- multi-root block Davidson (config C5's capability: 4 roots, blocked
    # sigma over vector pairs) on the same basis, a bounded number of
    # iterations; s/iter of the whole solver
    def roots_leg():
        rr = detci.davidson_roots(basis, args.roots, max_iter=args.roots_iters, want_vectors=False)
        nit = max(1, len(rr.iterations))
        return {"nroots": args.roots, "status": rr.status, "iterations": len(rr.iterations),
                "seconds": rr.seconds, "s_per_iter": rr.seconds / nit,
                "energies": [float(e) for e in rr.energies],
                "sigma_share": sum(i.matvec_seconds for i in rr.iterations) / max(rr.seconds, 1e-30)}

    roots = optional(roots_leg) if args.davidson and args.roots > 0 and world == 1 else None
    del dx, dy
    basis.close()
    torch.cuda.empty_cache()

    # ---- extra configs (C2 = BASELINE configs[1]): value and e2e
    extra = {}
    for cfg in [c for c in args.extra.split(",") if c and c != args.config]:
        def extra_leg(cfg=cfg):
            _, ea, eb, eb_basis, ebuild = open_basis(cfg)
            try:
                m = measure(cfg, eb_basis, len(ea), len(eb), args.steps, args.warmup)
                m.pop("tensors")
                return {"workload": WORKLOADS.get(cfg, cfg), "value": m["value"], "unit": "dets/s",
                        "ms_per_step": m["ms_per_step"], "e2e": m["e2e"], "phase_seconds": m["split"],
                        "parity_rows_max_rel_err": m["parity_rows_max_rel_err"], "build_seconds": ebuild}
            finally:
                eb_basis.close()
                torch.cuda.empty_cache()

        extra[cfg] = optional(extra_leg)

    # ---- full Davidson to convergence at C1 ("full-Davidson
    # wall time at C1"), energy against the reference pipeline's golden
    def c1_leg():
        ints1, a1, b1 = synth.synthetic_system("C1")
        with detci.GpuBasis(ints1.norbs, a1, b1, ints1.core, ints1.h1, ints1.eri,
                            detci.BasisOptions(device=local_rank)) as basis1:
            detci.davidson_solve(basis1, detci.DavidsonOptions(max_iter=2), want_vector=False)   # warm
            t1 = time.time()
            r1_ = detci.davidson_solve(basis1, want_vector=False)
            wall1 = time.time() - t1
            # stored-matrix method at C1 (Method::Stored):
            # CSR build and SpMV on device buffers; the SpMV is HBM-bound at
            # 12 B per nonzero + 24 B per row
            stored_c1 = None
            if args.stored:
                try:
                    tb = time.time()
                    sm = detci.build_stored_matrix(basis1, 0)
                    build_st = time.time() - tb
                    d1 = basis1.dimension()
                    sx = torch.from_numpy(synth.random_vector(d1, 11)).cuda()
                    sy = torch.empty_like(sx)
                    sm.use(True)
                    tms = []
                    for _ in range(6):
                        tmc = _lib.Timings()
                        assert lib.detci_gpu_sigma_device(basis1.handle, sx.data_ptr(), sy.data_ptr(), C.byref(tmc)) == 0
                        tms.append(tmc.total_seconds)
                    tfree = _lib.Timings()
                    sm.use(False)
                    assert lib.detci_gpu_sigma_device(basis1.handle, sx.data_ptr(), sy.data_ptr(), C.byref(tfree)) == 0
                    t_sp = float(np.median(tms[1:]))
                    bytes_sp = 12.0 * sm.nonzero_count() + 24.0 * d1
                    stored_c1 = {"nnz": sm.nonzero_count(), "build_seconds": build_st, "spmv_seconds": t_sp,
                                 "spmv_GBps": bytes_sp / t_sp / 1e9, "spmv_frac_of_hbm": bytes_sp / t_sp / 1e9 / hbm_peak,
                                 "matrix_free_sigma_seconds": tfree.total_seconds}
                    sm.release()
                    del sx, sy
                except Exception as e:   # noqa: BLE001 -- reported, not fatal
                    stored_c1 = {"error": str(e)}
        ref_e = None
        gpath = ROOT / "tests" / "golden" / "golden.json"
        if gpath.exists():
            ref_e = json.loads(gpath.read_text()).get("C1", {}).get("energy")
        return {"status": r1_.status, "iterations": len(r1_.iterations), "seconds": wall1, "energy": r1_.energy,
                "stored_matrix": stored_c1,
                "reference_energy": ref_e, "abs_err_vs_reference": abs(r1_.energy - ref_e) if ref_e else None,
                "reference_seconds_8core_container": json.loads(gpath.read_text()).get("C1", {}).get("davidson_seconds")
                if gpath.exists() else None}

    dav_c1 = optional(c1_leg) if args.davidson and world == 1 else None

    # ---- CPU baseline (reference on this host), rank 0 at N=1 only
    cpu = None
    if rank == 0 and world == 1 and args.cpu_baseline:
        try:
            v, secs, info = reference_cpu(args.config, args.ref_seconds, steps=1)
            cpu = {"value": v, "unit": "dets/s", "cores": info["threads"], "kind": "reference",
                   "cpu_model": cpu_model(), "host_cpus": os.cpu_count(),
                   "sample": f"{info['rows_per_step']} of {info['n_alpha']} alpha rows x all beta "
                             f"({100 * info['sample_fraction']:.2f}%) through the unmodified reference "
                             f"kernels, extrapolated by exact element counts; {secs[0]:.1f} s"}
        except Exception as exc:   # reference library missing on this box
            cpu = {"value": None, "unit": "dets/s", "cores": os.cpu_count(), "kind": "reference",
                   "cpu_model": cpu_model(), "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": main["value"], "unit": "dets/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": main["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS.get(args.config, args.config), "config": args.config,
                       "norbs": ints.norbs, "n_electrons": ints.nelec, "n_alpha": na, "n_beta": nb, "dim": dim,
                       "nnz_offdiag": nnz["total"], "nnz_alpha": nnz["alpha"], "nnz_beta": nnz["beta"],
                       "nnz_mixed": nnz["mixed"], "l2": "inputs larger than L2 (x, y = 8*dim bytes each)",
                       "parallelism": (f"alpha-block ring x{world} (NCCL send/recv)"
                                       if os.environ.get("DETCI_MULTI") == "ring" else
                                       f"alpha blocks x{world}: NCCL allgather of C, beta-column share of the "
                                       f"mixed term, point-to-point exchange; measured rebalance, 2 rounds") if world > 1 else "single GPU",
                       "build_seconds": build_s, "sigma_s_per_iter": per_step,
                       "phase_seconds": split, "parity_rows_max_rel_err": main["parity_rows_max_rel_err"],
                       "parity_rows_checked": main["parity_rows_checked"]},
            "roofline": roofline,
            "phases": phases,
            "roofline_gather_model": roofline_gather_model,
            "cpu_baseline": cpu,
            "e2e": main["e2e"],
            "e2e_pageable": main.get("e2e_pageable"),
            "gpu_launches": main["launches"],
            "clocks": main["clocks"],
            "extra_configs": extra,
            "davidson": dav,
            "davidson_c1_full": dav_c1,
            "davidson_roots": roots,
            "blocked_sigma": blocked,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(WORKLOADS))
    ap.add_argument("--extra", default="C2", help="comma list of extra configs timed after the main one ('' = none)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-seconds", type=float, default=8.0, help="target CPU seconds per reference sample")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-davidson", dest="davidson", action="store_false")
    ap.add_argument("--no-stored", dest="stored", action="store_false", help="skip the C1 stored-matrix leg")
    ap.add_argument("--roots", type=int, default=4, help="multi-root block Davidson leg (0 = skip)")
    ap.add_argument("--roots-iters", type=int, default=10)
    ap.add_argument("--block", type=int, default=4, help="vectors in the blocked-sigma measurement (0 = skip)")
    ap.add_argument("--davidson-iters", type=int, default=30,
                    help="Davidson iterations timed for s/iter (reference defaults otherwise)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        log("bench: warmup raised to 3 (timing rules)")
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
