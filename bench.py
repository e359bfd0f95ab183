"""Benchmark of the B200 POD-augmented CG hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--systems P] [--mode cg|fom]

Workload (BASELINE configs[2], the north-star sequence): Q1
hexahedral linear elasticity on 64^3 elements (N = 811,200, nnz =
63,695,790), 40 systems with drifting moduli and a rotating traction, Jacobi,
rtol 1e-5, POD basis <= 60 (pod-a-rbf, storage_cap = max_dim = 60,
nu_w = 1), CG recurrence. Seeded synthetic inputs with those shapes stand in
for the paper's unavailable Sierra matrices.

One step = one full sequence solve (all P systems through run_sequence).
``value`` is the device-resident sequence time (all matrices and right-hand
sides already in HBM); ``e2e`` is the same through the public API from host
CSR arrays (values + rhs H2D and every solution D2H inside the timed region).
Inputs (780 MB of CSR per SpMV) exceed L2, so no flush is needed.

``--impl reference`` times the CPU oracle port (the reference is pure Python,
so there is nothing to compile into oracle/_ref) on a bounded sample and
scales it to the same metric with the iteration schedule of the GPU run.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import subprocess
import sys
import threading
import time
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
warnings.simplefilter("ignore")

METRIC = "sequence solve time"
UNIT = "s"
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary_r02.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--systems", type=int, default=40)
    ap.add_argument("--mode", default="cg", choices=["cg", "fom"])
    ap.add_argument("--grid", type=int, default=64)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="c3", choices=["c3", "c1", "c2", "c4", "c5"],
                    help="c3 (default, the north-star sequence), c1 (64x64 Poisson, latency-bound), "
                         "c2 (128^3 diffusion sequence), "
                         "c4 (128x128x64 dynamic elasticity, snapshot to ~3000), c5 (POD truncation microbench)")
    ap.add_argument("--m", type=int, default=2048, help="c5: snapshot columns")
    args = ap.parse_args()
    if args.workload == "c2" and args.systems == 40:
        args.systems = 30
    if args.workload == "c1" and args.systems == 40:
        args.systems = 20
    if args.workload == "c4" and args.systems == 40:
        args.systems = 60
    return args


# BASELINE configs[1] (C2) and configs[2] (C3): sequence workloads
WORKLOADS = {
    "c3": {"rtol": 1e-5, "cap": 60, "data": "synthetic (seeded C3 generator, BASELINE configs[2] shapes)",
           "l2": "inputs larger than L2 (552 MB of 3x3-block matrix streamed per SpMV, 20 GB of matrices); no flush"},
    "c1": {"rtol": 1e-6, "cap": 20, "data": "synthetic (seeded C1 recipe, BASELINE configs[0])",
           "l2": "latency-bound: the 324 KB matrix and every vector stay in L2 (reported as us per iteration)"},
    "c2": {"rtol": 1e-4, "cap": 40, "data": "synthetic (seeded C2 generator, BASELINE configs[1] shapes)",
           "l2": "inputs larger than L2 (175 MB of CSR streamed per SpMV, 3.5 GB of matrices); no flush"},
    # C4: the snapshot accumulates Krylov vectors up to the storage cap (SURVEY 8d flags cap ~ 3000 as a
    # builder's choice); every accumulated column is a stage-1 column (nu_w = 1), max_dim 60 after truncation
    "c4": {"rtol": 1e-6, "cap": 3000, "max_dim": 60,
           "data": "synthetic (seeded C4 generator: K + M/dt^2, dt = 0.05, seeded load history; BASELINE configs[3])",
           "l2": "inputs larger than L2 (2.2 GB of 3x3-block matrix streamed per SpMV); no flush"},
}


def make_sequence(args, seed_offset=0, p=None):
    from paper_1512_05820_b200.problems import diffusion3d_sequence, elasticity_sequence

    p = args.systems if p is None else p
    if args.workload == "c1":
        from paper_1512_05820_b200.problems import poisson2d_sequence

        return poisson2d_sequence(64, p=p, rtol=1e-6, seed=0 + seed_offset)
    if args.workload == "c2":
        return diffusion3d_sequence(128, p=p, rtol=1e-4, seed=2 + seed_offset)
    if args.workload == "c4":
        return elasticity_sequence((128, 128, 64), p=p, rtol=1e-6, seed=4 + seed_offset, dynamic=True, dt=0.05)
    return elasticity_sequence((args.grid,) * 3, p=p, rtol=1e-5, seed=3 + seed_offset)


def workload_config(args, n=None, nnz=None):
    w = WORKLOADS[args.workload]
    name = {"c1": f"C1 2-D Poisson 64x64, {args.systems}-system recycled sequence",
            "c2": f"C2 variable-coefficient diffusion 128^3, {args.systems}-system recycled sequence",
            "c4": f"C4 Q1 elasticity 128x128x64 elements, K + M/dt^2, {args.systems}-system recycled sequence",
            }.get(args.workload, f"C3 Q1 elasticity {args.grid}^3 elements, {args.systems}-system recycled sequence")
    return {
        "workload": name,
        "systems": args.systems,
        "n": n,
        "nnz": nnz,
        "mode": args.mode,
        "preconditioner": "jacobi",
        "rtol": w["rtol"],
        "truncation": f"pod-a-rbf nu_y=1 nu_w=1 storage_cap={w['cap']} max_dim={w.get('max_dim', w['cap'])}",
        "l2": w["l2"],
        "parallelism": "replicas (the same seeded sequence solved independently on every GPU)",
    }


def solver_config(pk, args):
    w = WORKLOADS[args.workload]
    tr = pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=w["cap"],
                             max_dim=w.get("max_dim", w["cap"]))
    return pk.SolverConfig(truncation=tr, mode=args.mode)


def schedule_path(args):
    return os.path.join(ROOT, "profiles", f"{args.workload}_schedule.json")


# ---------------------------------------------------------------------------
# distributed plumbing (replicas only: no data-path collective)
# ---------------------------------------------------------------------------
def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws <= 1:
        return 0, 1, None
    import torch.distributed as dist

    backend = "nccl" if _cuda() else "gloo"
    dist.init_process_group(backend=backend)
    return dist.get_rank(), ws, dist


def _cuda():
    import torch

    return torch.cuda.is_available()


def max_over_ranks(value: float, dist) -> float:
    """Max of a per-rank scalar (device timing) over all ranks."""
    if dist is None:
        return value
    import torch

    dev = torch.device("cuda", torch.cuda.current_device()) if _cuda() else torch.device("cpu")
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ---------------------------------------------------------------------------
# clocks sampling during the timed region
# ---------------------------------------------------------------------------
_REASONS = [(0x1, "gpu_idle"), (0x2, "applications_clocks_setting"), (0x4, "sw_power_cap"), (0x8, "hw_slowdown"),
            (0x20, "sw_thermal_slowdown"), (0x40, "hw_thermal_slowdown"), (0x80, "hw_power_brake_slowdown"),
            (0x100, "display_clock_setting")]


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,utilization.gpu"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                f = [x.strip() for x in out.stdout.strip().split(",")]
                self.samples.append((float(f[0]), float(f[1]), int(f[2], 16) if f[2].startswith("0x") else int(f[2]),
                                     float(f[3])))
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [s for s in self.samples if s[3] > 10] or self.samples
        reasons = set()
        for s in loaded:
            for bit, name in _REASONS:
                if s[2] & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": float(np.median([s[0] for s in loaded])), "sm_max_mhz": max(s[1] for s in loaded),
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def spmv_bytes(n, nnz):
    """Algorithmic bytes of one CSR SpMV: fp64 value + int32 column
    per nonzero, the int32 row pointer, x read once, y written once."""
    return 12 * nnz + 4 * (n + 1) + 16 * n


def bsr3_bytes(n, nblk):
    """Algorithmic bytes of one 3x3-block SpMV in the format actually streamed:
    9 fp64 values + one int32 block column per block, the int32 block-row
    pointer, x read once, y written once."""
    return 76 * nblk + 4 * (n // 3 + 1) + 16 * n


def _shared_host_specs(args, seq, rank, world, dist):
    """The sequence's host arrays. With N > 1 replicas every rank solves the
    same seeded sequence; rank 0 generates it once into a file that all ranks
    map read-only, so the host holds one copy (C3: 20.6 GB of values) instead
    of one per rank (8 ranks would need ~170 GB of the box's host memory)."""
    if world <= 1:
        return list(seq)
    from paper_1512_05820_b200.problems import HostCsr, LinearSystemSpec

    first = next(iter(seq), None)
    if first is not None and getattr(first.A, "affine", None) is not None:
        return list(seq)  # C3: two value arrays per rank (1 GB), every system's values formed on the device
    del first

    base = os.path.join(os.environ.get("RK_BENCH_SHM", "/tmp"), f"rk_bench_{args.workload}_{args.grid}_{args.systems}")
    if rank == 0:
        specs = list(seq)
        uniq = []
        for s_ in specs:
            if not any(s_.A is u for u in uniq):
                uniq.append(s_.A)
        np.save(base + "_rp.npy", np.asarray(uniq[0].row_offsets))
        np.save(base + "_ci.npy", np.asarray(uniq[0].col_indices))
        vals = np.lib.format.open_memmap(base + "_vals.npy", mode="w+", dtype=np.float64,
                                         shape=(len(uniq), uniq[0].nnz))
        for i, u in enumerate(uniq):
            vals[i] = u.values
        vals.flush()
        which = np.array([next(i for i, u in enumerate(uniq) if s_.A is u) for s_ in specs])
        np.save(base + "_which.npy", which)
        np.save(base + "_b.npy", np.stack([s_.b for s_ in specs]))
        np.save(base + "_tol.npy", np.array([s_.tol for s_ in specs]))
        del specs, uniq, vals
    barrier(dist)
    rp = np.load(base + "_rp.npy", mmap_mode="r")
    ci = np.load(base + "_ci.npy", mmap_mode="r")
    vals = np.load(base + "_vals.npy", mmap_mode="r")
    which = np.load(base + "_which.npy")
    bs = np.load(base + "_b.npy", mmap_mode="r")
    tols = np.load(base + "_tol.npy")
    mats = [HostCsr(seq.n, rp, ci, vals[i]) for i in range(vals.shape[0])]
    return [LinearSystemSpec(A=mats[w], b=bs[j], xbar=None, tol=float(tols[j])) for j, w in enumerate(which)]


def run_b200(args, rank, world, dist):
    import torch

    import paper_1512_05820_b200 as pk
    from paper_1512_05820_b200 import _native as nat
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = nat.lib()
    seq = make_sequence(args, seed_offset=0 if world > 1 else rank)
    host_specs = _shared_host_specs(args, seq, rank, world, dist)  # host CSR values + rhs (the e2e inputs)
    n = seq.n
    nnz = host_specs[0].A.nnz
    # device-resident inputs for `value`
    dev_specs = []
    uploaded = {}  # invariant-matrix sequences (C4) share one device matrix
    for s in host_specs:
        if id(s.A) not in uploaded:
            uploaded[id(s.A)] = pk.SparseSpdMatrix.from_host(s.A)
        A = uploaded[id(s.A)]
        dev_specs.append(pk.LinearSystemSpec(A=A, b=torch.from_numpy(np.array(s.b)).to(dev), xbar=None, tol=s.tol))
    dseq = pk.SystemSequence(n, dev_specs, C=seq.C)
    cfg = solver_config(pk, args)
    jac = lambda A: pk.build_preconditioner("jacobi", A)  # noqa: E731
    torch.cuda.synchronize()

    for _ in range(args.warmup):
        pk.run_sequence(dseq, cfg, precond_factory=jac)
    torch.cuda.synchronize()

    from paper_1512_05820_b200 import _timing

    _timing.reset()
    stream = torch.cuda.current_stream()
    times = []
    reports = None
    launches0 = lib.rk_launch_count()
    lib.rk_profile_begin()
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            barrier(dist)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            xs, reports, _ = pk.run_sequence(dseq, cfg, precond_factory=jac)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
    ms = (ctypes.c_double * 4)()
    cnt = (ctypes.c_int64 * 4)()
    lib.rk_profile_end(ms, cnt)
    cl_ms, cl_n = ctypes.c_double(0.0), ctypes.c_int64(0)
    lib.rk_profile_cluster(ctypes.byref(cl_ms), ctypes.byref(cl_n))
    launches = (lib.rk_launch_count() - launches0) / max(args.steps, 1)
    t_step = max_over_ranks(float(np.mean(times)), dist)

    # q = c'x of the last timed sequence (D2H only after timing)
    q_last = float(seq.C[0] @ xs[-1].cpu().numpy())

    avg = [ms[i] / max(cnt[i], 1) for i in range(4)]
    peaks = _peaks()
    A0 = dev_specs[0].A
    if A0.bval is not None and A0.csr.bdim == 1:
        sell = A0._pattern.sell
        fmt = (f"scalar SELL-32 (one row per lane, fp64 values, int32 columns; {sell.nslot} slots for {nnz} "
               f"nonzeros, {100.0 * (sell.nslot - nnz) / sell.nslot:.1f}% padding)")
        alg_bytes = 12 * sell.nslot + 4 * ((n + 31) // 32 + 1) + 16 * n
    elif A0.bval is not None:
        bsr = A0._pattern.bsr
        fmt = (f"SELL-32 of 3x3 blocks (9x32 fp64 value tiles per slot row, int32 block columns; {bsr.nblk} slots for "
               f"{bsr.nreal} blocks, {100.0 * (bsr.nblk - bsr.nreal) / bsr.nblk:.1f}% padding)")
        alg_bytes = bsr3_bytes(n, bsr.nblk)
    else:
        fmt = "CSR (fp64 values, int32 columns)"
        alg_bytes = spmv_bytes(n, nnz)
    dev = A0.device
    # e2e: the public API from host CSR arrays; H2D of values+rhs and D2H of x inside
    e2e = None
    if not args.no_e2e and args.workload == "c4":
        # C4 fills HBM (two ~80 GB snapshot blocks): drop the device-resident
        # inputs of the `value` leg before the host-input run
        del dev_specs, dseq, xs, A0, A
        uploaded.clear()
        torch.cuda.empty_cache()
    if not args.no_e2e:
        hseq = pk.SystemSequence(n, host_specs, C=seq.C)
        # matrix bytes that cross PCIe: an affine sequence (C3) uploads its two
        # value arrays once, any other one every distinct matrix's values
        parts = {}
        for s in host_specs:
            aff = getattr(s.A, "affine", None)
            for arr in (aff[:2] if aff is not None else (s.A.values,)):
                parts[id(arr)] = arr.nbytes
        h2d = sum(s.b.nbytes for s in host_specs) + sum(parts.values())
        d2h = n * 8 * len(host_specs)
        from paper_1512_05820_b200 import linalg as _L

        with _L._affine_cache_lock:
            _L._affine_cache.clear()  # the `value` leg's setup uploaded them: the e2e run pays its own H2D
        barrier(dist)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        xs_e, reps_e, _ = pk.run_sequence(hseq, cfg, precond_factory=jac)  # host inputs -> numpy solutions
        assert all(isinstance(x, np.ndarray) for x in xs_e)
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(time.perf_counter() - t0, dist)
        del xs_e
        # cold: the same call once more with the pattern cache emptied, so the
        # int32 pattern upload and the SELL view build (on the device) are paid
        # inside the timed region, as by a first drop-in call in a fresh process
        _L.clear_upload_caches()
        barrier(dist)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        xs_c, _, _ = pk.run_sequence(hseq, cfg, precond_factory=jac)
        torch.cuda.synchronize()
        t_cold = max_over_ranks(time.perf_counter() - t0, dist)
        del xs_c
        e2e = {"value": round(t_e2e / world, 4), "unit": UNIT, "h2d_bytes_per_step": int(h2d * world),
               "d2h_bytes_per_step": int(d2h * world),
               "solve_wall_sum_s": round(sum(r.wall_time for r in reps_e), 3),
               "cold_value": round(t_cold / world, 4),
               "cold_note": "upload caches emptied first: the int32 pattern upload, the device SELL view build and "
                            "(C3) the upload of the two affine value arrays are inside the timed region (a first "
                            "call in a fresh process)",
               "path": "run_sequence over host CSR (reference-style SparseSpdMatrix fields); returns numpy solutions"}

    ach = alg_bytes / (avg[0] * 1e-3) / 1e9 if avg[0] > 0 else None  # C1: single-CTA batches, no per-kernel samples
    traffic = None
    if args.workload == "c3":  # the committed ncu capture is of the C3 SELL kernel
        try:
            with open(NCU_SUMMARY) as fh:
                traffic = json.load(fh).get("k_spmv_pcg", {}).get("dram_bytes_per_launch")
        except Exception:
            pass
    try:
        gram = _gram_roofline(n, dev, reports)
    except torch.cuda.OutOfMemoryError as exc:  # C4 fills HBM; the probe is measurement only
        torch.cuda.empty_cache()
        gram = {"kernel": "K7 k_gram_tma", "skipped": f"out of memory for the shape probe: {str(exc)[:80]}"}
    iters = [r.stage3_iters for r in reports]
    sched = {"stage3_iters": iters, "truncated": [bool(r.truncated) for r in reports],
             "basis_dim": [r.basis_dim for r in reports], "grown": [r.basis_dim + r.stage3_iters for r in reports]}
    line = {
        "metric": METRIC,
        "value": round(t_step / world, 4),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(t_step * 1e3, 2),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": WORKLOADS[args.workload]["data"],
        "config": workload_config(args, n, nnz),
        "roofline": {
            "kernel": "K1 SpMV fused with p'Ap, p'p (k_bsr3_spmv_pcg / k_spmv_pcg)",
            "format": fmt,
            "bound": "hbm",
            "achieved": round(ach, 1) if ach else None,
            "peak": peaks["hbm_gbs"],
            "unit": "GB/s",
            "frac": round(ach / peaks["hbm_gbs"], 3) if ach else None,
            "traffic": traffic,
            "algorithmic_bytes_per_launch": alg_bytes,
            "csr_equivalent_bytes": spmv_bytes(n, nnz),
            "avg_launch_ms": round(avg[0], 4),
            "peak_source": peaks["source"],
        },
        "gram": gram,
        "pcg_vectors": _pcg_vector_rooflines(n, reports, avg, peaks, args.mode),
        "kernels_ms_avg": {"spmv_pcg": round(avg[0], 4), "pcg_update": round(avg[1], 4),
                           "pcg_finish": round(avg[2], 4), "pcg_direction": round(avg[3], 4),
                           "launches": list(cnt)},
        "sequence": {"stage3_iters_total": int(sum(iters)), "cg_iters_per_s": round(sum(iters) / t_step, 1),
                     "us_per_iteration": round(t_step / max(sum(iters), 1) * 1e6, 2),
                     "per_system_iters": iters, "q_last": q_last,
                     "all_converged": bool(all(r.converged for r in reports))},
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    if cl_n.value:
        # small systems run in the persistent single-cluster solver (one launch
        # per solve, pcg_cluster.cu): no per-kernel slots; its event-timed
        # duration per iteration is the figure of merit (latency-bound: the
        # working set sits in L1 / shared memory, so the HBM fraction is tiny)
        tot_iters = max(int(sum(iters)) * args.steps, 1)
        us_it = cl_ms.value * 1e3 / tot_iters
        line["cluster_solver"] = {
            "kernel": "k_pcg_cluster (one thread-block cluster, DSMEM reductions, loops to convergence)",
            "launches": int(cl_n.value), "ms_total": round(cl_ms.value, 3),
            "us_per_iteration": round(us_it, 3),
            "share_of_step": round(cl_ms.value / 1e3 / max(sum(times), 1e-12), 3)}
        ach_c = alg_bytes / (us_it * 1e-6) / 1e9
        line["roofline"].update({"kernel": line["cluster_solver"]["kernel"], "achieved": round(ach_c, 1),
                                 "frac": round(ach_c / peaks["hbm_gbs"], 4),
                                 "avg_launch_ms": round(us_it * 1e-3, 5),
                                 "note": "per-iteration SpMV bytes over the cluster solver's time per iteration; "
                                         "latency-bound (matrix and vectors resident on chip)"})
    if _timing.ENABLED:  # diagnostic only: adds synchronisations, never on the reported line by default
        line["phases_s_per_step"] = {k: round(v / max(args.steps, 1), 4) for k, v in _timing.TIMES.items()}
    if rank == 0:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", f"{args.workload}_schedule.json"), "w") as fh:
            json.dump(sched, fh)
    return line, host_specs, sched


def _pcg_vector_rooflines(n, reports, avg, peaks, mode="cg"):
    """SURVEY 8d's fused-PCG GB/s: algorithmic bytes of the update kernel
    ((5 + m) 8N read + 3 * 8N written: x, p, r, Ap, 1/diag and the m columns of
    cross; x, r, z) and of the direction kernel ((3 + m) 8N: z, p_k and the m
    columns of B read, p_{k+1} written), averaged over the run's iterations
    with each system's projection width m, over the CUDA-event durations.
    In fom mode the direction slot also times the two re-orthogonalisation
    sweeps of iteration k (GEMV-T over A p_0..A p_k and p, GEMV-N over
    p_0..p_k reading and writing p: 2 (2k + 5) 8N bytes, SURVEY 8d's
    "4k 8N" plus the vector terms), so their bytes are counted there too."""
    iters = [r.stage3_iters for r in reports]
    widths = [r.basis_dim if r.basis_dim else 0 for r in reports]
    tot = max(sum(iters), 1)
    upd = sum(k * (8 + w) * 8 * n for k, w in zip(iters, widths)) / tot
    dirb = sum(k * (3 + w) * 8 * n for k, w in zip(iters, widths)) / tot
    if mode == "fom":  # sum over k < K of 2 (2k + 5) = 2 K^2 + 8 K
        dirb += sum((2 * k * k + 8 * k) * 8 * n for k in iters) / tot
    out = {}
    # avg[1]: the update kernel with its fused finish (widths <= 64; wider runs add
    # k_pcg_finish + k_pcg_musolve, sampled separately in avg[2])
    for name, b, ms in (("update", upd, avg[1]), ("direction", dirb, avg[3])):
        if ms > 0:
            gbs = b / (ms * 1e-3) / 1e9
            out[name] = {"algorithmic_bytes_per_launch": int(b), "avg_launch_ms": round(ms, 4),
                         "achieved_GB_s": round(gbs, 1), "frac": round(gbs / peaks["hbm_gbs"], 3)}
            if gbs > peaks["hbm_gbs"]:
                out[name]["note"] = ("a read-dominated stream (m columns read per vector written) against the "
                                     "measured COPY peak (read + write): fractions above 1 are real")
    return out


DMMA_PEAK_TFLOPS = 37.1  # B200 FP64 tensor (DMMA) peak measured by scripts/dmma_probe.cu (profiles/dmma_peak_r01.json)


def _gram_roofline(n, dev, reports):
    """BASELINE's second metric: the truncation Gram Z'AZ (rk_gram_upper from
    cached products, DMMA) at the sequence's own truncation width, timed with
    CUDA events after the timed region (3 launches, random data of that shape),
    against the measured DMMA peak. Flops counted for the upper triangle only,
    N m (m + 1)."""
    import torch

    from paper_1512_05820_b200.linalg import empty_block, symmetric_gram_from_products

    grown = [r.basis_dim + r.stage3_iters for r in reports if r.truncated]
    if not grown:
        return None
    m = int(np.median(grown))
    y_old = min(60, m - 1)
    note = None
    if 2 * n * m * 8 > 40e9:
        # C4: the sequence's own buffers already hold most of HBM; probe the same
        # width on fewer rows (split-K over rows: the rate does not depend on N here)
        n_full, n = n, int(20e9 / (2 * m * 8)) // 1024 * 1024
        note = f"rows reduced from {n_full} to {n} for the probe (two N x m blocks would need > 40 GB)"
    g = torch.Generator(device=dev).manual_seed(1)
    Z, AY, AV = empty_block(n, m, dev), empty_block(n, y_old, dev), empty_block(n, m - y_old, dev)
    for t in (Z, AY, AV):
        t.copy_(torch.randn(t.shape, generator=g, device=dev, dtype=torch.float64))
    symmetric_gram_from_products(Z, [(AY, 0), (AV, y_old)])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        symmetric_gram_from_products(Z, [(AY, 0), (AV, y_old)])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    tf = n * m * (m + 1) / (ms * 1e-3) / 1e12
    del Z, AY, AV
    out = {"kernel": "K7 k_gram_tma (rk_gram_upper_split, TMA-staged DMMA m8n8k4 f64)", "bound": "tensor", "n": n, "m": m,
           "ms": round(ms, 3), "achieved": round(tf, 2), "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
           "frac": round(tf / DMMA_PEAK_TFLOPS, 3),
           "peak_source": "measured DMMA register-only probe (scripts/dmma_probe.cu); cuBLAS DGEMM 35.5"}
    if note:
        out["note"] = note
    return out


# ---------------------------------------------------------------------------
# C5: POD truncation microbench (BASELINE configs[4])
# ---------------------------------------------------------------------------
C5_GRID = (128, 128, 256)
C5_BLOCK = 256


def _c5_flops(n, m):
    """Gram flops as computed: one triangle, N m (m + 1)."""
    return float(n) * m * (m + 1)


def run_c5(args, rank, world, dist):
    """One step = the POD truncation of a seeded N(0,1) snapshot block S
    (N = 4,194,304 x m) against the 7-point Laplacian on 128x128x256:
    A S and the upper triangle of S'(AS) column block by column block
    (assemble_gram_blocked, A S never held whole), the m x m eigenproblem
    (cuSOLVER), Phi = S V Sigma^-1 (DMMA), plus a 20-SpMV sweep on A.
    ``value`` = Gram flops / time of the A S + Gram phase."""
    import torch

    import paper_1512_05820_b200 as pk
    from paper_1512_05820_b200 import _native as nat
    from paper_1512_05820_b200.linalg import empty_block, spmv_into
    from paper_1512_05820_b200.problems import laplacian3d

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = nat.lib()
    L = laplacian3d(*C5_GRID)
    A = pk.SparseSpdMatrix(L.n, L.row_offsets, L.col_indices, L.values)
    n, m = L.n, args.m
    S = empty_block(n, m, dev)
    g = torch.Generator(device=dev).manual_seed(5 + rank)
    for j0 in range(0, m, 128):
        S[:, j0 : j0 + 128].normal_(generator=g)
    gamma = np.ones(m)
    x = S[:, 0].clone()
    y = torch.empty_like(x)
    torch.cuda.synchronize()

    def step(events=None):
        G = pk.assemble_gram_blocked(A, S, block=C5_BLOCK, events=events)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        res = pk.pod_evd_from_gram(G, S, gamma, 1.0)
        e2 = torch.cuda.Event(enable_timing=True)
        e2.record()
        a, b = x, y
        for _ in range(20):
            spmv_into(A, a, b)
            a, b = b, a
        e3 = torch.cuda.Event(enable_timing=True)
        e3.record()
        return G, res, (e1, e2, e3)

    for _ in range(args.warmup):
        _, res, _ = step()
        del res
    torch.cuda.synchronize()
    launches0 = lib.rk_launch_count()
    t_gram_phase, t_pod, t_spmv, t_spmm_k, t_gram_k, t_step = [], [], [], [], [], []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            barrier(dist)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
            evs = []
            G, res, (e1, e2, e3) = step(evs)
            torch.cuda.synchronize()
            t_gram_phase.append(e0.elapsed_time(e1) / 1e3)
            t_pod.append(e1.elapsed_time(e2) / 1e3)
            t_spmv.append(e2.elapsed_time(e3) / 1e3 / 20)
            t_step.append(e0.elapsed_time(e3) / 1e3)
            t_spmm_k.append(sum(a.elapsed_time(b) for a, b, _ in evs) / 1e3)
            t_gram_k.append(sum(b.elapsed_time(c) for _, b, c in evs) / 1e3)
            if _ < args.steps - 1:
                del res
    launches = (lib.rk_launch_count() - launches0) / max(args.steps, 1)
    tg = max_over_ranks(float(np.mean(t_gram_phase)), dist)
    flops = _c5_flops(n, m)
    y_kept = int(res.columns.shape[1])
    # size-independent checks (untimed): the POD basis is A-orthonormal,
    # Phi' A Phi = Sigma^-1 V' G V Sigma^-1 = I, on its leading 32 columns
    P = res.columns[:, :32]
    Gp, _ = pk.assemble_gram(A, P)
    orth = float((Gp - torch.eye(P.shape[1], dtype=torch.float64, device=dev)).abs().max())
    sig = res.singular_values
    e2e = None
    if not args.no_e2e:
        # public-API path from host memory: S H2D (pinned), the same truncation,
        # Phi D2H; the pinned host block is reused for Phi
        host = torch.empty((m, n), dtype=torch.float64, pin_memory=True)
        host.copy_(S.t())
        del res, G, P, Gp
        torch.cuda.empty_cache()
        torch.cuda.synchronize()
        barrier(dist)
        t0 = time.perf_counter()
        S.copy_(host.t())
        G = pk.assemble_gram_blocked(A, S, block=C5_BLOCK)
        res = pk.pod_evd_from_gram(G, S, gamma, 1.0)
        ph = host[: res.columns.shape[1]].t()
        ph.copy_(res.columns)
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(time.perf_counter() - t0, dist)
        e2e = {"value": round(flops / t_e2e / 1e12 * world, 3), "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(n * m * 8 * world),
               "d2h_bytes_per_step": int(n * int(res.columns.shape[1]) * 8 * world),
               "seconds_per_step": round(t_e2e, 4),
               "path": "S from pinned host memory -> assemble_gram_blocked -> pod_evd_from_gram -> Phi to host"}
        del host
    gk = float(np.mean(t_gram_k))
    achieved = flops / gk / 1e12
    spmv_b = spmv_bytes(n, L.nnz)
    if A.csr.bdim == 1:  # bytes of the format actually streamed (scalar SELL-32: no row pointers, padded slots)
        spmv_b = 12 * A._pattern.sell.nslot + 4 * ((n + 31) // 32 + 1) + 16 * n
    peaks = _peaks()
    spmv_gbs = spmv_b / float(np.mean(t_spmv)) / 1e9
    spmm_cols_bytes = (12 * L.nnz + 4 * (n + 1)) * math.ceil(C5_BLOCK / 8) * math.ceil(m / C5_BLOCK) + 16 * n * m
    line = {
        "metric": "snapshot-Gram FP64 TFLOP/s",
        "value": round(flops / tg / 1e12 * world, 3),
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(tg * 1e3, 2),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (S ~ N(0,1) from a seed on the device; 7-point Laplacian, BASELINE configs[4] shapes)",
        "config": {"workload": f"C5 POD truncation, Laplacian {C5_GRID[0]}x{C5_GRID[1]}x{C5_GRID[2]}, "
                               f"S {n} x {m}", "n": n, "nnz": L.nnz, "m": m, "column_block": C5_BLOCK,
                   "gamma": 1, "nu": 1.0,
                   "l2": "inputs larger than L2 (S is %.1f GB); no flush" % (n * m * 8 / 1e9),
                   "parallelism": "replicas (one independent truncation per GPU)"},
        "roofline": {"kernel": "K7 k_gram_tma (rk_gram_upper per column block, TMA-staged DMMA m8n8k4 f64)", "bound": "tensor",
                     "achieved": round(achieved, 2), "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": round(achieved / DMMA_PEAK_TFLOPS, 3), "traffic": None,
                     "flops_per_step": flops, "kernel_s": round(gk, 4),
                     "peak_source": "measured DMMA register-only probe (scripts/dmma_probe.cu); cuBLAS DGEMM 35.5"},
        "phases_s": {"spmm_plus_gram": round(tg, 4), "spmm_kernels": round(float(np.mean(t_spmm_k)), 4),
                     "gram_kernels": round(gk, 4), "evd_coef_reconstruction": round(float(np.mean(t_pod)), 4),
                     "pod_truncation_total": round(float(np.mean(t_step)) - 20 * float(np.mean(t_spmv)), 4)},
        "spmm": {"bytes_per_step": spmm_cols_bytes,
                 "GB_s": round(spmm_cols_bytes / float(np.mean(t_spmm_k)) / 1e9, 1)},
        "spmv": {"kernel": "rk_spmv (%s)" % ("scalar SELL-32 view" if A.csr.bdim == 1 else "CSR"), "bytes": spmv_b,
                 "avg_ms": round(float(np.mean(t_spmv)) * 1e3, 4), "GB_s": round(spmv_gbs, 1),
                 "frac": round(spmv_gbs / peaks["hbm_gbs"], 3), "peak": peaks["hbm_gbs"]},
        "pod": {"y": y_kept, "sigma_1": float(sig[0]), "sigma_m": float(sig[-1]),
                "phi_A_orthonormality_maxdev_32": orth},
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    return line


def cpu_sample_c5(m, cols=64):
    """The oracle's C5 operations (scipy A @ S, OpenBLAS S'(AS), LAPACK eigh,
    S @ coef) timed on `cols` columns of S (eigh at the full m) and scaled to m
    columns: the reference's assemble_gram computes the full m x m product."""
    from oracle import recycle_oracle as O
    from paper_1512_05820_b200.problems import laplacian3d

    L = laplacian3d(*C5_GRID)
    A = O.as_csr(L)
    n = L.n
    rng = np.random.default_rng(5)
    S = rng.standard_normal((n, cols))
    t0 = time.perf_counter()
    AS = A @ S
    t_spmm = (time.perf_counter() - t0) / cols
    t0 = time.perf_counter()
    _ = S.T @ AS
    t_pair = (time.perf_counter() - t0) / (cols * cols)
    G = rng.standard_normal((m, m))
    G = G @ G.T
    np.linalg.eigh(G[:64, :64])  # LAPACK / thread-pool warm-up
    t0 = time.perf_counter()
    np.linalg.eigh(G)
    t_evd = time.perf_counter() - t0
    C = rng.standard_normal((cols, cols))
    t0 = time.perf_counter()
    _ = S @ C
    t_rec_pair = (time.perf_counter() - t0) / (cols * cols)
    t_assemble = m * t_spmm + m * m * t_pair
    return {
        "value": round(_c5_flops(n, m) / t_assemble / 1e12, 4),
        "unit": "TFLOP/s",
        "cores": len(os.sched_getaffinity(0)),
        "kind": "port",
        "sample": (f"oracle ops on {cols} columns of S (N = {n}): A@S {t_spmm*1e3:.1f} ms/column, S'(AS) "
                   f"{t_pair*1e6:.1f} us per column pair, eigh({m}) {t_evd:.2f} s; scaled to m = {m} "
                   "(full m x m product as the reference computes it; extrapolated)"),
        "seconds": {"assemble_gram": round(t_assemble, 2), "eigh": round(t_evd, 2),
                    "reconstruction": round(m * m * t_rec_pair, 2),
                    "pod_truncation_total": round(t_assemble + t_evd + m * m * t_rec_pair, 2)},
    }


def run_reference_c5(args, world):
    vals, cb = [], None
    for _ in range(args.warmup):
        cpu_sample_c5(args.m)
    for _ in range(args.steps):
        cb = cpu_sample_c5(args.m)
        vals.append(cb["value"])
    v = float(np.mean(vals))
    cb["value"] = round(v, 4)
    n = C5_GRID[0] * C5_GRID[1] * C5_GRID[2]
    return {
        "impl": "reference", "metric": "snapshot-Gram FP64 TFLOP/s", "value": round(v, 4), "unit": "TFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (S ~ N(0,1) from a seed; 7-point Laplacian, BASELINE configs[4] shapes)",
        "config": {"workload": f"C5 POD truncation, Laplacian {C5_GRID[0]}x{C5_GRID[1]}x{C5_GRID[2]}, "
                               f"S {n} x {args.m}", "n": n, "m": args.m},
        "cpu_baseline": cb,
        "e2e": {"value": round(v, 4), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference = numpy/scipy (recykl); its operations timed through oracle/recycle_oracle.py on a "
                "bounded sample and scaled to m columns (extrapolated)",
    }


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "MEASURED_PEAKS.json (measured copy, burst)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback 6.65 TB/s (B200_PROFILING.md)"}


# ---------------------------------------------------------------------------
# CPU oracle sample, scaled to the metric
# ---------------------------------------------------------------------------
def cpu_sample(host_specs, sched, cap=60, label="C3", budget_s=20.0):
    """Time the oracle (numpy/scipy, as the reference) on a bounded sample of
    the sequence workload and scale it to one sequence with the GPU run's schedule:
    t = sum_j iters_j * t_iter(m_j) + sum_truncations t_trunc(grown_j)."""
    import scipy.sparse  # noqa: F401

    from oracle import recycle_oracle as O

    A = O.as_csr(host_specs[0].A)
    n = A.shape[0]
    b = host_specs[0].b
    dinv = 1.0 / A.diagonal()
    cores = len(os.sched_getaffinity(0))
    rng = np.random.default_rng(0)

    def iters_cost(Y, k):
        t = O.Tally()
        proj = None
        yh = None
        if Y is not None:
            proj = O.assembled_projection(lambda v: O.matvec(A, v, t), Y)
            yh = np.zeros(Y.shape[1])
        t0 = time.perf_counter()
        try:
            O.aug_pcg(lambda v: O.matvec(A, v, t), b, yh, Y, proj, dinv, 0.0, mode="cg", max_iter=k,
                      r0=b.copy(), tally=t)
        except O.OracleNotConverged:
            pass
        return (time.perf_counter() - t0) / k

    k0 = 12 if A.nnz < 10**8 else 6
    t_it0 = iters_cost(None, k0)
    ms = min(cap, 60)  # projected sample width; per-column cost scales the other widths
    Y = np.linalg.qr(rng.standard_normal((n, ms)))[0]
    t_itm = iters_cost(Y, 8 if A.nnz < 10**8 else 4)
    t_col = max(t_itm - t_it0, 0.0) / ms
    # truncation sample: SpMM + Gram with s_cols columns, eigh at full width, S @ coef sample
    s_cols = 32  # a 32 x 32 Gram sample: a narrower one understates BLAS efficiency (C4 at 8 columns: ~2x)
    Z = rng.standard_normal((n, s_cols))
    t0 = time.perf_counter()
    AZ = A @ Z
    t_spmm = (time.perf_counter() - t0) / s_cols
    t0 = time.perf_counter()
    _ = Z.T @ AZ
    t_gram_unit = (time.perf_counter() - t0) / (s_cols * s_cols)
    grown = max(sched["grown"]) if sched else 760
    G = rng.standard_normal((grown, grown))
    G = G + G.T
    t0 = time.perf_counter()
    np.linalg.eigh(G)
    t_evd = time.perf_counter() - t0
    t0 = time.perf_counter()
    _ = Z @ rng.standard_normal((s_cols, 60))
    t_rec_unit = (time.perf_counter() - t0) / s_cols

    total = 0.0
    if sched:
        widths = sched.get("basis_dim") or [0] + [cap] * (len(sched["stage3_iters"]) - 1)
        for k, g, w in zip(sched["stage3_iters"], sched["grown"], widths):
            total += k * (t_it0 + w * t_col)                      # stage-3 iterations projected against w
            if w:
                total += w * t_spmm + w * w * t_gram_unit        # stage-1 assemble_gram of W
            if g > cap:  # truncation: SpMM + Gram of the grown block, eigh, reconstruction
                total += g * t_spmm + g * g * t_gram_unit + t_evd * (g / grown) ** 3 + g * t_rec_unit
    return {
        "value": round(total, 2),
        "unit": UNIT,
        "cores": cores,
        "kind": "port",
        "sample": (f"oracle on {label} system 1: {k0} plain PCG iterations ({t_it0*1e3:.0f} ms/it), iterations "
                   f"projected against {ms} columns ({t_itm*1e3:.0f} ms/it), a {s_cols}-column SpMM+Gram, "
                   f"S@coef and eigh({grown}); scaled to the sequence with the GPU run's schedule "
                   f"({sum(sched['stage3_iters']) if sched else 0} stage-3 iterations, extrapolated)"),
        "components_s": {"t_iter_plain": t_it0, "t_iter_projected": t_itm, "t_per_projected_column": t_col,
                         "t_spmm_per_col": t_spmm, "t_gram_per_col2": t_gram_unit, "t_evd_full": t_evd},
    }


# ---------------------------------------------------------------------------
# The reference itself (recykl, installed into baseline/_ref), bounded sample
# ---------------------------------------------------------------------------
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _import_recykl():
    """recykl from baseline/_ref (pip install --target), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "recykl")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import recykl.linalg
    import recykl.preconditioners
    import recykl.threestage
    import recykl.truncation

    return recykl


class _CallTimer:
    """Accumulates the wall time of named module-level functions while the
    reference's own solve_system calls them (the functions are looked up by
    name at call time, so wrapping the module attribute times the real call)."""

    def __init__(self, module, names):
        self.module, self.names, self.t, self._orig = module, names, {}, {}

    def __enter__(self):
        for nm in self.names:
            f = getattr(self.module, nm)
            self._orig[nm] = f

            def wrap(*a, _f=f, _nm=nm, **k):
                t0 = time.perf_counter()
                try:
                    return _f(*a, **k)
                finally:
                    self.t[_nm] = self.t.get(_nm, 0.0) + time.perf_counter() - t0

            setattr(self.module, nm, wrap)
        return self

    def __exit__(self, *exc):
        for nm, f in self._orig.items():
            setattr(self.module, nm, f)


class ReferenceSample:
    """Times the unmodified reference (recykl.threestage.solve_system and the
    recykl.linalg primitives it calls) on a bounded sample of the sequence and
    scales it to the whole sequence with the GPU run's schedule (iterations,
    widths, truncations per system). Setup (untimed): systems 1-2 of the
    sequence as recykl matrices, and a 60-column recycled state made by
    recykl itself (system 1 for cap + 1 iterations, then its own POD
    truncation). One step:
      * solve_system(system 2, that state, max_iter = 8): stage 1 over the 60
        columns (direct_reduced_solve), 8 stage-3 iterations projected against
        them (augmented_pcg), update_basis with a POD truncation of 68 columns;
      * solve_system(system 1, empty state, max_iter = 8): 8 plain iterations;
      * assemble_gram on 8 columns (its SpMM per column), the Gram product
        Z' (A Z) at the schedule's typical truncation width (per column^2),
        symmetric_evd at the widest truncation of the schedule, S @ coef.
    The scaled sequence time is sum_j [stage 1(w_j) + k_j t_iter(w_j) +
    truncation(g_j)], labelled extrapolated."""

    K = 8

    def __init__(self, rk, host_specs, cap, mode, threads):
        self.rk, self.cap, self.mode = rk, cap, mode
        self.threads = threads
        L, P, T = rk.linalg, rk.preconditioners, rk.threestage
        self.mats = []
        for s in host_specs[:2]:
            self.mats.append(L.SparseSpdMatrix(s.A.n, np.asarray(s.A.row_offsets), np.asarray(s.A.col_indices),
                                               np.asarray(s.A.values)))
        self.specs = host_specs[:2]
        self.n = self.mats[0].n
        tr = rk.truncation.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=cap, max_dim=cap)
        self.cfg_run = lambda it: T.SolverConfig(truncation=tr, mode=mode, max_iter=it)
        A, s = self.mats[0], self.specs[0]
        t0 = time.perf_counter()
        _, rep, self.state60 = T.solve_system(A, s.b, None, T.RecycleState.empty(self.n),
                                              T.StageTolerances(eps=s.tol), self.cfg_run(cap + 1),
                                              M=P.build("jacobi", A), sink=L.InstrumentationSink())
        self.setup_s = time.perf_counter() - t0
        assert self.state60.basis_dim == cap, self.state60.basis_dim

    def step(self, gmax, gtyp):
        import copy

        rk, K = self.rk, self.K
        L, P, T = rk.linalg, rk.preconditioners, rk.threestage
        out = {}
        A, s = self.mats[1], self.specs[1]
        st = copy.deepcopy(self.state60)
        with _CallTimer(T, ["direct_reduced_solve", "augmented_pcg", "update_basis"]) as ct:
            t0 = time.perf_counter()
            _, rep, _ = T.solve_system(A, s.b, None, st, T.StageTolerances(eps=s.tol), self.cfg_run(K),
                                       M=P.build("jacobi", A), sink=L.InstrumentationSink())
            out["sys2_wall"] = time.perf_counter() - t0
        assert rep.stage3_iters == K and rep.truncated
        out["stage1"] = ct.t["direct_reduced_solve"]
        out["t_iter_proj"] = ct.t["augmented_pcg"] / K
        out["update_trunc"] = ct.t["update_basis"]
        A, s = self.mats[0], self.specs[0]
        with _CallTimer(T, ["augmented_pcg"]) as ct:
            T.solve_system(A, s.b, None, T.RecycleState.empty(self.n), T.StageTolerances(eps=s.tol),
                           self.cfg_run(K), M=P.build("jacobi", A), sink=L.InstrumentationSink())
        out["t_iter_plain"] = ct.t["augmented_pcg"] / K
        rng = np.random.default_rng(0)
        # assemble_gram(A, B) = A @ B (scipy csr_matvecs, per column) + B' (A B)
        # (BLAS dgemm, per column^2): the SpMM from an 8-column call, the
        # product at the schedule's typical truncation width (its efficiency
        # depends on the width)
        S = rng.standard_normal((self.n, 8))
        t0 = time.perf_counter()
        L.assemble_gram(A, S)
        t8 = time.perf_counter() - t0
        if getattr(self, "_gz", None) is None or self._gz[0].shape[1] != gtyp:
            # dgemm time does not depend on the values: filled once, reused by every step
            self._gz = (np.full((self.n, gtyp), 0.5), np.full((self.n, gtyp), 0.25))
        Z, AZ = self._gz
        t0 = time.perf_counter()
        _ = Z.T @ AZ
        out["gram_b"] = (time.perf_counter() - t0) / (gtyp * gtyp)
        out["gram_a"] = max(t8 - 64 * out["gram_b"], 0.0) / 8
        G = rng.standard_normal((gmax, gmax))
        t0 = time.perf_counter()
        L.symmetric_evd(G + G.T)
        out["evd_gmax"] = time.perf_counter() - t0
        S = rng.standard_normal((self.n, 8))
        t0 = time.perf_counter()
        _ = S @ rng.standard_normal((8, self.cap))
        out["recon_per_col"] = (time.perf_counter() - t0) / 8
        return out

    def scale(self, c, sched):
        """Sequence time from one step's components and the schedule."""
        cap, K = self.cap, self.K

        def gram(w):
            return c["gram_a"] * w + c["gram_b"] * w * w

        def trunc(g, gmax):
            return gram(g) + c["evd_gmax"] * (g / gmax) ** 3 + g * c["recon_per_col"]

        gmax = max(sched["grown"])
        g_s = cap + K
        # what update_basis costs beyond the modelled parts (hstack, weights, bookkeeping), per column
        over = max(c["update_trunc"] - trunc(g_s, gmax), 0.0) / g_s
        stage1_over = max(c["stage1"] - gram(cap), 0.0)  # Cholesky, solves, W' r0
        total = 0.0
        for k, g, w, tr in zip(sched["stage3_iters"], sched["grown"], sched["basis_dim"], sched["truncated"]):
            t_it = c["t_iter_plain"] + (c["t_iter_proj"] - c["t_iter_plain"]) * w / cap
            total += k * t_it
            if w:
                total += gram(w) + stage1_over * (w / cap) ** 2
            if tr:
                total += trunc(g, gmax) + over * g
        return total


def reference_baseline(args, host_specs, sched, steps=1, warmup=0):
    """cpu_baseline / --impl reference: the reference itself (baseline/_ref) on
    the bounded sample above, or the oracle port if it is not installed."""
    rk = _import_recykl()
    cap = WORKLOADS[args.workload]["cap"]
    if rk is None or sched is None or args.workload not in ("c2", "c3"):
        return None
    threads = len(os.sched_getaffinity(0))
    smp = ReferenceSample(rk, host_specs, cap, args.mode, threads)
    gmax = max(sched["grown"])
    gtyp = int(np.median([g for g, t in zip(sched["grown"], sched["truncated"]) if t] or [gmax]))
    for _ in range(warmup):
        smp.step(gmax, gtyp)
    vals, comps = [], None
    for _ in range(max(steps, 1)):
        comps = smp.step(gmax, gtyp)
        vals.append(smp.scale(comps, sched))
    v = float(np.mean(vals))
    return {
        "value": round(v, 2), "unit": UNIT, "cores": threads, "kind": "reference",
        "sample": (f"recykl (baseline/_ref, unmodified) on the {args.workload.upper()} sequence: solve_system of "
                   f"system 2 from a {cap}-column recycled state with max_iter {smp.K} (stage 1, {smp.K} projected "
                   f"iterations, a POD truncation of {cap + smp.K} columns) and of system 1 with max_iter {smp.K}, "
                   f"assemble_gram on 8 columns, the {gtyp}-column Gram product, symmetric_evd({gmax}); scaled to "
                   "the sequence with the GPU "
                   f"run's schedule ({sum(sched['stage3_iters'])} stage-3 iterations; extrapolated). scipy's SpMV is "
                   "single-threaded; BLAS uses every core"),
        "components_s": {k: round(x, 5) for k, x in comps.items()},
        "setup_s": round(smp.setup_s, 1),
        "steps_sampled": len(vals),
    }


def cpu_full_sequence(args):
    """C1: the oracle port runs the whole sequence (seconds), no extrapolation."""
    from oracle import recycle_oracle as O

    seq = make_sequence(args)
    cap = WORKLOADS[args.workload]["cap"]
    ocfg = O.Config(mode=args.mode, strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=cap, max_dim=cap)
    O.run_sequence(make_sequence(args, p=2), ocfg, precond="jacobi")  # warm-up
    t0 = time.perf_counter()
    _, reps, _ = O.run_sequence(seq, ocfg, precond="jacobi")
    t = time.perf_counter() - t0
    return {"value": round(t, 4), "unit": UNIT, "cores": len(os.sched_getaffinity(0)), "kind": "port",
            "sample": f"the whole {args.systems}-system C1 sequence through the oracle (numpy/scipy as the reference)"}


def run_reference(args, rank, world):
    """--impl reference: the oracle port on the box's host cores (rank 0 only)."""
    if rank != 0:
        return None
    if args.workload == "c5":
        return run_reference_c5(args, world)
    if args.workload == "c1":
        vals = [cpu_full_sequence(args)["value"] for _ in range(max(args.steps, 1))]
        cb = cpu_full_sequence(args)
        cb["value"] = round(float(np.mean(vals)), 4)
        return {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": False, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": WORKLOADS["c1"]["data"],
                "config": workload_config(args, 4096, 20224), "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    seq = make_sequence(args, p=2)
    host_specs = list(seq)
    try:
        with open(schedule_path(args)) as fh:
            sched = json.load(fh)
    except Exception:
        sched = None
    cap = WORKLOADS[args.workload]["cap"]
    label = args.workload.upper()
    # the reference itself when installed (a step is ~10 s of its own calls, so
    # the driver's K + W steps are capped at 12 samples to stay within minutes)
    cb = reference_baseline(args, host_specs, sched, steps=min(max(args.steps, 1), 8),
                            warmup=min(args.warmup, 1))
    if cb is None:
        vals = []
        for _ in range(args.warmup):
            cpu_sample(host_specs, sched, cap, label)
        for _ in range(args.steps):
            cb = cpu_sample(host_specs, sched, cap, label)
            vals.append(cb["value"])
        cb["value"] = round(float(np.mean(vals)), 2)
    v = float(cb["value"])
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(v, 2),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": WORKLOADS[args.workload]["data"],
        "config": workload_config(args, seq.n, host_specs[0].A.nnz),
        "cpu_baseline": cb,
        "e2e": {"value": round(v, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": (("reference = recykl itself (pure Python numpy/scipy, baseline/_ref) "
                  if cb.get("kind") == "reference" else
                  "reference = recykl's algorithm through its restatement oracle/recycle_oracle.py (baseline/_ref "
                  "missing) ") + f"on a bounded sample, scaled with profiles/{args.workload}_schedule.json "
                 "(extrapolated)"),
    }
    return line


def main():
    args = parse()
    rank, world, dist = dist_init()
    if args.impl == "reference":
        line = run_reference(args, rank, world)
        if rank == 0 and line is not None:
            print(json.dumps(line))
        if dist is not None:
            dist.destroy_process_group()
        return
    if args.workload == "c5":
        line = run_c5(args, rank, world, dist)
        if rank == 0:
            if world == 1 and not args.no_cpu:
                line["cpu_baseline"] = cpu_sample_c5(args.m)
            print(json.dumps(line))
        if dist is not None:
            dist.destroy_process_group()
        return
    line, host_specs, sched = run_b200(args, rank, world, dist)
    if rank == 0:
        if world == 1 and not args.no_cpu:
            if args.workload == "c1":
                line["cpu_baseline"] = cpu_full_sequence(args)
            else:
                cb = reference_baseline(args, host_specs, sched)
                line["cpu_baseline"] = cb or cpu_sample(host_specs, sched, WORKLOADS[args.workload]["cap"],
                                                        args.workload.upper())
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
