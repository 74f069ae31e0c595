#!/usr/bin/env python
"""Benchmark of the hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (z-slab strong scaling)

Workload (BASELINE.json metric "SIPG Laplace matvec DoF/s (fp64) and achieved HBM
GB/s vs peak, p=2..8"): for every degree p = 2..8 a
Cartesian [0,1]^3 mesh of N_p^3 cells, N_p = round(480/(p+1)) (108.5-112.7 M DoF,
0.87-0.90 GB per fp64 vector >> 126 MB L2), mirror Dirichlet, seeded uniform[-1,1)
vectors.  One STEP = the whole hot path once per degree:
    matvec y = A u  ->  basis change v = T^{x3} u  ->  degree-5 Chebyshev sweep
    (5 fused matvec + GL-Jacobi + update kernels, range [0.06, 1.2] lambda_max,
    lambda_max from 15 Lanczos steps at setup).
value = matvec DoF/s aggregated over the sweep = sum_p n_DoF(p) * K / (max over ranks
of the summed matvec kernel time, CUDA events on the launching stream).  The other
ops' rates, the step time, the roofline of the dominant kernel, e2e (host buffers,
H2D+D2H inside the timed region) and the CPU oracle baseline are extra keys.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synthetic import CONFIGS, c4_spec  # noqa: E402

METRIC = "SIPG Laplace matvec DoF/s (fp64) and achieved HBM GB/s vs peak, p=2..8"
UNIT = "DoF/s"
# lambda_max(P^-1 A_H) sanity values (Kronecker + Lanczos, Cartesian, mirror)
LMAX_SANITY = {2: 2.986, 3: 2.604, 4: 2.500, 5: 2.401, 6: 2.370, 7: 2.402, 8: 2.471}
BYTES_PER_DOF = {"matvec": 16.0, "basis_change": 16.0, "cheby_first": 32.0, "cheby": 40.0}


def args_():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--degrees", default="2,3,4,5,6,7,8")
    ap.add_argument("--workload", default="c4", choices=["c4", "c2", "c3", "c5"],
                    help="c4: degree sweep (default, the metric's configuration); c2/c3/c5: other BASELINE configs")
    ap.add_argument("--cheby-degree", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip peaks/e2e/cpu (profiling runs)")
    ap.add_argument("--no-extras", action="store_true", help="skip the C2/C3/C5 and paper-formulation extra keys")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, measured)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()   # nvidia-smi takes a moment to start: wait for its first sample
            while not self.lines and time.time() - t0 < 3.0:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


_ORACLE_CACHE = {}


def oracle_rate(p, budget_s, seed=0):
    """CPU oracle matvec DoF/s on a bounded random sample of cells of the C4 mesh
    (untimed setup: the oracle operator and the full seeded input vector)."""
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    from synthetic import uniform_vector
    spec = c4_spec(p)
    if p not in _ORACLE_CACHE:
        _ORACLE_CACHE[p] = (SIPG(mesh_from_spec(spec), p), uniform_vector(spec.n_dofs, spec.seed))
    op, u = _ORACLE_CACHE[p]
    n3 = (p + 1) ** 3
    rng = np.random.default_rng(seed + p)
    cells_done, t_used = 0, 0.0
    batch = max(1, int(2000 / n3 * 8))
    while t_used < budget_s:
        cells = rng.choice(spec.n_cells_total, size=batch, replace=False)
        t0 = time.perf_counter()
        op.apply(u, cells=cells)
        t_used += time.perf_counter() - t0
        cells_done += batch
    return cells_done * n3 / t_used, cells_done, t_used


def cpu_cores_used():
    return 1   # numpy c_einsum loops (the oracle's contractions) run on one thread


def _pool_worker(args):
    """One process of the all-core oracle sample: random cells of a 12^3-cell mesh of the
    same degree (the oracle's work per cell does not depend on the mesh size)."""
    p, budget_s, seed = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle.geometry import Mesh
    from oracle.sipg import SIPG
    from synthetic import uniform_vector
    N = 12
    op = SIPG(Mesh(N=(N, N, N)), p)
    u = uniform_vector(N ** 3 * (p + 1) ** 3, seed)
    rng = np.random.default_rng(seed)
    n3 = (p + 1) ** 3
    batch = max(1, int(2000 / n3 * 8))
    done, t_used = 0, 0.0
    while t_used < budget_s:
        cells = rng.choice(N ** 3, size=batch, replace=False)
        t0 = time.perf_counter()
        op.apply(u, cells=cells)
        t_used += time.perf_counter() - t0
        done += batch
    return done * n3, t_used


def oracle_rate_all_cores(degrees, budget_s):
    """Aggregate oracle matvec DoF/s with one process per host core (os.cpu_count()),
    each timing `budget_s` of naive quadrature per degree; returns (DoF/s, cores)."""
    import multiprocessing as mp_
    cores = os.cpu_count() or 1
    ctx = mp_.get_context("fork")
    rates = []
    with ctx.Pool(cores) as pool:
        for p in degrees:
            res = pool.map(_pool_worker, [(p, budget_s, 1000 * p + i) for i in range(cores)])
            # all processes run concurrently: aggregate rate = sum of per-process rates
            rates.append((p, sum(d / t for d, t in res)))
    # sweep rate: total DoF over total time, each degree weighted like the single-core figure
    inv = sum(1.0 / r for _, r in rates) / len(rates)
    return 1.0 / inv, cores, {p: r for p, r in rates}


# ----------------------------------------------------------------------------- reference arm
def run_reference(a, rank):
    """The reference arm (the tier's reference is the CPU oracle): the oracle as it stands,
    one process per host core, each step a bounded sample of every degree of the workload."""
    if rank != 0:
        return
    degrees = [int(x) for x in a.degrees.split(",")]
    per_degree_s = 0.4      # seconds of oracle work per degree per step, in every process
    oracle_rate_all_cores(degrees[:1], 0.05)   # warm-up (process start, imports)
    for _ in range(max(0, a.warmup - 1)):
        oracle_rate_all_cores(degrees, 0.05)
    rates = []
    t0 = time.perf_counter()
    for s in range(a.steps):
        r, cores, _ = oracle_rate_all_cores(degrees, per_degree_s)
        rates.append(r)
    wall = time.perf_counter() - t0
    value = float(np.mean(rates))
    sample = (f"oracle matvec (naive quadrature, numpy, untuned) with one process per host core "
              f"({cores}), each timing {per_degree_s}s per degree per step on random cells of a 12^3 mesh "
              f"of that degree (per-cell work equals the C4 mesh's); sweep rate = harmonic mean over degrees")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * wall / a.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded uniform[-1,1) fp64 vectors on Cartesian meshes",
            "config": {"workload": "C4 degree sweep p=2..8 (sampled cells, CPU oracle)",
                       "degrees": degrees},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def lanczos_lambda_max(m, iters=15):
    """15 Lanczos steps for lambda_max(P^{-1}A), start [-5.5..5.5] repeated,
    on the GPU through the library (dg_lanczos_lambda_max; setup, outside the timed region)."""
    return m.lanczos_lambda_max("gl_jacobi", iters)


def workload_specs(a):
    if a.workload == "c4":
        return [c4_spec(int(x)) for x in a.degrees.split(",")]
    if a.workload == "c2":
        return [CONFIGS["C2"], CONFIGS["C2_GL"]]
    if a.workload == "c3":
        return [CONFIGS["C3"]]
    return [CONFIGS["C5"]]


def geometry_bytes_per_dof(spec):
    """Algorithmic geometry bytes per DoF read by one operator pass (each datum once):
    per-q-point merged tensor 6 words/q-point + per face point 4 words (3 faces per cell)."""
    if spec.geometry != "per_qpoint":
        return 0.0
    n = spec.n
    return 6 * 8 + 3 * 4 * 8 * n * n / n ** 3


def measured_traffic(workload, kernel, degrees, alg_bytes_per_step):
    """kernel: one name, or a dict degree -> name (the per-degree kernel of a kernel family)."""
    names = kernel if isinstance(kernel, dict) else {q: kernel for q in degrees}
    return _measured_traffic(workload, names, degrees)


def _measured_traffic(workload, names, degrees):
    """DRAM bytes (read + write) per launch of the dominant kernel, from the committed
    ncu capture profiles/r1_traffic.json (one `ncu --metrics dram__bytes_read.sum,
    dram__bytes_write.sum` pass of this workload, per degree), averaged over the degrees
    like `achieved`; None if the capture does not cover this workload/kernel."""
    caps = []
    for fn in ("r2s5_traffic.json", "r2s4_traffic.json", "r2_traffic.json", "r1_traffic.json"):   # newest capture first
        p = os.path.join(ROOT, "profiles", fn)
        if os.path.exists(p):
            with open(p) as f:
                caps.append(json.load(f))
    if not caps:
        return None, "no committed ncu traffic capture"
    per, alg, srcs = [], [], set()
    for q in degrees:
        ent = next((e for e in (d.get(workload, {}).get(names[q]) for d in caps)
                    if e and str(q) in e["per_launch_bytes"]), None)
        if ent is None:
            return None, "ncu traffic capture does not cover this configuration"
        per.append(ent["per_launch_bytes"][str(q)])
        alg.append(ent["algorithmic_bytes"][str(q)])
        srcs.add(ent["source"])
    return float(np.mean(per)), (f"ncu dram read+write per launch, mean over degrees ({', '.join(sorted(srcs))}); "
                                 f"measured/algorithmic = {sum(per) / sum(alg):.3f}")


WORKLOAD_TEXT = {
    "c4": "C4 degree sweep p=2..8, N_p=round(480/(p+1)) cells per direction, matvec + H->GL basis change "
          "+ degree-5 Chebyshev (GL-Jacobi) per degree; Cartesian meshes run the Kronecker form of the same "
          "operator (Eq. (14); the cell-per-thread kernel k_kron3c at p=2, k_kron4 otherwise; the Chebyshev "
          "steps at p=3,4,6,7,8 on the transformed residual (T^-T)^(x)3 (b - Au)), the paper's quadrature "
          "formulation is measured separately as c4_paper_formulation",
    "c2": "C2 p=4 32^3 Cartesian, Hermite-like vs nodal Gauss-Lobatto (full-neighbour reads)",
    "c3": "C3 p=5 48^3 curved (amp 0.05), per-quadrature-point geometry, general quadrature kernel",
    "c5": "C5 p=5 128^3 Cartesian (453M DoF), z-slabs",
}


OPS_H = {2: 190.7, 3: 218.0, 4: 205.6, 5: 225.3, 6: 223.8, 7: 241.0, 8: 244.0}   # tab:operations opsH,
# FLOP per DoF of the paper's general-geometry matvec in the Hermite-like basis


def make_setups(specs, rank, world, dev, P, torch, nccl_id=None, need_lmax=True):
    setups = []
    for spec in specs:
        p = spec.degree
        m = P.mesh_from_spec(spec, rank=rank, nranks=world, nccl_unique_id=nccl_id)
        nl = m.n_local_dofs
        g = torch.Generator(device=dev)
        g.manual_seed(spec.seed * 1000 + rank)
        u = torch.rand(nl, dtype=torch.float64, device=dev, generator=g).mul_(2).sub_(1)
        g.manual_seed((100 + p) * 1000 + rank)
        b = torch.rand(nl, dtype=torch.float64, device=dev, generator=g).mul_(2).sub_(1)
        x = torch.zeros(nl, dtype=torch.float64, device=dev)
        y = torch.empty_like(u)
        v = torch.empty_like(u)
        work2 = torch.empty(2 * nl, dtype=torch.float64, device=dev)
        lmax = lanczos_lambda_max(m) if need_lmax else None
        setups.append(dict(p=p, spec=spec, m=m, u=u, b=b, x=x, y=y, v=v, work2=work2, lmax=lmax,
                           n_global=m.n_global_dofs, key=f"p{p}" + ("-gl" if spec.basis == "gl" else "")
                           + ("-curved" if spec.deform_amp else "")))
    torch.cuda.synchronize()
    return setups


def time_steps(setups, a, stream, torch, barrier, ops=("matvec", "basis_change", "cheby"), apply_flags=0):
    """W warm-up + K timed steps of the listed ops per setup; CUDA events per op on `stream`
    (each op bracketed by its own events; an L2 flush outside the events when the vectors
    are smaller than 2x L2).  Returns (per-setup op ms lists, total ms, launches, clocks,
    l2 flush note)."""
    dev = setups[0]["u"].device
    small = min(s["m"].n_local_dofs for s in setups) * 8 < (256 << 20)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if small else None

    def l2_flush():
        if flush is not None:
            flush.fill_(1)

    def run_op(s, op):
        if op == "matvec":
            s["m"].apply_laplace(s["u"], s["y"], flags=apply_flags)
        elif op == "basis_change":
            if s["spec"].basis == "hermite":
                s["m"].basis_change("T", s["u"], s["v"])
        else:
            s["m"].chebyshev_smooth(s["b"], s["x"], s["lmax"], degree=a.cheby_degree, work2=s["work2"])

    def step(record):
        for s in setups:
            for op in ops:
                l2_flush()
                if record:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                run_op(s, op)
                if record:
                    e1.record(stream)
                    s.setdefault("ev", {}).setdefault(op, []).append((e0, e1))

    for s in setups:
        s["ev"] = {}
    for _ in range(a.warmup):
        step(False)
    launches0 = sum(s["m"].launch_count for s in setups)
    barrier()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index or 0) as clk:
        t_start.record(stream)
        for _ in range(a.steps):
            step(True)
        t_end.record(stream)
        barrier()
    launches = sum(s["m"].launch_count for s in setups) - launches0
    ms = {}
    for s in setups:
        ms[s["key"]] = {op: sum(e0.elapsed_time(e1) for e0, e1 in s["ev"][op]) for op in ops}
        # per-repeat times too: the paper reports the best of its repeats (Eq. (10))
        ms[s["key"]].update({op + "_each": [e0.elapsed_time(e1) for e0, e1 in s["ev"][op]] for op in ops})
    note = ("256 MB buffer overwritten before every timed op (outside its events; vectors < 2x L2)" if small else
            f"inputs larger than L2 ({min(s['m'].n_local_dofs for s in setups) * 8 / 1e9:.2f} GB or more per "
            "vector >> 126 MB)")
    return ms, t_start.elapsed_time(t_end), launches, clk.summary(), note


def run_ours(a, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1907_08492_b200 as P

    specs = workload_specs(a)
    degrees = [sp.degree for sp in specs]
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    hbm_peak, hbm_src = load_peaks()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    fp64_peak = None
    fp64_peaks = {}
    if not a.quick:
        fp64_peak = P.measure_peak("fp64")
        # the FP64 tensor cores (DMMA) against the DFMA roof, measured
        fp64_peaks = {"dfma_tflops": fp64_peak, "dmma_tflops": P.measure_peak("dmma"),
                      "dmma_and_dfma_interleaved_tflops": P.measure_peak("dmma+dfma")}
    # ---------------------------------------------------------------- setup per degree
    nccl_id = None
    if world > 1:   # one unique id: every degree's mesh shares one NCCL communicator
        obj = [P.get_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    setups = make_setups(specs, rank, world, dev, P, torch, nccl_id)
    op_ms, total_ms, launches, clocks, flush_note = time_steps(setups, a, stream, torch, barrier)
    total_ms = allmax(total_ms)
    ops = {}
    t_mv_sum = 0.0
    dom = {"matvec": [0.0, 0.0], "basis_change": [0.0, 0.0], "chebyshev_step": [0.0, 0.0]}  # bytes, ms
    for s in setups:
        mv, bc, ch = (allmax(op_ms[s["key"]][k]) for k in ("matvec", "basis_change", "cheby"))
        t_mv_sum += mv
        nd = s["n_global"]
        K = a.steps
        cd = a.cheby_degree
        gb = geometry_bytes_per_dof(s["spec"])
        herm = s["spec"].basis == "hermite"
        ch_bytes = nd * (BYTES_PER_DOF["cheby_first"] + (cd - 1) * BYTES_PER_DOF["cheby"] + cd * gb)
        mv_bytes = nd * (BYTES_PER_DOF["matvec"] + gb)
        each = op_ms[s["key"]]["matvec_each"]
        ops[s["key"]] = {
            "n_dofs": nd, "lambda_max": s["lmax"],
            "matvec_dofs_per_s": nd * K / (mv * 1e-3),
            "matvec_dofs_per_s_max": nd / (min(each) * 1e-3),         # best repeat (the paper's convention)
            "matvec_dofs_per_s_median": nd / (float(np.median(each)) * 1e-3),
            "matvec_gbs": mv_bytes * K / (mv * 1e-3) / 1e9,
            "matvec_frac_hbm": mv_bytes * K / (mv * 1e-3) / 1e9 / world / hbm_peak,
            "matvec_bytes_per_dof": mv_bytes / nd,
            "basis_change_dofs_per_s": nd * K / (bc * 1e-3) if herm else None,
            "basis_change_gbs": nd * BYTES_PER_DOF["basis_change"] * K / (bc * 1e-3) / 1e9 if herm else None,
            "cheby_step_dofs_per_s": nd * cd * K / (ch * 1e-3),
            "cheby_sweep_gbs": ch_bytes * K / (ch * 1e-3) / 1e9,
            "cheby_frac_hbm": ch_bytes * K / (ch * 1e-3) / 1e9 / world / hbm_peak,
        }
        if s["spec"].basis == "hermite" and not s["spec"].deform_amp and s["p"] in LMAX_SANITY:
            ops[s["key"]]["lambda_max_sanity"] = LMAX_SANITY[s["p"]]
        dom["matvec"][0] += mv_bytes * K
        dom["matvec"][1] += mv
        if herm:
            dom["basis_change"][0] += nd * BYTES_PER_DOF["basis_change"] * K
            dom["basis_change"][1] += bc
        dom["chebyshev_step"][0] += ch_bytes * K
        dom["chebyshev_step"][1] += ch
    n_sum = sum(s["n_global"] for s in setups)
    value = n_sum * a.steps / (t_mv_sum * 1e-3)
    dom_name = max(dom, key=lambda k: dom[k][1])
    dom = {k: v if v[1] > 0 else [0.0, 1e-30] for k, v in dom.items()}
    ach = dom[dom_name][0] / (dom[dom_name][1] * 1e-3) / 1e9 / world   # per-GPU GB/s
    cart = all(sp.geometry == "constant" and sp.deform_amp == 0 for sp in specs)
    if cart:
        kname = "k_kron4"   # p = 3..8; p = 2 runs the cell-per-thread kernel k_kron3c
    elif all(sp.geometry in ("constant", "per_qpoint") for sp in specs) and os.environ.get("DG_QUAD") != "1":
        kname = "k_quad3"
    else:
        kname = "k_quad"
    # default: the warp-private pipelined kernels of k_bchgw.cu (plane mode k_bchgp at p = 2..7, line mode
    # k_bchgw at p = 8)
    bname = {"4": "k_bchg4", "5": "k_bchgp/k_bchgw", "1": "k_bchg"}.get(os.environ.get("DG_BCHG", ""), "k_bchgp/k_bchgw")
    kernel = {"matvec": f"{kname}<APPLY>", "basis_change": bname,
              "chebyshev_step": f"{kname}<CHEBY_GL>"}[dom_name]
    kper = {q: kernel for q in degrees}
    k3c = os.environ.get("DG_K3C", "1") != "0"
    if cart and dom_name == "chebyshev_step":
        # transformed-residual step (KMODE_CHEBY_GLT) where bit n-3 of DG_CHEBY_GLT is set (the
        # library's default mask 0x77: every n but 6), after one basis-change pass b~ = (T^-T)^(x)3 b per sweep
        glt = int(os.environ.get("DG_CHEBY_GLT", "119"))
        for q in degrees:
            if (glt >> (q - 2)) & 1 and not (q == 2 and k3c):
                kper[q] = "k_kron4<CHEBY_GLT>"
        gq = [q for q in degrees if kper[q].endswith("GLT>")]
        if gq:
            dq = [q for q in degrees if q not in gq and not (q == 2 and k3c)]
            kernel = (f"k_kron4<CHEBY_GLT> (p={','.join(map(str, gq))}; + one basis-change pass per sweep)"
                      + (f" + k_kron4<CHEBY_GL> (p={','.join(map(str, dq))})" if dq else ""))
    if cart and dom_name != "basis_change" and 2 in degrees and k3c:
        kper[2] = f"k_kron3c<{'APPLY' if dom_name == 'matvec' else 'CHEBY_GL'}>"
        kernel = kernel + (" (p=3..8)" if "(p=" not in kernel else "") + " + " + kper[2] + " (p=2)"
    traffic, traffic_note = measured_traffic(a.workload, kper, degrees, dom[dom_name][0] / max(1, a.steps))
    roofline = {"bound": "hbm", "kernel": kernel,
                "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                "traffic": traffic, "traffic_note": traffic_note, "peak_source": hbm_src,
                "per_degree_frac": {k: (o["cheby_frac_hbm"] if dom_name == "chebyshev_step" else o["matvec_frac_hbm"])
                                    for k, o in ops.items()},
                "note": "achieved = algorithmic bytes (matvec/basis change 16 B/DoF, Chebyshev step "
                        "40 B/DoF, first step 32; the transformed-residual sweep's extra basis-change pass on b "
                        "is not counted) / summed CUDA-event time of that op, per GPU"}
    mv_gbs = dom["matvec"][0] / (dom["matvec"][1] * 1e-3) / 1e9 / world
    matvec_roof = {"achieved_gbs": mv_gbs, "frac_hbm": mv_gbs / hbm_peak}
    if fp64_peak:
        matvec_roof["fp64_peak_tflops_measured"] = fp64_peak
        matvec_roof["fp64_peaks_measured"] = fp64_peaks
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded uniform[-1,1) fp64 vectors on Cartesian [0,1]^3 meshes (mirror Dirichlet)",
            "config": {"workload": WORKLOAD_TEXT[a.workload],
                       "degrees": degrees, "n_dofs_total": n_sum,
                       "l2_flush": flush_note,
                       "parallelism": f"z-slab x{world}"},
            "roofline": roofline, "matvec_roofline": matvec_roof, "ops": ops,
            "gpu_launches": launches, "clocks": clocks}

    # ---------------------------------------------------------------- the paper's formulation on C4
    # The general quadrature kernel (cell + face quadrature with a constant merged tensor,
    # PAPER.md:798-804) on the same C4 meshes, matvec only (the paper's benchmark); its roof is
    # FP64: tab:operations FLOP/DoF x DoF/s vs the measured DFMA peak.
    if a.workload == "c4" and not a.quick and world == 1 and not a.no_extras:
        qms, _, _, qclk, _ = time_steps(setups, a, stream, torch, barrier, ops=("matvec",),
                                        apply_flags=P.APPLY_QUADRATURE)
        per = {}
        for s in setups:
            r = s["n_global"] * a.steps / (qms[s["key"]]["matvec"] * 1e-3)
            per[s["key"]] = {"matvec_dofs_per_s": r, "flop_per_dof": OPS_H.get(s["p"]),
                             "tflops": r * OPS_H.get(s["p"], 0) / 1e12,
                             "frac_fp64": (r * OPS_H.get(s["p"], 0) / 1e12 / fp64_peak) if fp64_peak else None,
                             "frac_hbm": r * 16 / 1e9 / hbm_peak}
        line["c4_paper_formulation"] = {
            "workload": "C4 meshes through the general quadrature kernel k_quad3 (DG_APPLY_QUADRATURE): "
                        "cell + face quadrature with the constant merged tensor, the paper's benchmark setup",
            "value": sum(s["n_global"] for s in setups) * a.steps
            / (sum(qms[s["key"]]["matvec"] for s in setups) * 1e-3),
            "unit": UNIT, "ops": per, "clocks": qclk,
            "roof": "fp64: tab:operations opsH FLOP/DoF x DoF/s over dg_measure_peak(fp64)"}

    # ---------------------------------------------------------------- FDM smoother (extra)
    # the same fused Chebyshev sweep around the FDM block-Jacobi
    # inner preconditioner (Eqs. (13)-(15)); measured after the timed region, not part of
    # `value`.  Algorithmic bytes 32 B/DoF per step (b, u_j, u_{j-1} in, u_{j+1} out; the
    # FDM diagonal is computed in the kernel), first step 24.
    if a.workload in ("c4", "c5") and not a.quick:
        for s in setups:
            m_ = s["m"]
            x2 = torch.zeros_like(s["x"])
            m_.chebyshev_smooth(s["b"], x2, 1.7, degree=a.cheby_degree, work2=s["work2"], inner="fdm")
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(a.steps):
                m_.chebyshev_smooth(s["b"], x2, 1.7, degree=a.cheby_degree, work2=s["work2"], inner="fdm")
            e1.record(stream)
            barrier()
            ms = allmax(e0.elapsed_time(e1))
            nd, cd = s["n_global"], a.cheby_degree
            ops[s["key"]]["cheby_fdm_step_dofs_per_s"] = nd * cd * a.steps / (ms * 1e-3)
            ops[s["key"]]["cheby_fdm_sweep_gbs"] = nd * (24.0 + 32.0 * (cd - 1)) * a.steps / (ms * 1e-3) / 1e9
    # ---------------------------------------------------------------- fp32 path (extra)
    # the same matvec and GL-Jacobi Chebyshev sweep in fp32 (8 B/DoF
    # per vector access: matvec 8 B/DoF, Chebyshev step 20 B/DoF); after the timed region,
    # not part of `value`.
    if a.workload in ("c4", "c5") and not a.quick and world == 1:
        for s in setups:
            m_ = s["m"]
            u32, b32 = s["u"].float(), s["b"].float()
            y32 = torch.empty_like(u32)
            x32 = torch.zeros_like(u32)
            w32 = torch.empty(2 * u32.numel(), dtype=torch.float32, device=dev)
            m_.apply_laplace_f32(u32, y32)
            m_.chebyshev_smooth_f32(b32, x32, s["lmax"], degree=a.cheby_degree, work2=w32)
            barrier()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(stream)
            for _ in range(a.steps):
                m_.apply_laplace_f32(u32, y32)
            e[1].record(stream)
            for _ in range(a.steps):
                m_.chebyshev_smooth_f32(b32, x32, s["lmax"], degree=a.cheby_degree, work2=w32)
            e[2].record(stream)
            barrier()
            nd, cd = s["n_global"], a.cheby_degree
            ops[s["key"]]["matvec_f32_dofs_per_s"] = nd * a.steps / (e[0].elapsed_time(e[1]) * 1e-3)
            ops[s["key"]]["cheby_f32_step_dofs_per_s"] = nd * cd * a.steps / (e[1].elapsed_time(e[2]) * 1e-3)
            del u32, b32, y32, x32, w32
    # ---------------------------------------------------------------- e2e (host buffers)
    if not a.no_e2e and not a.quick:
        h2d = d2h = 0
        e2e_ms = 0.0
        for s in setups:
            nl = s["m"].n_local_dofs
            uh = torch.empty(nl, dtype=torch.float64, pin_memory=True)
            uh.copy_(s["u"].cpu())
            yh = torch.empty(nl, dtype=torch.float64, pin_memory=True)
            for _ in range(max(1, a.warmup)):   # warm-up: staging buffers, streams
                s["m"].apply_laplace_host(uh, yh, stream=stream)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(a.steps):
                s["m"].apply_laplace_host(uh, yh, stream=stream)
            e1.record(stream)
            barrier()
            e2e_ms += allmax(e0.elapsed_time(e1))
            h2d += 8 * s["n_global"]
            d2h += 8 * s["n_global"]
            del uh, yh
        line["e2e"] = {"value": n_sum * a.steps / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h,
                       "note": f"{a.steps} steps of: per degree, dg_apply_laplace_host on pinned host vectors "
                               "(H2D of u, matvec, D2H of y in overlapped z-plane chunks inside the call); "
                               "CUDA events around the K steps, summed over the sweep"}
    # ---------------------------------------------------------------- other BASELINE configs
    # C3 (curved, per-q-point geometry, k_quad3), C5 (453M DoF, one GPU) and C2 (Hermite vs nodal
    # GL): the same step (matvec, basis change, degree-5 Chebyshev) with their own clocks; extra
    # keys, not part of `value`.
    if a.workload == "c4" and not a.quick and world == 1 and not a.no_extras:
        del setups
        torch.cuda.empty_cache()
        extras = {}
        for name, specs_x in (("c3", [CONFIGS["C3"]]), ("c5", [CONFIGS["C5"]]),
                              ("c2", [CONFIGS["C2"], CONFIGS["C2_GL"]])):
            sx = make_setups(specs_x, 0, 1, dev, P, torch)
            xms, xtot, xl, xclk, xnote = time_steps(sx, a, stream, torch, barrier)
            per = {}
            for s_ in sx:
                nd, K, cd = s_["n_global"], a.steps, a.cheby_degree
                gb = geometry_bytes_per_dof(s_["spec"])
                mv, bc, ch = (xms[s_["key"]][k] for k in ("matvec", "basis_change", "cheby"))
                mvb = nd * (16.0 + gb)
                chb = nd * (BYTES_PER_DOF["cheby_first"] + (cd - 1) * BYTES_PER_DOF["cheby"] + cd * gb)
                herm = s_["spec"].basis == "hermite"
                per[s_["key"]] = {
                    "n_dofs": nd, "lambda_max": s_["lmax"], "bytes_per_dof_matvec": mvb / nd,
                    "matvec_dofs_per_s": nd * K / (mv * 1e-3), "matvec_gbs": mvb * K / (mv * 1e-3) / 1e9,
                    "matvec_frac_hbm": mvb * K / (mv * 1e-3) / 1e9 / hbm_peak,
                    "basis_change_gbs": nd * 16.0 * K / (bc * 1e-3) / 1e9 if herm else None,
                    "cheby_step_dofs_per_s": nd * cd * K / (ch * 1e-3),
                    "cheby_sweep_gbs": chb * K / (ch * 1e-3) / 1e9,
                    "cheby_frac_hbm": chb * K / (ch * 1e-3) / 1e9 / hbm_peak}
            extras[name] = {"workload": WORKLOAD_TEXT[name], "ops": per, "clocks": xclk, "l2_flush": xnote,
                            "ms_per_step": xtot / a.steps, "gpu_launches": xl}
            del sx
            torch.cuda.empty_cache()
        line["workloads"] = extras

    # ---------------------------------------------------------------- CPU oracle baseline
    if rank == 0 and world == 1 and not a.no_cpu_baseline and not a.quick:
        dofs = secs = 0.0
        cells = {}
        for p in sorted(set(degrees)):
            r, c, t = oracle_rate(p, 2.0)
            dofs += r * t
            secs += t
            cells[p] = c
        single = dofs / secs
        try:
            allc, ncores, per_deg = oracle_rate_all_cores(sorted(set(degrees)), 1.5)
        except Exception as e:   # noqa: BLE001 - a host without fork keeps the single-core figure
            allc, ncores, per_deg = None, 1, {"error": str(e)}
        value_cpu = allc if allc else single
        line["cpu_baseline"] = {"value": value_cpu, "unit": UNIT, "cores": ncores if allc else 1,
                                "kind": "oracle",
                                "host_cpu_count": os.cpu_count(),
                                "single_core_value": single,
                                "all_core_per_degree": per_deg,
                                "sample": f"naive numpy quadrature matvec (oracle, untuned). all-core value: one "
                                          f"process per host core, each ~1.5 s per degree on random cells of a "
                                          f"12^3-cell mesh of that degree (per-cell work is size-independent); "
                                          f"single_core_value: one thread, ~2 s per degree on random cells of "
                                          f"each C4 mesh, cells {cells}; sweep rate = harmonic mean over degrees"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    a = args_()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank)
        return
    if world > 1:
        # NCCL init log (ranks, channels, NVLS) for the scaling runs; INIT subsystem only
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ours(a, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
