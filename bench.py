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
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
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


# ----------------------------------------------------------------------------- reference arm
def run_reference(a, rank):
    if rank != 0:
        return
    degrees = [int(x) for x in a.degrees.split(",")]
    per_step_budget = 0.35      # seconds of oracle work per degree per step
    for _ in range(a.warmup):
        for p in degrees:
            oracle_rate(p, 0.05)
    dofs, secs, cells = 0.0, 0.0, {}
    t0 = time.perf_counter()
    for s in range(a.steps):
        for p in degrees:
            r, c, t = oracle_rate(p, per_step_budget, seed=s)
            dofs += r * t
            secs += t
            cells[p] = cells.get(p, 0) + c
    wall = time.perf_counter() - t0
    value = dofs / secs
    sample = (f"oracle matvec (naive quadrature, numpy) on random cells of the C4 meshes, "
              f"{per_step_budget}s per degree per step; cells per degree: {cells}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * wall / a.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded uniform[-1,1) fp64 vectors on Cartesian meshes",
            "config": {"workload": "C4 degree sweep p=2..8 (sampled cells, CPU oracle)",
                       "degrees": degrees},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu_cores_used(), "kind": "oracle",
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
    """DRAM bytes (read + write) per launch of the dominant kernel, from the committed
    ncu capture profiles/r1_traffic.json (one `ncu --metrics dram__bytes_read.sum,
    dram__bytes_write.sum` pass of this workload, per degree), averaged over the degrees
    like `achieved`; None if the capture does not cover this workload/kernel."""
    p = os.path.join(ROOT, "profiles", "r1_traffic.json")
    if not os.path.exists(p):
        return None, "no committed ncu traffic capture"
    with open(p) as f:
        d = json.load(f)
    ent = d.get(workload, {}).get(kernel)
    if not ent or any(str(q) not in ent["per_launch_bytes"] for q in degrees):
        return None, "ncu traffic capture does not cover this configuration"
    per = [ent["per_launch_bytes"][str(q)] for q in degrees]
    alg = [ent["algorithmic_bytes"][str(q)] for q in degrees]
    return float(np.mean(per)), (f"ncu dram read+write per launch, mean over degrees ({ent['source']}); "
                                 f"measured/algorithmic = {sum(per) / sum(alg):.3f}")


WORKLOAD_TEXT = {
    "c4": "C4 degree sweep p=2..8, N_p=round(480/(p+1)) cells per direction, matvec + H->GL basis change "
          "+ degree-5 Chebyshev (GL-Jacobi) per degree",
    "c2": "C2 p=4 32^3 Cartesian, Hermite-like vs nodal Gauss-Lobatto (full-neighbour reads)",
    "c3": "C3 p=5 48^3 curved (amp 0.05), per-quadrature-point geometry, general quadrature kernel",
    "c5": "C5 p=5 128^3 Cartesian (453M DoF), z-slabs",
}


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
    if not a.quick:
        fp64_peak = P.measure_peak("fp64")
    # ---------------------------------------------------------------- setup per degree
    setups = []
    for spec in specs:
        p = spec.degree
        nccl_id = None
        if world > 1:
            obj = [P.get_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nccl_id = obj[0]
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
        lmax = lanczos_lambda_max(m)
        setups.append(dict(p=p, spec=spec, m=m, u=u, b=b, x=x, y=y, v=v, work2=work2, lmax=lmax,
                           n_global=m.n_global_dofs, key=f"p{p}" + ("-gl" if spec.basis == "gl" else "")
                           + ("-curved" if spec.deform_amp else "")))
    torch.cuda.synchronize()
    # L2 (126 MB): vectors smaller than 2x L2 (C2: 33 MB) would stay resident between the timed
    # ops, so then a 256 MB buffer is overwritten before every op, outside its event bracket
    small = min(s["m"].n_local_dofs for s in setups) * 8 < (256 << 20)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if small else None

    def l2_flush():
        if flush is not None:
            flush.fill_(1)

    def step(record):
        for s in setups:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)] if record else None
            l2_flush()
            if record:
                ev[0].record(stream)
            s["m"].apply_laplace(s["u"], s["y"])
            if record:
                ev[1].record(stream)
            l2_flush()
            if record:
                ev[2].record(stream)
            if s["spec"].basis == "hermite":
                s["m"].basis_change("T", s["u"], s["v"])
            if record:
                ev[3].record(stream)
            l2_flush()
            if record:
                ev[4].record(stream)
            s["m"].chebyshev_smooth(s["b"], s["x"], s["lmax"], degree=a.cheby_degree, work2=s["work2"])
            if record:
                ev[5].record(stream)
                s.setdefault("events", []).append(ev)

    for _ in range(a.warmup):
        step(False)
    launches0 = sum(s["m"].launch_count for s in setups)
    barrier()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        t_start.record(stream)
        for _ in range(a.steps):
            step(True)
        t_end.record(stream)
        barrier()
    launches = sum(s["m"].launch_count for s in setups) - launches0
    total_ms = allmax(t_start.elapsed_time(t_end))
    ops = {}
    t_mv_sum = 0.0
    dom = {"matvec": [0.0, 0.0], "basis_change": [0.0, 0.0], "chebyshev_step": [0.0, 0.0]}  # bytes, ms
    for s in setups:
        mv = sum(e[0].elapsed_time(e[1]) for e in s["events"])
        bc = sum(e[2].elapsed_time(e[3]) for e in s["events"])
        ch = sum(e[4].elapsed_time(e[5]) for e in s["events"])
        mv, bc, ch = allmax(mv), allmax(bc), allmax(ch)
        t_mv_sum += mv
        nd = s["n_global"]
        K = a.steps
        cd = a.cheby_degree
        gb = geometry_bytes_per_dof(s["spec"])
        herm = s["spec"].basis == "hermite"
        ch_bytes = nd * (BYTES_PER_DOF["cheby_first"] + (cd - 1) * BYTES_PER_DOF["cheby"] + cd * gb)
        mv_bytes = nd * (BYTES_PER_DOF["matvec"] + gb)
        ops[s["key"]] = {
            "n_dofs": nd, "lambda_max": s["lmax"],
            "matvec_dofs_per_s": nd * K / (mv * 1e-3),
            "matvec_gbs": mv_bytes * K / (mv * 1e-3) / 1e9,
            "matvec_bytes_per_dof": mv_bytes / nd,
            "basis_change_dofs_per_s": nd * K / (bc * 1e-3) if herm else None,
            "basis_change_gbs": nd * BYTES_PER_DOF["basis_change"] * K / (bc * 1e-3) / 1e9 if herm else None,
            "cheby_step_dofs_per_s": nd * cd * K / (ch * 1e-3),
            "cheby_sweep_gbs": ch_bytes * K / (ch * 1e-3) / 1e9,
        }
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
    if all(sp.geometry == "constant" and sp.deform_amp == 0 for sp in specs):
        kname = "k_kron4"
    elif all(sp.geometry in ("constant", "per_qpoint") for sp in specs) and os.environ.get("DG_QUAD") != "1":
        kname = "k_quad3"
    else:
        kname = "k_quad"
    bname = "k_bchg4" if os.environ.get("DG_BCHG") == "4" else "k_bchg"   # k_bchg4 default only at p=2, 8
    kernel = {"matvec": f"{kname}<APPLY>", "basis_change": bname,
              "chebyshev_step": f"{kname}<CHEBY_GL>"}[dom_name]
    traffic, traffic_note = measured_traffic(a.workload, kernel, degrees, dom[dom_name][0] / max(1, a.steps))
    roofline = {"bound": "hbm", "kernel": kernel,
                "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                "traffic": traffic, "traffic_note": traffic_note, "peak_source": hbm_src,
                "note": "achieved = algorithmic bytes (matvec/basis change 16 B/DoF, Chebyshev step "
                        "40 B/DoF, first step 32) / summed CUDA-event time of that op, per GPU"}
    mv_gbs = dom["matvec"][0] / (dom["matvec"][1] * 1e-3) / 1e9 / world
    matvec_roof = {"achieved_gbs": mv_gbs, "frac_hbm": mv_gbs / hbm_peak}
    if fp64_peak:
        matvec_roof["fp64_peak_tflops_measured"] = fp64_peak
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded uniform[-1,1) fp64 vectors on Cartesian [0,1]^3 meshes (mirror Dirichlet)",
            "config": {"workload": WORKLOAD_TEXT[a.workload],
                       "degrees": degrees, "n_dofs_total": n_sum,
                       "l2_flush": ("256 MB buffer overwritten before every timed op (outside its events; "
                                    "vectors < 2x L2)" if small else
                                    f"inputs larger than L2 ({min(s['m'].n_local_dofs for s in setups) * 8 / 1e9:.2f}"
                                    " GB or more per vector >> 126 MB)"),
                       "parallelism": f"z-slab x{world}"},
            "roofline": roofline, "matvec_roofline": matvec_roof, "ops": ops,
            "gpu_launches": launches, "clocks": clk.summary()}

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
            s["m"].apply_laplace_host(uh, yh, stream=stream)   # warm-up: staging buffers, streams
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            s["m"].apply_laplace_host(uh, yh, stream=stream)
            e1.record(stream)
            barrier()
            e2e_ms += allmax(e0.elapsed_time(e1))
            h2d += 8 * s["n_global"]
            d2h += 8 * s["n_global"]
        line["e2e"] = {"value": n_sum / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h,
                       "note": "per degree: dg_apply_laplace_host on pinned host vectors (H2D of u, matvec, D2H "
                               "of y in overlapped z-plane chunks inside the call); summed over the sweep"}
    # ---------------------------------------------------------------- CPU oracle baseline
    if rank == 0 and world == 1 and not a.no_cpu_baseline and not a.quick:
        dofs = secs = 0.0
        cells = {}
        for p in sorted(set(degrees)):
            r, c, t = oracle_rate(p, 3.0)
            dofs += r * t
            secs += t
            cells[p] = c
        line["cpu_baseline"] = {"value": dofs / secs, "unit": UNIT, "cores": cpu_cores_used(),
                                "kind": "oracle",
                                "sample": f"naive numpy quadrature matvec on random cells of each C4 mesh, "
                                          f"~3 s per degree; cells {cells}"}
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
