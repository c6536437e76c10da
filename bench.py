"""Benchmark of the explicit-step hot path (BASELINE.json metric:
explicit-step DoF-updates/s (fp64) + % of the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
    python bench.py --impl reference ...     # CPU oracle port, rank 0 only

Default workload: BASELINE configs[1] (128x128x32 Q2 cells, 4,293,185
DoFs, k(T) + latent heat + radiation/convection, 70 W beam on a 5-track
hatch, dt = 0.5 us).  A step is one forward-Euler update of the whole
mesh: operator apply + lumped-capacity update (apparent heat capacity) +
moving source + top-surface losses + Dirichlet pin + stability check.

Timing: W untimed warm-up steps, then K steps each bracketed by CUDA
events on the library's stream, with L2 flushed (256 MiB write) before
every timed step outside the events; per-rank time = sum of the step
times, job time = max over ranks.  ``sweep`` adds BASELINE configs[2]
(~50M DoFs at degree 1..4, inputs larger than L2) measured the same way.

Under torchrun (N > 1) the global box is the workload box repeated N
times along x and split into x-slabs, one per GPU (weak scaling); every
step exchanges the rank-interface partial sums over NCCL on the
library's stream (paper_2302_05164_b200/distributed.py).  value = DoF-
updates of the whole box / max over ranks of the summed step times.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

from workloads import (CELLS_50M, WORKLOADS, _st, build_part, build_problem,  # noqa: F401
                       schedule, workload_config0, workload_config1, workload_config2)

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_FLUSH_BYTES = 256 << 20
L2_NOTE = ("flushed before every timed step: 256 MiB write, then a 256 MiB read of a second "
           "buffer (the flush's dirty lines are written back outside the timed region)")
METRIC = "explicit-step DoF-updates/s (fp64)"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class Clocks:
    """SM clock and throttle reasons sampled during the timed region: NVML
    every millisecond (the timed regions are tens of ms), nvidia-smi as a
    fallback."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            phys = int(vis.split(",")[index]) if vis and vis.split(",")[0].isdigit() else index
            h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            bits = [pynvml.nvmlClocksEventReasonHwSlowdown,
                    pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwPowerCap]
            self._nvml = (pynvml, h, bits)
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h, bits = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        return [str(sm), str(mx)] + ["Active" if r & bt else "Not Active" for bt in bits]

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml:
                    self.samples.append(self._sample_nvml())
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                          f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.001 if self._nvml else 0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [v for v in (num(s[0]) for s in self.samples) if v is not None]
        mx = [v for v in (num(s[1]) for s in self.samples) if v is not None]
        reasons = sorted({self.NAMES[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def fp64_peak_tflops(flop_per_cycle=None):
    """Measured fp64 peak of this B200 pool (tools/fp64_peak.cu: independent
    DFMA chains on every SM, CUDA events; profiles/r2/fp64_peak.json), else
    148 SMs x 64 DFMA lanes x 2 flop x max SM clock.  Returns (TF/s, how)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2", "fp64_peak.json")) as f:
            vals = [json.loads(l) for l in f if l.strip()]
        best = max(v["tflops"] for v in vals if "tflops" in v)
        return best, "measured (profiles/r2/fp64_peak.json, tools/fp64_peak.cu)"
    except Exception:
        pass
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f)["sm_max_mhz"])
    except Exception:
        mhz = 1965.0
    return (flop_per_cycle or 148 * 64 * 2) * mhz * 1e6 / 1e12, "computed (lanes x clock)"


# algorithmic bytes per DoF-update of the explicit step on a
# structured mesh -- T_n read + T_{n+1} write + one per-DoF diagonal (C~^-1)
# read.  The kernel here evaluates C~^-1 from the tensor-product lumped mass
# instead of reading it, so 16 B is the least it must move; the roofline is
# reported at the contract's 24 B with the 16 B figure alongside.
B_ALG = 24.0


def measured_hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# CPU: the oracle port (numpy restatement of the reference path)
# ---------------------------------------------------------------------------

class CpuSample:
    """The oracle on a bounded sub-box of the workload (same physics,
    same degree); rates are per DoF so the sub-box is representative."""

    def __init__(self, w):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from cpu_oracle import OracleOperator, structured_tables
        nx, ny, nz = w["sample"]
        self.dims = (nx, ny, nz)
        origin = w.get("sample_origin", (0.0, 0.0, None))
        self.orc = OracleOperator(structured_tables(nx, ny, nz, w["h"], w["degree"],
                                                    origin=origin), w["params"])
        q = w["degree"] + 1
        self.rc = np.ones((self.orc.n, q, q, q))
        self.T = w["T0"](self.orc.nv)
        self.dts, beams = schedule(w, 64)
        from cpu_oracle import beam_tuple
        self.beams = [[beam_tuple(b) for b in row] for row in beams]
        self.n_dofs = self.orc.nv
        self.i = 0
        self.w = w

    def step(self):
        k = self.i % len(self.dts)
        self.T = self.orc.explicit_step(self.T, float(self.dts[k]), self.rc, self.beams[k])
        self.rc = self.orc.update_history(self.rc, self.T)
        self.i += 1

    def describe(self, n):
        nx, ny, nz = self.dims
        return (f"{n} explicit steps (+history) on a {nx}x{ny}x{nz}-cell Q{self.w['degree']} "
                f"block ({self.n_dofs} DoFs, same h, material, dt and beams, under the first "
                f"beam) of {self.w['name']} with the numpy oracle port (oracle/cpu_oracle.py); "
                f"the rate is per DoF")


def cpu_baseline(w, seconds=15.0):
    from threadpoolctl import threadpool_limits
    cores = os.cpu_count() or 1
    s = CpuSample(w)
    with threadpool_limits(limits=cores):
        s.step()  # warm (capacity cache, imports)
        n = 0
        t0 = time.perf_counter()
        while n < 1 or time.perf_counter() - t0 < seconds:
            s.step()
            n += 1
        el = time.perf_counter() - t0
    return {"value": s.n_dofs * n / el, "unit": "DoF-updates/s", "cores": cores,
            "kind": "port", "sample": s.describe(n) + f", BLAS threads <= {cores}"}


# ---------------------------------------------------------------------------
# GPU runs
# ---------------------------------------------------------------------------

def ncu_traffic(key, kernel):
    """DRAM bytes per launch of the hot kernel from the committed ncu
    capture of the same workload (profiles/traffic.json), if it is the
    kernel that ran."""
    try:
        idx = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except (OSError, ValueError):
        return None
    e = idx.get(key or "")
    if not e or not kernel or kernel.split("<")[0] not in e["kernel"]:
        return None
    return e


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def gpu_measure(w, steps, warmup, device, clocks=True):
    st = _st()
    box = build_part(w)
    op = st.ThermalOperator(box, box, w["params"], st.SolverSettings(), device=device)
    dts, beams = schedule(w, warmup + steps)
    T0 = w["T0"](box.n_vertices)
    op.set_state(T0, 1.0)           # consolidated material: r_c = 1 everywhere
    op.bench_explicit(dts[:warmup], beams[:warmup], 0)
    launches0 = op.launches
    clk = Clocks(device) if clocks else None
    if clk:
        clk.__enter__()
    step_ms, main_ms = op.bench_explicit(dts[warmup:], beams[warmup:], L2_FLUSH_BYTES)
    if clk:
        clk.__exit__()
    launches = op.launches - launches0
    bpd_kernel = op.bytes_per_dof()
    bpd = max(B_ALG, bpd_kernel)
    main_avg_s = float(np.mean(main_ms)) * 1e-3
    peak, peak_kind = measured_hbm_peak()
    achieved = bpd * box.n_dofs / main_avg_s / 1e9
    _, _, main_name = op.profile_read()
    ncu = ncu_traffic(w.get("key"), main_name)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu.get("dram_bytes") if ncu else None,
                "kernel": main_name,
                "bytes_per_dof": bpd, "peak_source": peak_kind,
                "kernel_min_bytes_per_dof": bpd_kernel,
                "frac_at_kernel_min_bytes": bpd_kernel * box.n_dofs / main_avg_s / 1e9 / peak,
                "step_frac": bpd * box.n_dofs / (float(np.mean(step_ms)) * 1e-3) / 1e9 / peak,
                "kernel_ms": float(np.mean(main_ms)),
                "kernel_share_of_step": float(np.sum(main_ms) / np.sum(step_ms))}
    if ncu:
        roofline["ncu"] = {k: ncu[k] for k in ("fp64_pipe_pct", "issue_active_pct", "duration_us",
                                               "source") if k in ncu}
        if ncu.get("fp64_flop"):
            # the kernel is fp64-issue bound, not HBM bound: its
            # fp64 flop per launch (ncu instruction counts of the same
            # workload) over the live-measured launch time, against the fp64
            # peak (64 DFMA lanes per SM x 2 flop x SMs x max SM clock)
            peak, how = fp64_peak_tflops(ncu.get("fp64_peak_flop_per_cycle"))
            ach = ncu["fp64_flop"] / main_avg_s / 1e12
            roofline["fp64"] = {"achieved": ach, "peak": peak, "unit": "TFLOP/s",
                                "frac": ach / peak, "peak_source": how,
                                "flop_per_dof": ncu["fp64_flop"] / box.n_dofs}
    return dict(op=op, box=box, dts=dts, beams=beams, T0=T0, step_ms=step_ms,
                launches=launches, roofline=roofline, clocks=clk.summary() if clk else None)


def run_slabs(args):
    """N > 1, one x-slab per GPU.  Default (config 4): strong scaling -- the
    957M-DoF part cut into N slabs balanced by cumulative DoFs
    (distributed.balanced_partition); ``--scaling weak`` repeats a box
    workload N times along x instead.  Every step: interface chunks, packed
    interface planes, NCCL exchange on a communication stream overlapping
    the interior chunks, seam pass; a cross-rank MAX stability check every
    32 steps.  The timed region is the whole K-step loop (checks included)
    between CUDA events on every rank, max over ranks; the per-rank inputs
    (>= 1.2e8 DoFs of T) are larger than L2, no flush."""
    import torch
    import torch.distributed as dist
    from paper_2302_05164_b200.distributed import (GpuSlabStepper, SlabDriver,
                                                   balanced_partition, partition, slab_of,
                                                   torch_exchange, torch_max_reducer)
    st = _st()
    ws, rank, local = dist_env()
    # ST_DIST_BACKEND=gloo: functional check of this path where the ranks
    # cannot have a GPU each (the exchange is staged through the host and
    # the ranks share the visible GPUs round-robin); never a measurement
    backend = os.environ.get("ST_DIST_BACKEND", "nccl")
    if backend == "gloo":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if backend == "gloo":
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    red_dev = "cpu" if backend == "gloo" else "cuda"
    w = dict(WORKLOADS[args.workload](), key=args.workload)
    weak = args.scaling == "weak" or w.get("xext") is None
    if weak:
        nx, ny, nz = w["dims"]
        glob = st.StructuredBox(nx * ws, ny, nz, w["h"], degree=w["degree"])
        parts = partition(glob.nx, ws)
    else:
        glob = build_part(w)
        parts = balanced_partition(glob, ws)
    box = slab_of(glob, *parts[rank], rank, ws)
    op = st.ThermalOperator(box, box, w["params"], st.SolverSettings(), device=local)
    if hasattr(box, "g_lo") and "T0_slice" in w:
        T_loc = w["T0_slice"](box.g_lo, box.g_hi)
    else:
        T_loc = box.local_of(w["T0"](glob.n_vertices))
    op.set_state(T_loc, 1.0)
    stepper = GpuSlabStepper(op)
    drv = SlabDriver(stepper, torch_exchange(rank, ws), reduce_max=torch_max_reducer())
    dts, beams = schedule(w, args.warmup + args.steps)
    with torch.cuda.stream(stepper.stream):
        drv.run(dts[:args.warmup], beams[:args.warmup], check_every=32)
        torch.cuda.synchronize()
        dist.barrier()
        launches0 = op.launches
        clk = Clocks(local)
        clk.__enter__()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tmax = drv.run(dts[args.warmup:], beams[args.warmup:], check_every=32)
        e1.record()
        torch.cuda.synchronize()
        clk.__exit__()
    launches = op.launches - launches0
    total_ms = e0.elapsed_time(e1)
    t = torch.tensor([total_ms], device=red_dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    # end to end: host slab in -> K split steps with the exchange -> host out
    # (pinned host buffers, as in the single-GPU line)
    T_host = torch.empty(len(T_loc), dtype=torch.float64, pin_memory=True).numpy()
    T_host[:] = T_loc
    T_buf = torch.empty(len(T_loc), dtype=torch.float64, pin_memory=True).numpy()
    dist.barrier()
    t0 = time.perf_counter()
    op.set_state(T_host, 1.0)
    with torch.cuda.stream(stepper.stream):
        drv.run(dts[args.warmup:], beams[args.warmup:], check_every=32)
    T_out, rc_out = op.get_state(out=T_buf)
    e2e_s = torch.tensor([time.perf_counter() - t0], device=red_dev)
    dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    nb = beams.shape[1]
    dofs_total = glob.n_dofs
    e2e = {"value": dofs_total * args.steps / float(e2e_s.item()), "unit": "DoF-updates/s",
           "h2d_bytes_per_step": (T_host.nbytes + args.steps * nb * 40) / args.steps,
           "d2h_bytes_per_step": (T_out.nbytes + (0 if rc_out.strides == (0,) else rc_out.nbytes))
           / args.steps,
           "api": "per rank: set_state + split steps (NCCL exchange, stability check every "
                  "32 steps) + get_state; max over ranks"}
    value = dofs_total * args.steps / (total_ms * 1e-3)
    # per GPU, over the whole split step (cells, exchange, seam pass, stability
    # checks) -- the kernel alone is the N = 1 line's roofline
    peak, peak_kind = measured_hbm_peak()
    ach = B_ALG * value / ws / 1e9
    roofline = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "traffic": None, "bytes_per_dof": B_ALG,
                "peak_source": peak_kind,
                "scope": "per GPU, whole split step (max over ranks), not the kernel alone"}
    dist.barrier()
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "DoF-updates/s", "n_gpus": ws,
               "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": total_ms / args.steps, "higher_is_better": True,
               "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic",
               "config": dict(workload=w["name"] + (f"_x{ws}" if weak else ""), dofs=dofs_total,
                              backend="structured x-slabs",
                              partition=[list(p) for p in parts],
                              parallelism=f"x-slab dp{ws}, NCCL partial-sum interface exchange "
                                          "overlapped with the interior chunks"
                                          + (" [ST_DIST_BACKEND=gloo: host-staged functional "
                                             "check, not a measurement]"
                                             if backend == "gloo" else ""),
                              l2="inputs larger than L2 (no flush)", **w["cfg"]),
               "e2e": e2e, "roofline": roofline, "gpu_launches": int(launches),
               "clocks": clk.summary(), "t_max": tmax}
        print(json.dumps(out), flush=True)
    op.close()
    dist.destroy_process_group()


def implicit_measure(device, n_steps=10, cpu=True):
    """Backward-Euler cool-down steps (Newton + Jacobi-PCG on the device,
    SURVEY §8 rows a14-a18) on a BASELINE configs[3]-sized Q1 mesh: a
    40x40x14 box through the unstructured (Forest/DofMap) backend, 24,600
    DoFs, reference default material, krylov_tol 1e-10, dt 1 ms, from a
    synthetic post-scan field (300 K + a 1700 K Gaussian bump at the top).
    Returns ms per BE step, iterations, and (CPU-baseline leg) the oracle
    port's time for one step on the host."""
    st = _st()
    h = 80e-6
    box = st.StructuredBox(40, 40, 14, h, degree=1)
    forest, dm = box.to_forest_dofmap()
    params = st.ProcessParams(st.MaterialParams(), st.BoundaryParams(), st.HeatSourceParams(),
                              st.MeshParams(h_coarse=h, n_refine=0, h_powder=h))
    s = st.SolverSettings(explicit_cooldown_steps=0, dt_implicit=1e-3, krylov_tol=1e-10,
                          preconditioner="diagonal")
    op = st.ThermalOperator(forest, dm, params, s, device=device)
    n = op.nv
    NY, NZ = box.ny + 1, box.nz + 1  # vertex lattice, x-major / z-fastest (mesh.py:712-715)
    idx = np.arange(n)
    x, y, z = (idx // (NY * NZ)) * h, ((idx // NZ) % NY) * h, (idx % NZ - box.nz) * h
    r2 = (x - 20 * h) ** 2 + (y - 20 * h) ** 2 + z ** 2
    T0 = 300.0 + 1700.0 * np.exp(-r2 / (4e-4) ** 2)
    rc0 = np.ones(op.n_cells * op.qpc)
    op.set_state(T0, rc0)
    op.implicit_step(1e-3, s)
    op.finish_implicit_step()
    op.set_state(T0, rc0)
    nn = nk = 0
    t0 = time.perf_counter()
    for _ in range(n_steps):
        out = op.implicit_step(1e-3, s)
        if out is None:
            raise RuntimeError("implicit step did not converge")
        op.finish_implicit_step()
        nn += out[0]
        nk += out[1]
    el = time.perf_counter() - t0
    # the PCG solve alone (st_pcg: one persistent cooperative launch on this
    # backend), krylov_tol 1e-13 for a longer solve
    rhs = op.evaluate_rhs(T0, rc0, None, faces=False, source=False)
    rhs[dm.is_dirichlet] = 0.0
    op.solve_jacobian(rhs, T0, rc0, 1e-3, 1e-13, 2000)
    tp = time.perf_counter()
    _, pcg_it, _ = op.solve_jacobian(rhs, T0, rc0, 1e-3, 1e-13, 2000)
    el_p = time.perf_counter() - tp
    # the explicit scan steps of the same backend (config 3 integrates 40k
    # of them per layer): 2 x 512 device-resident steps of a 1 m/s track
    lp = st.LayerPath(0, 0.0, [st.Segment(5 * h, 20 * h, 35 * h, 20 * h, 1.0, 70.0)], 0.0)
    dts_e, bm_e = st.flatten_schedule(lp, 1e-6, 1024)
    op.set_state(T0, rc0)
    op.run_explicit(dts_e[:512], bm_e[:512])  # returns after the batch's stability read
    te = time.perf_counter()
    fail, _, _ = op.run_explicit(dts_e[512:], bm_e[512:])
    el_e = time.perf_counter() - te
    res_e = {"explicit_us_per_step": el_e / 512 * 1e6, "explicit_fail": int(fail)}
    # step criteria (row a19 / §8f row 4): the whole power iteration on the
    # device, once per layer in the reference driver (driver.py:225)
    st.compute_step_criteria(op)
    tc = time.perf_counter()
    crit = st.compute_step_criteria(op)
    el_c = time.perf_counter() - tc
    res_c = {"step_criteria_ms": el_c * 1e3, "power_iterations": op.last_power_iterations,
             "dt_stability": crit.dt_stability}
    res = {"workload": "config3-sized cool-down: 40x40x14 Q1 box, unstructured backend",
           "dofs": int(n), "be_steps": n_steps, "ms_per_be_step": el / n_steps * 1e3,
           "newton_per_step": nn / n_steps, "cg_per_step": nk / n_steps,
           "us_per_cg_iteration": el / max(nk, 1) * 1e6,
           "pcg_solve": {"iterations": int(pcg_it), "ms": el_p * 1e3,
                         "us_per_iteration": el_p / max(pcg_it, 1) * 1e6,
                         "note": "st_pcg alone (krylov_tol 1e-13), wall clock incl. the "
                                 "vector copies in and out"},
           **res_e, **res_c}
    if cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from cpu_oracle import OracleOperator, implicit_step, structured_tables
        orc = OracleOperator(structured_tables(box.nx, box.ny, box.nz, h, 1), params)
        t1 = time.perf_counter()
        implicit_step(orc, T0, rc0.reshape(-1, 2, 2, 2), 1e-3, s)
        res["cpu_baseline"] = {"value": (time.perf_counter() - t1) * 1e3, "unit": "ms per BE step",
                               "cores": os.cpu_count() or 1, "kind": "port",
                               "sample": "one BE step of oracle/cpu_oracle.py implicit_step on "
                                         "the same box (the CPU-baseline leg of this entry)"}
        # oracle power iteration: 20 applies timed, scaled to the device's count
        from cpu_oracle import spectral_radius
        mat = params.material
        kf = max(mat.k_m, mat.k_s)
        cinv = orc.capacity_inverse()
        isd = orc.M["is_dirichlet"]

        def apply(v):
            vd = v.copy()
            vd[isd] = 0.0
            w = -orc.evaluate_rhs(vd, None, faces=False, source=False, frozen_k=kf) * cinv
            w[isd] = 0.0
            return w
        t2 = time.perf_counter()
        spectral_radius(apply, orc.nv, max_iter=20)
        per = (time.perf_counter() - t2) / 20
        res["cpu_step_criteria_ms"] = per * op.last_power_iterations * 1e3
        res["cpu_step_criteria_sample"] = ("20 oracle power-iteration applies, scaled to the "
                                           f"{op.last_power_iterations} the device ran")
    op.close()
    return res


def config3_build_measure(cpu=True):
    """BASELINE configs[3] end to end on the device (workloads.run_config3_build:
    the reference's run_build layer loop): ten layers, each = native mesh
    advance + transfer + operator rebuild, device step criteria, the full
    20-track scan (40,000 explicit steps at dt = 1 us) and the 1 s
    backward-Euler cool-down (1000 steps at 1 ms, Jacobi-PCG, krylov_tol
    1e-10).  Wall clock per layer.  CPU leg: the oracle port's explicit step
    and BE step on the layer-0 mesh, scaled to a layer's step counts."""
    import workloads as wl
    t0 = time.perf_counter()
    state, recs = wl.run_config3_build()
    total = time.perf_counter() - t0
    walls = [r["wall_amr"] + r["wall_criteria"] + r["wall_scan"] + r["wall_cool"] for r in recs]
    res = {"workload": "config3: 2x2 mm chamber on a 2 mm plate, Q1, 1 refinement level, "
                       "10 layers x (40,000 explicit + 1000 BE steps), 70 W hatch, rotation 0/90",
           "layers": len(recs), "wall_s_total": total,
           "wall_s_per_layer": float(np.mean(walls)),
           "per_layer": [{k: (round(v, 5) if isinstance(v, float) else v) for k, v in r.items()}
                         for r in recs],
           "scan_steps_per_layer": recs[0]["scan_steps"], "cool_steps_per_layer": recs[0]["cool_steps"],
           "dofs_last_layer": recs[-1]["n_dofs"]}
    state.op.close()
    if cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from cpu_oracle import OracleOperator, implicit_step, tables_from_arrays
        mesh, geo, params, settings = wl.config3_setup()
        st0 = wl.config3_initial_state(mesh, geo, params, settings)
        wl.advance_mesh(st0, params, settings)
        f, dm = st0.forest, st0.dofmap
        from paper_2302_05164_b200.mesh import interface_faces
        fs = interface_faces(f)
        rows = dm.active_rows
        pos = np.full(f.n_cells, -1, dtype=np.int64)
        pos[rows] = np.arange(len(rows))
        M = tables_from_arrays(dm.n_vertices, dm.cell_verts, f.size_m(rows),
                               f.anchor[rows] * f.h_fine, dm.is_slave, dm.is_dirichlet,
                               dm.slaves, dm.slave_ptr, dm.slave_masters, dm.slave_weights,
                               pos[fs.cell_rows], fs.offset, fs.fsize, f.size(rows))
        orc = OracleOperator(M, params)
        paths = wl.config3_layer_paths(geo, mesh)
        from paper_2302_05164_b200.physics import flatten_schedule
        from cpu_oracle import beam_tuple
        dts, bm = flatten_schedule(paths[0], 1e-6, 20)
        T, rc = st0.T.copy(), st0.history.r_c.copy()
        orc.explicit_step(T, 1e-6, rc, [])
        te = time.perf_counter()
        for i in range(20):
            T = orc.explicit_step(T, float(dts[i]), rc, [beam_tuple(b) for b in bm[i]])
            rc = orc.update_history(rc, T)
        t_exp = (time.perf_counter() - te) / 20
        tb = time.perf_counter()
        implicit_step(orc, T, rc, 1e-3, settings)
        t_be = time.perf_counter() - tb
        st0.op.close()
        per_layer = 40000 * t_exp + 1000 * t_be
        res["cpu_baseline"] = {
            "value": per_layer, "unit": "s per layer (extrapolated)", "cores": os.cpu_count() or 1,
            "kind": "port", "sample": f"20 explicit steps ({t_exp * 1e3:.1f} ms each) and one BE "
            f"step ({t_be:.2f} s) of oracle/cpu_oracle.py on the layer-0 mesh, scaled to 40,000 + "
            f"1000 steps (the reference itself measured 2.4-3 h per layer, SURVEY §8d)"}
        res["speedup_per_layer_vs_port"] = per_layer / res["wall_s_per_layer"]
    return res


def snapshot_measure(device, steps=60):
    """the output / checkpoint phase as an asynchronous
    snapshot.  Config 1, K device-resident steps in one st_explicit_steps
    call, with and without a snapshot of T (into pinned host memory) taken
    after the first third: wall clock of the whole call sequence (the
    drain overlaps the steps queued after the snapshot)."""
    import torch
    st = _st()
    w = workload_config1()
    box = build_part(w)
    op = st.ThermalOperator(box, box, w["params"], st.SolverSettings(), device=device)
    dts, beams = schedule(w, steps)
    T0 = w["T0"](box.n_vertices)
    buf = torch.empty(op.nv, dtype=torch.float64, pin_memory=True).numpy()
    k = steps // 3
    res = {}
    for with_snap in (False, True, False, True):
        op.set_state(T0, 1.0)
        t0 = time.perf_counter()
        op.run_explicit(dts[:k], beams[:k])
        if with_snap:
            op.snapshot(buf)
        op.run_explicit(dts[k:], beams[k:])
        if with_snap:
            op.snapshot_wait()
        res["with_snapshot" if with_snap else "without"] = (time.perf_counter() - t0) * 1e3
    Tk = None
    op.set_state(T0, 1.0)
    op.run_explicit(dts[:k], beams[:k])
    Tk, _ = op.get_state()
    op.close()
    return {"workload": w["name"], "steps": steps, "snapshot_after": k,
            "ms_without": res["without"], "ms_with_snapshot": res["with_snapshot"],
            "snapshot_bytes": int(buf.nbytes), "snapshot_equals_state": bool(np.array_equal(buf, Tk)),
            "note": "wall clock of the K-step sequence; the snapshot's D2H drain runs on a copy "
                    "stream while the later steps run"}


def measure_summary(r, steps):
    return {"dofs": r["box"].n_dofs,
            "value": r["box"].n_dofs * steps / (float(np.sum(r["step_ms"])) * 1e-3),
            "ms_per_step": float(np.mean(r["step_ms"])), "roofline": r["roofline"]}


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        return run_slabs(args)
    w = dict(WORKLOADS[args.workload](), key=args.workload)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    r = gpu_measure(w, args.steps, args.warmup, local)
    torch.cuda.synchronize()
    total_ms = float(np.sum(r["step_ms"]))
    if ws > 1:
        t = torch.tensor([total_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
        torch.distributed.barrier()
    dofs = r["box"].n_dofs
    value = dofs * args.steps * ws / (total_ms * 1e-3)

    # end to end through the public API: host T in -> K steps -> host T, r_c out
    op = r["op"]
    dts, beams = r["dts"][args.warmup:], r["beams"][args.warmup:]
    # pinned host buffers for the state in / out (the caller's arrays)
    T_host = torch.empty(len(r["T0"]), dtype=torch.float64, pin_memory=True).numpy()
    T_host[:] = r["T0"]
    T_buf = torch.empty(len(r["T0"]), dtype=torch.float64, pin_memory=True).numpy()
    # one untimed pass (first-touch of the pinned pages and the beam
    # schedule buffer), then the median of three timed passes (wall clock)
    e2e_runs = []
    for rep in range(4):
        t0 = time.perf_counter()
        op.set_state(T_host, 1.0)
        fail, _, _ = op.run_explicit(dts, beams)
        T_out, rc_out = op.get_state(out=T_buf)
        if rep:
            e2e_runs.append(time.perf_counter() - t0)
        if fail or not np.all(np.isfinite(T_out)):
            raise RuntimeError("end-to-end run diverged")
    e2e_s = float(np.median(e2e_runs))
    nb = beams.shape[1]
    h2d = T_host.nbytes + args.steps * (nb * 40 + 8)
    # r_c = 1 stays uniform on the device (never stored, never copied):
    # count only the bytes that crossed the bus
    rc_bytes = 0 if rc_out.strides == (0,) else rc_out.nbytes
    d2h = T_out.nbytes + rc_bytes + args.steps * 16
    e2e = {"value": dofs * args.steps / e2e_s, "unit": "DoF-updates/s",
           "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
           "api": "ThermalOperator.set_state(T pinned host) + run_explicit(K steps, "
                  "st_explicit_steps; per step dt + beams in, stability maxima out) + "
                  "get_state(T into pinned host; uniform r_c as a scalar); wall clock, "
                  "median of 3 passes after one untimed pass"}
    op.close()  # config 4 holds ~150 GB of HBM; the extras below need room
    del T_host, T_buf
    cfg = dict(workload=w["name"], dofs=dofs, backend="structured",
               l2=L2_NOTE,
               parallelism=f"replicas x{ws}", **w["cfg"])
    out = {"metric": METRIC, "value": value, "unit": "DoF-updates/s", "n_gpus": ws,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": cfg, "e2e": e2e, "roofline": r["roofline"],
           "gpu_launches": int(r["launches"]), "clocks": r["clocks"]}
    if rank == 0 and ws == 1 and args.sweep and args.workload != "config1":
        w1 = dict(workload_config1(), key="config1")
        r1 = gpu_measure(w1, args.sweep_steps * 2, 5, local, clocks=False)
        out["config1"] = dict(measure_summary(r1, args.sweep_steps * 2), workload=w1["name"])
        r1["op"].close()
    if rank == 0 and ws == 1 and args.sweep:
        sweep = {}
        for p in (1, 2, 3, 4):
            wp = dict(workload_config2(p), key=f"config2_p{p}")
            rp = gpu_measure(wp, args.sweep_steps, 3, local, clocks=False)
            sweep[f"q{p}"] = {"dofs": rp["box"].n_dofs,
                              "value": rp["box"].n_dofs * args.sweep_steps
                              / (float(np.sum(rp["step_ms"])) * 1e-3),
                              "ms_per_step": float(np.mean(rp["step_ms"])),
                              "roofline_frac": rp["roofline"]["frac"],
                              "kernel": rp["roofline"]["kernel"],
                              "traffic": rp["roofline"]["traffic"],
                              "achieved_GBps": rp["roofline"]["achieved"],
                              "fp64": rp["roofline"].get("fp64")}
            rp["op"].close()
        out["sweep_config2"] = sweep
    if rank == 0 and ws == 1 and args.sweep:
        out["implicit_config3"] = implicit_measure(local, cpu=not args.no_cpu_baseline)
        out["config3_build"] = config3_build_measure(cpu=not args.no_cpu_baseline)
        out["snapshot_config1"] = snapshot_measure(local)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(w, seconds=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def run_reference(args):
    """The reference's CPU path (oracle port; the reference itself is a
    Python package that is not installed on the GPU box) on the same
    workload: each step is one explicit step of a bounded sub-box."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits
    w = dict(WORKLOADS[args.workload](), key=args.workload)
    cores = os.cpu_count() or 1
    s = CpuSample(w)
    with threadpool_limits(limits=cores):
        for _ in range(args.warmup):
            s.step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            s.step()
        el = time.perf_counter() - t0
    v = s.n_dofs * args.steps / el
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "DoF-updates/s",
           "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": dict(workload=w["name"], **w["cfg"]),
           "cpu_baseline": {"value": v, "unit": "DoF-updates/s", "cores": cores, "kind": "port",
                            "sample": s.describe(args.steps) + f", BLAS threads <= {cores}"},
           "e2e": {"value": v, "unit": "DoF-updates/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config4", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sweep", type=int, default=1, help="also measure configs[2], p=1..4")
    ap.add_argument("--sweep-steps", type=int, default=10)
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: strong (config 4 split by DoFs) or weak (box per GPU)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        args.steps = min(args.steps, 20)   # bounded CPU sample per the contract
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
