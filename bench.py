"""Benchmark of the explicit-step hot path (BASELINE.json metric:
explicit-step DoF-updates/s (fp64) + % of the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
    python bench.py --impl reference ...     # CPU oracle port, rank 0 only

A step is one forward-Euler update of the whole mesh (operator apply +
lumped-capacity update + moving source + top-surface losses + Dirichlet
pin + stability check + history).  Timing: W untimed warm-up steps, then
K steps each bracketed by CUDA events on the library's stream, with L2
flushed (256 MiB write) before every timed step outside the events; the
per-rank time is the sum, the job time the max over ranks.

Under torchrun (N > 1) every rank runs its own copy of the workload on
its GPU ("replicas"; the z-slab partition with halo exchange is
DESIGN.md §6 work in progress), value = DoF-updates of all ranks / max
time.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_FLUSH_BYTES = 256 << 20


# ---------------------------------------------------------------------------
# workloads (BASELINE.json configs; synthetic inputs of the stated shapes)
# ---------------------------------------------------------------------------

def workload_config0(n_steps):
    """configs[0]: 64x64x32 Q1 (139,425 DoFs), k = 6.7, 70 W beam at
    1 m/s along y = 1 mm, dt = 1 us, bottom Dirichlet 300 K."""
    import paper_2302_05164_b200 as st
    h = 31.25e-6
    box = st.StructuredBox(64, 64, 32, h, degree=1)
    mat = st.MaterialParams(k_p=6.7, k_m=6.7, k_s=6.7, rho=4430.0, c=526.0)
    bnd = st.BoundaryParams(emissivity=0.0, T_inf=300.0, T_v=1e9)
    las = st.HeatSourceParams(radius=50e-6, h_powder=40e-6, power=70.0, scan_velocity=1.0)
    params = st.ProcessParams(mat, bnd, las, st.MeshParams(h_coarse=h, n_refine=0, h_powder=h))
    T0 = 300.0 + np.random.default_rng(0).uniform(0.0, 1.0, box.n_vertices)
    dt = 1e-6
    # the beam crosses the plate: 2 mm at 1 m/s = 2000 steps of 1 us
    lp = st.LayerPath(0, 0.0, [st.Segment(0.0, 1e-3, 2e-3, 1e-3, 1.0, 70.0)], 0.0)
    return dict(name="config0_q1_64x64x32", box=box, params=params, T0=T0, rc=1.0,
                dt=dt, paths=[lp], degree=1, dofs=box.n_dofs,
                cfg={"mesh": "64x64x32 Q1", "dofs": box.n_dofs, "dt": dt,
                     "material": "k=6.7 const", "beams": 1})


WORKLOADS = {"config0": workload_config0}


def make_operator(w):
    import paper_2302_05164_b200 as st
    box = w["box"]
    try:
        op = st.ThermalOperator(box, box, w["params"], st.SolverSettings())
        backend = "structured"
    except Exception:
        if w["degree"] != 1:
            raise
        forest, dm = box.to_forest_dofmap()
        op = st.ThermalOperator(forest, dm, w["params"], st.SolverSettings())
        backend = "unstructured"
    return op, backend


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

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
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def measured_hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port (numpy restatement of the reference path)
# ---------------------------------------------------------------------------

def cpu_baseline(w, seconds=15.0):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from cpu_oracle import OracleOperator, structured_tables
    from threadpoolctl import threadpool_limits
    box = w["box"]
    cores = os.cpu_count() or 1
    orc = OracleOperator(structured_tables(box.nx, box.ny, box.nz, box.h, w["degree"]),
                         w["params"])
    q = w["degree"] + 1
    rc = np.ones((box.n_cells, q, q, q))
    T = w["T0"].copy()
    from paper_2302_05164_b200.physics import flatten_schedule
    dts, beams = flatten_schedule(w["paths"], w["dt"], 200)
    from cpu_oracle import beam_tuple
    n = 0
    with threadpool_limits(limits=cores):
        orc.capacity_inverse()
        t0 = time.perf_counter()
        while True:
            T = orc.explicit_step(T, float(dts[n % 200]), rc,
                                  [beam_tuple(b) for b in beams[n % 200]])
            rc = orc.update_history(rc, T)
            n += 1
            if time.perf_counter() - t0 > seconds:
                break
        el = time.perf_counter() - t0
    return {"value": w["dofs"] * n / el, "unit": "DoF-updates/s", "cores": cores,
            "kind": "port",
            "sample": f"{n} full explicit steps (+history) of {w['name']} with the numpy oracle "
                      f"port (oracle/cpu_oracle.py), BLAS threads <= {cores}"}


# ---------------------------------------------------------------------------
# runs
# ---------------------------------------------------------------------------

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    from paper_2302_05164_b200.physics import flatten_schedule
    w = WORKLOADS[args.workload](args.warmup + args.steps)
    op, backend = make_operator(w)
    dts, beams = flatten_schedule(w["paths"], w["dt"], args.warmup + args.steps)
    op.set_state(w["T0"], w["rc"])
    # warm-up (untimed)
    op.bench_explicit(dts[:args.warmup], beams[:args.warmup], 0)
    launches0 = op.launches
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        step_ms, main_ms = op.bench_explicit(dts[args.warmup:], beams[args.warmup:],
                                             L2_FLUSH_BYTES)
    torch.cuda.synchronize()
    launches = op.launches - launches0
    total_ms = float(np.sum(step_ms))
    if ws > 1:
        t = torch.tensor([total_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
        torch.distributed.barrier()
    dof_updates = w["dofs"] * args.steps * ws
    value = dof_updates / (total_ms * 1e-3)

    # end to end through the public API: host T in, K steps, host T out
    T_host = np.ascontiguousarray(w["T0"])
    t0 = time.perf_counter()
    op.set_state(T_host, w["rc"])
    fail, _, _ = op.run_explicit(dts[args.warmup:], beams[args.warmup:])
    T_out, rc_out = op.get_state()
    e2e_s = time.perf_counter() - t0
    assert fail == 0 and np.all(np.isfinite(T_out))
    nb = beams.shape[1]
    h2d = T_host.nbytes + (0 if np.isscalar(w["rc"]) else np.asarray(w["rc"]).nbytes) \
        + args.steps * (nb * 40 + 8)
    d2h = T_out.nbytes + rc_out.nbytes
    e2e = {"value": w["dofs"] * args.steps / e2e_s, "unit": "DoF-updates/s",
           "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
           "api": "ThermalOperator.set_state + run_explicit (st_explicit_steps) + get_state, "
                  "host buffers, wall clock"}

    bpd = op.bytes_per_dof()
    main_avg_s = float(np.mean(main_ms)) * 1e-3
    peak, peak_kind = measured_hbm_peak()
    achieved = bpd * w["dofs"] / main_avg_s / 1e9
    _, _, main_name = op.profile_read()
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None, "kernel": main_name,
                "bytes_per_dof": bpd, "peak_source": peak_kind,
                "kernel_share_of_step": float(np.sum(main_ms) / np.sum(step_ms))}
    out = {"metric": "explicit-step DoF-updates/s (fp64)", "value": value,
           "unit": "DoF-updates/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": total_ms / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": dict(workload=w["name"], backend=backend, l2="flushed (256 MiB write) "
                          "before every timed step", parallelism=f"replicas x{ws}", **w["cfg"]),
           "e2e": e2e, "roofline": roofline, "gpu_launches": int(launches),
           "clocks": clk.summary()}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(w, seconds=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    w = WORKLOADS[args.workload](200)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    per = []
    for _ in range(args.warmup + args.steps):
        r = cpu_baseline(w, seconds=args.cpu_seconds / max(1, args.steps))
        per.append(r)
    vals = [r["value"] for r in per[args.warmup:]]
    v = float(np.mean(vals))
    cb = dict(per[-1])
    cb["value"] = v
    out = {"impl": "reference", "metric": "explicit-step DoF-updates/s (fp64)", "value": v,
           "unit": "DoF-updates/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": w["dofs"] / v * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": dict(workload=w["name"], **w["cfg"]), "cpu_baseline": cb,
           "e2e": {"value": v, "unit": "DoF-updates/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config0", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
