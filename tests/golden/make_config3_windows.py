"""Config-3 parity windows, made by running the REFERENCE here:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_config3_windows.py

BASELINE configs[3]: 2 x 2 mm chamber on a 2 mm plate, Q1,
MeshParams(h_coarse=80e-6, n_refine=1, h_powder=40e-6), default material
and boundary, 70 W beam, hatch_path(d_h=100 um, v=1 m/s, rotation 0/90),
dt = 1 us.  Windows:
  * layer 0 after its activation: the first 1000 explicit scan steps
    (run_scan_phase, stopped by its on_step hook);
  * then 20 backward-Euler steps (dt_implicit 1 ms, krylov_tol 1e-13,
    Jacobi, no explicit pre-phase) via run_cooldown_phase on a 20 ms
    window;
  * the layer-0 step criteria (rho, dt_stability).
Writes tests/golden/config3_windows.npz (T and r_c at each window end,
iteration counts, rho).
"""

import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import scantherm as st  # noqa: E402
from scantherm.driver import hatch_path  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


class _Stop(Exception):
    pass


def main():
    mesh = st.MeshParams(h_coarse=80e-6, n_refine=1, h_powder=40e-6)
    geo = st.PartGeometry.chamber((2e-3, 2e-3), 10 * 40e-6, 2e-3, mesh)
    params = st.ProcessParams(st.MaterialParams(), st.BoundaryParams(),
                              st.HeatSourceParams(power=70.0, scan_velocity=1.0), mesh)
    settings = st.SolverSettings(explicit_cooldown_steps=0, dt_implicit=1e-3,
                                 krylov_tol=1e-13, preconditioner="diagonal")
    path = hatch_path(geo, mesh, 1e-4, 1.0, 70.0, 1.0, rotation=(0.0, 90.0))
    forest = st.build_coarse_grid(geo, mesh)
    history = st.initial_history(forest)
    dofmap = st.build_dofmap(forest)
    T = np.full(dofmap.n_vertices, params.T_0)
    plan = st.advance_layer(forest, history)
    forest, fields, history = st.apply_update(forest, plan, [st.NodalField(T, forest.epoch)],
                                              history, T_0=params.T_0)
    dofmap = st.build_dofmap(forest)
    op = st.ThermalOperator(forest, dofmap, params, settings)
    state = st.SimulationState(forest, dofmap, op, fields[0].values.copy(), history)
    t0 = time.perf_counter()
    crit = st.compute_step_criteria(op, settings)
    t_crit = time.perf_counter() - t0
    snap = {}

    def hook(s, step, tau):
        if step == 1000:
            snap["T"] = s.T.copy()
            snap["rc"] = s.history.r_c.copy()
            raise _Stop()

    lp = path.layers[0]
    t0 = time.perf_counter()
    try:
        st.run_scan_phase(state, lp, 1e-6, on_step=hook)
    except _Stop:
        pass
    t_scan = time.perf_counter() - t0
    print(f"1000 scan steps in {t_scan:.1f} s, T max {snap['T'].max():.1f}")
    state.T = snap["T"].copy()
    state.history.r_c[...] = snap["rc"]
    win = st.LayerPath(0, lp.z, [], 20e-3)
    t0 = time.perf_counter()
    cool = st.run_cooldown_phase(state, win, 1e-6, settings)
    t_cool = time.perf_counter() - t0
    print(f"{cool.n_steps} BE steps in {t_cool:.1f} s: newton {cool.newton_iters}, "
          f"krylov {cool.krylov_iters}; rho {crit.dt_stability}")
    np.savez_compressed(
        os.path.join(OUT, "config3_windows.npz"),
        T_scan1000=snap["T"], rc_scan1000=snap["rc"], T_be20=state.T.copy(),
        rc_be20=state.history.r_c.copy(),
        be_iters=np.array([cool.n_steps, cool.newton_iters, cool.krylov_iters]),
        dt_stability=np.array(crit.dt_stability), n_vertices=np.array(dofmap.n_vertices),
        wall=np.array([t_crit, t_scan, t_cool]))


if __name__ == "__main__":
    main()
