"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_golden.py [--skip-config0]

Writes tests/golden/*.npz.  The GPU box never runs this script; it only
reads the committed fixtures.  Every array here is an output of the
reference's own code path (scantherm 0.1.0), so the fixtures pin both
the oracle restatement (oracle/cpu_oracle.py) and the CUDA operator.
"""

import argparse
import dataclasses
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import scantherm as st  # noqa: E402
from scantherm import interface_faces  # noqa: E402
from scantherm.timestepping import _implicit_step  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def params_json(params):
    return json.dumps({
        "material": dataclasses.asdict(params.material),
        "boundary": dataclasses.asdict(params.boundary),
        "laser": dataclasses.asdict(params.laser),
        "T_0": params.T_0,
    })


def mesh_arrays(prefix, forest, dofmap):
    fs = interface_faces(forest)
    out = {
        "level": forest.level, "anchor": forest.anchor, "active": forest.active,
        "init_consol": forest.init_consol,
        "meta": np.array([forest.depth, forest.cpl, forest.geometry.z_min(),
                          int(forest.mesh_params.dirichlet_bottom), forest.epoch,
                          forest.current_layer], dtype=np.int64),
        "h_fine": np.array(forest.h_fine),
        "vertices": dofmap.vertices, "cell_verts": dofmap.cell_verts,
        "active_rows": dofmap.active_rows, "is_slave": dofmap.is_slave,
        "is_dirichlet": dofmap.is_dirichlet, "slaves": dofmap.slaves,
        "slave_ptr": dofmap.slave_ptr, "slave_masters": dofmap.slave_masters,
        "slave_weights": dofmap.slave_weights,
        "face_rows": fs.cell_rows, "face_offset": fs.offset, "face_fsize": fs.fsize,
    }
    return {f"{prefix}{k}": np.asarray(v) for k, v in out.items()}


def beam_arr(b):
    return np.array([b.position[0], b.position[1], b.z_top, b.power,
                     1.0 if b.active else 0.0])


def operator_outputs(prefix, op, T, r_c, beam, dt, rng):
    o = {}
    o["rhs_beam"] = op.evaluate_rhs(T, r_c, beam)
    o["rhs_nobeam"] = op.evaluate_rhs(T, r_c, None)
    o["rhs_diff"] = op.evaluate_rhs(T, r_c, None, faces=False, source=False)
    o["rhs_faces"] = op.evaluate_rhs(T, r_c, None, diffusion=False, source=False)
    o["rhs_src"] = op.evaluate_rhs(T, r_c, beam, diffusion=False, faces=False)
    o["rhs_frozen"] = op.evaluate_rhs(T, None, None, faces=False, source=False,
                                      frozen_k=20.0)
    o["lumped"] = op.lumped_capacity()
    v = rng.standard_normal(op.dofmap.n_vertices)
    v[op.dofmap.is_slave] = 0.0
    o["v"] = v
    o["mass_v"] = op.apply_mass(v)
    o["jac_v"] = op.apply_jacobian(v, T, r_c, dt)
    o["jac_diag"] = op.jacobian_diagonal(T, r_c, dt)
    o["step"] = op.explicit_fused_step(T.copy(), 2e-7, r_c, beam)
    h = st.HistoryField(r_c.copy(), op.epoch)
    op.update_history(h, T)
    o["history"] = h.r_c
    o["T"] = T
    o["r_c"] = r_c
    o["beam"] = beam_arr(beam)
    o["dt"] = np.array(dt)
    return {f"{prefix}{k}": np.asarray(v) for k, v in o.items()}


def make_oracle_cases():
    from conftest import oracle_cases, random_state
    rng = np.random.default_rng(2024)
    data = {}
    names = []
    for name, forest, dofmap, history, params in oracle_cases():
        op = st.ThermalOperator(forest, dofmap, params, st.SolverSettings())
        T, r_c = random_state(dofmap, history, rng)
        xyz = dofmap.vertices_m()
        cx = 0.5 * (xyz[:, 0].min() + xyz[:, 0].max())
        cy = 0.5 * (xyz[:, 1].min() + xyz[:, 1].max())
        beam = st.BeamState(np.array([cx + 13e-6, cy - 7e-6]),
                            float(xyz[:, 2].max()), 100.0, True)
        data.update(mesh_arrays(f"{name}/", forest, dofmap))
        data.update(operator_outputs(f"{name}/", op, T, r_c, beam, 1e-4, rng))
        data[f"{name}/params"] = np.array(params_json(params))
        names.append(name)
    data["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "oracle_cases.npz"), **data)
    print("oracle_cases:", names)


def config0_setup():
    h = 31.25e-6
    mesh = st.MeshParams(h_coarse=h, n_refine=0, h_powder=h)
    geo = st.PartGeometry.chamber((2e-3, 2e-3), h, 1e-3, mesh)
    mat = st.MaterialParams(k_p=6.7, k_m=6.7, k_s=6.7, rho=4430.0, c=526.0)
    bnd = st.BoundaryParams(emissivity=0.0, T_inf=300.0, T_v=1e9)
    las = st.HeatSourceParams(radius=50e-6, h_powder=40e-6, power=70.0,
                              scan_velocity=1.0)
    params = st.ProcessParams(mat, bnd, las, mesh)
    forest = st.build_coarse_grid(geo, mesh)
    history = st.initial_history(forest)
    dofmap = st.build_dofmap(forest)
    op = st.ThermalOperator(forest, dofmap, params, st.SolverSettings())
    T0 = 300.0 + np.random.default_rng(0).uniform(0.0, 1.0, dofmap.n_vertices)
    lp = st.LayerPath(0, 0.0, [st.Segment(0.0, 1e-3, 2e-4, 1e-3, 1.0, 70.0)], 0.0)
    return forest, dofmap, params, history, op, T0, lp


def make_config0():
    forest, dofmap, params, history, op, T0, lp = config0_setup()
    snaps = {}

    def hook(state, step, t):
        if step in (1, 20, 200):
            snaps[step] = state.T.copy()

    state = st.SimulationState(forest, dofmap, op, T0.copy(), history)
    t0 = time.perf_counter()
    stats = st.run_scan_phase(state, lp, 1e-6, on_step=hook)
    wall = time.perf_counter() - t0
    print(f"config0: {stats.n_steps} steps in {wall:.1f} s, T_max {state.T.max():.1f}")
    np.savez_compressed(os.path.join(OUT, "config0.npz"),
                        T1=snaps[1], T20=snaps[20], T200=snaps[200],
                        n_dofs=np.array(dofmap.n_dofs), wall_s=np.array(wall),
                        rc_all_one=np.array(bool(np.all(state.history.r_c == 1.0))))


def make_growing():
    """Config-3-like growing domain on a small footprint: per-layer
    activation tables, transfers, an explicit window and BE steps."""
    from conftest import make_params
    mesh = st.MeshParams(h_coarse=80e-6, n_refine=1, h_powder=40e-6)
    geo = st.PartGeometry.chamber((0.48e-3, 0.32e-3), 0.16e-3, 0.32e-3, mesh)
    params = make_params(mesh, power=70.0)
    settings = st.SolverSettings(explicit_cooldown_steps=0, dt_implicit=1e-3,
                                 krylov_tol=1e-13, preconditioner="diagonal")
    forest = st.build_coarse_grid(geo, mesh)
    history = st.initial_history(forest)
    dofmap = st.build_dofmap(forest)
    T = np.full(dofmap.n_vertices, params.T_0)
    data = {"params": np.array(params_json(params))}
    data.update(mesh_arrays("L0/", forest, dofmap))
    rng = np.random.default_rng(7)
    for layer in range(1, 3):
        # a non-trivial field/history so transfer and coarsening paths run
        xyz = dofmap.vertices_m()
        T = 303.0 + 1500.0 * np.exp(-((xyz[:, 0] - 0.2e-3) ** 2) / (1e-4) ** 2)
        dofmap.distribute(T)
        history.r_c[:] = np.maximum(history.r_c,
                                    rng.uniform(0.0, 1.0, history.r_c.shape))
        data[f"L{layer}/pre_T"] = T.copy()
        data[f"L{layer}/pre_rc"] = history.r_c.copy()
        plan = st.advance_layer(forest, history)
        forest, fields, history = st.apply_update(
            forest, plan, [st.NodalField(T, forest.epoch)], history, T_0=params.T_0)
        T = fields[0].values
        dofmap = st.build_dofmap(forest)
        data.update(mesh_arrays(f"L{layer}/", forest, dofmap))
        data[f"L{layer}/post_T"] = T.copy()
        data[f"L{layer}/post_rc"] = history.r_c.copy()
        data[f"L{layer}/transfer_source"] = plan.transfer_report.vertex_source

    # explicit window with a moving beam on the last mesh
    op = st.ThermalOperator(forest, dofmap, params, settings)
    segs = st.generate_hatch([(0.0, 0.0, 0.48e-3, 0.32e-3)], 1e-4, 1.0, 70.0)
    lp = st.LayerPath(2, 2 * 40e-6, segs, 0.0)
    state = st.SimulationState(forest, dofmap, op, T.copy(), history.copy())
    data["expl/T0"] = state.T.copy()
    data["expl/rc0"] = state.history.r_c.copy()
    lp_short = st.LayerPath(2, 2 * 40e-6, [st.Segment(
        segs[0].x0, segs[0].y0, segs[0].x0 + 60e-6, segs[0].y1, 1.0, 70.0)], 0.0)
    stats = st.run_scan_phase(state, lp_short, 1e-6)
    data["expl/n_steps"] = np.array(stats.n_steps)
    data["expl/T"] = state.T.copy()
    data["expl/rc"] = state.history.r_c.copy()
    data["expl/seg"] = np.array([lp_short.segments[0].x0, lp_short.segments[0].y0,
                                 lp_short.segments[0].x1, lp_short.segments[0].y1,
                                 1.0, 70.0, lp_short.z])

    # backward Euler steps from the hot end-of-scan field
    Tn = state.T.copy()
    rc = state.history.r_c.copy()
    t0 = time.perf_counter()
    bes = []
    for i in range(3):
        out = _implicit_step(state, 1e-3, settings)
        Tn1, nn, nk = out
        Tn1 = Tn1.copy()
        Tn1[dofmap.is_dirichlet] = params.boundary.T_inf
        bes.append((nn, nk))
        data[f"be/T{i + 1}"] = Tn1.copy()
        state.T = Tn1
        op.update_history(state.history, state.T)
    print(f"growing: 3 BE steps in {time.perf_counter() - t0:.1f} s, iters {bes}")
    data["be/T0"] = Tn
    data["be/rc0"] = rc
    data["be/iters"] = np.array(bes)
    data["be/rc_final"] = state.history.r_c.copy()
    # single jacobian pieces at the BE linearisation point
    v = rng.standard_normal(dofmap.n_vertices)
    v[dofmap.is_slave] = 0.0
    data["be/v"] = v
    data["be/jac_v"] = op.apply_jacobian(v, Tn, rc, 1e-3)
    data["be/jac_diag"] = op.jacobian_diagonal(Tn, rc, 1e-3)
    np.savez_compressed(os.path.join(OUT, "growing.npz"), **data)


def make_pointwise():
    """Material law and surface fluxes on lanes covering every branch."""
    from scantherm.material import (conductivity, conductivity_derivative,
                                    liquid_fraction)
    from scantherm.physics import (evaporation_flux, radiation_flux,
                                   volumetric_source)
    rng = np.random.default_rng(99)
    mat = st.MaterialParams()
    bp = st.BoundaryParams()
    T = np.concatenate([rng.uniform(250.0, 4500.0, 4000),
                        [mat.T_s, mat.T_l, bp.T_v, bp.T_v + 1000.0, 0.5]])
    rc = rng.uniform(0.0, 1.0, len(T))
    hs = st.HeatSourceParams(radius=50e-6, h_powder=40e-6, power=100.0)
    beam = st.BeamState(np.array([1e-4, 2e-4]), 40e-6, 100.0, True)
    pts = np.stack([rng.uniform(-1e-4, 3e-4, 2000), rng.uniform(0, 4e-4, 2000),
                    rng.uniform(-2e-5, 6e-5, 2000)], axis=1)
    segs = st.generate_hatch([(0.0, 0.0, 4e-4, 3e-4)], 1e-4, 1.0, 70.0)
    lp = st.LayerPath(0, 4e-5, segs, 1e-4)
    taus = np.arange(0, int(lp.duration() / 1e-6)) * 1e-6
    bs = [st.layer_beam_state(lp, t) for t in taus]
    np.savez_compressed(
        os.path.join(OUT, "pointwise.npz"), T=T, rc=rc,
        g=liquid_fraction(T, mat), k=conductivity(T, rc, mat),
        dk=conductivity_derivative(T, rc, mat),
        rad=radiation_flux(T, bp), evap=evaporation_flux(T, bp, mat.c),
        pts=pts, src=volumetric_source(pts, beam, hs),
        hatch=np.array([[s.x0, s.y0, s.x1, s.y1, s.v, s.power] for s in segs]),
        taus=taus, beam_pos=np.array([b.position for b in bs]),
        beam_on=np.array([b.active for b in bs]),
        beam_power=np.array([b.power for b in bs]))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-config0", action="store_true")
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    jobs = {"pointwise": make_pointwise, "oracle_cases": make_oracle_cases,
            "growing": make_growing, "config0": make_config0}
    for name, fn in jobs.items():
        if a.only and name != a.only:
            continue
        if name == "config0" and a.skip_config0:
            continue
        fn()
