"""Synthetic BASELINE workloads (bench.py and the tests; not part of the
product package).

BASELINE.json defines its scan patterns through the reference's hatch
generator (driver.py:85-111: n = max(1, floor(width / spacing)) tracks per
box, centred, serpentine across tracks and boxes; 0 deg along x, 90 along
y).  ``hatch_segments`` produces the same segments (the same float
operations per coordinate, tests/test_workloads.py pins it against the
reference's output) with the track grid computed per box in one go.
"""

import math

import numpy as np


def hatch_segments(boxes, spacing, v, power, direction_deg=0.0):
    """Serpentine hatch over (x0, y0, x1, y1) boxes -> list of Segment."""
    from paper_2302_05164_b200.physics import Segment
    if direction_deg not in (0, 90):
        raise ValueError("hatch direction must be 0 or 90 degrees")
    across = 1 if direction_deg == 0 else 0  # axis the tracks are stacked along
    out = []
    parity = 0
    for box in boxes:
        lo, hi = (box[1], box[3]) if across else (box[0], box[2])
        a0, a1 = (box[0], box[2]) if across else (box[1], box[3])
        width = hi - lo
        n = max(1, int(math.floor(width / spacing + 1e-9)))
        margin = (width - (n - 1) * spacing) / 2.0
        pos = [lo + (margin + i * spacing) for i in range(n)]
        for i, c in enumerate(pos):
            fwd = (parity + i) % 2 == 0
            s, e = (a0, a1) if fwd else (a1, a0)
            out.append(Segment(s, c, e, c, v, power) if across else Segment(c, s, c, e, v, power))
        parity = (parity + n) % 2
    return out


# --- BASELINE configs[0..2] (structured boxes) ---------------------------------

def _st():
    import paper_2302_05164_b200 as st
    return st


def workload_config0():
    """configs[0]: 64x64x32 Q1 (139,425 DoFs), k = 6.7 const, 70 W beam at
    1 m/s along y = 1 mm, dt = 1 us, bottom Dirichlet 300 K."""
    st = _st()
    h = 31.25e-6
    mat = st.MaterialParams(k_p=6.7, k_m=6.7, k_s=6.7, rho=4430.0, c=526.0)
    bnd = st.BoundaryParams(emissivity=0.0, T_inf=300.0, T_v=1e9)
    las = st.HeatSourceParams(radius=50e-6, h_powder=40e-6, power=70.0, scan_velocity=1.0)
    params = st.ProcessParams(mat, bnd, las, st.MeshParams(h_coarse=h, n_refine=0, h_powder=h))
    lp = st.LayerPath(0, 0.0, [st.Segment(0.0, 1e-3, 2e-3, 1e-3, 1.0, 70.0)], 0.0)
    return dict(name="config0_q1_64x64x32", dims=(64, 64, 32), h=h, degree=1,
                params=params, T0=lambda n: 300.0 + np.random.default_rng(0).uniform(0, 1, n),
                dt=1e-6, paths=[lp], sample=(64, 64, 32),
                cfg={"mesh": "64x64x32 Q1", "dt": 1e-6, "material": "k=6.7 const",
                     "beams": 1})


def _config1_params():
    st = _st()
    h = 31.25e-6
    # k(T) = g k_m + (1-g) k_s with r_c = 1, c_app with latent heat
    mat = st.MaterialParams(k_p=6.7, k_m=32.0, k_s=6.7, rho=4430.0, c=526.0, T_s=300.0,
                            T_l=1928.0, latent_heat=2.86e5, T_lat_s=1878.0, T_lat_l=1928.0)
    bnd = st.BoundaryParams(emissivity=0.3, T_inf=300.0, T_v=1e9, h_conv=10.0)
    las = st.HeatSourceParams(radius=50e-6, h_powder=40e-6, power=70.0, scan_velocity=1.0)
    return st.ProcessParams(mat, bnd, las, st.MeshParams(h_coarse=h, n_refine=0, h_powder=h))


def workload_config1():
    """configs[1]: 4x4x1 mm, 128x128x32 Q2 cells (4,293,185 DoFs), k(T)
    6.7 -> 32 W/mK over 300-1928 K, apparent heat capacity (latent
    2.86e5 J/kg over 1878-1928 K), top radiation eps 0.3 + convection
    h = 10, 70 W beam on a 5-track serpentine hatch (100 um), dt = 0.5 us."""
    st = _st()
    h = 31.25e-6
    segs = hatch_segments([(1.5e-3, 1.75e-3, 2.5e-3, 2.25e-3)], 1e-4, 1.0, 70.0)
    lp = st.LayerPath(0, 0.0, segs, 0.0)
    return dict(name="config1_q2_128x128x32", dims=(128, 128, 32), h=h, degree=2,
                params=_config1_params(),
                T0=lambda n: 300.0 + np.random.default_rng(0).uniform(0, 1, n),
                dt=0.5e-6, paths=[lp], sample=(32, 32, 32),
                cfg={"mesh": "128x128x32 Q2", "dt": 0.5e-6,
                     "material": "k(T) 6.7->32, c_app latent 2.86e5, rad 0.3 + conv 10",
                     "beams": 1, "hatch": "5 tracks x 1 mm, 100 um"})


CELLS_50M = {1: 367, 2: 184, 3: 122, 4: 92}


def workload_config2(p):
    """configs[2]: unit cube, ~50M DoFs at degree p, T ~ U[300, 2500],
    material as config 1, beam off, dt = 1 ms."""
    st = _st()
    n = CELLS_50M[p]
    h = 1.0 / n
    lp = st.LayerPath(0, 0.0, [], 0.0)
    return dict(name=f"config2_q{p}_{n}^3", dims=(n, n, n), h=h, degree=p,
                params=_config1_params(),
                T0=lambda m: np.random.default_rng(2).uniform(300.0, 2500.0, m),
                dt=1e-3, paths=[lp], sample=(24, 24, 24),
                cfg={"mesh": f"{n}^3 Q{p} unit cube", "dt": 1e-3,
                     "material": "as config 1", "beams": 0})


WORKLOADS = {"config0": workload_config0, "config1": workload_config1,
             "config2_p1": lambda: workload_config2(1), "config2_p2": lambda: workload_config2(2),
             "config2_p3": lambda: workload_config2(3), "config2_p4": lambda: workload_config2(4)}


def build_problem(w, dims=None):
    st = _st()
    nx, ny, nz = dims or w["dims"]
    box = st.StructuredBox(nx, ny, nz, w["h"], degree=w["degree"])
    return box


def schedule(w, n):
    from paper_2302_05164_b200.physics import flatten_schedule
    paths = w["paths"]
    if not paths[0].segments:       # beam off: an empty layer of n steps
        dts = np.full(n, w["dt"])
        from paper_2302_05164_b200.physics import BEAM_DTYPE
        return dts, np.zeros((n, 0), dtype=BEAM_DTYPE)
    return flatten_schedule(paths, w["dt"], n)



# --- BASELINE configs[4]: partitioned large part -------------------------------

def workload_config4(scale=1, steps_hint=100):
    """configs[4]: a cantilever-like part of 75 x 5 x 12 mm -- a 20 mm base
    of the full 12 mm height plus a 2.4 mm thin overhang slab on top that
    reaches out to 75 mm -- Q2 at h = 25 um (scale 1: 3000 x 200 x 480 cell
    lattice, 957,492,161 DoFs; ``scale`` coarsens h by that factor for the
    replicas, 4 = the 1/64-volume replica), material as config 1 (k(T),
    latent heat, radiation + convection), r_c = 1, T0 = 300 K + U[0, 1]
    (seed 0), four 70 W spots at 1 m/s each hatching its own 10 x 4 mm
    patch of the top surface (tracks along x, 100 um apart), dt = 2 us."""
    from paper_2302_05164_b200.mesh import FittedPart
    from paper_2302_05164_b200.physics import LayerPath
    h = 25e-6 * scale
    nx, ny, nz = 3000 // scale, 200 // scale, 480 // scale
    base, over = 800 // scale, 96 // scale
    xext = [base] * (nz - over) + [nx] * over
    paths = []
    for x0 in (2e-3, 22e-3, 42e-3, 62e-3):
        segs = hatch_segments([(x0, 0.5e-3, x0 + 10e-3, 4.5e-3)], 1e-4, 1.0, 70.0)
        paths.append(LayerPath(0, 0.0, segs, 0.0))
    return dict(name=f"config4_q2_cantilever{'' if scale == 1 else f'_1:{scale ** 3}'}",
                dims=(nx, ny, nz), h=h, degree=2, xext=xext,
                params=_config1_params(),
                T0=lambda n: 300.0 + np.random.default_rng(0).uniform(0, 1, n),
                T0_slice=lambda lo, hi: 300.0 + _uniform_slice(0, lo, hi),
                dt=2e-6, paths=paths, sample=(32, 32, 32),
                sample_origin=(2e-3 - 16 * h, 0.5e-3 - 16 * h, -32 * h),
                cfg={"mesh": f"{nx}x{ny}x{nz} Q2 lattice, 20 mm base + 2.4 mm overhang to 75 mm",
                     "h_um": 25.0 * scale, "dt": 2e-6,
                     "material": "as config 1 (k(T), latent 2.86e5, rad 0.3 + conv 10)",
                     "beams": 4, "hatch": "4 patches 10 x 4 mm, 100 um, 1 m/s"})


def _uniform_slice(seed, lo, hi):
    """Entries [lo, hi) of default_rng(seed).uniform(0, 1, n) for any n >= hi
    without drawing the prefix (PCG64 jump-ahead: one 64-bit draw per
    double), so every rank builds only its slab of the global T0."""
    g = np.random.default_rng(seed)
    g.bit_generator.advance(lo)
    return g.uniform(0.0, 1.0, hi - lo)


def build_part(w):
    """The mesh object of a workload (box or fitted part)."""
    import paper_2302_05164_b200 as st
    from paper_2302_05164_b200.mesh import FittedPart
    nx, ny, nz = w["dims"]
    if w.get("xext") is not None:
        return FittedPart(nx, ny, nz, w["h"], w["xext"], degree=w["degree"])
    return st.StructuredBox(nx, ny, nz, w["h"], degree=w["degree"])


WORKLOADS["config4"] = workload_config4
WORKLOADS["config4_s2"] = lambda: workload_config4(2)  # 1/8 volume (1.2e8 DoFs)


# --- BASELINE configs[3]: growing domain with cool-down ------------------------

def config3_setup(krylov_tol=1e-10):
    """2 x 2 mm chamber on a 2 mm plate, Q1, h_coarse 80 um / one refinement
    level / 40 um layers, ten layers; reference default material and
    boundary, 70 W beam at 1 m/s; backward-Euler cool-down at 1 ms with
    Jacobi-PCG."""
    import paper_2302_05164_b200 as st
    from paper_2302_05164_b200.mesh import chamber_geometry
    mesh = st.MeshParams(h_coarse=80e-6, n_refine=1, h_powder=40e-6)
    geo = chamber_geometry((2e-3, 2e-3), 10 * 40e-6, 2e-3, mesh)
    params = st.ProcessParams(st.MaterialParams(), st.BoundaryParams(),
                              st.HeatSourceParams(power=70.0, scan_velocity=1.0), mesh)
    settings = st.SolverSettings(explicit_cooldown_steps=0, dt_implicit=1e-3,
                                 krylov_tol=krylov_tol, preconditioner="diagonal")
    return mesh, geo, params, settings


def config3_layer_paths(geo, mesh, d_h=1e-4, v=1.0, power=70.0, cool_time=1.0,
                        rotation=(0, 90)):
    """Per layer: the footprint hatched at d_h, direction cycling through
    ``rotation``, the beam at the layer top (the reference's hatch_path,
    driver.py:114-130)."""
    from paper_2302_05164_b200.physics import LayerPath
    out = []
    for k in range(geo.n_layers):
        boxes = geo.footprints[k] * mesh.h_fine
        segs = hatch_segments(boxes, d_h, v, power, rotation[k % len(rotation)])
        out.append(LayerPath(k, (k + 1) * mesh.h_powder, segs, cool_time))
    return out


def config3_initial_state(mesh, geo, params, settings):
    import paper_2302_05164_b200 as st
    from paper_2302_05164_b200.mesh import build_coarse_grid
    forest = build_coarse_grid(geo, mesh)
    history = st.initial_history(forest)
    dofmap = st.build_dofmap(forest)
    op = st.ThermalOperator(forest, dofmap, params, settings)
    return st.SimulationState(forest, dofmap, op, np.full(dofmap.n_vertices, params.T_0),
                              history)


def advance_mesh(state, params, settings):
    """One deposition step: plan, transfer T and r_c, new tables and a new
    operator (the reference's _advance_mesh + _rebuild_operator,
    driver.py:162-194)."""
    import paper_2302_05164_b200 as st
    from paper_2302_05164_b200.mesh import NodalField, advance_layer, apply_update
    plan = advance_layer(state.forest, state.history)
    forest, fields, history = apply_update(state.forest, plan,
                                           [NodalField(state.T, state.forest.epoch)],
                                           state.history, T_0=params.T_0)
    state.op.close()
    state.forest, state.T, state.history = forest, fields[0].values, history
    state.dofmap = st.build_dofmap(forest)
    state.op = st.ThermalOperator(forest, state.dofmap, params, settings)
    return plan


def run_config3_build(n_layers=None, dt=1e-6, scan_steps=None, cool_time=None,
                      krylov_tol=1e-10, on_layer=None):
    """The reference's run_build layer loop (driver.py:197-254) for
    config 3 on the B200 operator: per layer advance the mesh, step
    criteria, the scan (dt = 1 us) and the backward-Euler cool-down.
    ``scan_steps`` / ``cool_time`` truncate a layer for quick runs.
    Returns per-layer records with wall times."""
    import time

    import paper_2302_05164_b200 as st
    from paper_2302_05164_b200.physics import LayerPath, Segment
    mesh, geo, params, settings = config3_setup(krylov_tol)
    paths = config3_layer_paths(geo, mesh)
    state = config3_initial_state(mesh, geo, params, settings)
    recs = []
    for lp in paths[:n_layers]:
        rec = {"layer": lp.layer_index}
        t0 = time.perf_counter()
        advance_mesh(state, params, settings)
        rec["wall_amr"] = time.perf_counter() - t0
        rec["n_dofs"] = int(state.dofmap.n_dofs)
        rec["n_cells"] = int(state.forest.active.sum())
        t0 = time.perf_counter()
        crit = st.compute_step_criteria(state.op, settings)
        rec["wall_criteria"] = time.perf_counter() - t0
        rec["dt_stability"] = crit.dt_stability
        scan_lp = lp
        if scan_steps is not None:
            # the same schedule, stopped after scan_steps steps
            keep, t_left = [], scan_steps * dt
            for s in lp.segments:
                if t_left <= 0:
                    break
                if s.duration <= t_left + 1e-15:
                    keep.append(s)
                    t_left -= s.duration
                else:
                    f = t_left / s.duration
                    keep.append(Segment(s.x0, s.y0, s.x0 + f * (s.x1 - s.x0),
                                        s.y0 + f * (s.y1 - s.y0), s.v, s.power))
                    t_left = 0
            scan_lp = LayerPath(lp.layer_index, lp.z, keep, lp.cool_time)
        cool_lp = lp if cool_time is None else LayerPath(lp.layer_index, lp.z, [], cool_time)
        scan = st.run_scan_phase(state, scan_lp, dt)
        cool = st.run_cooldown_phase(state, cool_lp, dt, settings)
        rec.update(scan_steps=scan.n_steps, wall_scan=scan.wall_time, t_max=scan.t_max_seen,
                   cool_steps=cool.n_steps, newton=cool.newton_iters, krylov=cool.krylov_iters,
                   wall_cool=cool.wall_time)
        recs.append(rec)
        if on_layer is not None:
            on_layer(state, rec)
    return state, recs
