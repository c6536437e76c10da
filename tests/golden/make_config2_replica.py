"""Config-2 replica at p = 1 against the REFERENCE (run here):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_config2_replica.py

BASELINE configs[2] at degree 1 on a 128^3-cell unit cube (2,146,689
DoFs; the full 367^3 case needs ~52 GB in the reference): the reference
expresses the config-1 conductivity exactly (k_s = 6.7, k_m = 32 over
300-1928 K with r_c = 1) but has no latent heat or convection, so the
replica runs without those; top radiation eps 0.3, evaporation off,
Dirichlet bottom, beam off, T = default_rng(2).uniform(300, 2500),
dt = 1 ms.  Stored (the full vectors are 17 MB each): 20,000 seeded
sample entries and three checksums of the rhs and of one explicit step.
"""

import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import scantherm as st  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
N = 128


def checks(v, idx, u):
    return v[idx], np.array([v.sum(), np.abs(v).sum(), v @ u])


def main():
    h = 1.0 / N
    mesh = st.MeshParams(h_coarse=h, n_refine=0, h_powder=h)
    geo = st.PartGeometry.chamber((1.0, 1.0), h, 1.0, mesh)
    mat = st.MaterialParams(k_p=6.7, k_m=32.0, k_s=6.7, rho=4430.0, c=526.0, T_s=300.0,
                            T_l=1928.0)
    bnd = st.BoundaryParams(emissivity=0.3, T_inf=300.0, T_v=1e9)
    las = st.HeatSourceParams(radius=50e-6, h_powder=40e-6, power=70.0)
    params = st.ProcessParams(mat, bnd, las, mesh)
    forest = st.build_coarse_grid(geo, mesh)
    history = st.initial_history(forest)
    dofmap = st.build_dofmap(forest)
    assert np.all(history.r_c == 1.0)
    op = st.ThermalOperator(forest, dofmap, params, st.SolverSettings())
    nv = dofmap.n_vertices
    T = np.random.default_rng(2).uniform(300.0, 2500.0, nv)
    idx = np.sort(np.random.default_rng(3).choice(nv, 20000, replace=False))
    u = np.random.default_rng(5).standard_normal(nv)
    t0 = time.perf_counter()
    f = op.evaluate_rhs(T, history.r_c)
    t1 = time.perf_counter()
    T1 = op.explicit_fused_step(T.copy(), 1e-3, history.r_c)
    t2 = time.perf_counter()
    fs, fc = checks(f, idx, u)
    ss, sc = checks(T1 - T, idx, u)
    print(f"{nv} DoFs: rhs {t1 - t0:.1f} s, step {t2 - t1:.1f} s")
    np.savez_compressed(os.path.join(OUT, "config2_replica_q1.npz"), n=np.array(N),
                        nv=np.array(nv), idx=idx, f_samples=fs, f_checks=fc,
                        dT_samples=ss, dT_checks=sc, f_absmax=np.array(np.abs(f).max()),
                        dT_absmax=np.array(np.abs(T1 - T).max()),
                        wall=np.array([t1 - t0, t2 - t1]))


if __name__ == "__main__":
    main()
