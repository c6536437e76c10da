"""Golden step criteria from the REFERENCE.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_criteria_golden.py

For every `conftest.oracle_cases` mesh (the same meshes as
oracle_cases.npz, whose tables the tests already load) and for the
uniform plate of `test_timestepping.py::test_step_criteria_on_a_uniform_plate`
this runs the reference's `compute_step_criteria` (timestepping.py:70-99,
power iteration `estimate_spectral_radius` :49-67 with seed 0) and records
rho = 2 / dt_stability, dt_accuracy, the number of operator applies, and
the Rayleigh quotients of every iteration.  Writes tests/golden/criteria.npz.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import scantherm as st  # noqa: E402
from scantherm import timestepping as ts  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def run(op):
    """compute_step_criteria with the power iteration instrumented: the
    reference's own estimate_spectral_radius, called through a counting
    wrapper of its apply callback."""
    lams = []
    orig = ts.estimate_spectral_radius

    def counting(apply_fn, n, **kw):
        def wrapped(v):
            w = apply_fn(v)
            lams.append(float(np.dot(v, w)))
            return w
        return orig(wrapped, n, **kw)

    ts.estimate_spectral_radius = counting
    try:
        crit = ts.compute_step_criteria(op)
    finally:
        ts.estimate_spectral_radius = orig
    return crit, np.array(lams)


def main():
    from conftest import oracle_cases
    from test_timestepping import _plate_state
    data = {}
    names = []
    for name, forest, dofmap, history, params in oracle_cases():
        op = st.ThermalOperator(forest, dofmap, params, st.SolverSettings())
        crit, lams = run(op)
        data[f"{name}/rho"] = np.array(2.0 / crit.dt_stability)
        data[f"{name}/dt_stability"] = np.array(crit.dt_stability)
        data[f"{name}/dt_accuracy"] = np.array(crit.dt_accuracy)
        data[f"{name}/lams"] = lams
        names.append(name)
        print(name, dofmap.n_vertices, len(lams), 2.0 / crit.dt_stability)
    state, params = _plate_state(nx=8, ny=8, nz=4)
    crit, lams = run(state.op)
    from make_golden import mesh_arrays, params_json
    data.update(mesh_arrays("plate/", state.op.forest, state.op.dofmap))
    data["plate/params"] = np.array(params_json(params))
    data["plate/rho"] = np.array(2.0 / crit.dt_stability)
    data["plate/dt_stability"] = np.array(crit.dt_stability)
    data["plate/dt_accuracy"] = np.array(crit.dt_accuracy)
    data["plate/lams"] = lams
    m = params.material
    h = params.mesh.h_fine
    data["plate/analytic"] = np.array(m.rho * m.c * h * h / (2.0 * max(m.k_m, m.k_s)))
    print("plate", len(lams), crit.dt_stability, float(data["plate/analytic"]))
    data["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "criteria.npz"), **data)


if __name__ == "__main__":
    sys.path.insert(0, OUT)
    main()
