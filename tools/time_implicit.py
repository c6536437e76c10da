"""Time backward-Euler cool-down steps (Newton + Jacobi-PCG on the device)
on the growing-domain fixture (BASELINE config 3 mesh, layer 2, hanging
nodes).  Dev tool: python tools/time_implicit.py [n_steps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]

import numpy as np  # noqa: E402

import paper_2302_05164_b200 as st  # noqa: E402
from fixtures import forest_dofmap, load, params_from_json  # noqa: E402


def main(n=10):
    d = load("growing")
    params = params_from_json(d["params"])
    forest, dm, _ = forest_dofmap(d, "L2/")
    s = st.SolverSettings(explicit_cooldown_steps=0, dt_implicit=1e-3, krylov_tol=1e-10)
    op = st.ThermalOperator(forest, dm, params, s)
    op.set_state(d["be/T0"], d["be/rc0"])
    out = op.implicit_step(1e-3, s)  # warm-up
    op.finish_implicit_step()
    t0 = time.perf_counter()
    nn = nk = 0
    for _ in range(n):
        a, b = op.implicit_step(1e-3, s)
        op.finish_implicit_step()
        nn += a
        nk += b
    el = time.perf_counter() - t0
    print(f"nv {op.nv} BE steps {n}: {el / n * 1e3:.2f} ms/step, newton {nn / n:.1f}, "
          f"cg {nk / n:.1f} /step, {el / max(nk, 1) * 1e6:.1f} us per CG iteration")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 10)
