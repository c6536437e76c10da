"""Time the config-3 explicit scan on layer 0 (device-resident batches) for
the launch-list capture: wall per step with and without PDL."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import workloads as w
import paper_2302_05164_b200 as st
from paper_2302_05164_b200.physics import flatten_schedule

mesh, geo, params, settings = w.config3_setup()
state = w.config3_initial_state(mesh, geo, params, settings)
w.advance_mesh(state, params, settings)
paths = w.config3_layer_paths(geo, mesh)
n = int(os.environ.get("NSTEPS", "2048"))
dts, beams = flatten_schedule(paths[0], 1e-6, n)
op = state.op
op.set_state(state.T, state.history.r_c)
op.run_explicit(dts[:512], beams[:512])
t0 = time.perf_counter()
op.run_explicit(dts, beams)
el = time.perf_counter() - t0
print(f"config3 layer 0: {op.nv} DoFs, {len(op.dofmap.slaves)} hanging, {n} steps "
      f"{el / n * 1e6:.2f} us/step")
op.close()
