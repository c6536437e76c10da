"""Step-by-step reproduction of tests/test_gpu_slabs_overlap.py (box, 2
slabs) with progress prints, to localise a host crash."""
import faulthandler
import os
import sys

faulthandler.enable(all_threads=True)
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
os.environ.setdefault("ST_LX", "4")
import numpy as np

import paper_2302_05164_b200 as st
from paper_2302_05164_b200.distributed import (GpuSlabStepper, local_exchange,
                                               local_exchange_overlapped, partition, slab_of)

mode = sys.argv[1] if len(sys.argv) > 1 else "overlap"
H = 40e-6


def log(*a):
    print("[repro]", *a, file=sys.stderr, flush=True)


mat = st.MaterialParams(k_p=6.7, k_m=32.0, k_s=6.7, T_s=300.0, T_l=1928.0, latent_heat=2.86e5)
bnd = st.BoundaryParams(emissivity=0.3, T_inf=300.0, T_v=1e9, h_conv=10.0)
las = st.HeatSourceParams(radius=60e-6, h_powder=40e-6, power=150.0)
params = st.ProcessParams(mat, bnd, las)
glob = st.StructuredBox(36, 9, 18, H, degree=2)
T0 = 300.0 + np.random.default_rng(7).uniform(0.0, 1800.0, glob.n_vertices)
lp = st.LayerPath(0, 0.0, [st.Segment(0.0, 4.5 * H, 36 * H, 4.5 * H, 1.0, 150.0)], 0.0)
dts, beams = st.flatten_schedule(lp, 2e-8, 10)
log("single")
op = st.ThermalOperator(glob, glob, params, st.SolverSettings())
op.set_state(T0, 1.0)
log("run", op.run_explicit(dts, beams))
op.close()
parts = partition(glob.nx, 2)
boxes = [slab_of(glob, *parts[r], r, 2) for r in range(2)]
log("slab ops")
ops = [st.ThermalOperator(b, b, params, st.SolverSettings()) for b in boxes]
for b, o in zip(boxes, ops):
    o.set_state(b.local_of(T0), 1.0)
log("steppers")
steppers = [GpuSlabStepper(o, overlap=(mode == "overlap")) for o in ops]
step = (local_exchange_overlapped if mode == "overlap" else local_exchange)(steppers)
for i in range(len(dts)):
    log("step", i)
    step(float(dts[i]), beams[i])
log("maxima")
for s in steppers:
    log(s.maxima_history(len(dts)))
log("done")
