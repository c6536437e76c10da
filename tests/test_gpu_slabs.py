"""Multi-slab split steps on one GPU: several slab contexts of the same
box exchange their interface partials in-process (no cross-process
waits), which exercises exactly the kernels and host logic of the
multi-GPU path; the assembled field must match the single-domain run."""

import numpy as np
import pytest

import paper_2302_05164_b200 as st
from paper_2302_05164_b200.distributed import (GpuSlabStepper, SlabBox, gather_global,
                                               local_exchange, partition)
from fixtures import rel

pytestmark = pytest.mark.gpu
H = 40e-6


def _params(latent):
    mat = st.MaterialParams(k_p=6.7, k_m=32.0, k_s=6.7, T_s=300.0, T_l=1928.0,
                            latent_heat=2.86e5 if latent else 0.0)
    bnd = st.BoundaryParams(emissivity=0.3, T_inf=300.0, T_v=1e9, h_conv=10.0)
    las = st.HeatSourceParams(radius=60e-6, h_powder=40e-6, power=150.0)
    return st.ProcessParams(mat, bnd, las)


@pytest.mark.parametrize("p,world,latent", [(1, 2, False), (2, 2, True), (2, 3, True),
                                            (3, 2, False)])
def test_gpu_slabs_match_single_domain(p, world, latent):
    dims = {1: (40, 9, 35), 2: (21, 7, 18), 3: (12, 5, 9)}[p]
    glob = st.StructuredBox(*dims, H, degree=p)
    params = _params(latent)
    rng = np.random.default_rng(p)
    T0 = 300.0 + rng.uniform(0.0, 1800.0, glob.n_vertices)
    T0[glob.is_dirichlet] = 300.0
    lp = st.LayerPath(0, 0.0, [st.Segment(0.0, dims[1] * H / 2, dims[0] * H, dims[1] * H / 2,
                                          1.0, 150.0)], 0.0)
    dts, beams = st.flatten_schedule(lp, 2e-8, 12)
    # single domain
    op = st.ThermalOperator(glob, glob, params, st.SolverSettings())
    op.set_state(T0, 1.0)
    fail, _, _ = op.run_explicit(dts, beams)
    assert fail == 0
    T_ref, _ = op.get_state()
    # slabs on the same device
    boxes = [SlabBox(glob, *partition(glob.nx, world)[r], r, world) for r in range(world)]
    ops = [st.ThermalOperator(b, b, params, st.SolverSettings()) for b in boxes]
    for b, o in zip(boxes, ops):
        o.set_state(b.local_of(T0), 1.0)
    steppers = [GpuSlabStepper(o) for o in ops]
    step = local_exchange(steppers)
    for i in range(len(dts)):
        step(float(dts[i]), beams[i])
    T_slab = gather_global(boxes, [o.get_state()[0] for o in ops])
    assert rel(T_slab, T_ref) < 1e-12
    # the shared interface planes are bitwise identical on both sides
    NYZ = glob.node_dims[1] * glob.node_dims[2]
    for r in range(world - 1):
        hi = ops[r].get_state()[0][-NYZ:]
        lo = ops[r + 1].get_state()[0][:NYZ]
        assert np.array_equal(hi, lo)
    am, tm = steppers[0].maxima()
    assert np.isfinite(am) and am >= tm > 300.0
