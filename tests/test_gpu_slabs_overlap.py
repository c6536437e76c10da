"""The overlapped multi-GPU schedule on one device: interface chunks first,
packed planes behind an event, the exchange on a communication stream
while the interior chunks run, then the seam pass -- for boxes and for a
fitted part (config 4's base + overhang) cut by cumulative DoFs; the
assembled field must equal the single-domain run, interface planes
bitwise equal on both sides, and the cross-rank stability check must
report the diverging step."""

import numpy as np
import pytest

import paper_2302_05164_b200 as st
from paper_2302_05164_b200.distributed import (GpuSlabStepper, SlabDriver, balanced_partition,
                                               gather_global, local_exchange,
                                               local_exchange_overlapped, partition, slab_of)
from paper_2302_05164_b200.mesh import FittedPart
from fixtures import rel

pytestmark = pytest.mark.gpu
H = 40e-6


def _params():
    mat = st.MaterialParams(k_p=6.7, k_m=32.0, k_s=6.7, T_s=300.0, T_l=1928.0,
                            latent_heat=2.86e5)
    bnd = st.BoundaryParams(emissivity=0.3, T_inf=300.0, T_v=1e9, h_conv=10.0)
    las = st.HeatSourceParams(radius=60e-6, h_powder=40e-6, power=150.0)
    return st.ProcessParams(mat, bnd, las)


def _glob(kind):
    if kind == "box":
        return st.StructuredBox(36, 9, 18, H, degree=2)
    # base of 10 layers under 16 rows, overhang rows to 36
    return FittedPart(36, 9, 24, H, [10] * 16 + [36] * 8, degree=2)


@pytest.mark.parametrize("kind,world,overlap", [("box", 2, True), ("box", 3, True),
                                               ("fitted", 2, True), ("fitted", 3, True),
                                               ("fitted", 3, False)])
def test_overlapped_slabs_match_single_domain(kind, world, overlap, monkeypatch):
    monkeypatch.setenv("ST_LX", "4")  # several chunks per slab: interface + interior
    glob = _glob(kind)
    params = _params()
    rng = np.random.default_rng(7)
    T0 = 300.0 + rng.uniform(0.0, 1800.0, glob.n_vertices)
    T0[glob.is_dirichlet] = 300.0
    lp = st.LayerPath(0, 0.0, [st.Segment(0.0, 4.5 * H, 36 * H, 4.5 * H, 1.0, 150.0)], 0.0)
    dts, beams = st.flatten_schedule(lp, 2e-8, 10)
    op = st.ThermalOperator(glob, glob, params, st.SolverSettings())
    op.set_state(T0, 1.0)
    assert op.run_explicit(dts, beams)[0] == 0
    T_ref, _ = op.get_state()
    op.close()
    parts = balanced_partition(glob, world) if kind == "fitted" else partition(glob.nx, world)
    boxes = [slab_of(glob, *parts[r], r, world) for r in range(world)]
    ops = [st.ThermalOperator(b, b, params, st.SolverSettings()) for b in boxes]
    for b, o in zip(boxes, ops):
        o.set_state(b.local_of(T0), 1.0)
    steppers = [GpuSlabStepper(o, overlap=overlap) for o in ops]
    step = (local_exchange_overlapped if overlap else local_exchange)(steppers)
    for i in range(len(dts)):
        step(float(dts[i]), beams[i])
    for s in steppers:
        am, tm = s.maxima_history(len(dts))
        assert np.all(np.isfinite(am)) and am.max() < 1e4
    T_slab = gather_global(boxes, [o.get_state()[0] for o in ops])
    assert rel(T_slab, T_ref) < 1e-12
    for r in range(world - 1):
        a, b = ops[r].get_state()[0], ops[r + 1].get_state()[0]
        if kind == "fitted":
            lo, hi = boxes[r].owned_range()
            n = boxes[r].n_vertices - (hi - lo)   # the shared interface plane
        else:
            n = glob.node_dims[1] * glob.node_dims[2]
        assert np.array_equal(a[-n:], b[:n])
    for o in ops:
        o.close()


def test_slab_driver_reports_the_diverging_step():
    glob = _glob("box")
    params = _params()
    T0 = np.full(glob.n_vertices, 300.0)
    parts = partition(glob.nx, 2)
    boxes = [slab_of(glob, *parts[r], r, 2) for r in range(2)]
    ops = [st.ThermalOperator(b, b, params, st.SolverSettings()) for b in boxes]
    for b, o in zip(boxes, ops):
        o.set_state(b.local_of(T0), 1.0)
    steppers = [GpuSlabStepper(o) for o in ops]
    step = local_exchange_overlapped(steppers)

    class Both:  # a two-rank driver in one process: steps both, checks both
        def __init__(self):
            self.steps = 0

        def begin(self, dt, beams):
            step(dt, beams)
            return {}

        def end(self, recv):
            pass

        def maxima_history(self, n):
            a = [s.maxima_history(n) for s in steppers]
            return np.maximum(a[0][0], a[1][0]), np.maximum(a[0][1], a[1][1])

    drv = SlabDriver(Both(), lambda p: {})
    lp = st.LayerPath(0, 0.0, [st.Segment(0.0, 4.5 * H, 36 * H, 4.5 * H, 1.0, 150.0)], 0.0)
    dts, beams = st.flatten_schedule(lp, 2e-8, 12)
    dts = dts.copy()
    dts[7:] = 1e3  # far above the stability bound from step 8 on
    with pytest.raises(st.InstabilityError) as e:
        drv.run(dts, beams, check_every=5)
    assert e.value.step == 8
    for o in ops:
        o.close()
