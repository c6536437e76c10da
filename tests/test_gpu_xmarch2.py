"""k_xmarch2 (the lean Q2 explicit-step kernel) against k_xmarch<2> (the
general kernel, ST_XMARCH2=0): the same arithmetic in the same order, so the
fields after several steps are bitwise equal (zeros may differ in sign) --
boxes with full and ragged tiles, several x chunks, a fitted part with its
re-entrant edge, latent heat on and off, a melt pool that crosses the latent
interval, and the stability maxima."""

import numpy as np
import pytest

import paper_2302_05164_b200 as st
from paper_2302_05164_b200.mesh import FittedPart
from paper_2302_05164_b200.physics import BEAM_DTYPE, BeamState, pack_beams

pytestmark = pytest.mark.gpu

H = 40e-6


def _params(latent):
    mat = st.MaterialParams(k_p=0.3, k_m=30.0, k_s=22.0, T_s=1450.0, T_l=1900.0,
                            latent_heat=2.86e5 if latent else 0.0, T_lat_s=1878.0,
                            T_lat_l=1928.0)
    bnd = st.BoundaryParams(emissivity=0.4, T_inf=300.0, T_v=2900.0, h_conv=10.0)
    las = st.HeatSourceParams(radius=60e-6, h_powder=40e-6, power=90.0)
    return st.ProcessParams(mat, bnd, las, st.MeshParams(h_coarse=H, n_refine=0, h_powder=H))


def _run(mesh, latent, lx, x2, monkeypatch, steps=6, inseam=False, nbeams=2, pipe=0):
    monkeypatch.setenv("ST_XMARCH2", "1" if x2 else "0")
    # the pipelined seam pass is for parts of many waves of CTAs: off here
    # unless a test forces it on (groups of any size)
    monkeypatch.setenv("ST_SEAM_PIPE", str(pipe))
    if pipe:
        monkeypatch.setenv("ST_X2_ADAPT", "0")   # stay on k_xmarch2 on this latent-dense field
    monkeypatch.setenv("ST_SEAM_PIPE_MINWAVES", "0")
    monkeypatch.setenv("ST_INSEAM", "1" if inseam else "0")
    # the general kernel runs on the original seam layout (split f / dc slot
    # arrays), the lean one on the round's layout ((f, dc) pairs)
    monkeypatch.setenv("ST_SEAM_PAIR", "1" if x2 else "0")
    if lx:
        monkeypatch.setenv("ST_LX", lx)
    else:
        monkeypatch.delenv("ST_LX", raising=False)
    op = st.ThermalOperator(mesh, mesh, _params(latent), st.SolverSettings())
    rng = np.random.default_rng(7)
    # a field that crosses the latent interval (1878-1928 K) in many cells
    T = rng.uniform(1700.0, 2100.0, op.nv)
    T[rng.random(op.nv) < 0.5] = rng.uniform(300.0, 600.0)
    op.set_state(T, 1.0)
    lx_m, ly_m = mesh.nx * H, mesh.ny * H
    recs = np.zeros((steps, nbeams), dtype=BEAM_DTYPE)
    for s in range(steps):
        beams = [BeamState(np.array([lx_m * 0.3 + s * 4e-6, ly_m * 0.5]), 0.0, 90.0, True),
                 BeamState(np.array([lx_m * 0.7, ly_m * 0.3 + s * 2e-6]), 0.0, 60.0, s % 2 == 0)]
        beams += [BeamState(np.array([lx_m * (0.1 + 0.1 * b), ly_m * (0.9 - 0.1 * b)]), 0.0,
                            20.0 + 5.0 * b, True) for b in range(2, nbeams)]
        if nbeams:
            recs[s] = pack_beams(beams[:nbeams])
    fail, amax, tmax = op.run_explicit(np.full(steps, 2e-8), recs)
    Tout, _ = op.get_state()
    _run.launches = op.launches
    op.close()
    return fail, amax, tmax, Tout


CASES = {
    "box_full": lambda: st.StructuredBox(12, 16, 32, H, degree=2),
    "box_ragged": lambda: st.StructuredBox(9, 11, 19, H, degree=2),
    "box_single_tile": lambda: st.StructuredBox(5, 7, 9, H, degree=2),
    "fitted": lambda: FittedPart(13, 11, 40, H, [5] * 16 + [9] * 16 + [13] * 8, degree=2),
}


@pytest.mark.parametrize("inseam", [False, True])
@pytest.mark.parametrize("lx", [None, "3"])
@pytest.mark.parametrize("latent", [True, False])
@pytest.mark.parametrize("case", list(CASES))
def test_lean_kernel_equals_general_kernel_bitwise(case, latent, lx, inseam, monkeypatch):
    """inseam: the opt-in in-kernel seam completion (last-arriving CTA sums
    the slots in the seam pass's order) instead of the seam pass."""
    # (the general kernel on the round's layout is covered by the oracle
    # comparisons of test_gpu_structured / test_gpu_fitted: rhs mode and
    # stored histories run it)
    mesh = CASES[case]()
    f0, a0, t0, T0 = _run(mesh, latent, lx, False, monkeypatch)
    f1, a1, t1, T1 = _run(mesh, latent, lx, True, monkeypatch, inseam=inseam)
    assert f0 == f1
    assert a0 == a1 and t0 == t1
    assert np.array_equal(T0, T1)


PIPE_CASES = {
    # (mesh, x chunk length): 12 / 5 / 3 chunks of a box, a fitted part whose
    # tile rows end inside different groups, two chunks (two groups of one)
    "box_12_chunks": (lambda: st.StructuredBox(12, 16, 32, H, degree=2), "1"),
    "box_ragged": (lambda: st.StructuredBox(9, 11, 19, H, degree=2), "2"),
    "box_3_chunks": (lambda: st.StructuredBox(9, 11, 19, H, degree=2), "3"),
    "fitted": (lambda: FittedPart(13, 11, 40, H, [5] * 16 + [9] * 16 + [13] * 8, degree=2), "2"),
    "two_chunks": (lambda: st.StructuredBox(4, 9, 17, H, degree=2), "2"),
}


@pytest.mark.parametrize("groups", [2, 3, 16])
@pytest.mark.parametrize("latent", [True, False])
@pytest.mark.parametrize("case", list(PIPE_CASES))
def test_pipelined_seam_pass_bitwise(case, latent, groups, monkeypatch):
    """The step with the x chunks launched as groups on two streams and the
    seam entries of each group's planes on a third (xmarch_piped) against the
    single launch followed by the whole pass: same kernels and summation
    order, so the fields, the stability maxima and the sign of zeros agree."""
    make, lx = PIPE_CASES[case]
    monkeypatch.setenv("ST_X2_ADAPT", "0")
    f0, a0, t0, T0 = _run(make(), latent, lx, True, monkeypatch, steps=8)
    n0 = _run.launches
    f1, a1, t1, T1 = _run(make(), latent, lx, True, monkeypatch, steps=8, pipe=groups)
    assert _run.launches >= n0 + 8 * 2   # at least two groups per step ran
    assert f0 == f1
    assert a0 == a1 and t0 == t1
    assert np.array_equal(T0, T1)
    assert np.array_equal(np.signbit(T0), np.signbit(T1))


EDGE_CASES = {
    # one cell layer (a chunk is its first and last plane only), two layers in
    # one-layer chunks, no Dirichlet plane and no radiating top, thin in z
    "one_layer": (lambda: st.StructuredBox(1, 9, 17, H, degree=2), None),
    "chunks_of_one": (lambda: st.StructuredBox(2, 9, 17, H, degree=2), "1"),
    "insulated": (lambda: st.StructuredBox(6, 10, 18, H, degree=2, dirichlet_bottom=False,
                                           top_faces=False), "2"),
    "one_cell_high": (lambda: st.StructuredBox(7, 20, 1, H, degree=2), "3"),
}


@pytest.mark.parametrize("nbeams", [0, 8])
@pytest.mark.parametrize("case", list(EDGE_CASES))
def test_lean_kernel_edge_cases_bitwise(case, nbeams, monkeypatch):
    """Degenerate extents and boundary switches, without beams and with the
    eight beams the kernel's source tables hold."""
    make, lx = EDGE_CASES[case]
    f0, a0, t0, T0 = _run(make(), True, lx, False, monkeypatch, steps=4, nbeams=nbeams)
    f1, a1, t1, T1 = _run(make(), True, lx, True, monkeypatch, steps=4, nbeams=nbeams)
    assert f0 == f1
    assert a0 == a1 and t0 == t1
    assert np.array_equal(T0, T1)


def test_adaptive_dispatch_on_a_latent_dense_field(monkeypatch):
    """A field in which every tile gathers latent increments in most layers
    (config 2's situation) makes the context fall back to the general kernel
    (the kernels count their latent CTA-layers, the host reads the counter
    asynchronously); a field with no latent cell stays on k_xmarch2; the
    fields are bitwise those of a run pinned to k_xmarch2."""
    monkeypatch.setenv("ST_XMARCH2", "1")
    mesh = st.StructuredBox(12, 16, 32, H, degree=2)
    rng = np.random.default_rng(3)
    dense = rng.uniform(1700.0, 2100.0, mesh.n_vertices)   # 1/8 of the Gauss points latent
    cold = rng.uniform(300.0, 600.0, mesh.n_vertices)
    empty = np.zeros((1, 0), dtype=BEAM_DTYPE)

    def run(T0, adapt):
        monkeypatch.setenv("ST_X2_ADAPT", "1" if adapt else "0")
        op = st.ThermalOperator(mesh, mesh, _params(True), st.SolverSettings())
        op.set_state(T0, 1.0)
        names = []
        for _ in range(12):   # one step per call: the counter is read between calls
            fail, _, _ = op.run_explicit(np.full(1, 2e-8), empty)
            assert fail == 0
            names.append(op.profile_read()[2])
        T, _ = op.get_state()
        op.close()
        return T, names

    Td_pinned, n0 = run(dense, False)
    Td_adapt, n1 = run(dense, True)
    assert set(n0) == {"k_xmarch2"}
    assert n1[0] == "k_xmarch2" and n1[-1] == "k_xmarch"
    assert np.array_equal(Td_pinned, Td_adapt)
    _, n2 = run(cold, True)
    assert set(n2) == {"k_xmarch2"}
