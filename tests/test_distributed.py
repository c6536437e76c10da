"""x-slab decomposition (paper_2302_05164_b200.distributed) on CPU with
gloo, world size 2 and 3: each rank advances its slab with the CPU oracle
through the same split-step driver and exchange code the GPU path uses;
the assembled field must equal the single-domain run."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from cpu_oracle import OracleOperator, structured_tables

import paper_2302_05164_b200 as st
from paper_2302_05164_b200.distributed import (Partials, SlabBox, SlabDriver,
                                               balanced_partition, gather_global, layer_dofs,
                                               partition, slab_of, torch_exchange,
                                               torch_max_reducer)
from paper_2302_05164_b200.mesh import FittedPart

H = 40e-6


def _params():
    mat = st.MaterialParams(k_p=0.3, k_m=30.0, k_s=22.0, T_s=1450.0, T_l=1900.0,
                            latent_heat=2.86e5)
    bnd = st.BoundaryParams(emissivity=0.4, T_inf=300.0, T_v=2900.0, h_conv=10.0)
    las = st.HeatSourceParams(radius=60e-6, h_powder=40e-6, power=150.0)
    return st.ProcessParams(mat, bnd, las)


class OracleSlabStepper:
    """CPU split step of one slab: partial f and lumped capacity on the
    interface planes are exchanged and summed low + high."""

    def __init__(self, box, params, T0, rc0):
        self.box = box
        M = structured_tables(box.nx, box.ny, box.nz, box.h, box.degree,
                              origin=(box.origin[0], box.origin[1], None))
        self.orc = OracleOperator(M, params)
        self.M = M
        self.T = T0.copy()
        self.rc = rc0.copy()
        self.plane = box.node_dims[1] * box.node_dims[2]
        self.sides = [s for s, on in ((0, box.iface_lo), (1, box.iface_hi)) if on]
        self.params = params
        self.hist = []          # per-step (max |T|, max T), unchecked
        self.poison_at = None   # step number at which this rank diverges (tests)
        self.n = 0

    def _planes(self, v):
        return {0: v[:self.plane], 1: v[-self.plane:]}

    def begin(self, dt, beams):
        self.dt = dt
        self.f = self.orc.evaluate_rhs(self.T, self.rc, beams)
        self.C = self.orc.lumped_capacity(self.T)
        pf, pc = self._planes(self.f), self._planes(self.C)
        return {s: Partials(torch.from_numpy(pf[s].copy()), torch.from_numpy(pc[s].copy()))
                for s in self.sides}

    def end(self, recv):
        f, C = self.f, self.C
        if 0 in recv:
            f[:self.plane] = recv[0].f.numpy() + f[:self.plane]
            C[:self.plane] = recv[0].c.numpy() + C[:self.plane]
        if 1 in recv:
            f[-self.plane:] = f[-self.plane:] + recv[1].f.numpy()
            C[-self.plane:] = C[-self.plane:] + recv[1].c.numpy()
        out = self.T + self.dt * ((1.0 / C) * f)
        out[self.M["is_dirichlet"]] = self.params.boundary.T_inf
        self.n += 1
        if self.poison_at is not None and self.n >= self.poison_at:
            out[len(out) // 2] = np.nan
        self.T = out
        self.hist.append((float(np.max(np.abs(out))) if np.all(np.isfinite(out)) else np.nan,
                          float(np.max(out))))
        self.rc = self.orc.update_history(self.rc, np.nan_to_num(self.T, nan=300.0))

    def maxima_history(self, n):
        h, self.hist = self.hist[:n], self.hist[n:]
        return np.array([a for a, _ in h]), np.array([b for _, b in h])


def _problem(p=2):
    glob = st.StructuredBox(7, 3, 3, H, degree=p)
    rng = np.random.default_rng(4)
    T0 = 300.0 + rng.uniform(0.0, 1500.0, glob.n_vertices)
    T0[glob.is_dirichlet] = 300.0
    lp = st.LayerPath(0, 0.0, [st.Segment(0.0, 1.5 * H, 7 * H, 1.5 * H, 1.0, 150.0)], 0.0)
    dts, beams = st.flatten_schedule(lp, 2e-7, 6)
    return glob, T0, dts, beams


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    glob, T0, dts, beams = _problem()
    c0, c1 = partition(glob.nx, world)[rank]
    box = SlabBox(glob, c0, c1, rank, world)
    qd = glob.degree + 1
    rc0 = np.ones((box.n_cells, qd, qd, qd))
    stepper = OracleSlabStepper(box, _params(), box.local_of(T0), rc0)
    drv = SlabDriver(stepper, torch_exchange(rank, world))
    from cpu_oracle import beam_tuple
    for i in range(len(dts)):
        drv.step(float(dts[i]), [beam_tuple(b) for b in beams[i]])
    out = [None] * world
    dist.all_gather_object(out, (rank, stepper.T))
    if rank == 0:
        q.put(gather_global([SlabBox(glob, *partition(glob.nx, world)[r], r, world)
                             for r in range(world)], [t for _, t in sorted(out)]))
    dist.barrier()
    dist.destroy_process_group()


def _diverge_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    glob, T0, dts, beams = _problem()
    c0, c1 = partition(glob.nx, world)[rank]
    box = SlabBox(glob, c0, c1, rank, world)
    qd = glob.degree + 1
    stepper = OracleSlabStepper(box, _params(), box.local_of(T0), np.ones((box.n_cells, qd, qd, qd)))
    if rank == world - 1:
        stepper.poison_at = 4          # only the last rank diverges
    drv = SlabDriver(stepper, torch_exchange(rank, world), reduce_max=torch_max_reducer())
    from cpu_oracle import beam_tuple
    try:
        drv.run(dts, [[beam_tuple(b) for b in row] for row in beams], check_every=3)
        q.put((rank, None))
    except st.InstabilityError as e:
        q.put((rank, e.step))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3])
def test_slab_decomposition_matches_single_domain(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    got, t0 = None, time.time()
    while got is None:
        try:
            got = q.get(timeout=2)
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs) or time.time() - t0 > 300:
                for p in procs:
                    p.kill()
                pytest.fail("slab worker failed")
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    glob, T0, dts, beams = _problem()
    M = structured_tables(glob.nx, glob.ny, glob.nz, H, glob.degree)
    orc = OracleOperator(M, _params())
    from cpu_oracle import beam_tuple, run_explicit
    qd = glob.degree + 1
    T, _ = run_explicit(orc, T0, np.ones((glob.n_cells, qd, qd, qd)), dts,
                        [[beam_tuple(b) for b in row] for row in beams])
    assert np.max(np.abs(got - T)) / np.max(np.abs(T)) < 1e-13


def _spawn(target, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_cross_rank_stability_check(world):
    """One rank diverges at step 4; the MAX all-reduce of the per-step
    maxima makes every rank raise InstabilityError at step 4."""
    got = _spawn(_diverge_worker, world)
    assert sorted(got) == [(r, 4) for r in range(world)]


def test_fitted_balanced_partition_and_gather():
    g = FittedPart(36, 9, 24, H, [10] * 16 + [36] * 8, degree=2)
    ld = layer_dofs(g)
    assert ld.sum() + g.node_dims[1] * (g.node_dims[2] - g.kmin[-1]) == g.n_vertices
    for w in (2, 3, 4):
        parts = balanced_partition(g, w)
        assert parts[0][0] == 0 and parts[-1][1] == g.nx
        boxes = [slab_of(g, *parts[r], r, w) for r in range(w)]
        T = np.arange(g.n_vertices, dtype=float)
        assert np.array_equal(gather_global(boxes, [b.local_of(T) for b in boxes]), T)
        for b in boxes:  # each slab's own numbering is the global one, shifted
            assert b.n_vertices == len(b.local_of(T))
    with pytest.raises(ValueError):
        slab_of(g, 0, 10, 0, 2)  # a cut exactly where the base ends


def test_partition_is_balanced_and_contiguous():
    for nx, w in [(128, 8), (7, 3), (100, 7)]:
        parts = partition(nx, w)
        assert parts[0][0] == 0 and parts[-1][1] == nx
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        sizes = [b - a for a, b in parts]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        partition(3, 4)
