"""x-slab decomposition of a structured box over ranks (one GPU per rank).

The explicit step is a cell-local apply plus a node scatter, so ranks
need exactly one neighbour exchange per step (option (ii)
"partial-sum"): rank r owns cell layers [c_r, c_{r+1}) of the box; the
node plane on a rank interface receives partial sums from both sides.
Each side sends its partial plane to the other and both add them in the
fixed order low-rank + high-rank, so the interface plane is bitwise the
same on both ranks and no second (halo) exchange is needed.  x is the
slowest axis of the node numbering, so a slab's nodes and every
interface plane are contiguous in memory.

The step is split around the exchange (``st_explicit_step_begin`` /
``st_explicit_step_end``).  ``begin`` launches the x chunks that touch a
rank interface first, packs the interface planes, records an event and
then launches the interior chunks; the exchange runs on a separate
communication stream that waits only for that event, so the NCCL transfer
overlaps the interior sweep (the paper's ghost exchange overlapped with
local compute), and the seam pass waits for the received
planes.  :class:`SlabDriver` holds the rank logic -- including the
cross-rank stability check, a MAX all-reduce of the per-step maxima every
``check_every`` steps (timestepping.py:186-192) -- and is shared by the
GPU path and the CPU reference path used by the gloo tests.

Fitted parts (config 4's base + overhang) split into :class:`SlabPart`
slices, balanced by cumulative DoFs (:func:`balanced_partition`) at cuts
where both sides see the same node column.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from .mesh import FittedPart, StructuredBox


def partition(nx, world):
    """Contiguous, balanced cell-layer ranges [(c0, c1), ...] per rank."""
    if world < 1 or nx < world:
        raise ValueError("need at least one cell layer per rank")
    base, extra = divmod(nx, world)
    out, c = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((c, c + n))
        c += n
    return out


def _cut_ok(glob, c):
    """A fitted part may be cut before cell layer c when node plane p*c
    holds the same rows seen from either side."""
    if not isinstance(glob, FittedPart):
        return True
    x = glob.xext
    return np.searchsorted(x, max(c, 1)) == np.searchsorted(x, c + 1)


def layer_dofs(glob):
    """DoFs per cell layer in x (the nodes of its p node planes)."""
    p = glob.degree
    NX, NY, NZ = glob.node_dims
    kmin = glob.kmin if isinstance(glob, FittedPart) else np.zeros(NX, dtype=np.int64)
    per_plane = NY * (NZ - kmin)
    return per_plane[:-1].reshape(glob.nx, p).sum(axis=1)


def balanced_partition(glob, world):
    """Cell-layer ranges per rank balanced by cumulative DoFs (SURVEY
    §8e), each cut moved to the nearest layer a fitted part may be cut at."""
    if world < 1 or glob.nx < world:
        raise ValueError("need at least one cell layer per rank")
    cum = np.concatenate([[0], np.cumsum(layer_dofs(glob))])
    cuts = [0]
    for r in range(1, world):
        c = int(np.searchsorted(cum, cum[-1] * r / world))
        best = None
        for d in range(glob.nx):
            for cand in (c - d, c + d):
                if cuts[-1] < cand < glob.nx - (world - r) + 1 and _cut_ok(glob, cand):
                    best = cand
                    break
            if best is not None:
                break
        if best is None:
            raise ValueError("no admissible cut for this world size")
        cuts.append(best)
    cuts.append(glob.nx)
    return list(zip(cuts[:-1], cuts[1:]))


class SlabBox(StructuredBox):
    """Cells [c0, c1) in x of a global StructuredBox, as its own box.

    Node plane 0 of the slab is global plane p*c0, the last one p*c1; the
    planes shared with a neighbour rank are marked as interfaces."""

    def __init__(self, glob, c0, c1, rank, world):
        p = glob.degree
        ox = glob.origin[0] + c0 * glob.h
        super().__init__(c1 - c0, glob.ny, glob.nz, glob.h, degree=p,
                         origin=(ox, glob.origin[1], glob.origin[2]),
                         dirichlet_bottom=glob.dirichlet_bottom, top_faces=glob.top_faces,
                         epoch=glob.epoch)
        self.glob = glob
        self.c0, self.c1 = c0, c1
        self.rank, self.world = rank, world
        self.gx0 = p * c0
        self.gNX = glob.node_dims[0]
        self.iface_lo = rank > 0
        self.iface_hi = rank < world - 1

    def local_of(self, T_global):
        """Slab part (including both boundary planes) of a global field."""
        NX, NY, NZ = self.glob.node_dims
        g = np.asarray(T_global).reshape(NX, NY * NZ)
        return np.ascontiguousarray(g[self.gx0:self.gx0 + self.node_dims[0]].reshape(-1))

    def owned_planes(self):
        """Global node planes this rank owns (the upper interface belongs
        to the upper rank; the last rank owns the top plane)."""
        n = self.node_dims[0]
        return range(self.gx0, self.gx0 + (n if not self.iface_hi else n - 1))


class SlabPart(FittedPart):
    """Cells [c0, c1) in x of a global FittedPart, as its own fitted part:
    the local row extents are the global ones clipped to the slab, rows
    with no cell in the slab (the base's rows past its end) dropped.  Its
    nodes are one contiguous range of the global numbering."""

    def __init__(self, glob, c0, c1, rank, world):
        if not ((c0 == 0 or _cut_ok(glob, c0)) and (c1 == glob.nx or _cut_ok(glob, c1))):
            raise ValueError("a fitted part cannot be cut where its extent steps")
        p = glob.degree
        ext = np.clip(glob.xext - c0, 0, c1 - c0)
        drop = int(np.searchsorted(ext, 1))
        ox = glob.origin[0] + c0 * glob.h
        oz = glob.origin[2] + drop * glob.h
        super().__init__(c1 - c0, glob.ny, glob.nz - drop, glob.h, ext[drop:], degree=p,
                         origin=(ox, glob.origin[1], oz),
                         dirichlet_bottom=glob.dirichlet_bottom and drop == 0,
                         top_faces=glob.top_faces, epoch=glob.epoch)
        self.glob, self.c0, self.c1, self.drop = glob, c0, c1, drop
        self.rank, self.world = rank, world
        self.gx0 = p * c0
        self.gNX = glob.node_dims[0]
        self.iface_lo = rank > 0
        self.iface_hi = rank < world - 1
        g = glob
        self.g_lo = int(g.plane_offset[p * c0])
        self.g_hi = int(g.plane_offset[p * c1] + g.node_dims[1] * (g.node_dims[2] - g.kmin[p * c1]))
        assert self.g_hi - self.g_lo == self.n_vertices

    def local_of(self, T_global):
        return np.ascontiguousarray(np.asarray(T_global)[self.g_lo:self.g_hi])

    def owned_range(self):
        """Global node ids this rank owns (the upper interface plane is the
        upper rank's)."""
        g, p = self.glob, self.degree
        hi = self.g_hi
        if self.iface_hi:
            hi = int(g.plane_offset[p * self.c1])
        return self.g_lo, hi


def slab_of(glob, c0, c1, rank, world):
    """The rank-local mesh of cells [c0, c1) of a box or a fitted part."""
    if isinstance(glob, FittedPart):
        return SlabPart(glob, c0, c1, rank, world)
    return SlabBox(glob, c0, c1, rank, world)


def gather_global(boxes, locals_):
    """Assemble the global field from every rank's slab field."""
    glob = boxes[0].glob
    if isinstance(glob, FittedPart):
        out = np.empty(glob.n_vertices)
        for b, v in zip(boxes, locals_):
            lo, hi = b.owned_range()
            out[lo:hi] = np.asarray(v)[:hi - lo]
        return out
    NX, NY, NZ = glob.node_dims
    out = np.empty((NX, NY * NZ))
    for b, v in zip(boxes, locals_):
        v = np.asarray(v).reshape(b.node_dims[0], NY * NZ)
        planes = list(b.owned_planes())
        out[planes[0]:planes[-1] + 1] = v[:len(planes)]
    return out.reshape(-1)


class _CudaPlane:
    """Zero-copy view of a device plane for torch (__cuda_array_interface__)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


@dataclass
class Partials:
    f: object          # partial f on the interface plane (array / tensor)
    c: object = None   # partial latent capacity increment (or None)


class SlabDriver:
    """Rank-side logic of one split step: begin -> exchange -> end.

    ``stepper`` implements begin(dt, beams) -> {side: Partials} for the
    sides with a neighbour (0 = lower, 1 = upper), end(recv) where recv
    maps side -> the neighbour's Partials, and maxima_history(n) -> the
    (max |T|, max T) arrays of its n oldest unchecked steps; a stepper
    with ``exchange_on(exchange, parts)`` runs the exchange itself (the
    GPU stepper: on its communication stream).  ``exchange`` maps
    {side: Partials} -> {side: Partials} (torch.distributed or local);
    ``reduce_max`` maps a float64 array to its elementwise maximum over
    the ranks (None: this rank only)."""

    def __init__(self, stepper, exchange, reduce_max=None):
        self.stepper = stepper
        self.exchange = exchange
        self.reduce_max = reduce_max
        self.steps = 0
        self.checked = 0

    def step(self, dt, beams):
        parts = self.stepper.begin(dt, beams)
        if hasattr(self.stepper, "exchange_on"):
            recv = self.stepper.exchange_on(self.exchange, parts)
        else:
            recv = self.exchange(parts)
        self.stepper.end(recv)
        self.steps += 1

    def check(self, t0=0.0, dts=None, base=0):
        """Cross-rank stability check of the steps since the last one
        (timestepping.py:186-192): max |T| of each step, MAX over ranks;
        raises InstabilityError at the first step that is non-finite or
        above 1e7 K, numbered from ``base`` (the run's first step) with
        its time from t0 and ``dts`` (the run's steps).  Returns the
        largest T seen."""
        from .timestepping import InstabilityError, _T_DIVERGED
        n = self.steps - self.checked
        if n == 0:
            return -np.inf
        am, tm = self.stepper.maxima_history(n)
        v = np.concatenate([np.where(np.isfinite(am), am, np.inf), tm])
        if self.reduce_max is not None:
            v = self.reduce_max(v)
        am, tm = v[:n], v[n:]
        bad = np.flatnonzero(~(am <= _T_DIVERGED))
        first = self.checked
        self.checked = self.steps
        if bad.size:
            s = first + int(bad[0]) + 1 - base
            dt = float(dts[s - 1]) if dts is not None else float("nan")
            t = t0 + (float(np.sum(dts[:s - 1])) if dts is not None else 0.0)
            raise InstabilityError(s, t, dt, float(am[bad[0]]))
        return float(np.max(tm))

    def run(self, dts, beams, check_every=32, t0=0.0):
        """Integrate len(dts) split steps with a cross-rank stability check
        every ``check_every`` (<= 64) steps and after the last; returns the
        largest T seen."""
        tmax = -np.inf
        base = self.steps
        for i in range(len(dts)):
            self.step(float(dts[i]), beams[i])
            if (i + 1) % check_every == 0 or i + 1 == len(dts):
                tmax = max(tmax, self.check(t0, dts, base))
        return tmax


def torch_max_reducer(group=None):
    """Elementwise MAX all-reduce of a float64 array over the ranks."""
    import torch
    import torch.distributed as dist

    def red(v):
        dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.as_tensor(np.asarray(v, dtype=np.float64), device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return t.cpu().numpy()
    return red


def torch_exchange(rank, world, group=None):
    """Exchange with torch.distributed point-to-point (NCCL or gloo).

    Sends side-1 partials to rank+1 and side-0 partials to rank-1; returns
    what the neighbours sent.  For NCCL the caller runs this with the
    library stream as torch's current stream so the transfer is ordered
    after the sweep and before the seam pass."""
    import torch
    import torch.distributed as dist

    def ex(parts):
        # gloo has no device point-to-point: device planes are staged through
        # the host there (functional checks on a box without a GPU per rank)
        staged = dist.get_backend(group) != "nccl"
        host = lambda t: t.cpu() if staged and torch.is_tensor(t) and t.is_cuda else t
        ops, recv = [], {}
        for side, peer in ((0, rank - 1), (1, rank + 1)):
            if side not in parts or not (0 <= peer < world):
                continue
            mine = parts[side]
            sf, sc = host(mine.f), (host(mine.c) if mine.c is not None else None)
            rf = torch.empty_like(sf)
            rc = torch.empty_like(sc) if sc is not None else None
            ops.append(dist.P2POp(dist.isend, sf, peer, group))
            ops.append(dist.P2POp(dist.irecv, rf, peer, group))
            if sc is not None:
                ops.append(dist.P2POp(dist.isend, sc, peer, group))
                ops.append(dist.P2POp(dist.irecv, rc, peer, group))
            recv[side] = (Partials(rf, rc), mine)
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        back = lambda t, like: (t.to(like.device) if torch.is_tensor(like) and like.is_cuda
                                and not t.is_cuda else t)
        return {s: Partials(back(r.f, m.f), back(r.c, m.c) if r.c is not None else None)
                for s, (r, m) in recv.items()}

    return ex


class GpuSlabStepper:
    """Split step on a B200 slab operator (ThermalOperator on a SlabBox)."""

    def __init__(self, op, overlap=True):
        import torch
        self.op = op
        self.torch = torch
        self.stream = torch.cuda.ExternalStream(op.stream_ptr())
        # the exchange runs here, started by the interface-planes event of
        # st_explicit_step_begin, while the interior chunks run on self.stream
        self.comm = torch.cuda.Stream() if overlap else self.stream
        self._keep = None
        lib = op._lib
        self._planes = {}
        box = op.forest
        self.sides = [s for s, on in ((0, box.iface_lo), (1, box.iface_hi)) if on]
        for side in self.sides:
            f = ctypes.POINTER(ctypes.c_double)()
            c = ctypes.POINTER(ctypes.c_double)()
            n = ctypes.c_int64()
            from . import _lib
            _lib.check(lib.st_iface_partials(op._ctx, side, ctypes.byref(f), ctypes.byref(c),
                                             ctypes.byref(n)), "iface_partials")
            fp = ctypes.cast(f, ctypes.c_void_p).value
            cp = ctypes.cast(c, ctypes.c_void_p).value if c else None
            tf = torch.as_tensor(_CudaPlane(fp, n.value), device="cuda")
            tc = torch.as_tensor(_CudaPlane(cp, n.value), device="cuda") if cp else None
            self._planes[side] = Partials(tf, tc)

    def begin(self, dt, beams):
        from . import _lib
        bp, nb = _lib.beams_array(beams)
        _lib.check(self.op._lib.st_explicit_step_begin(self.op._ctx, float(dt), bp, nb),
                   "step_begin")
        return {s: self._planes[s] for s in self.sides}

    def end(self, recv):
        from . import _lib
        ptr = lambda t: None if t is None else t.data_ptr()
        lo, hi = recv.get(0), recv.get(1)
        _lib.check(self.op._lib.st_explicit_step_end(
            self.op._ctx, ptr(lo.f) if lo else None, ptr(lo.c) if lo else None,
            ptr(hi.f) if hi else None, ptr(hi.c) if hi else None), "step_end")

    def exchange_on(self, exchange, parts):
        """Run ``exchange`` on the communication stream once this step's
        interface partials are packed; the library stream waits for the
        received planes before its seam pass."""
        from . import _lib
        torch = self.torch
        if self.comm is self.stream:
            with torch.cuda.stream(self.stream):
                return exchange(parts)
        _lib.check(self.op._lib.st_iface_wait(self.op._ctx, self.comm.cuda_stream), "iface_wait")
        with torch.cuda.stream(self.comm):
            recv = exchange(parts)
            done = torch.cuda.Event()
            done.record(self.comm)
        self.stream.wait_event(done)
        # the received planes are read by this step's seam pass on the
        # library stream: keep them until the next exchange, whose comm-stream
        # work is ordered after that seam pass (it waits for the next step's
        # packed-planes event); no record_stream on the library's stream,
        # which the context destroys before torch frees these buffers
        self._keep = recv
        return recv

    def maxima(self):
        am, tm = ctypes.c_double(), ctypes.c_double()
        from . import _lib
        _lib.check(self.op._lib.st_step_maxima(self.op._ctx, ctypes.byref(am),
                                               ctypes.byref(tm)), "step_maxima")
        return am.value, tm.value

    def maxima_history(self, n):
        from . import _lib
        am, tm = np.empty(n), np.empty(n)
        _lib.check(self.op._lib.st_step_maxima_history(self.op._ctx, n, _lib.dptr(am),
                                                       _lib.dptr(tm)), "step_maxima_history")
        return am, tm


def local_exchange(steppers):
    """In-process exchange among slabs on one device (tests / emulation):
    copies each slab's partial planes into fresh buffers for its peer."""
    import torch

    def run_step(dt, beams):
        parts = [s.begin(dt, beams) for s in steppers]
        torch.cuda.synchronize()     # every slab stream has finished its sweep
        for r, s in enumerate(steppers):
            recv = {}
            if 0 in parts[r]:
                p = parts[r - 1][1]
                recv[0] = Partials(p.f.clone(), None if p.c is None else p.c.clone())
            if 1 in parts[r]:
                p = parts[r + 1][0]
                recv[1] = Partials(p.f.clone(), None if p.c is None else p.c.clone())
            s._recv = recv
        torch.cuda.synchronize()
        for s in steppers:
            s.end(s._recv)
    return run_step


def local_exchange_overlapped(steppers):
    """In-process emulation of the overlapped schedule on one device: every
    slab's exchange runs on its communication stream after its own and its
    neighbour's interface events (st_iface_wait), while the interior chunks
    are still queued on the slab streams; the seam passes follow."""
    import torch
    from . import _lib

    def run_step(dt, beams):
        parts = [s.begin(dt, beams) for s in steppers]
        for r, s in enumerate(steppers):
            def ex(_, r=r, s=s):
                recv = {}
                for side, peer, pside in ((0, r - 1, 1), (1, r + 1, 0)):
                    if side not in parts[r]:
                        continue
                    o = steppers[peer].op
                    _lib.check(o._lib.st_iface_wait(o._ctx, s.comm.cuda_stream), "iface_wait")
                    p = parts[peer][pside]
                    recv[side] = Partials(p.f.clone(), None if p.c is None else p.c.clone())
                return recv
            s._recv = s.exchange_on(ex, parts[r])
        # a neighbour's packed planes are rewritten by its next step: this
        # emulation orders that by a device sync (NCCL does by stream order)
        torch.cuda.synchronize()
        for s in steppers:
            s.end(s._recv)
    return run_step
