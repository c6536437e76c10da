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
``st_explicit_step_end``); :class:`SlabDriver` holds the rank logic and
is shared by the GPU path (NCCL through ``torch.distributed`` on the
library's own stream) and the CPU reference path used by the gloo tests
(:class:`tests`' oracle slabs).
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from .mesh import StructuredBox


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


def gather_global(boxes, locals_):
    """Assemble the global field from every rank's slab field."""
    glob = boxes[0].glob
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
    sides with a neighbour (0 = lower, 1 = upper) and end(recv) where
    recv maps side -> the neighbour's Partials.  ``exchange`` maps
    {side: Partials} -> {side: Partials} (torch.distributed or local)."""

    def __init__(self, stepper, exchange):
        self.stepper = stepper
        self.exchange = exchange

    def step(self, dt, beams):
        parts = self.stepper.begin(dt, beams)
        recv = self.exchange(parts)
        self.stepper.end(recv)


def torch_exchange(rank, world, group=None):
    """Exchange with torch.distributed point-to-point (NCCL or gloo).

    Sends side-1 partials to rank+1 and side-0 partials to rank-1; returns
    what the neighbours sent.  For NCCL the caller runs this with the
    library stream as torch's current stream so the transfer is ordered
    after the sweep and before the seam pass."""
    import torch
    import torch.distributed as dist

    def ex(parts):
        ops, recv = [], {}
        for side, peer in ((0, rank - 1), (1, rank + 1)):
            if side not in parts or not (0 <= peer < world):
                continue
            mine = parts[side]
            rf = torch.empty_like(mine.f)
            rc = torch.empty_like(mine.c) if mine.c is not None else None
            ops.append(dist.P2POp(dist.isend, mine.f, peer, group))
            ops.append(dist.P2POp(dist.irecv, rf, peer, group))
            if mine.c is not None:
                ops.append(dist.P2POp(dist.isend, mine.c, peer, group))
                ops.append(dist.P2POp(dist.irecv, rc, peer, group))
            recv[side] = Partials(rf, rc)
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return recv

    return ex


class GpuSlabStepper:
    """Split step on a B200 slab operator (ThermalOperator on a SlabBox)."""

    def __init__(self, op):
        import torch
        self.op = op
        self.torch = torch
        self.stream = torch.cuda.ExternalStream(op.stream_ptr())
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

    def maxima(self):
        am, tm = ctypes.c_double(), ctypes.c_double()
        from . import _lib
        _lib.check(self.op._lib.st_step_maxima(self.op._ctx, ctypes.byref(am),
                                               ctypes.byref(tm)), "step_maxima")
        return am.value, tm.value


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
