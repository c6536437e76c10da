"""Drop-in ThermalOperator running on a B200 through libscantherm_b200.

Mirrors the public surface of the reference class
``scantherm.operators.ThermalOperator`` (operators.py:84-459): same
constructor ``(forest, dofmap, params, settings)``, same attributes
(forest, dofmap, params, settings, epoch, n_cells) and same methods with
the same argument meaning, array shapes and error behaviour, so the
reference time integrators (timestepping.py) and driver run on it
unchanged.  Every numeric method is one call into the C ABI
(include/scantherm_b200.h); the host only stages arrays.

Additions beyond the reference surface:
  * ``beam`` may also be a list of BeamStates (concurrent spots);
  * ``explicit_steps`` and the resident-state methods (``set_state``,
    ``run_explicit``, ``implicit_step``) keep T and r_c in HBM across
    steps — the host loop of the reference remains valid, only slower;
  * :class:`paper_2302_05164_b200.mesh.StructuredBox` meshes (degree
    1..4) run on the structured backend.
"""

import ctypes

import numpy as np

from . import _lib
from .mesh import interface_faces
from .physics import BEAM_DTYPE, pack_beams

_SQ3 = np.sqrt(3.0)
GAUSS_1D = np.array([-1.0 / _SQ3, 1.0 / _SQ3])


def _beams(beam):
    if beam is None:
        return np.zeros(0, dtype=BEAM_DTYPE)
    if isinstance(beam, np.ndarray) and beam.dtype == BEAM_DTYPE:
        return np.ascontiguousarray(beam)
    if isinstance(beam, (list, tuple)):
        return pack_beams(list(beam))
    return pack_beams([beam])


class _Tangent:
    """Opaque linearisation handle: the kernels recompute k, dk/dT and
    grad T at the quadrature points from T_lin (operators.py:373-378)."""

    def __init__(self, T_lin, r_c):
        self.T_lin = _lib.as_f64(T_lin)
        self.r_c = None if r_c is None else _lib.as_f64(r_c)


class ThermalOperator:
    """All finite element kernels for one mesh epoch, on the GPU."""

    def __init__(self, forest, dofmap, params, settings, device=0):
        if dofmap.h_fine != forest.h_fine:
            raise ValueError("dofmap does not belong to this forest")
        self.forest = forest
        self.dofmap = dofmap
        self.params = params
        self.settings = settings
        self.epoch = forest.epoch
        self._lib = _lib.load()
        self._ctx = ctypes.c_void_p()
        self._cinv = None
        self._uniform_rc = 1.0  # the context's uniform r_c (st_set_uniform_rc)
        pst = _lib.params_struct(params)
        if getattr(forest, "structured", False):
            self.structured = True
            m = _lib.StStructuredMesh(forest.nx, forest.ny, forest.nz, forest.degree,
                                      forest.h, forest.origin[0], forest.origin[1],
                                      forest.origin[2], int(forest.dirichlet_bottom),
                                      int(forest.top_faces), int(getattr(forest, "gx0", 0)),
                                      int(getattr(forest, "gNX", 0)),
                                      int(bool(getattr(forest, "iface_lo", False))),
                                      int(bool(getattr(forest, "iface_hi", False))))
            xext = getattr(forest, "xext", None)
            if xext is not None:
                self._xext = np.ascontiguousarray(xext, dtype=np.int32)
                m.xext = self._xext.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            _lib.check(self._lib.st_ctx_create_structured(
                device, ctypes.byref(m), ctypes.byref(pst), ctypes.byref(self._ctx)),
                "st_ctx_create_structured")
            self.n_cells = forest.n_cells
        else:
            self.structured = False
            self._create_unstructured(device, pst)
        self.nv = int(self._lib.st_ctx_n_vertices(self._ctx))
        self.qpc = int(self._lib.st_ctx_qp_per_cell(self._ctx))
        _lib.check(self._lib.st_ctx_set_deterministic(
            self._ctx, int(getattr(settings, "deterministic", True))), "set_deterministic")

    # -- construction ------------------------------------------------------------
    def _create_unstructured(self, device, pst):
        forest, dm = self.forest, self.dofmap
        rows = np.asarray(dm.active_rows)
        self.n_cells = len(rows)
        h_m = np.ascontiguousarray(forest.size_m(rows), dtype=np.float64)
        anchor_m = np.ascontiguousarray(forest.anchor[rows] * forest.h_fine, dtype=np.float64)
        cv = np.ascontiguousarray(dm.cell_verts, dtype=np.int32)
        # facet quadrature exactly as the reference builds it (operators.py:118-134)
        fs = interface_faces(forest)
        pos = np.full(forest.n_cells, -1, dtype=np.int64)
        pos[rows] = np.arange(len(rows))
        cell_pos = pos[fs.cell_rows]
        if len(cell_pos):
            size = forest.size(fs.cell_rows).astype(np.float64)
            r0 = fs.offset / size[:, None]
            rr = fs.fsize / size
            u = r0[:, :, None] + (GAUSS_1D[None, None, :] + 1.0) / 2.0 * rr[:, None, None]
            Vx = np.stack([1.0 - u[:, 0], u[:, 0]], axis=1)
            Vy = np.stack([1.0 - u[:, 1], u[:, 1]], axis=1)
            area = (fs.fsize * forest.h_fine / 2.0) ** 2
        else:
            Vx = Vy = np.zeros((0, 2, 2))
            area = np.zeros(0)
        keep = dict(
            cv=cv, h=h_m, anc=anchor_m,
            sl=np.ascontiguousarray(dm.is_slave, dtype=np.uint8),
            di=np.ascontiguousarray(dm.is_dirichlet, dtype=np.uint8),
            slaves=np.ascontiguousarray(dm.slaves, dtype=np.int64),
            sptr=np.ascontiguousarray(dm.slave_ptr, dtype=np.int64),
            smast=np.ascontiguousarray(dm.slave_masters, dtype=np.int64),
            sw=np.ascontiguousarray(dm.slave_weights, dtype=np.float64),
            fc=np.ascontiguousarray(cell_pos, dtype=np.int64),
            vx=np.ascontiguousarray(Vx, dtype=np.float64),
            vy=np.ascontiguousarray(Vy, dtype=np.float64),
            area=np.ascontiguousarray(area, dtype=np.float64))
        P = ctypes.POINTER
        m = _lib.StUnstructuredMesh(
            len(rows), dm.n_vertices,
            keep["cv"].ctypes.data_as(P(ctypes.c_int32)), _lib.dptr(keep["h"]),
            _lib.dptr(keep["anc"]), keep["sl"].ctypes.data_as(P(ctypes.c_uint8)),
            keep["di"].ctypes.data_as(P(ctypes.c_uint8)), len(keep["slaves"]),
            keep["slaves"].ctypes.data_as(P(ctypes.c_int64)),
            keep["sptr"].ctypes.data_as(P(ctypes.c_int64)),
            keep["smast"].ctypes.data_as(P(ctypes.c_int64)), _lib.dptr(keep["sw"]),
            len(keep["fc"]), keep["fc"].ctypes.data_as(P(ctypes.c_int64)),
            _lib.dptr(keep["vx"]), _lib.dptr(keep["vy"]), _lib.dptr(keep["area"]))
        _lib.check(self._lib.st_ctx_create_unstructured(
            device, ctypes.byref(m), ctypes.byref(pst), ctypes.byref(self._ctx)),
            "st_ctx_create_unstructured")
        self._faces_cell_pos = cell_pos

    # -- SIMD-batch view of the reference (API parity, not on the device path) --
    @property
    def verts8(self):
        """(n_cells, 8) int64 corner vertex ids (reference attribute)."""
        if getattr(self.forest, "structured", False):
            return self.forest.cell_node_ids()
        return np.asarray(self.dofmap.cell_verts, dtype=np.int64)

    def _batch_colors(self):
        """First-fit colouring of n_lanes-wide cell batches such that the
        batches of one colour share no vertex (the reference's CPU SIMD
        scatter schedule, operators.py:136-156).  The device never needs
        it: its non-deterministic mode scatters with fp64 atomics.  Each
        vertex carries a bit set of the colours already touching it; a
        batch takes the lowest colour absent from the union of its
        vertices' sets."""
        if getattr(self, "_colors", None) is not None:
            return self._colors
        lanes = int(getattr(self.settings, "n_lanes", 8))
        v8 = self.verts8
        used = [0] * int(self.nv)
        groups = {}
        for start in range(0, len(v8), lanes):
            verts = np.unique(v8[start:start + lanes]).tolist()
            taken = 0
            for v in verts:
                taken |= used[v]
            color = (~taken & (taken + 1)).bit_length() - 1
            for v in verts:
                used[v] |= 1 << color
            groups.setdefault(color, []).append(slice(start, min(start + lanes, len(v8))))
        self._colors = [groups[c] for c in sorted(groups)]
        return self._colors

    def close(self):
        if getattr(self, "_ctx", None) is not None and self._ctx.value:
            self._lib.st_ctx_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers ---------------------------------------------------------------------
    def _vec(self, v, name="vector"):
        v = _lib.as_f64(v)
        if v.shape != (self.nv,):
            raise ValueError(f"{name} must have shape ({self.nv},), got {v.shape}")
        return v

    def _rc(self, r_c):
        if r_c is None:
            return None
        r = _lib.as_f64(r_c)
        if r.size != self.n_cells * self.qpc:
            raise ValueError("r_c does not match the active cells of this operator")
        return r.reshape(-1)

    def _call_rc(self, r_c):
        """r_c for a per-call entry point: a structured context evaluates a
        uniform consolidated history (every entry equal to the context's
        uniform value, 1 unless set_state set another) without a per-point
        array (NULL), which a fitted part requires; else the array."""
        r = self._rc(r_c)
        if (r is not None and self.structured and r.size and r[0] >= 1.0
                and r[0] == self._uniform_rc and np.all(r == r[0])):
            return None, True
        return r, False

    @property
    def launches(self):
        """Kernels launched by this operator so far."""
        return int(self._lib.st_ctx_launches(self._ctx))

    def check_epoch(self, field):
        if getattr(field, "epoch", self.epoch) != self.epoch:
            raise ValueError("field epoch does not match operator epoch")

    # -- history (operators.py:219-225) ---------------------------------------------------
    def update_history(self, history, T):
        self.check_epoch(history)
        T = self._vec(T, "T")
        rc = np.ascontiguousarray(history.r_c, dtype=np.float64)
        flat = rc.reshape(-1)
        if self.structured and flat.size and flat[0] >= 1.0 and np.all(flat == flat[0]):
            # max(r_c, g) with g <= 1 <= r_c: a consolidated history is a
            # fixed point (and a fitted part stores none)
            return history
        _lib.check(self._lib.st_update_history(self._ctx, _lib.dptr(T), _lib.dptr(flat)),
                   "update_history")
        history.r_c[...] = rc.reshape(history.r_c.shape)
        return history

    # -- rhs (operators.py:247-321) ---------------------------------------------------
    def evaluate_rhs(self, T, r_c, beam=None, diffusion=True, faces=True, source=True,
                     frozen_k=None):
        T = self._vec(T, "T")
        flags = 0
        if diffusion:
            flags |= _lib.ST_RHS_DIFFUSION
            if frozen_k is not None:
                flags |= _lib.ST_RHS_FROZEN_K
            elif r_c is None:
                raise ValueError("evaluate_rhs needs r_c unless frozen_k is given")
        if faces:
            flags |= _lib.ST_RHS_FACES
        if source:
            flags |= _lib.ST_RHS_SOURCE
        rc = self._call_rc(r_c)[0] if (diffusion and frozen_k is None) else None
        b = _beams(beam if source else None)
        bp, nb = _lib.beams_array(b)
        out = np.empty(self.nv)
        _lib.check(self._lib.st_evaluate_rhs(
            self._ctx, _lib.dptr(T), _lib.dptr(rc), flags,
            float(frozen_k) if frozen_k is not None else 0.0, bp, nb, _lib.dptr(out)),
            "evaluate_rhs")
        return out

    # -- capacity (operators.py:325-348) -----------------------------------------------
    def lumped_capacity(self, T=None):
        out = np.empty(self.nv)
        Tp = self._vec(T, "T") if T is not None else None
        _lib.check(self._lib.st_lumped_capacity(self._ctx, _lib.dptr(Tp), _lib.dptr(out)),
                   "lumped_capacity")
        return out

    def capacity_inverse(self):
        if self._cinv is None:
            self._cinv = 1.0 / self.lumped_capacity()
        return self._cinv

    def apply_mass(self, v):
        v = self._vec(v, "v")
        out = np.empty(self.nv)
        _lib.check(self._lib.st_apply_mass(self._ctx, _lib.dptr(v), _lib.dptr(out)),
                   "apply_mass")
        return out

    # -- explicit step (operators.py:352-369) ---------------------------------------------
    def explicit_fused_step(self, T, dt, r_c, beam=None, fused=True):
        """One forward Euler step; returns a new array (T is not modified).
        ``fused`` is accepted for interface parity: the device kernel
        always evaluates T + dt * (cinv * f) in one pass."""
        T = self._vec(T, "T")
        if r_c is None:
            raise ValueError("explicit step needs r_c")
        rc, _ = self._call_rc(r_c)
        b = _beams(beam)
        bp, nb = _lib.beams_array(b)
        out = np.empty(self.nv)
        _lib.check(self._lib.st_explicit_step(self._ctx, _lib.dptr(T), float(dt),
                                              _lib.dptr(rc), bp, nb, _lib.dptr(out)),
                   "explicit_fused_step")
        return out

    # -- Newton pieces (operators.py:373-459) --------------------------------------------
    def _tangent_fields(self, T_lin, r_c):
        return _Tangent(T_lin, r_c)

    def apply_jacobian(self, v, T_lin, r_c, dt, tangent=None):
        if isinstance(tangent, _Tangent):
            T_lin, r_c = tangent.T_lin, tangent.r_c
        v = self._vec(v, "v")
        T_lin = self._vec(T_lin, "T_lin")
        rc = self._rc(r_c)
        out = np.empty(self.nv)
        _lib.check(self._lib.st_apply_jacobian(self._ctx, _lib.dptr(v), _lib.dptr(T_lin),
                                               _lib.dptr(rc), float(dt), _lib.dptr(out)),
                   "apply_jacobian")
        return out

    def jacobian_diagonal(self, T_lin, r_c, dt, tangent=None):
        if isinstance(tangent, _Tangent):
            T_lin, r_c = tangent.T_lin, tangent.r_c
        T_lin = self._vec(T_lin, "T_lin")
        rc = self._rc(r_c)
        out = np.empty(self.nv)
        _lib.check(self._lib.st_jacobian_diagonal(self._ctx, _lib.dptr(T_lin), _lib.dptr(rc),
                                                  float(dt), _lib.dptr(out)),
                   "jacobian_diagonal")
        return out

    def solve_jacobian(self, b, T_lin, r_c, dt, tol, max_iter, precondition=True,
                       diag_inv=None):
        """Device PCG for J(T_lin) x = b (krylov_solve, timestepping.py:102):
        Jacobi with the caller's ``diag_inv`` when given, else with the
        exact Jacobian diagonal (``precondition``), or none."""
        b = self._vec(b, "b")
        di = None if diag_inv is None else self._vec(diag_inv, "diag_inv")
        T_lin = self._vec(T_lin, "T_lin")
        rc = self._rc(r_c)
        x = np.empty(self.nv)
        it = ctypes.c_int()
        ok = ctypes.c_int()
        _lib.check(self._lib.st_pcg(self._ctx, _lib.dptr(T_lin), _lib.dptr(rc), float(dt),
                                    _lib.dptr(b), float(tol), int(max_iter),
                                    int(bool(precondition) or di is not None), _lib.dptr(di),
                                    _lib.dptr(x), ctypes.byref(it),
                                    ctypes.byref(ok)), "pcg")
        return x, it.value, bool(ok.value)

    def spectral_radius(self, k_frozen, seed=0, tol=1e-9, max_iter=500):
        """rho(C~^-1 K) at conductivity k_frozen by power iteration on the
        device (timestepping.py:49-99): the start vector is the reference's
        (default_rng(seed), normalised on the host), the apply is the
        reference's (close constraints, zero Dirichlet entries, diffusion-only
        rhs, scale by C~^-1, zero Dirichlet/slave rows).  The number of
        operator applies is kept in ``last_power_iterations``."""
        v0 = np.random.default_rng(seed).standard_normal(self.nv)
        v0 /= np.linalg.norm(v0)
        rho = ctypes.c_double()
        it = ctypes.c_int()
        _lib.check(self._lib.st_spectral_radius(self._ctx, float(k_frozen), _lib.dptr(v0),
                                                float(tol), int(max_iter), ctypes.byref(rho),
                                                ctypes.byref(it)), "spectral_radius")
        self.last_power_iterations = it.value
        return rho.value

    # -- resident state ----------------------------------------------------------------
    def set_state(self, T, r_c):
        """Upload (T, r_c) to HBM; r_c may be a scalar >= 1 (consolidated)."""
        T = self._vec(T, "T")
        _lib.check(self._lib.st_set_field(self._ctx, _lib.ST_FIELD_T, _lib.dptr(T), T.size),
                   "set T")
        if np.isscalar(r_c):
            _lib.check(self._lib.st_set_uniform_rc(self._ctx, float(r_c)), "set r_c")
            self._uniform_rc = float(r_c)
            return
        rc = self._rc(r_c)
        if np.all(rc >= 1.0) and np.all(rc == rc[0]) if rc.size else False:
            _lib.check(self._lib.st_set_uniform_rc(self._ctx, float(rc[0])), "set r_c")
            self._uniform_rc = float(rc[0])
        else:
            _lib.check(self._lib.st_set_field(self._ctx, _lib.ST_FIELD_RC, _lib.dptr(rc),
                                              rc.size), "set r_c")

    def get_state(self, r_c_shape=None, out=None):
        """Download (T, r_c).  `out` may be a caller-owned float64 array of
        n_vertices (e.g. pinned host memory) that receives T.  A uniform
        resident r_c (st_set_uniform_rc, r_c >= 1) is never stored on the
        device, so it comes back as a read-only broadcast of that value
        instead of an expanded copy."""
        T = np.empty(self.nv) if out is None else out
        _lib.check(self._lib.st_get_field(self._ctx, _lib.ST_FIELD_T, _lib.dptr(T), T.size),
                   "get T")
        n = self.n_cells * self.qpc
        v = ctypes.c_double()
        uni = self._lib.st_get_uniform_rc(self._ctx, ctypes.byref(v))
        if uni < 0:
            _lib.check(uni, "get r_c")
        if uni == 1:
            rc = np.broadcast_to(np.float64(v.value), (n,))
        else:
            rc = np.empty(n)
            _lib.check(self._lib.st_get_field(self._ctx, _lib.ST_FIELD_RC, _lib.dptr(rc), n),
                       "get r_c")
        if r_c_shape is not None:
            rc = rc.reshape(r_c_shape) if uni != 1 else np.broadcast_to(np.float64(v.value),
                                                                          r_c_shape)
        return T, rc

    def _seg_args(self, layer_paths):
        from .physics import segment_table
        counts, segs, z = segment_table(layer_paths)
        keep = (counts, segs if len(segs) else np.zeros((1, 9)), z)
        return keep, (len(counts), keep[0].ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                      keep[1].ctypes.data_as(ctypes.POINTER(_lib.StSegment)), _lib.dptr(keep[2]))

    def run_scan(self, layer_paths, dt, n_steps, step0=1):
        """Forward-Euler steps step0 .. step0+n_steps-1 of a scan phase on
        the resident state with the beams of ``layer_paths`` (one or several
        concurrently scanned LayerPaths) evaluated on the device
        (st_scan_layer).  Returns (fail_step, t_extreme, t_max)."""
        paths = layer_paths if isinstance(layer_paths, (list, tuple)) else [layer_paths]
        keep, (np_, cnt, seg, z) = self._seg_args(paths)
        fail, ext, tmax = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
        _lib.check(self._lib.st_scan_layer(self._ctx, int(n_steps), int(step0), float(dt),
                                           float(paths[0].scan_duration()), np_, cnt, seg, z,
                                           ctypes.byref(fail), ctypes.byref(ext),
                                           ctypes.byref(tmax)), "scan_layer")
        return fail.value, ext.value, tmax.value

    def beam_schedule(self, layer_paths, dt, n_steps, step0=1):
        """The device-evaluated beam records (n_steps, n_paths) BEAM_DTYPE."""
        from .physics import BEAM_DTYPE
        paths = layer_paths if isinstance(layer_paths, (list, tuple)) else [layer_paths]
        keep, (np_, cnt, seg, z) = self._seg_args(paths)
        out = np.zeros((int(n_steps), np_), dtype=BEAM_DTYPE)
        _lib.check(self._lib.st_beam_schedule(self._ctx, int(n_steps), int(step0), float(dt), np_,
                                              cnt, seg, z,
                                              out.ctypes.data_as(ctypes.POINTER(_lib.StBeam))),
                   "beam_schedule")
        return out

    def snapshot(self, T_out, r_c_out=None):
        """Start an asynchronous snapshot of the resident state into the
        caller's arrays (pinned host memory keeps it asynchronous): the
        device copy is ordered after the steps queued so far, the drain to
        the host overlaps the steps queued after it.  Complete it with
        :meth:`snapshot_wait` before reading the arrays."""
        if T_out.dtype != np.float64 or T_out.shape != (self.nv,) or \
                not T_out.flags["C_CONTIGUOUS"]:
            raise ValueError("T_out must be a contiguous float64 array of n_vertices")
        rc = None
        if r_c_out is not None:
            if r_c_out.dtype != np.float64 or r_c_out.size != self.n_cells * self.qpc or \
                    not r_c_out.flags["C_CONTIGUOUS"]:
                raise ValueError("r_c_out must be a contiguous float64 array of n_cells * qp")
            rc = r_c_out.reshape(-1)
        self._snap = (T_out, r_c_out)  # keep the buffers alive until the drain ends
        _lib.check(self._lib.st_snapshot_begin(self._ctx, _lib.dptr(T_out), _lib.dptr(rc)),
                   "snapshot")

    def snapshot_wait(self, block=True):
        """True when the last snapshot is on the host (block: wait for it)."""
        r = self._lib.st_snapshot_wait(self._ctx, int(bool(block)))
        if r < 0:
            _lib.check(r, "snapshot_wait")
        return bool(r)

    def run_explicit(self, dts, beams):
        """Forward-Euler steps on the resident state (timestepping.py:211-221).

        dts (n,), beams (n, n_beams) BEAM_DTYPE.  Returns (fail_step,
        t_extreme, t_max); fail_step = 0 when every step was stable."""
        dts = _lib.as_f64(dts)
        n = len(dts)
        beams = np.ascontiguousarray(beams)
        nb = beams.shape[1] if beams.ndim == 2 else 0
        bp = beams.ctypes.data_as(ctypes.POINTER(_lib.StBeam)) if nb else None
        fail = ctypes.c_int()
        ext = ctypes.c_double()
        tmax = ctypes.c_double()
        _lib.check(self._lib.st_explicit_steps(self._ctx, n, _lib.dptr(dts), bp, nb,
                                               ctypes.byref(fail), ctypes.byref(ext),
                                               ctypes.byref(tmax)), "explicit_steps")
        return fail.value, ext.value, tmax.value

    def implicit_step(self, dt, settings):
        """One backward-Euler step on the resident state; returns
        (newton_iters, krylov_iters) or None when Newton failed."""
        nn, nk, ok = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        pre = 1 if settings.preconditioner == "diagonal" else 0
        _lib.check(self._lib.st_implicit_step(
            self._ctx, float(dt), settings.newton_tol, settings.newton_abs_tol,
            settings.newton_max_iter, settings.krylov_tol, settings.krylov_max_iter, pre,
            ctypes.byref(nn), ctypes.byref(nk), ctypes.byref(ok)), "implicit_step")
        if not ok.value:
            return None
        return nn.value, nk.value

    def finish_implicit_step(self):
        _lib.check(self._lib.st_finish_implicit_step(self._ctx), "finish_implicit_step")

    # -- measurement --------------------------------------------------------------------
    def profile(self, enable=True):
        _lib.check(self._lib.st_profile_enable(self._ctx, int(enable)), "profile")

    def profile_read(self):
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        name = ctypes.create_string_buffer(64)
        _lib.check(self._lib.st_profile_read(self._ctx, ctypes.byref(ms), ctypes.byref(n),
                                             name, 64), "profile_read")
        return ms.value, n.value, name.value.decode()

    def bench_explicit(self, dts, beams, flush_bytes=0):
        """Device-timed explicit steps on the resident state; returns
        per-step (total_ms, main_kernel_ms) arrays (st_bench_explicit)."""
        dts = _lib.as_f64(dts)
        n = len(dts)
        beams = np.ascontiguousarray(beams)
        nb = beams.shape[1] if beams.ndim == 2 else 0
        bp = beams.ctypes.data_as(ctypes.POINTER(_lib.StBeam)) if nb else None
        step_ms = np.zeros(n, dtype=np.float32)
        main_ms = np.zeros(n, dtype=np.float32)
        fp = ctypes.POINTER(ctypes.c_float)
        _lib.check(self._lib.st_bench_explicit(self._ctx, n, _lib.dptr(dts), bp, nb,
                                               int(flush_bytes), step_ms.ctypes.data_as(fp),
                                               main_ms.ctypes.data_as(fp)), "bench_explicit")
        return step_ms, main_ms

    def bytes_per_dof(self):
        return float(self._lib.st_algorithmic_bytes_per_dof(self._ctx))

    def stream_ptr(self):
        return self._lib.st_ctx_stream(self._ctx)


def close_constraints(dofmap, values):
    """Overwrite hanging-vertex entries with their master interpolation."""
    return dofmap.distribute(values)
