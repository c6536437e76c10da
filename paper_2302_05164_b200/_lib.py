"""ctypes binding of libscantherm_b200.so (include/scantherm_b200.h).

The library is built in-tree (``__graft_entry__.build()`` or
``python -m paper_2302_05164_b200._build``).  There is no CPU fallback:
importing the operator without the shared library, or using it without
a CUDA device, raises.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libscantherm_b200.so")
if os.environ.get("ST_VARIANT"):  # kernel A/B experiments (see _build.py)
    LIB_PATH = os.path.join(_HERE, "libscantherm_b200_" + os.environ["ST_VARIANT"] + ".so")

ST_RHS_DIFFUSION = 1
ST_RHS_FACES = 2
ST_RHS_SOURCE = 4
ST_RHS_FROZEN_K = 8
ST_FIELD_T = 0
ST_FIELD_RC = 1

_dp = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u8p = ctypes.POINTER(ctypes.c_uint8)


class StMaterial(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in
                ("k_p", "k_m", "k_s", "rho", "c", "T_s", "T_l",
                 "latent_heat", "T_lat_s", "T_lat_l")]


class StBoundary(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in
                ("emissivity", "sigma_s", "T_inf", "T_v", "C_P", "C_T", "C_M",
                 "h_v", "T_h0", "T_max", "h_conv")]


class StLaser(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("radius", "h_powder", "cutoff_radii")]


class StParams(ctypes.Structure):
    _fields_ = [("mat", StMaterial), ("bnd", StBoundary), ("las", StLaser)]


class StBeam(ctypes.Structure):
    _fields_ = [("x", ctypes.c_double), ("y", ctypes.c_double),
                ("z_top", ctypes.c_double), ("power", ctypes.c_double),
                ("active", ctypes.c_int32), ("_pad", ctypes.c_int32)]


class StUnstructuredMesh(ctypes.Structure):
    _fields_ = [("n_cells", ctypes.c_int64), ("n_vertices", ctypes.c_int64),
                ("cell_verts", _i32p), ("cell_h", _dp), ("cell_anchor", _dp),
                ("is_slave", _u8p), ("is_dirichlet", _u8p),
                ("n_slaves", ctypes.c_int64), ("slaves", _i64p),
                ("slave_ptr", _i64p), ("slave_masters", _i64p),
                ("slave_weights", _dp), ("n_faces", ctypes.c_int64),
                ("face_cell", _i64p), ("face_vx", _dp), ("face_vy", _dp),
                ("face_area", _dp)]


class StStructuredMesh(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
                ("nz", ctypes.c_int32), ("degree", ctypes.c_int32),
                ("h", ctypes.c_double), ("x0", ctypes.c_double),
                ("y0", ctypes.c_double), ("z0", ctypes.c_double),
                ("dirichlet_bottom", ctypes.c_int32), ("top_faces", ctypes.c_int32),
                ("gx0", ctypes.c_int32), ("gNX", ctypes.c_int32),
                ("iface_lo", ctypes.c_int32), ("iface_hi", ctypes.c_int32),
                ("xext", _i32p)]


class StSegment(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in
                ("x0", "y0", "x1", "y1", "v", "power", "length", "duration", "t_start")]


class StLeaves(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("depth", ctypes.c_int32), ("cpl", ctypes.c_int32),
                ("level", ctypes.POINTER(ctypes.c_int8)), ("anchor", _i64p),
                ("active", _u8p), ("init_consol", _u8p)]


_i8p = ctypes.POINTER(ctypes.c_int8)
_DT = {1: np.int8, 2: np.uint8, 3: np.int32, 4: np.int64, 5: np.float64}


# (name, restype, argtypes) for every symbol of include/scantherm_b200.h
_VP = ctypes.c_void_p
SIGNATURES = [
    ("st_version", ctypes.c_int, []),
    ("st_last_error", ctypes.c_char_p, []),
    ("st_device_count", ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    ("st_ctx_create_unstructured", ctypes.c_int,
     [ctypes.c_int, ctypes.POINTER(StUnstructuredMesh), ctypes.POINTER(StParams),
      ctypes.POINTER(_VP)]),
    ("st_ctx_create_structured", ctypes.c_int,
     [ctypes.c_int, ctypes.POINTER(StStructuredMesh), ctypes.POINTER(StParams),
      ctypes.POINTER(_VP)]),
    ("st_ctx_destroy", ctypes.c_int, [_VP]),
    ("st_ctx_n_vertices", ctypes.c_int64, [_VP]),
    ("st_ctx_n_cells", ctypes.c_int64, [_VP]),
    ("st_ctx_qp_per_cell", ctypes.c_int, [_VP]),
    ("st_ctx_launches", ctypes.c_int64, [_VP]),
    ("st_ctx_stream", _VP, [_VP]),
    ("st_ctx_set_deterministic", ctypes.c_int, [_VP, ctypes.c_int]),
    ("st_set_field", ctypes.c_int, [_VP, ctypes.c_int, _dp, ctypes.c_int64]),
    ("st_get_field", ctypes.c_int, [_VP, ctypes.c_int, _dp, ctypes.c_int64]),
    ("st_set_uniform_rc", ctypes.c_int, [_VP, ctypes.c_double]),
    ("st_get_uniform_rc", ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_double)]),
    ("st_field_device_ptr", _VP, [_VP, ctypes.c_int]),
    ("st_snapshot_begin", ctypes.c_int, [_VP, _dp, _dp]),
    ("st_scan_layer", ctypes.c_int,
     [_VP, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int, _i32p,
      ctypes.POINTER(StSegment), _dp, ctypes.POINTER(ctypes.c_int), _dp, _dp]),
    ("st_beam_schedule", ctypes.c_int,
     [_VP, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int, _i32p,
      ctypes.POINTER(StSegment), _dp, ctypes.POINTER(StBeam)]),
    ("st_snapshot_wait", ctypes.c_int, [_VP, ctypes.c_int]),
    ("st_evaluate_rhs", ctypes.c_int,
     [_VP, _dp, _dp, ctypes.c_int, ctypes.c_double, ctypes.POINTER(StBeam),
      ctypes.c_int, _dp]),
    ("st_lumped_capacity", ctypes.c_int, [_VP, _dp, _dp]),
    ("st_apply_mass", ctypes.c_int, [_VP, _dp, _dp]),
    ("st_explicit_step", ctypes.c_int,
     [_VP, _dp, ctypes.c_double, _dp, ctypes.POINTER(StBeam), ctypes.c_int, _dp]),
    ("st_update_history", ctypes.c_int, [_VP, _dp, _dp]),
    ("st_apply_jacobian", ctypes.c_int, [_VP, _dp, _dp, _dp, ctypes.c_double, _dp]),
    ("st_jacobian_diagonal", ctypes.c_int, [_VP, _dp, _dp, ctypes.c_double, _dp]),
    ("st_explicit_steps", ctypes.c_int,
     [_VP, ctypes.c_int, _dp, ctypes.POINTER(StBeam), ctypes.c_int,
      ctypes.POINTER(ctypes.c_int), _dp, _dp]),
    ("st_implicit_step", ctypes.c_int,
     [_VP, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
      ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
      ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    ("st_finish_implicit_step", ctypes.c_int, [_VP]),
    ("st_pcg", ctypes.c_int,
     [_VP, _dp, _dp, ctypes.c_double, _dp, ctypes.c_double, ctypes.c_int,
      ctypes.c_int, _dp, _dp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    ("st_spectral_radius", ctypes.c_int,
     [_VP, ctypes.c_double, _dp, ctypes.c_double, ctypes.c_int, _dp,
      ctypes.POINTER(ctypes.c_int)]),
    ("st_profile_enable", ctypes.c_int, [_VP, ctypes.c_int]),
    ("st_profile_read", ctypes.c_int,
     [_VP, _dp, _i64p, ctypes.c_char_p, ctypes.c_int]),
    ("st_algorithmic_bytes_per_dof", ctypes.c_double, [_VP]),
    ("st_explicit_step_begin", ctypes.c_int,
     [_VP, ctypes.c_double, ctypes.POINTER(StBeam), ctypes.c_int]),
    ("st_iface_partials", ctypes.c_int,
     [_VP, ctypes.c_int, ctypes.POINTER(_dp), ctypes.POINTER(_dp), _i64p]),
    ("st_explicit_step_end", ctypes.c_int, [_VP, _VP, _VP, _VP, _VP]),
    ("st_step_maxima", ctypes.c_int, [_VP, _dp, _dp]),
    ("st_step_maxima_history", ctypes.c_int, [_VP, ctypes.c_int, _dp, _dp]),
    ("st_iface_wait", ctypes.c_int, [_VP, _VP]),
    ("st_bench_explicit", ctypes.c_int,
     [_VP, ctypes.c_int, _dp, ctypes.POINTER(StBeam), ctypes.c_int, ctypes.c_int64,
      ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]),
    # leaf tables (host C++, st_forest.cpp)
    ("st_tables_get", ctypes.c_int,
     [_VP, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), _i64p,
      ctypes.POINTER(_VP)]),
    ("st_tables_free", None, [_VP]),
    ("st_coarse_grid", ctypes.c_int,
     [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, _i64p, _u8p, ctypes.POINTER(_VP)]),
    ("st_build_dofmap", ctypes.c_int,
     [ctypes.POINTER(StLeaves), ctypes.c_int64, ctypes.c_int, ctypes.POINTER(_VP)]),
    ("st_interface_faces", ctypes.c_int, [ctypes.POINTER(StLeaves), ctypes.POINTER(_VP)]),
    ("st_plan_layer", ctypes.c_int,
     [ctypes.POINTER(StLeaves), ctypes.c_int32, _dp, ctypes.c_int32, ctypes.POINTER(_VP)]),
    ("st_transfer_nodal", ctypes.c_int,
     [ctypes.POINTER(StLeaves), _i64p, ctypes.c_int64, _i32p, _i64p, ctypes.c_int64, _i64p,
      _i64p, ctypes.c_int64, _i64p, _dp, ctypes.c_int32, _dp, ctypes.c_double, _dp, _i8p]),
    ("st_transfer_history", ctypes.c_int,
     [ctypes.POINTER(StLeaves), ctypes.POINTER(StLeaves), _i64p, _i64p, ctypes.c_int64, _i64p,
      _i64p, _i64p, _dp, _dp]),
    ("st_host_distribute", ctypes.c_int, [ctypes.c_int64, _i64p, _i64p, _i64p, _dp, _dp]),
    ("st_host_condense", ctypes.c_int, [ctypes.c_int64, _i64p, _i64p, _i64p, _dp, _dp]),
]

_lib = None


class StError(RuntimeError):
    """A libscantherm_b200 call failed."""


def load():
    """Load and type the shared library (raises if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'`; "
            "there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc, what=""):
    if rc != 0:
        msg = load().st_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        raise StError(f"{what} failed ({rc}): {msg}")


def tables_dict(t):
    """Copy every array of an st_tables bag into numpy (names probed from
    the known result sets)."""
    lib = load()
    names = ("level", "anchor", "active", "init_consol", "same_src", "ancestor_src",
             "group_rows", "group_ptr", "group_kids", "coarsened_min_rc", "vertices",
             "cell_verts", "active_rows", "is_slave", "is_dirichlet", "slaves", "slave_ptr",
             "slave_masters", "slave_weights", "cell_rows", "offset", "fsize")
    out = {}
    dt, nd = ctypes.c_int(), ctypes.c_int()
    dims = (ctypes.c_int64 * 4)()
    data = ctypes.c_void_p()
    for n in names:
        if lib.st_tables_get(t, n.encode(), ctypes.byref(dt), ctypes.byref(nd), dims,
                             ctypes.byref(data)) != 0:
            continue
        shape = tuple(dims[i] for i in range(nd.value))
        typ = _DT[dt.value]
        count = int(np.prod(shape)) if shape else 0
        if count == 0:
            out[n] = np.zeros(shape, dtype=typ)
            continue
        buf = (ctypes.c_char * (count * np.dtype(typ).itemsize)).from_address(data.value)
        out[n] = np.frombuffer(buf, dtype=typ).reshape(shape).copy()
    return out


def dptr(a):
    """float64 C-contiguous array -> double* (None passes NULL)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], "need contiguous float64"
    return a.ctypes.data_as(_dp)


def as_f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def params_struct(params):
    """Reference-compatible ProcessParams -> StParams (extensions default off)."""
    m, b, l = params.material, params.boundary, params.laser
    mat = StMaterial(m.k_p, m.k_m, m.k_s, m.rho, m.c, m.T_s, m.T_l,
                     float(getattr(m, "latent_heat", 0.0) or 0.0),
                     float(getattr(m, "T_lat_s", 1878.0)),
                     float(getattr(m, "T_lat_l", 1928.0)))
    bnd = StBoundary(b.emissivity, b.sigma_s, b.T_inf, b.T_v, b.C_P, b.C_T, b.C_M,
                     b.h_v, b.T_h0, b.T_v + b.T_max_offset,
                     float(getattr(b, "h_conv", 0.0) or 0.0))
    las = StLaser(l.radius, l.h_powder, l.cutoff_radii)
    return StParams(mat, bnd, las)


def beams_array(beams):
    """BEAM_DTYPE structured array -> (pointer, count)."""
    if beams is None or len(beams) == 0:
        return None, 0
    assert beams.dtype.itemsize == ctypes.sizeof(StBeam)
    return beams.ctypes.data_as(ctypes.POINTER(StBeam)), int(beams.size)
