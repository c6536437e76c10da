/*
 * scantherm_b200 — C ABI of the B200 (sm_100a) heat-operator library.
 *
 * Drop-in boundary for the hot path of the reference package
 * `scantherm` (arXiv 2302.05164 re-implementation, Python/numpy).  The
 * reference has no native FFI; its operator interface is the Python
 * class ThermalOperator (pkg/src/scantherm/operators.py:84).  Each entry
 * point below replaces one method of that class or of the time
 * integrator, and is bound from Python with ctypes
 * (paper_2302_05164_b200/_lib.py; INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - plain pointers and sizes; float64 fields, int32/int64 indices;
 *  - every function returns 0 on success and a negative ST_E* code on
 *    failure; st_last_error() gives the message of the calling thread's
 *    last failure (reference errors are ValueError / RuntimeError /
 *    InstabilityError; the Python layer re-raises the same types);
 *  - host pointers ("const double* T", "double* out") are copied
 *    host<->device inside the call on the context's stream and the call
 *    returns after the result is on the host;
 *  - the context owns its device buffers; one context per mesh epoch
 *    (the reference rebuilds its operator per mesh update,
 *    driver.py:162-164); calls on one context are stream-ordered and
 *    not thread-safe.
 */
#ifndef SCANTHERM_B200_H
#define SCANTHERM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ST_OK 0
#define ST_EINVAL (-1)
#define ST_ECUDA (-2)
#define ST_ENOMEM (-3)
#define ST_EUNSUPPORTED (-4)
#define ST_ENOCONV (-5)

typedef struct st_ctx st_ctx;

/* Material law (reference params.py:17 MaterialParams) + extension:
 * latent_heat > 0 turns on the apparent heat capacity
 * c_app = c + latent_heat / (T_lat_l - T_lat_s) strictly inside
 * (T_lat_s, T_lat_l). */
typedef struct st_material {
  double k_p, k_m, k_s, rho, c, T_s, T_l;
  double latent_heat, T_lat_s, T_lat_l;
} st_material;

/* Top-surface losses (reference params.py:37 BoundaryParams; T_max =
 * T_v + T_max_offset) + extension h_conv (convection). */
typedef struct st_boundary {
  double emissivity, sigma_s, T_inf, T_v, C_P, C_T, C_M, h_v, T_h0, T_max;
  double h_conv;
} st_boundary;

/* Beam model (reference params.py:63 HeatSourceParams). */
typedef struct st_laser {
  double radius, h_powder, cutoff_radii;
} st_laser;

typedef struct st_params {
  st_material mat;
  st_boundary bnd;
  st_laser las;
} st_params;

/* One beam at one step (reference physics.py:96 BeamState); a beam
 * contributes only when active != 0 and power > 0 (operators.py:270).
 * 40 bytes, matching physics.BEAM_DTYPE. */
typedef struct st_beam {
  double x, y, z_top, power;
  int32_t active;
  int32_t _pad;
} st_beam;

/* One straight scan segment (reference physics.py:32 Segment) with the
 * values the reference derives from it: length (np.hypot), duration
 * (length / v) and the start time within its layer path (the running
 * sum of the earlier durations), all as the caller's Python computes them. */
typedef struct st_segment {
  double x0, y0, x1, y1, v, power, length, duration, t_start;
} st_segment;

/* Tables of an arbitrary (adaptive, hanging-node) Q1 mesh: reference
 * DofMap (mesh.py:619-638) + per-cell geometry (operators.py:104-112)
 * + facet quadrature (operators.py:118-134, FaceSet mesh.py:980). */
typedef struct st_unstructured_mesh {
  int64_t n_cells, n_vertices;
  const int32_t* cell_verts;   /* (n_cells, 8), corner ix*4+iy*2+iz   */
  const double* cell_h;        /* (n_cells,)  edge length (m)          */
  const double* cell_anchor;   /* (n_cells,3) min corner (m)           */
  const uint8_t* is_slave;     /* (n_vertices,)                        */
  const uint8_t* is_dirichlet; /* (n_vertices,)                        */
  int64_t n_slaves;
  const int64_t* slaves;       /* (n_slaves,) ascending                */
  const int64_t* slave_ptr;    /* (n_slaves+1,)                        */
  const int64_t* slave_masters;
  const double* slave_weights;
  int64_t n_faces;             /* +z facets, sorted by cell            */
  const int64_t* face_cell;    /* (n_faces,) active-cell position      */
  const double* face_vx;       /* (n_faces,2,2) Vx[f][i][q]            */
  const double* face_vy;       /* (n_faces,2,2)                        */
  const double* face_area;     /* (n_faces,) area per facet qp         */
} st_unstructured_mesh;

/* Uniform box of degree-p cells (p = 1..4), nodes numbered x-major,
 * z-fastest on the p-refined lattice (reference rule mesh.py:712-715);
 * GLL nodes, (p+1)^3 Gauss points.  Bottom node plane Dirichlet, top
 * faces radiating. */
typedef struct st_structured_mesh {
  int32_t nx, ny, nz, degree;
  double h, x0, y0, z0;
  int32_t dirichlet_bottom, top_faces;
  /* x-slab of a larger box (multi-GPU): global index of local node plane
   * 0 and the global node-plane count (gNX = 0: not a slab); iface_lo /
   * iface_hi mark local node planes 0 / NX-1 as rank interfaces whose
   * partial sums are exchanged between st_explicit_step_begin/_end. */
  int32_t gx0, gNX, iface_lo, iface_hi;
  /* Fitted part (BASELINE configs[4]): NULL for the full box, else nz
   * x extents -- cell row k holds the cells i < xext[k], non-decreasing
   * in k (a base with overhanging slabs on top; extents may change only at
   * tile-row boundaries of the kernel).  Nodes are those of the active
   * cells, numbered by the reference's sorted-key rule: node plane I
   * holds rows K >= kmin(I) of every J. */
  const int32_t* xext;
} st_structured_mesh;

/* evaluate_rhs term flags (operators.py:247 diffusion/faces/source). */
#define ST_RHS_DIFFUSION 1
#define ST_RHS_FACES 2
#define ST_RHS_SOURCE 4
#define ST_RHS_FROZEN_K 8

/* resident fields */
#define ST_FIELD_T 0
#define ST_FIELD_RC 1

int st_version(void);
const char* st_last_error(void);
int st_device_count(int* n);

/* ThermalOperator.__init__ (operators.py:91-114) */
int st_ctx_create_unstructured(int device, const st_unstructured_mesh* mesh,
                               const st_params* params, st_ctx** out);
int st_ctx_create_structured(int device, const st_structured_mesh* mesh,
                             const st_params* params, st_ctx** out);
int st_ctx_destroy(st_ctx* ctx);
int64_t st_ctx_n_vertices(const st_ctx* ctx);
int64_t st_ctx_n_cells(const st_ctx* ctx);
int st_ctx_qp_per_cell(const st_ctx* ctx);
/* number of kernels this context has launched so far */
int64_t st_ctx_launches(const st_ctx* ctx);
/* the cudaStream_t the context launches on (as an opaque pointer) */
void* st_ctx_stream(const st_ctx* ctx);
/* deterministic (fixed-order gather) vs atomic scatter, SolverSettings.deterministic */
int st_ctx_set_deterministic(st_ctx* ctx, int deterministic);

/* Resident state (T: n_vertices, r_c: n_cells * qp_per_cell). */
int st_set_field(st_ctx* ctx, int field, const double* host, int64_t n);
int st_get_field(st_ctx* ctx, int field, double* host, int64_t n);
/* r_c == value everywhere (e.g. a fully consolidated plate); the
 * structured backend then stores no history at all. */
int st_set_uniform_rc(st_ctx* ctx, double value);
/* 1 (and *value) when the resident r_c is uniform (st_set_uniform_rc with
 * value >= 1: the history is a fixed point and is never stored), else 0;
 * < 0 on error.  Lets a caller read the state without expanding r_c. */
int st_get_uniform_rc(st_ctx* ctx, double* value);
/* A layer's scan phase (run_scan_phase, timestepping.py:195-226) with the
 * beam schedule evaluated on the device: n_paths concurrently scanned
 * layer paths (seg_count[k] segments each, concatenated in segs; beam z
 * z_top[k]), steps step0 .. step0+n_steps-1 at tau = (step-1) dt with
 * dt_step = min(dt, duration - tau); layer_beam_state's closed windows
 * (physics.py:135-151).  Otherwise as st_explicit_steps. */
int st_scan_layer(st_ctx* ctx, int n_steps, int step0, double dt, double duration, int n_paths,
                  const int32_t* seg_count, const st_segment* segs, const double* z_top,
                  int* fail_step, double* t_extreme, double* t_max);
/* the device-evaluated beam records of those steps (n_steps x n_paths) */
int st_beam_schedule(st_ctx* ctx, int n_steps, int step0, double dt, int n_paths,
                     const int32_t* seg_count, const st_segment* segs, const double* z_top,
                     st_beam* out);

/* Asynchronous snapshot of the resident state (the output / checkpoint
 * phase, driver.py:275-337, io/vtu.py:58-145, without stalling the step
 * loop): T (and r_c, after the owed history update; host_rc nullable) is
 * copied on the device on the context stream and drained to the (pinned)
 * host buffers on a separate copy stream while later steps run.
 * st_snapshot_wait returns 1 when the snapshot is on the host (wait != 0
 * blocks until then), 0 while it is in flight. */
int st_snapshot_begin(st_ctx* ctx, double* host_T, double* host_rc);
int st_snapshot_wait(st_ctx* ctx, int wait);
/* raw device pointer of a resident field (for zero-copy interop) */
double* st_field_device_ptr(st_ctx* ctx, int field);

/* --- per-call operator methods on host arrays (drop-in API) --------- */
/* evaluate_rhs (operators.py:318): condensed f, Dirichlet rows kept.
 * rc may be NULL with ST_RHS_FROZEN_K, without ST_RHS_DIFFUSION, or on a
 * structured context (then the context's uniform history, 1 unless
 * st_set_uniform_rc set another value). */
int st_evaluate_rhs(st_ctx* ctx, const double* T, const double* rc, int flags,
                    double frozen_k, const st_beam* beams, int n_beams,
                    double* out);
/* lumped_capacity (operators.py:325); with latent heat the capacity
 * depends on T (pass T), else T may be NULL. */
int st_lumped_capacity(st_ctx* ctx, const double* T, double* out);
/* apply_mass (operators.py:341) */
int st_apply_mass(st_ctx* ctx, const double* v, double* out);
/* explicit_fused_step (operators.py:352-369) */
int st_explicit_step(st_ctx* ctx, const double* T, double dt, const double* rc,
                     const st_beam* beams, int n_beams, double* out);
/* update_history (operators.py:219-225), rc updated in place */
int st_update_history(st_ctx* ctx, const double* T, double* rc);
/* apply_jacobian (operators.py:380-410) */
int st_apply_jacobian(st_ctx* ctx, const double* v, const double* T_lin,
                      const double* rc, double dt, double* out);
/* jacobian_diagonal (operators.py:426-459) */
int st_jacobian_diagonal(st_ctx* ctx, const double* T_lin, const double* rc,
                         double dt, double* out);

/* --- device-resident time integration ------------------------------- */
/* n_steps forward-Euler steps of run_scan_phase (timestepping.py:211-
 * 221) on the resident (T, r_c): step, stability check, history update.
 * dts[n_steps]; beams[n_steps * n_beams].  On divergence (|T| > 1e7 or
 * non-finite, timestepping.py:186-192) the state is left exactly at the
 * failing step and *fail_step (1-based within the call) / *t_extreme
 * are set; otherwise *fail_step = 0.  *t_max receives max(T) over all
 * accepted steps (PhaseStats.t_max_seen). */
int st_explicit_steps(st_ctx* ctx, int n_steps, const double* dts,
                      const st_beam* beams, int n_beams, int* fail_step,
                      double* t_extreme, double* t_max);
/* One backward-Euler step of run_cooldown_phase on the resident state
 * (_implicit_step, timestepping.py:229-283: f_re frozen at T_n, Newton
 * with Jacobi-PCG).  On success the resident T is the new iterate (not
 * yet Dirichlet-pinned, like the reference) and *converged = 1. */
int st_implicit_step(st_ctx* ctx, double dt, double newton_tol,
                     double newton_abs_tol, int newton_max_iter,
                     double krylov_tol, int krylov_max_iter, int precond,
                     int* newton_iters, int* krylov_iters, int* converged);
/* Dirichlet pin of the resident T + history update (run_cooldown_phase
 * :357-362). */
int st_finish_implicit_step(st_ctx* ctx);
/* krylov_solve (timestepping.py:102-131) for J(T_lin) x = b: no
 * preconditioner (precond = 0), or z = diag_inv * r with the caller's
 * diag_inv (precond = 1, diag_inv != NULL) or with the inverse of the
 * exact Jacobian diagonal (precond = 1, diag_inv == NULL). */
int st_pcg(st_ctx* ctx, const double* T_lin, const double* rc, double dt,
           const double* b, double tol, int max_iter, int precond,
           const double* diag_inv, double* x, int* iters, int* converged);
/* compute_step_criteria / estimate_spectral_radius (timestepping.py:49-99):
 * rho(C~^-1 K) at conductivity k_frozen by power iteration, entirely on the
 * device.  v0 is the caller's normalised start vector (the reference draws
 * default_rng(0).standard_normal(n) / norm); each apply closes constraints,
 * zeroes Dirichlet entries, evaluates the diffusion-only rhs, scales by
 * C~^-1 and zeroes Dirichlet/slave rows; stop when two Rayleigh quotients
 * agree to tol or after max_iter applies.  *rho = max(|lam|, |lam_prev|)
 * (0 when an apply returns the zero vector), *iters = applies. */
int st_spectral_radius(st_ctx* ctx, double k_frozen, const double* v0, double tol,
                       int max_iter, double* rho, int* iters);

/* --- multi-GPU slabs (structured backend) ------------------------------ */
/* One explicit step split around the rank-interface exchange: _begin runs
 * the cell sweep on the resident state leaving the interface planes as
 * partial sums; st_iface_partials gives the device pointers of this
 * rank's partial f (and latent dC, or NULL) on local plane 0 (side 0) or
 * NX-1 (side 1), NY*NZ doubles each; _end adds the neighbours' partials
 * (device pointers, NULL where there is no neighbour) in the fixed order
 * low rank + high rank, finalises all seams and commits the step. */
int st_explicit_step_begin(st_ctx* ctx, double dt, const st_beam* beams, int n_beams);
int st_iface_partials(st_ctx* ctx, int side, double** f_plane, double** c_plane,
                      int64_t* n);
int st_explicit_step_end(st_ctx* ctx, const double* recv_lo_f, const double* recv_lo_c,
                         const double* recv_hi_f, const double* recv_hi_c);
/* max |T| and max T over the steps committed since the last call */
/* max |T'| and max T' over the split steps since the last read */
int st_step_maxima(st_ctx* ctx, double* absmax, double* tmax);
/* per-step maxima of the n oldest unread split steps (n <= 64; read at
 * least every 64 split steps) -- the rank-local half of the cross-rank
 * stability check (timestepping.py:186-192) */
int st_step_maxima_history(st_ctx* ctx, int n, double* absmax, double* tmax);
/* make `stream` (a cudaStream_t) wait until this step's rank-interface
 * partials are packed: the exchange may start while the interior chunks
 * of the sweep still run (st_explicit_step_begin launches the interface
 * chunks first) */
int st_iface_wait(st_ctx* ctx, void* stream);

/* --- measurement ------------------------------------------------------ */
/* When enabled, the step loop brackets its dominant kernel with CUDA
 * events on the context stream; st_profile_read returns the summed
 * device milliseconds and launch count of that kernel since enabling. */
int st_profile_enable(st_ctx* ctx, int enable);
int st_profile_read(st_ctx* ctx, double* main_ms, int64_t* main_launches,
                    char* main_name, int name_len);
/* Algorithmic HBM bytes per DoF-update the dominant kernel must move. */
double st_algorithmic_bytes_per_dof(const st_ctx* ctx);
/* Benchmark loop: like st_explicit_steps (no divergence replay), but
 * every step is bracketed by CUDA events on the context stream and,
 * when flush_bytes > 0, preceded (outside the events) by a write of
 * flush_bytes to a scratch buffer to evict L2.  step_ms[n_steps]
 * receives each step's device time; main_ms[n_steps] (nullable) the
 * dominant kernel's time within the step. */
int st_bench_explicit(st_ctx* ctx, int n_steps, const double* dts, const st_beam* beams,
                      int n_beams, int64_t flush_bytes, float* step_ms, float* main_ms);

/* --- leaf tables of the growing adaptive mesh (host C++, st_forest.cpp) --
 * The reference keeps these in numpy (pkg/src/scantherm/mesh.py); these
 * entry points build bit-identical tables from a leaf set.  No device
 * work, no context: they run on any host. */

/* Leaf table (reference Forest, mesh.py:143-157): lattice anchors in
 * finest units, level in [.., depth], canonical order (key, level). */
typedef struct st_leaves {
  int64_t n;
  int32_t depth;  /* finest level (MeshParams.total_depth)        */
  int32_t cpl;    /* finest cells per powder layer                */
  const int8_t* level;
  const int64_t* anchor;      /* (n, 3) */
  const uint8_t* active;
  const uint8_t* init_consol; /* nullable */
} st_leaves;

/* Variable-size results: a bag of named arrays owned by the library. */
typedef struct st_tables st_tables;
#define ST_DT_I8 1
#define ST_DT_U8 2
#define ST_DT_I32 3
#define ST_DT_I64 4
#define ST_DT_F64 5
/* dims has room for 4 entries; *data stays valid until st_tables_free. */
int st_tables_get(const st_tables* t, const char* name, int* dtype, int* ndim, int64_t* dims,
                  const void** data);
void st_tables_free(st_tables* t);

/* Level-0 tiling of integer boxes (m, 6) [x0 y0 z0 x1 y1 z1], each box
 * active (plate) or void (build volume): replaces build_coarse_grid
 * (mesh.py:289-333).  Arrays: level, anchor, active, init_consol. */
int st_coarse_grid(int32_t depth, int32_t cpl, int64_t n_boxes, const int64_t* boxes,
                   const uint8_t* box_active, st_tables** out);
/* Vertex numbering by packed lattice key, hanging-node constraints with
 * chains expanded, Dirichlet on the z_min plane: replaces build_dofmap
 * (mesh.py:706-779).  Arrays: vertices, cell_verts, active_rows,
 * is_slave, is_dirichlet, slaves, slave_ptr, slave_masters,
 * slave_weights. */
int st_build_dofmap(const st_leaves* leaves, int64_t z_min, int dirichlet_bottom,
                    st_tables** out);
/* Radiating +z facets (full or quarter): replaces interface_faces
 * (mesh.py:998-1072).  Arrays: cell_rows, offset, fsize. */
int st_interface_faces(const st_leaves* leaves, st_tables** out);
/* Plan of the update activating layer new_layer: replaces advance_layer
 * (mesh.py:439-549) and _lineage (:552-602).  rc: the history
 * (n_active, nq) of the old leaves, or NULL (no coarsening gate).
 * Arrays: level, anchor, active, init_consol, same_src, ancestor_src,
 * group_rows, group_ptr, group_kids (coarse_groups as CSR),
 * coarsened_min_rc. */
int st_plan_layer(const st_leaves* leaves, int32_t new_layer, const double* rc, int32_t nq,
                  st_tables** out);
/* Nodal transfer of n_fields fields (field-major) onto the new vertices:
 * copy / trilinear from the old containing cell / T_0, then the new
 * slaves re-interpolated; source[v] = 0 / 1 / 2 (TransferReport).
 * Replaces the nodal half of apply_update (mesh.py:823-866). */
int st_transfer_nodal(const st_leaves* old_leaves, const int64_t* old_verts, int64_t nv_old,
                      const int32_t* old_cell_verts, const int64_t* new_verts, int64_t nv_new,
                      const int64_t* slave_ptr, const int64_t* slaves, int64_t n_slaves,
                      const int64_t* slave_masters, const double* slave_weights, int32_t n_fields,
                      const double* fields_old, double T_0, double* fields_new, int8_t* source);
/* History transfer (n_active, 8): octant copy down, octant mean up;
 * replaces mesh.py:868-896. */
int st_transfer_history(const st_leaves* old_leaves, const st_leaves* new_leaves,
                        const int64_t* same_src, const int64_t* ancestor_src, int64_t n_groups,
                        const int64_t* group_rows, const int64_t* group_ptr,
                        const int64_t* group_kids, const double* rc_old, double* rc_new);

/* Host constraint plumbing on a vertex vector, in place (replaces
 * DofMap.distribute / DofMap.condense, mesh.py:652-670). */
int st_host_distribute(int64_t n_slaves, const int64_t* slaves, const int64_t* slave_ptr,
                       const int64_t* slave_masters, const double* slave_weights, double* values);
int st_host_condense(int64_t n_slaves, const int64_t* slaves, const int64_t* slave_ptr,
                     const int64_t* slave_masters, const double* slave_weights, double* values);

#ifdef __cplusplus
}
#endif
#endif
