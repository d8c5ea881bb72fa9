/*
 * stb200.h -- C ABI of the B200-native stencil_tb hot path (libstb200.so).
 *
 * Drop-in boundary for the reference package `stencil_tb`
 * (/root/reference/pkg/src/stencil_tb).  The reference is pure Python/NumPy,
 * so its "plugin interface" for this path is the set of Python functions
 * named beside each entry point below; the host mirror in
 * paper_2010_10248_b200/ (Python, same names, same argument meaning and
 * exceptions) binds these symbols with ctypes.  See INTEGRATION.md for the
 * binding a stencil_tb maintainer would add.
 *
 * Conventions
 *  - extern "C", POD arguments only; every call returns an int status
 *    (STB_OK == 0).  No C++ exception or CUDA error crosses the ABI; the
 *    message of the last failure on the calling thread is returned by
 *    stb_last_error().
 *  - Host arrays are caller-owned (NumPy) and C-contiguous; they are read or
 *    filled only during the call.  Device memory is owned by the opaque
 *    handles and released by the matching *_destroy.
 *  - Grid index (i, j, k) <-> C-order (x, y, z), z fastest, exactly the
 *    interior layout of grid.py:173-225 (the zero halo of the reference is
 *    realised on the device by zero-fill, never stored on the host side).
 *  - Calls on one handle are not re-entrant; different handles may be used
 *    from different threads (one CUDA device per thread via stb_set_device).
 */
#ifndef STB200_H
#define STB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STB_ABI_VERSION 1

/* Status codes; the Python mirror maps them to stencil_tb.errors
 * (errors.py:4-28). */
enum {
  STB_OK = 0,
  STB_ERR_ARG = 1,      /* ValueError                                      */
  STB_ERR_DOMAIN = 2,   /* OutOfDomainError  (sparse.py:146-150, 224-238)   */
  STB_ERR_CUDA = 3,     /* RuntimeError: CUDA failure / no device           */
  STB_ERR_UNSTABLE = 4, /* StabilityError    (engine.py:354-360)            */
  STB_ERR_PLAN = 5,     /* InvalidPlanError  (schedule.py:181-199)          */
  STB_ERR_NOMEM = 6,    /* MemoryError       (grid.py:193-198)              */
  STB_ERR_CONFIG = 7    /* ConfigError       (engine.py:102-117)            */
};

int stb_abi_version(void);
const char* stb_last_error(void);
int stb_device_count(int* count);
int stb_set_device(int device);

/* Page-locked host memory for the arrays that cross the boundary (media in,
 * fields and traces out).  No reference counterpart: stencil_tb's arrays are
 * plain NumPy (grid.py:173-198, engine.py:430-447).  Every entry point takes
 * pageable memory too (staged through the library's own pinned ring); arrays
 * from stb_host_alloc are read and written by the copy engine directly.
 * Freed blocks are cached by size (the cache holds at most 6 GiB). */
int stb_host_alloc(int64_t bytes, void** out);
int stb_host_free(void* p);

/* ------------------------------------------------------------------------
 * Geometry of a regular grid: index i sits at origin + i * spacing
 * (grid.py:22-74).
 * ---------------------------------------------------------------------- */
typedef struct {
  int64_t shape[3];
  double spacing[3];
  double origin[3];
} stb_geometry;

/* Trilinear 2x2x2 stencils of n off-grid points, computed on the GPU.
 * Replaces sparse.interp_stencil (sparse.py:136-173) for many points at
 * once; with margin >= 0 it also applies validate_coords_in_extent
 * (sparse.py:224-238) with that margin.  idx_out: n*8*3 int64, w_out: n*8
 * f64, corners in (bx, by, bz) lexicographic order.  Out-of-extent ->
 * STB_ERR_DOMAIN (message names the first offending point). */
int stb_interp_stencils(const double* coords, int64_t n, const stb_geometry* g,
                        int64_t margin, int64_t* idx_out, double* w_out);

/* ------------------------------------------------------------------------
 * Inspector: the paper's Alg. 2-3/5 (precompute.py:103-316) on the GPU.
 * ---------------------------------------------------------------------- */
typedef struct stb_support_s* stb_support_t;

/* Build the on-grid footprint of n sparse points: stencils, the union of
 * corners with weight > 0 (keep_zero_weights = 0; find_support "geometric",
 * precompute.py:114-125) or of all 8 corners (keep_zero_weights = 1),
 * lexicographic point ids and the per-(x, y) column compression
 * (build_masks + compress, precompute.py:150-180). */
int stb_support_create(const double* coords, int64_t n, const stb_geometry* g,
                       int32_t keep_zero_weights, stb_support_t* out);
/* Support of an explicit set of grid points (build_masks on a given set,
 * precompute.py:150-165): duplicates are merged, ids are lexicographic.
 * Indices outside the interior -> STB_ERR_ARG (ValueError). */
int stb_support_from_points(const int64_t* points, int64_t n, const stb_geometry* g,
                            stb_support_t* out);
/* K = number of affected points, M = number of kept (point, owner) entries. */
int stb_support_info(stb_support_t s, int64_t* n_affected, int64_t* n_entries);
/* points: K*3 int64, lexicographically sorted (SparseSupport.points). */
int stb_support_points(stb_support_t s, int64_t* points);
/* compress(): nnz_mask (nx*ny int32), _row_ptr (nx*ny+1 int64), _flat_z (K
 * int64), _flat_id (K int32).  Any pointer may be NULL to skip it. */
int stb_support_compress(stb_support_t s, int32_t* nnz_mask, int64_t* row_ptr,
                         int64_t* flat_z, int32_t* flat_id);
/* build_masks(): dense sm (uint8) and sid (int32, -1 sentinel), nx*ny*nz. */
int stb_support_masks(stb_support_t s, uint8_t* sm, int32_t* sid);
/* precompute_receivers() entry table (precompute.py:267-284): M entries
 * sorted by (point, owner): point (M*3 int64), owner id (M int64), w (M f64). */
int stb_support_entries(stb_support_t s, int64_t* entry_points, int64_t* entry_owner,
                        double* entry_w);
/* decompose_wavefields() (precompute.py:183-206): src_dcmp (nt*K f64) with
 * src_dcmp[t, id] = sum over kept entries in source-major order of
 * (w * scale[s]) * wavelets[t, s]; wavelets is (nt_w, n) f64, nt >= nt_w,
 * rows >= nt_w are zero. */
int stb_support_decompose(stb_support_t s, const double* wavelets, int64_t nt_w,
                          const double* scale, int64_t nt, double* src_dcmp);
int stb_support_destroy(stb_support_t s);

/* ------------------------------------------------------------------------
 * Propagators: the engine.run hot loop (engine.py:362-376, 426-434).
 * ---------------------------------------------------------------------- */
typedef struct stb_prop_s* stb_prop_t;

/* Isotropic acoustic (AcousticModel / acoustic_update, physics.py:124-213).
 * All coefficients are passed in f64 exactly as the reference computes
 * them in Python and are rounded once to the field dtype on the device. */
typedef struct {
  stb_geometry geom;
  int32_t space_order;       /* even, 2..16                                  */
  int32_t precision;         /* 32 or 64                                     */
  double dt;
  double center;             /* sum_{active a} w_0 / h_a^2   (physics.py:159) */
  double coef[3][8];         /* w_r / h_a^2, r = 1..R; 0 on inactive axes    */
  int32_t active[3];         /* axis has more than one point                 */
  double dt2;                /* dt**2 as evaluated by the host (Python float) */
  const double* velocity;    /* per-point velocity (nx*ny*nz, f64): the device
                                forms m = 1/v**2 and dt2/m (engine.py:243,
                                physics.py:151) -- or NULL                    */
  const double* m;           /* per-point squared slowness, used when
                                velocity == NULL; NULL -> inv_scalar         */
  double inv_scalar;         /* dt**2/m of a homogeneous medium              */
  const double* damp[3];     /* per-axis 1/(1+dt*profile_a) tables (f64), or
                                NULL for no sponge (physics.py:66-115)       */
  int32_t arithmetic;        /* 0 = EXACT: reference IEEE operation order,
                                bitwise equal to stencil_tb; 1 = FMA: the
                                Laplacian accumulates with fused multiply-add
                                (within 1e-5 relative L2 of the reference)   */
  int64_t x_begin;           /* x-slab handles (multi-GPU): the handle holds
                                global planes [x_begin, x_begin + nx_local);
                                geom stays the GLOBAL grid (stencils, sponge
                                tables and supports are global), velocity/m
                                are the local slab.  nx_local == 0: whole grid */
  int64_t nx_local;
} stb_acoustic_desc;

/* Isotropic elastic velocity-stress (ElasticModel, physics.py:216-429). */
typedef struct {
  stb_geometry geom;
  int32_t space_order;
  int32_t precision;
  double dt;
  double d1[3][8];           /* c_j / h_a, j = 1..R; 0 on inactive axes      */
  int32_t active[3];
  const double* lam;         /* Lame lambda per point (Pa) or NULL -> scalar */
  const double* mu;          /* shear modulus per point or NULL -> scalar    */
  const double* rho;         /* density per point or NULL -> scalar          */
  double lam_scalar, mu_scalar, rho_scalar;
  /* the device forms dt/rho, dt*lam, dt*mu, 2*dt*mu (physics.py:251-257);
     f32(2*dt*mu) == 2*f32(dt*mu) exactly, so only three streams are kept. */
  const double* damp[3];
  int64_t x_begin;           /* x slab, as in stb_acoustic_desc (materials are
                                the local slab; geometry, tables global)     */
  int64_t nx_local;
  /* from_velocities = 1: lam/mu are formed on the device from vp, vs, rho
     exactly as engine.py:247-255 does in f64 (mu = rho*vs^2, lam =
     rho*vp^2 - 2*mu) and checked as physics.py:229-236 does; lam/mu above
     are ignored.  The handle also records max(vp) (stb_prop_velocity_max). */
  int32_t from_velocities;
  const double* vp;          /* per point or NULL -> vp_scalar               */
  const double* vs;
  double vp_scalar, vs_scalar;
} stb_elastic_desc;

/* Pseudo-acoustic TTI, coupled p and q (eq. 2).  Not in
 * the reference: the discrete operator is this repo's, defined
 * by oracle/stencil_oracle.py:TTI (parity unpinned).  All material values are
 * formed in f64 by the host and rounded once on the device:
 *   inv = dt2 / (1/vp^2), e2 = 1 + 2 eps, d2 = sqrt(1 + 2 delta),
 *   axis = (sin t cos f, sin t sin f, cos t).
 * Fields: 0 = p, 1 = q.  Receivers record p; sources inject into p and q. */
typedef struct {
  stb_geometry geom;
  int32_t space_order;       /* multiple of 4 in [4, 16]                     */
  int32_t precision;         /* 32 or 64                                     */
  double dt;
  double d1[3][4];           /* centred first-derivative weights a_k / h_a,
                                k = 1..so/4 (order so/2); 0 on inactive axes */
  int32_t active[3];
  double dt2;
  const double* velocity;    /* vp per point (compact slab, f64) or NULL     */
  double inv_scalar;         /* dt2/m of a homogeneous medium                */
  const double* e2;          /* 1 + 2 epsilon per point, or NULL -> scalar   */
  double e2_scalar;
  const double* d2;          /* sqrt(1 + 2 delta) per point, or NULL         */
  double d2_scalar;
  const double* axis[3];     /* symmetry-axis components per point, or NULL  */
  double axis_scalar[3];
  const double* damp[3];     /* per-axis sponge tables, as acoustic          */
  int64_t x_begin;           /* x slab, as in stb_acoustic_desc              */
  int64_t nx_local;
  int32_t arithmetic;        /* 0 = EXACT (the oracle's operation order,
                                bitwise); 1 = FMA (contracted products, within
                                1e-5 relative L2; fused f32 3-D kernel only)  */
  int32_t raw_eps_delta;     /* 1: e2 / d2 carry epsilon / delta per point and
                                the device forms 1 + 2 eps and
                                sqrt(1 + 2 delta) in f64 (same IEEE ops)     */
  const float* axis32[3];    /* precision 32: axis components already rounded
                                to f32 on the host (overrides axis[a])      */
} stb_tti_desc;

int stb_acoustic_create(const stb_acoustic_desc* d, stb_prop_t* out);
int stb_elastic_create(const stb_elastic_desc* d, stb_prop_t* out);
int stb_tti_create(const stb_tti_desc* d, stb_prop_t* out);

/* Sources: fused injection of the decomposed series (Alg. 4/5,
 * precompute.py:209-252).  Decomposition runs on the device from the
 * support handle (which must come from the same geometry). */
int stb_prop_set_sources(stb_prop_t p, stb_support_t s, const double* wavelets,
                         int64_t nt_w, const double* scale, int64_t nt);
/* Receivers: per-step trilinear gather (record_receivers, sparse.py:197-207),
 * summed per receiver with NumPy's 8-wide pairwise order.  Coordinates
 * must already be validated (margin = boundary_layers, engine.py:282-290). */
int stb_prop_set_receivers(stb_prop_t p, const double* coords, int64_t nrec);

/* Field the receivers record (same indices as stb_prop_read_field).  Default
 * = the reference's: acoustic u, elastic txx (engine.py:327-332), TTI p.
 * Extension for BASELINE cfg5 (vx / vz receivers). */
int stb_prop_set_receiver_field(stb_prop_t p, int32_t field);

/* Sponge tables after creation (acoustic; replaces the desc's damp[]):
 * _damp_factor's per-axis f64 tables (physics.py:66-115, engine.py:211-218),
 * global x table as in the desc; NULL = no damping on that axis.  Lets the
 * host compute v_max (the default decay needs it) while the model uploads. */
int stb_prop_set_damping(stb_prop_t p, const double* fx, const double* fy, const double* fz);
/* Advance steps [t0, t0 + nsteps), time_height steps fused per HBM pass
 * (schedule.py:171-207 semantics; 0 = library default).  rec_out, when not
 * NULL, receives the (nsteps, nrec) f64 traces.  On a non-finite field at a
 * guard step (multiple of 32) returns STB_ERR_UNSTABLE and sets *bad_step. */
int stb_prop_run(stb_prop_t p, int64_t t0, int64_t nsteps, int32_t time_height,
                 double* rec_out, int64_t* bad_step);
/* Field `field` (acoustic: 0 = u; elastic: 0..8 = vx vy vz txx tyy tzz txy
 * txz tyz; tti: 0 = p, 1 = q) at time level t (the last two written levels are resident),
 * copied to a host (nx, ny, nz) array of the handle's dtype. */
int stb_prop_read_field(stb_prop_t p, int32_t field, int64_t t, void* out);
/* Device address of time level t of field `field` (x-slab halo exchange):
 * *dev points at local plane 0; planes are contiguous blocks of
 * *plane_elems elements (ny rows of *pitch_elems, z fastest). */
int stb_prop_level_ptr(stb_prop_t p, int32_t field, int64_t t, void** dev,
                       int64_t* plane_elems, int64_t* pitch_elems);
/* Write field `field` at level t to `path` in stencil_tb's snapshot format
 * (engine.py:553-577): a 32-byte header -- "STBSNAP\0", uint32 bits (32 or
 * 64), int32 nx, ny, nz, uint32 t, zero padding -- then the (nx, ny, nz)
 * C-order little-endian samples.  Device -> file without Python. */
int stb_prop_write_snapshot(stb_prop_t p, int32_t field, int64_t t, const char* path);
/* Asynchronous stepping for x-slab multi-GPU runs (fused acoustic path).
 * Work is enqueued on the handle's stream (stb_prop_stream; the caller
 * orders its halo exchange against it) with no host synchronisation:
 *   stb_prop_async_begin(p, t0, n)           window of steps [t0, t0 + n)
 *   stb_prop_step_async(p, t, kb, lo, hi)    kb fused steps from t over
 *                                            local planes [lo, hi)
 *   stb_prop_gather_async(p, t, kb)          receiver rows of levels t..t+kb-1
 *   stb_prop_async_finish(p, rec_out, &bad)  sync, (n, nrec) traces, NaN guard
 * Replaces the engine.py:426-434 loop when the caller interleaves the halo
 * exchange (slabs.py); stb_prop_run is the synchronous whole-window form. */
int stb_prop_stream(stb_prop_t p, void** stream);
int stb_prop_async_begin(stb_prop_t p, int64_t t0, int64_t nsteps);
int stb_prop_step_async(stb_prop_t p, int64_t t, int32_t kb, int64_t x_lo, int64_t x_hi);
/* Elastic x slabs: one half step of step t (phase 0: v, physics.py:334-368;
 * phase 1: tau + injection, physics.py:371-429) over local planes
 * [x_lo, x_hi), so R ghost planes of the half step's fields can be exchanged
 * between the halves (step_async runs both). */
int stb_prop_half_step_async(stb_prop_t p, int64_t t, int32_t phase, int64_t x_lo, int64_t x_hi);
/* Fused halo exchange (x slabs, one process driving several GPUs with peer
 * access): the K = 1 step over [x_lo, x_hi) also stores its boundary planes
 * straight into the neighbours' ghost planes over NVLink -- local plane
 * p < lo_end goes to `lo` (the lower neighbour's level-t buffer, from its
 * stb_prop_level_ptr) at its local plane p + lo_shift; p >= hi_begin to
 * `hi` at p + hi_shift.  NULL pointers: no neighbour on that side.  The
 * caller orders the neighbours' next launches after this one (events). */
typedef struct {
  void* lo;
  int64_t lo_end, lo_shift;
  void* hi;
  int64_t hi_begin, hi_shift;
} stb_peer_halo;
int stb_prop_step_async_peers(stb_prop_t p, int64_t t, int64_t x_lo, int64_t x_hi,
                              const stb_peer_halo* peers);
int stb_prop_gather_async(stb_prop_t p, int64_t t, int32_t kb);
int stb_prop_async_finish(stb_prop_t p, double* rec_out, int64_t* bad_step);
/* Zero all time levels (reuse a handle for another shot). */
int stb_prop_reset(stb_prop_t p);
/* Device-side timing of the last stb_prop_run (CUDA events on the launching
 * stream), for bench.py: stencil-kernel launches and their summed duration,
 * grid-point updates, all kernels launched, and the whole run's duration. */
int stb_prop_stats(stb_prop_t p, int64_t* launches, double* kernel_ms,
                   int64_t* updates, int64_t* all_launches, double* run_ms);
/* Kernel configuration chosen for time_height k (name, bytes per point). */
int stb_prop_describe(stb_prop_t p, int32_t time_height, char* buf, int64_t buflen);
/* Deepest time_height one fused pass of this handle computes (acoustic fp32
 * 3-D: 2 at so 2/4/8, 1 otherwise).  Longer wavefront heights
 * (schedule.py:171-207) run as consecutive blocks of this depth; run()
 * reports the depth used in RunReport.schedule["time_height"]. */
int stb_prop_max_time_height(stb_prop_t p, int32_t* k);
/* max of the velocity array the handle was created from, as np.max
 * (engine.py:160-169; NaN if it holds a NaN or was not recorded): acoustic
 * handles reduce it on the device in the kernel that forms inv, so the host
 * need not read the 1.7 GB velocity a second time for the sponge decay. */
int stb_prop_velocity_max(stb_prop_t p, double* vmax);
int stb_prop_destroy(stb_prop_t p);

/* ------------------------------------------------------------------------
 * Step-level operators (stepping.cu) on the reference's halo-padded level
 * layout: TimeBufferedField.level(t) (grid.py:173-218) is a C-order
 * (nx+2h, ny+2h, nz+2h) array with a zero halo.  All pointers below are
 * DEVICE pointers in that layout (caller-owned, e.g. torch CUDA tensors);
 * work is enqueued on `stream` (a cudaStream_t, NULL = legacy default) and
 * not synchronised.  Boxes are half-open interior index ranges
 * (grid.py:228-262).  Materials (inv, buoy, lam, mu, mu2) and the sponge
 * factor are padded arrays of the same layout or NULL (scalar / no sponge),
 * exactly as the reference models store them (physics.py:90-115).
 * ------------------------------------------------------------------------ */
typedef struct {
  int64_t padded[3];   /* nx + 2h, ny + 2h, nz + 2h */
  int32_t halo;        /* h */
  int32_t precision;   /* 32 or 64 */
} stb_layout;

typedef struct {
  int64_t lo[3], hi[3];
} stb_box;

/* acoustic_update (physics.py:181-213).  active[3]: axes with > 1 point;
 * weights[a*8 + r-1] = w_r / h_a^2, center = sum_a w_0 / h_a^2 (Python
 * floats, rounded to the field dtype like NumPy's weak scalars). */
int stb_box_acoustic_update(const stb_layout* L, void* dst, const void* u1, const void* u0,
                            int32_t radius, const int32_t* active, double center,
                            const double* weights, const void* inv, double inv_scalar,
                            const void* dampfac, const stb_box* box, void* stream);
/* elastic_update_v (physics.py:334-368): v_out/v_prev = vx vy vz at t / t-1,
 * tau_prev = txx tyy tzz txy txz tyz at t-1; d1[a*8 + j-1] = c_j / h_a. */
int stb_box_elastic_v(const stb_layout* L, void* const* v_out, const void* const* v_prev,
                      const void* const* tau_prev, int32_t radius, const int32_t* active,
                      const double* d1, const void* buoy, double buoy_scalar,
                      const void* dampfac, const stb_box* box, void* stream);
/* elastic_update_tau (physics.py:371-429): v_cur = vx vy vz at t. */
int stb_box_elastic_tau(const stb_layout* L, void* const* tau_out, const void* const* tau_prev,
                        const void* const* v_cur, int32_t radius, const int32_t* active,
                        const double* d1, const void* lam, double lam_scalar, const void* mu,
                        double mu_scalar, const void* mu2, double mu2_scalar,
                        const void* dampfac, const stb_box* box, void* stream);
/* scatter_box / fused_inject_row / inject_direct (precompute.py:209-252,
 * sparse.py:176-194): dst[p_k] += T(values[k]) for the K support points
 * (points K*3 int64, lexicographic, each once) that lie in the box. */
int stb_box_scatter(const stb_layout* L, void* dst, const int64_t* points,
                    const double* values, int64_t K, const stb_box* box, void* stream);
/* gather_box (precompute.py:287-308): contrib[m] = w[m] * level[p_m] (f64)
 * and in_box[m] = 1 for entries in the box, 0 (contrib 0) otherwise. */
int stb_box_gather(const stb_layout* L, const void* src, const int64_t* points,
                   const double* weights, int64_t M, const stb_box* box, double* contrib,
                   uint8_t* in_box, void* stream);
/* record_receivers (sparse.py:197-207): out[r] = sum of the 8 corner
 * products w * level[corner] in NumPy's pairwise order; idx n*8*3, w n*8. */
int stb_record_receivers(const stb_layout* L, const void* src, const int64_t* idx,
                         const double* w, int64_t n, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* STB200_H */
