/*
 * surriga_b200 -- C ABI of the B200 (sm_100a) surrogate / full-quadrature IGA assembly path.
 *
 * The reference (arXiv 1904.06971 "surriga", pure Python) exposes the hot path as two
 * Python functions; this library sits behind exactly those two calls:
 *
 *   assemble(form, disc, rows=None, coefficient=1.0) -> SparseMatrix
 *        reference: pkg/src/surriga/assembly.py:579-651      -> sg_assemble()
 *   build_surrogate_matrix(form, disc, strategy=None, q=3, mode=None, coefficient=1.0)
 *        -> (SparseMatrix, AssemblyReport)
 *        reference: pkg/src/surriga/surrogate.py:538-691     -> sg_surrogate()
 *
 * The Python host (paper_1904_06971_b200/) validates arguments with the reference's error
 * messages, performs the exact-rational setup (knots, Gauss points, lattice), and calls these
 * entry points through ctypes.  All O(nnz) and O(elements * Q * L^2) work runs on the GPU.
 *
 * Conventions: plain pointers and sizes only; every input pointer is a HOST pointer that is
 * borrowed for the duration of the call (copied to the device inside the call).  Results live
 * on the device behind an opaque handle until sg_result_free().  Every function returns 0 on
 * success and a negative status on failure; sg_last_error() gives a thread-local message:
 * -1 invalid argument (the reference's ValueError), -2 unsupported configuration, -3 CUDA
 * error, -4 allocation failure, -5 I/O error, -6 index out of bounds (the reference's
 * IndexError, e.g. surrogate.py:673-680's positional reset after an exact-zero drop).
 * Multi-index / flat-index order is colex (first direction fastest), as in bspline.py:306-339.
 */
#ifndef SURRIGA_B200_H
#define SURRIGA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* assembly.py:51-58 FormKind.  STOKES_VELOCITY is Poisson times a coefficient (assembly.py:533). */
enum sg_form { SG_POISSON = 0, SG_MASS = 1, SG_BIHARMONIC = 2 };

/* surrogate.py:36-41 SurrogateMode */
enum sg_mode { SG_GENERAL = 0, SG_SYMMETRIC = 1, SG_SYMMETRIC_KERNEL_PRESERVING = 2 };

/* Everything the hot path reads from a Discretization (assembly.py:133-176). */
typedef struct sg_problem {
    int32_t n;              /* parametric dimension 1..3                                 */
    int32_t p;              /* solution degree (all directions), 1..SG_MAX_P             */
    int32_t form;           /* enum sg_form                                              */
    int32_t m[3];           /* basis functions per direction (m = spans + p)             */
    int32_t g;              /* Gauss points per direction (assembly.py:173)               */
    const double* knots[3]; /* solution knots per direction, m+p+1 each (float of exact)  */
    const double* qpts[3];  /* Gauss points per direction, (m-p)*g each (assembly.py:108)  */
    const double* qwts[3];  /* per-direction point weights, g each (w * h/2)              */
    const double* sol_w;    /* N solution weights (colex) or NULL when `weights.is_unit`  */
    int32_t geo_p;          /* geometry degree                                            */
    int32_t geo_m[3];       /* geometry basis functions per direction                     */
    const double* geo_knots[3];
    const double* geo_hom;  /* Ng x (n+1): control*w | w, colex (geometry.py:193-195)      */
    double coefficient;     /* Poisson / Stokes-velocity multiplier (assembly.py:606-610)  */
} sg_problem;

/* Row-slab / device options for one call. */
typedef struct sg_exec {
    int32_t device;         /* CUDA device ordinal                                        */
    void* stream;           /* cudaStream_t to run on, or NULL for a per-call stream      */
    int64_t slab_lo;        /* rows [slab_lo, slab_hi) assembled on this device (row slab) */
    int64_t slab_hi;        /* slab_hi <= 0 means "all rows"                               */
} sg_exec;

/* Surrogate parameters (host-resolved: M from the sampling strategy, lattice from tilde box). */
typedef struct sg_surrogate_params {
    int32_t M;              /* sampling stride (surrogate.py:236-253)                     */
    int32_t q;              /* requested interpolation order                              */
    int32_t mode;           /* enum sg_mode                                               */
    int32_t nlat[3];        /* lattice sites per direction                                */
    const int64_t* lat_idx[3];   /* 0-based lattice basis indices per direction           */
    int32_t qd[3];          /* per-direction interpolation degree (lowered, 0 = constant)  */
    const double* interp_knots[3]; /* averaged knots per direction (nlat+qd+1) or NULL    */
    const double* colloc_inv[3];   /* nlat x nlat inverse collocation matrix (row-major)  */
    const double* box_pts[3];      /* in-box midpoints per direction (box count each)     */
} sg_surrogate_params;

/* Integer/float facts the host needs to build AssemblyReport (surrogate.py:478-502). */
typedef struct sg_surrogate_stats {
    int64_t n_interp_rows;
    int64_t n_quad_rows;
    int64_t n_interp_entries;   /* (interp row, offset) pairs filled from an interpolant  */
    int64_t n_zero_dropped;     /* exact zeros removed by the CSR merge (surrogate.py:670) */
    int64_t n_reset_rows;       /* kernel-preserving diagonal resets (surrogate.py:673)    */
} sg_surrogate_stats;

typedef struct sg_result sg_result;

/* Full or row-restricted assembly.  rows == NULL: all rows (the reference's rows=None).
 * rows != NULL: nrows sorted unique 0-based rows; only their entries are emitted
 * (assembly.py:613-622,638-640), bitwise equal to the full rows. */
int sg_assemble(const sg_problem* prob, const int64_t* rows, int64_t nrows, const sg_exec* ex, sg_result** out);

/* Surrogate assembly (quadrature rows + interpolated interior rows + merge + SKP diagonal). */
int sg_surrogate(const sg_problem* prob, const sg_surrogate_params* sp, const sg_exec* ex, sg_result** out,
                 sg_surrogate_stats* stats);

/* Surrogate assembly on a row slab in two phases, for several devices sharing one matrix (SURVEY
 * §8e): every device assembles only its slab's quadrature rows (and their p-plane halo), so the
 * samples of the lattice rows outside its slab come from the devices that own them.
 *   sg_surrogate_begin : the slab's quadrature rows (K4) and the samples of the lattice rows inside
 *       [slab_lo, slab_hi), written into the state's device table *samples = S[o][lattice colex]
 *       (P * *nlat doubles, P = (2p+1)^n; the other lattice columns are zero).  Returns after the
 *       table is complete on the device.
 *   [the caller fills the other lattice columns on the device, e.g. an all-gather of every slab's
 *    own columns over NCCL, and synchronises]
 *   sg_surrogate_finish : collocation solves, interpolation, merge, SKP diagonal; `params` must be
 *       the same as for begin.  Frees the state (also on error).
 * sg_surrogate() on a slab is begin + a row-restricted assembly of the other lattice rows + finish.
 * Results are bitwise those of the whole-matrix call, whatever the slabs. */
typedef struct sg_surrogate_state sg_surrogate_state;
int sg_surrogate_begin(const sg_problem* prob, const sg_surrogate_params* params, const sg_exec* exec,
                       sg_surrogate_state** state, double** samples, int64_t* nlat);
int sg_surrogate_finish(sg_surrogate_state* state, const sg_surrogate_params* params, sg_result** out,
                        sg_surrogate_stats* stats);
int sg_surrogate_state_free(sg_surrogate_state* state);

/* Result inspection / transfer. */
int sg_result_sizes(const sg_result* r, int64_t* nrows, int64_t* nnz);
/* Copy CSR to host: indptr int32[nrows+1] (or int64 if *_i64 variant), indices int32[nnz], data f64[nnz]. */
int sg_result_copy(const sg_result* r, int32_t* indptr, int32_t* indices, double* data);
int sg_result_copy_i64(const sg_result* r, int64_t* indptr, int32_t* indices, double* data);
/* Mixed divergence pairing (replaces surriga/assembly.py:654-725 `assemble_divergence(stokes, rows=None)`):
   `velocity` describes the velocity discretisation (degree pp+1 on the halved mesh, its Gauss points and weights,
   the geometry), `pressure` the pressure space (degree pp; only n, p, m and knots are read).  Writes n results,
   one per velocity component c (out[0..n-1]): rows = pressure functions, columns = velocity functions, entry
   sum_q w_q P_i sum_a d_a V_j adj(J)[a][c].  `rows` (sorted, unique) restricts to pressure rows as the reference's
   `rows=` (bitwise equal to the full assembly).  B-spline or NURBS spaces (sol_w of either problem);
   sg_exec slab_lo/hi: pressure rows [lo, hi) only (not with `rows`). */
int sg_assemble_divergence(const sg_problem* velocity, const sg_problem* pressure, const int64_t* rows, int64_t nrows,
                           const sg_exec* exec, sg_result** out);
/* Surrogate divergence pairing, general mode (replaces surriga/surrogate.py:702-819 `build_surrogate_divergence`):
   `params` as for sg_surrogate over the pressure space (lattice, per-direction degree, averaged knots, inverse
   collocation matrices, in-box midpoints); `shifts` the P mixed offsets [-2pp, pp+2]^n (colex, n ints each);
   `quad_rows` the host-classified quadrature rows (not in the one-index-shrunk box, or on the lattice).  Quadrature
   rows by quadrature, the others interpolated per offset; exact zeros dropped per component.  sg_exec slab_lo/hi:
   pressure rows [lo, hi) only (the slab's quadrature rows and every lattice row are assembled). */
int sg_surrogate_divergence(const sg_problem* velocity, const sg_problem* pressure, const sg_surrogate_params* params,
                            const int32_t* shifts, const int64_t* quad_rows, int64_t nquad, const sg_exec* exec,
                            sg_result** out, sg_surrogate_stats* stats);
/* Load vector (replaces surriga/assembly.py:728-759 `assemble_load(disc, f)`), split at the caller's callable f:
   sg_map_points writes the physical quadrature points phi(x_q) element-major, shape (E, Q, n) with E colex elements
   and Q colex points per element (the array the reference passes to f); sg_assemble_load takes f's values (E, Q)
   and writes vec[N] = sum_e sum_q f det(J) w_q N_i (rational N_i for non-unit sol_w). */
int sg_map_points(const sg_problem* problem, const sg_exec* exec, double* phi_out);
int sg_assemble_load(const sg_problem* problem, const double* fvals, const sg_exec* exec, double* vec_out);
/* Quadrature fields (replaces surriga/assembly.py:839-907 `quadrature_fields(disc, coefs, nu, gauss)`): for the
   coefficient vector coefs[N] of the problem's space, writes at every element quadrature point (element-major,
   T = E * g^n points): x_out[T][n] physical points, w_out[T] = w_q det J, val_out[T] field values and, for nu >= 1,
   grad_out[T][n] physical gradients, for nu >= 2, hess_out[T][n][n] physical Hessians (NULL when not requested).
   The problem's `form` is ignored; rational solution spaces use the NURBS basis. */
int sg_quadrature_fields(const sg_problem* problem, const double* coefs, int32_t nu, const sg_exec* exec, double* x_out,
                         double* w_out, double* val_out, double* grad_out, double* hess_out);
/* MatrixMarket coordinate output (replaces surriga/assembly.py:304-312 `save_matrix_market(path, A)`): header,
   "%", "nrows ncols count", 1-based "i j value" lines; symmetric != 0 writes the lower triangle under the
   `symmetric` tag as scipy's mmwrite does.  Values are printed in the shortest form that reads back to the same
   double (the reference's 16 digits do not always round-trip).  Rows are formatted by `nthreads` host threads
   (<= 0: all cores).  The device variant copies the result to the host first; ncols <= 0 means square. */
int sg_write_matrix_market_host(const char* path, int64_t nrows, int64_t ncols, const int64_t* indptr, const int32_t* indices,
                                const double* data, int32_t symmetric, int32_t nthreads);
int sg_write_matrix_market(const sg_result* A, int64_t ncols, const char* path, int32_t symmetric, int32_t nthreads);
/* Optional: allocate the calling thread's pinned D2H staging ring and host copy pool for `device` up
   front (otherwise done by the first large sg_result_copy*; not part of the reference interface). */
int sg_host_staging_init(int device);
/* Optional: pin / unpin a host range with the driver (cudaHostRegister); sg_result_copy* DMAs straight into
   registered destinations.  Used by the Python layer for reused result buffers. */
int sg_host_register(void* ptr, size_t bytes);
int sg_host_unregister(void* ptr);
/* Device pointers (for device-resident consumers and timing). */
int sg_result_device_ptrs(const sg_result* r, void** indptr_i64, void** indices_i32, void** data_f64);
/* Deterministic fp64 checksums {nnz, sum a, sum a^2, sum |a|, sum of row sums} of the rows in the result. */
int sg_result_checksum(const sg_result* r, double out[5]);
int sg_result_free(sg_result* r);

/* ---- Device-resident consumer of the CSR (surriga/solvers.py:74-155) ---- */
/* Upload a host CSR (e.g. a SparseMatrix built elsewhere) into a result handle on `device`. */
int sg_result_from_host(int32_t device, int64_t nrows, int64_t nnz, const int64_t* indptr, const int32_t* indices,
                        const double* data, sg_result** out);
/* y = A x for a whole square result (host x, y of nrows doubles); replaces scipy's `mat @ x`. */
int sg_spmv(const sg_result* A, const double* x, double* y, const sg_exec* exec);

enum sg_cg_status {
    SG_CG_CONVERGED = 0,             /* |r| <= tol |b| (solvers.py:144-145)                      */
    SG_CG_NEGATIVE_CURVATURE = 1,    /* d.Ad <= 0 at `iterations` (solvers.py:138-141)           */
    SG_CG_NONPOSITIVE_DIAGONAL = 2,  /* diagonal preconditioner with a diagonal entry <= 0 (:123) */
    SG_CG_MAX_ITERATIONS = 3         /* no convergence in max_iterations (solvers.py:146-155)     */
};
typedef struct sg_cg_stats {
    int32_t status;          /* enum sg_cg_status                                         */
    int64_t iterations;      /* iterations run (the failing one for NEGATIVE_CURVATURE)   */
    double norm_b;           /* |b|                                                       */
    double rel_residual;     /* |A x - b| / |b| of the returned x (solvers.py:108-110,151) */
} sg_cg_stats;
/* Conjugate gradient of solvers.py:118-155 on a device-resident square CSR: x0 = 0, relative
   tolerance `tol`, at most `maxit` iterations, precond 0 = "none", 1 = "diagonal" (Jacobi).  b, x are
   host arrays of nrows doubles; x receives the final iterate.  The caller maps the status to the
   reference's RuntimeError messages. */
int sg_cg_solve(const sg_result* A, const double* b, double* x, double tol, int64_t maxit, int32_t precond,
                const sg_exec* exec, sg_cg_stats* stats);

/* Device-time of the kernels of the last call on this thread (ms), and their launch count. */
int sg_last_timing(double* ms_total, int32_t* launches);
/* fp64 tensor-core (DMMA m8n8k4, 512 flops each) instructions the assembly kernel executed in the last
   call on this thread: the hardware-work figure next to the reference-algorithm flop count. */
int sg_last_dmma_count(int64_t* count);
/* Per-kernel breakdown of the last call: name list (comma separated) and ms values. */
int sg_last_kernel_times(char* names, int32_t names_cap, double* ms, int32_t cap, int32_t* count);

const char* sg_last_error(void);
const char* sg_version(void);
int sg_max_degree(void);

#ifdef __cplusplus
}
#endif
#endif /* SURRIGA_B200_H */
