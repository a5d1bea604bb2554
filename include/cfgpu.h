/*
 * cfgpu.h -- C ABI of the B200-native cavityflow hot path (libcfgpu.so).
 *
 * The reference (cfdSCOPE / `cavityflow`, a Python+numba package) has no
 * FFI: its plugin surface is the Python kernel/operator API.  Each entry
 * point below replaces one reference function (cited as src/<file>:<line>,
 * src = /root/reference/pkg/src/cavityflow); the Python package
 * paper_2504_03697_b200 binds them with ctypes and keeps the reference's
 * names, argument order and exceptions (INTEGRATION.md shows the binding).
 *
 * Conventions
 *   - All pointers are DEVICE pointers to fp64 (or int32 index) arrays,
 *     except where a name ends in _host.  `stream` is a cudaStream_t.
 *   - Scalar (cell-centred) fields are flat with x (i) fastest:
 *     index = i + nx*(j + ny*k)  (src/grid.py:44-48).
 *   - Velocity components are x-fastest with a padded row pitch `ld`
 *     (elements) and plane pitch ld*ny_c, where the component extents are
 *     u:(n+1,n,n)  v:(n,n+1,n)  w:(n,n,n+1)  (src/grid.py:51-65).
 *   - Return value: CF_OK (0) on success, CF_BREAKDOWN / CF_NOT_CONVERGED
 *     for solver outcomes, a negative code for errors; cf_last_error()
 *     returns the message of the calling thread's last error.
 */
#ifndef CFGPU_H
#define CFGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CF_OK 0
#define CF_BREAKDOWN 1      /* p^T A p <= 0            (src/solver.py:151-152) */
#define CF_NOT_CONVERGED 2  /* max_iter reached        (src/solver.py:147, :171) */
#define CF_EINVAL (-1)      /* bad argument            (ValueError in the reference) */
#define CF_ECUDA (-2)       /* CUDA runtime failure */
#define CF_ENOMEM (-3)
#define CF_EIO (-4)         /* file I/O failure        (OSError in the reference) */

/* SpMV summation order: CSR order is src/sparse.py:194-201 over the columns
 * of src/sim.py:306-308 (k-1, j-1, i-1, diag, i+1, j+1, k+1); SYM order is
 * src/sparse.py:204-213 (diag, i+1, j+1, k+1, k-1, j-1, i-1). */
#define CF_ORDER_CSR 0
#define CF_ORDER_SYM 1

#define CF_PRECOND_NONE 0        /* src/solver.py:71-76 (z = r) */
#define CF_PRECOND_JACOBI 1      /* src/precond.py:77-95 (z = r * inv_diag) */
#define CF_PRECOND_DIC 2         /* src/precond.py:98-124 */

const char *cf_last_error(void);
int cf_version(void);
int cf_device_sms(void);

/* ---- vector kernels (src/sparse.py:270-301) ---------------------------- */
/* dot: writes the fp64 result to *result_host (synchronises `stream`).
 * Replaces sparse.dot (src/sparse.py:270). */
int cf_dot(const double *x, const double *y, int64_t n, double *result_host, void *stream);
/* y += alpha * x (unfused mul+add).  Replaces multiply_add_inplace (:284). */
int cf_axpy(double *y, double alpha, const double *x, int64_t n, void *stream);
/* out = x + y.  Replaces add (:293). */
int cf_add(const double *x, const double *y, double *out, int64_t n, void *stream);
/* out = alpha * x.  Replaces scale (:299). */
int cf_scale(double alpha, const double *x, double *out, int64_t n, void *stream);
/* out = x * y (elementwise).  Replaces JacobiPreconditioner.apply
 * (src/precond.py:89-95). */
int cf_mul(const double *x, const double *y, double *out, int64_t n, void *stream);
/* max |x| -> *result_host (synchronises). Used for div_pre (src/sim.py:394). */
int cf_max_abs(const double *x, int64_t n, double *result_host, void *stream);

/* ---- operators ---------------------------------------------------------- */
/* y = A x for full CSR with int32 indices, serial per-row order.
 * Replaces spmv (src/sparse.py:236-247). */
int cf_csr_spmv(int64_t n_rows, const int32_t *row_ptr, const int32_t *col_idx,
                const double *values, const double *x, double *y, void *stream);
/* y = (D + U + U^T) x with the transpose gathered through t_perm.
 * Replaces spmv_sym (src/sparse.py:250-267). */
int cf_sym_spmv(int64_t n, const double *diag, const int32_t *row_ptr, const int32_t *col_idx,
                const double *values, const int32_t *t_row_ptr, const int32_t *t_col_idx,
                const int32_t *t_perm, const double *x, double *y, void *stream);
/* Matrix-free 7-point operator of src/sim.py:296-333 (diag 6/h^2, neighbours
 * -1/h^2, Dirichlet-ghost neighbours dropped) on an nx*ny*nz block.  With
 * `order` = CF_ORDER_CSR the result equals cf_csr_spmv on poisson_full_csr
 * bit for bit, with CF_ORDER_SYM it equals spmv_sym on poisson_symmetric. */
int cf_stencil7_apply(int nx, int ny, int nz, double h, int order, const double *x, double *y,
                      void *stream);

/* ---- simplified DIC preconditioner (src/precond.py:24-54, :141-151) ----- */
/* Level schedule of a strictly lower triangle given as HOST int64 CSR
 * (level = 1 + max level of the row's lower columns; for the 7-point
 * operator level(i,j,k) = i+j+k).  Host-only, no CUDA call. */
int cf_level_schedule(int64_t n, const int64_t *lower_ptr, const int64_t *lower_col, int32_t *level_host,
                      int32_t *nlevels_host);
/* Modified diagonal d~ (src/precond.py:24-34) by level-scheduled launches
 * over the strict lower triangle (lp, lc, lv: int32/fp64 device CSR).
 * level_rows: rows sorted by level (device); level_ptr_host: nlevels+1
 * offsets (host).  Returns CF_EINVAL with the first failing row in
 * *bad_row_host when a diagonal becomes <= 0 (else -1). */
int cf_dic_factor(int64_t n, const int32_t *lp, const int32_t *lc, const double *lv, const double *diag,
                  const int32_t *level_rows, const int64_t *level_ptr_host, int nlevels, double *d,
                  int64_t *bad_row_host, void *stream);
/* z = M^-1 r, M = (L + D~) D~^-1 (D~ + L^T) (src/precond.py:37-54, :116-124):
 * forward sweep over levels ascending into w, backward over levels
 * descending into z.  (up, uc, uv) is the strict upper triangle. */
int cf_dic_apply(int64_t n, const int32_t *lp, const int32_t *lc, const double *lv, const int32_t *up,
                 const int32_t *uc, const double *uv, const double *d, const int32_t *level_rows,
                 const int64_t *level_ptr_host, int nlevels, const double *r, double *w, double *z,
                 void *stream);
/* q[i] = a[i] / d[i] computed the way the skewed DIC sweeps divide (the
 * reciprocal refinement of the compiler's fp64 division hoisted out of the
 * sweep, its last three operations per cell; src/precond.py:44, :54 `s / d[i]`).
 * Bit-identical to IEEE division; exposed so the tests can check exactly that. */
int cf_dic_divide(int64_t n, const double *a, const double *d, double *q, void *stream);

/* ---- fused conjugate gradient (src/solver.py:33-171) -------------------- */
typedef struct cf_cg cf_cg;
/* One workspace per grid, like PoissonCache (src/sim.py:336-349): owns the
 * CG vectors, block partials, device scalars and the captured CUDA graph. */
int cf_cg_create(cf_cg **ws, int nx, int ny, int nz, double h, int order, void *stream);
int cf_cg_destroy(cf_cg *ws);
/* Solve A x = b.  x0 may be NULL (x = 0).  precond: CF_PRECOND_*; for
 * JACOBI, inv_diag may be NULL to mean the operator's constant h^2/6.
 * The iteration loop runs on the device (CUDA graph with a conditional WHILE
 * node); stats are returned through the *_host pointers.  Returns CF_OK,
 * CF_NOT_CONVERGED (x is the last iterate) or CF_BREAKDOWN. */
int cf_cg_solve(cf_cg *ws, const double *b, double *x, const double *x0, double tol,
                int64_t max_iter, int precond, const double *inv_diag, int64_t *iters_host,
                double *res_host, void *stream);
/* Device time (ms) of the last solve's iteration loop, CUDA-event timed. */
int cf_cg_last_loop_ms(cf_cg *ws, float *ms_host);
/* The kernel form the last solve ran and how many kernels it launched
 * (no reference counterpart: measurement support for bench.py). */
enum {
    CF_CG_FORM_SMALL = 0,    /* n^3 <= 5120: the whole solve in one block */
    CF_CG_FORM_TWO = 1,      /* two fused kernels per iteration (the reference recurrence) */
    CF_CG_FORM_SPASS = 2,    /* one TMA-fed single-reduction pass per iteration (default) */
    CF_CG_FORM_PASS = 3,     /* opt-in single-reduction pass kernels (CF_CG_ALGO=pass) */
    CF_CG_FORM_PERSIST = 4,  /* opt-in persistent single launch (CF_PERSIST=1) */
    CF_CG_FORM_TWO_DIC = 5   /* two-kernel loop with the DIC sweeps */
};
int cf_cg_last_form(cf_cg *ws, int *form_host, int64_t *launches_host);
/* Attach a DIC factor (arguments as cf_dic_apply; device arrays must stay
 * alive) so cf_cg_solve accepts CF_PRECOND_DIC: each iteration then runs the
 * level sweeps inside the same device loop. */
int cf_cg_set_dic(cf_cg *ws, const int32_t *lp, const int32_t *lc, const double *lv, const int32_t *up,
                  const int32_t *uc, const double *uv, const double *d, const int32_t *level_rows,
                  const int64_t *level_ptr_host, int nlevels);

/* ---- z-slab conjugate gradient (multi-GPU; SURVEY.md §5.8, §8 e) -------- */
typedef struct cf_dcg cf_dcg;
/* 128-byte NCCL unique id (rank 0 creates it and broadcasts it). */
int cf_nccl_unique_id(void *out128);
/* CG over z-slabs of an nx*ny*nz grid (nx even >= 32).  This process owns
 * `nslabs` consecutive slabs with global plane bounds slab_bounds[0..nslabs]
 * on the current device; lo_rank / hi_rank are the ranks owning the slabs
 * below / above (-1: none).  nccl_id NULL (or nranks 1) runs without NCCL --
 * several slabs in one process is the single-device emulation of the
 * decomposition.  The reference has no distributed solver; the iterates are
 * the reference's CG (src/solver.py:128-171) up to reduction order. */
int cf_dcg_create(cf_dcg **ws, int nx, int ny, int nz, double h, int order, int nranks, int rank,
                  const void *nccl_id, int nslabs, const int *slab_bounds, int lo_rank, int hi_rank,
                  void *stream);
int cf_dcg_destroy(cf_dcg *ws);
/* b_slabs / x_slabs: per local slab, device pointers to its owned planes
 * (nx*ny*(z1-z0) doubles, x fastest).  precond: CF_PRECOND_NONE or
 * CF_PRECOND_JACOBI (constant diagonal).  Same return codes as cf_cg_solve. */
int cf_dcg_solve(cf_dcg *ws, const double *const *b_slabs, double *const *x_slabs, double tol,
                 int64_t max_iter, int precond, int64_t *iters_host, double *res_host, void *stream);
int cf_dcg_last_loop_ms(cf_dcg *ws, float *ms_host);

/* ---- z-slab CG with the collectives fused into the kernels (peer memory) --
 * Same solve as cf_dcg, but each iteration is two kernels per GPU: the r
 * halo planes are stored straight into the neighbours' memory by the update
 * kernel, and each reduction is posted to every rank's mailbox and summed
 * (rank order) by the kernels' last blocks -- no NCCL, no extra launches
 * (csrc/cf_p2p.cu).  nslabs == 1: this process is `rank` of `nranks`, one GPU
 * each; link the ranks with cf_pcg_export (publish this rank's IPC handles)
 * and cf_pcg_import (all ranks' blobs in rank order) before solving.
 * nslabs == nranks (rank 0): every slab in this process on one device, the
 * single-device verification of the same kernels.  nx even, <= 8 ranks. */
typedef struct cf_pcg cf_pcg;
int cf_pcg_create(cf_pcg **ws, int nx, int ny, int nz, double h, int order, int nranks, int rank, int nslabs,
                  const int *slab_bounds, void *stream);
int cf_pcg_export_size(void);
int cf_pcg_export(cf_pcg *ws, void *out, int cap);
int cf_pcg_import(cf_pcg *ws, const void *all_blobs, int nranks);
int cf_pcg_destroy(cf_pcg *ws);
int cf_pcg_solve(cf_pcg *ws, const double *const *b_slabs, double *const *x_slabs, double tol, int64_t max_iter,
                 int precond, int64_t *iters_host, double *res_host, void *stream);
int cf_pcg_last_loop_ms(cf_pcg *ws, float *ms_host);
/* The slab CG form (CF_CG_FORM_SPASS: the single pass, default; CF_CG_FORM_TWO:
 * the two-kernel form, CF_PCG_ALGO=two or slabs thinner than 4 planes). */
int cf_pcg_form(cf_pcg *ws, int *form_host);
/* Diagnostics (tests): which 0 = this rank's r allocation incl. halo planes
 * (read or write), 1 / 2 = the peer plane this rank's bottom / top r plane is
 * stored into (read only); 3 = the single pass's r0 array (nzl + 4 planes,
 * two halo planes each side), 4 / 5 = the two peer planes its bottom /
 * top two planes are stored into -- checks the IPC linking without running
 * kernels. */
int cf_pcg_debug_io(cf_pcg *ws, int which, int write, double *host, int64_t n);

/* ---- time-step kernels (src/sim.py:134-289, :352-449) ------------------- */
/* Lid forcing u[1:n, n-1, :] += lid_dv, then zero the six wall-normal face
 * planes.  Replaces apply_forces + enforce_boundaries (:134-149).
 * lid_dv = 0 gives enforce_boundaries alone. */
int cf_forces_bc(double *u, double *v, double *w, int n, int ldu, int ldv, int ldw,
                 double lid_dv, int apply_lid, void *stream);
/* Semi-Lagrangian advection of all three components (src/sim.py:259-289),
 * wall-normal planes of the result zeroed.  Inputs and outputs must not
 * alias. */
int cf_advect(const double *u, const double *v, const double *w, double *nu, double *nv,
              double *nw, int n, int ldu, int ldv, int ldw, double h, double dt, void *stream);
/* out = scale * divergence (src/grid.py:145-154; scale = -rho/dt gives the
 * Poisson right-hand side of src/sim.py:359-360).  max|out| is written to
 * *maxabs_host when non-NULL (synchronises). */
int cf_divergence(const double *u, const double *v, const double *w, int n, int ldu, int ldv,
                  int ldw, double h, double scale, double *out, double *maxabs_host,
                  void *stream);
/* Pressure-gradient correction with ghost p = 0 (src/sim.py:426-449), read
 * from (u, v, w) and written out of place to (nu, nv, nw) (same pitches; the
 * correction of each face reads neighbouring faces, so in-place would race).
 * The post-correction max cell |divergence| (before the wall clamp) goes to
 * *div_post_host (synchronises); the written field is wall-clamped. */
int cf_pressure_correct(const double *u, const double *v, const double *w, double *nu, double *nv,
                        double *nw, const double *p, int n, int ldu, int ldv, int ldw, double h,
                        double coef, double *div_post_host, void *stream);
/* Box (nx x ny x nz; the reference's cube is nx = ny = nz = n, other boxes
 * are the SURVEY.md §8 f2 extension) and z-slab forms of the step kernels
 * (multi-GPU): the slab owns global planes [z0, z1) of nz and
 * its velocity arrays hold planes z0-halo .. (u, v: z1+halo-1; w: z1+halo),
 * pointers at the first stored plane; scalar arrays (out, p) are slab-local
 * with plane 0 = z0 and, for p, readable halo planes -1 / z1-z0 where
 * neighbours exist.  Owned w faces are [z0, z1) plus face nz on the last
 * slab.  z0 = 0, z1 = nz, halo = 0 is the whole box. */
int cf_forces_bc_slab(double *u, double *v, double *w, int nx, int ny, int nz, int z0, int z1, int halo,
                      int ldu, int ldv, int ldw, double lid_dv, int apply_lid, void *stream);
int cf_advect_slab(const double *u, const double *v, const double *w, double *nu, double *nv, double *nw,
                   int nx, int ny, int nz, int z0, int z1, int halo, int ldu, int ldv, int ldw, double h,
                   double dt, void *stream);
int cf_divergence_slab(const double *u, const double *v, const double *w, int nx, int ny, int nz, int z0,
                       int z1, int halo, int ldu, int ldv, int ldw, double h, double scale, double *out,
                       double *maxabs_host, void *stream);
int cf_pressure_correct_slab(const double *u, const double *v, const double *w, double *nu, double *nv,
                             double *nw, const double *p, int nx, int ny, int nz, int z0, int z1, int halo,
                             int ldu, int ldv, int ldw, double h, double coef, double *div_post_host,
                             void *stream);
/* Physics extension beyond the (inviscid) reference, SURVEY.md §8 f2:
 * explicit viscous diffusion of every non-wall-normal face,
 *   new = c + kdt*((((((xm + xp) + ym) + yp) + zm) + zp) - 6c),  kdt = nu*dt/h^2,
 * tangential ghosts mirrored (free slip) or negated (no_slip), the lid
 * (y = Ly) a Dirichlet wall when lid_dirichlet (ghost u = 2*lid_u - c,
 * ghost w = -c).  Out of place.  Stable for kdt <= 1/6. */
int cf_diffuse(const double *u, const double *v, const double *w, double *nu, double *nv, double *nw, int n,
               int ldu, int ldv, int ldw, double kdt, double lid_u, int lid_dirichlet, int no_slip,
               void *stream);
int cf_diffuse_slab(const double *u, const double *v, const double *w, double *nu, double *nv, double *nw,
                    int nx, int ny, int nz, int z0, int z1, int halo, int ldu, int ldv, int ldw, double kdt,
                    double lid_u, int lid_dirichlet, int no_slip, void *stream);
/* Implicit (backward-Euler) diffusion operator of one component (comp 0/1/2
 * = u/v/w) on its physical padded array (row pitch ld): (I - kdt L) with the
 * ghost rules of cf_diffuse folded into the diagonal and, for the moving lid,
 * the right-hand side.  mode 0: y = A x; mode 1: y = diag(A); mode 2: y = the
 * right-hand side for x = u*.  Fixed faces and padding are identity rows. */
int cf_helmholtz(int mode, int comp, const double *x, double *y, int nx, int ny, int nz, int ld, double kdt,
                 double lid_u, int lid_dirichlet, int no_slip, void *stream);
/* Trilinear sample of all three components at one point (src/grid.py:124-142);
 * result (3 doubles) to out_host. */
int cf_sample_velocity(const double *u, const double *v, const double *w, int n, int ldu,
                       int ldv, int ldw, double h, double px, double py, double pz,
                       double *out_host, void *stream);

/* ---- snapshots (src/snapshots.py) --------------------- */
/* Cell-centred view of the state (src/snapshots.py:46-62): out (device,
 * 4*nx*ny*nz doubles) = [uc | vc | wc | p], each i-fastest, uc = 0.5*(u[i] +
 * u[i+1]) etc.  p is the flat pressure vector. */
int cf_snapshot_cells(const double *u, const double *v, const double *w, const double *p, int nx, int ny, int nz,
                      int ldu, int ldv, int ldw, double *out, void *stream);
/* repr(float(v)) minus a trailing ".0" (src/snapshots.py:65-70) into out
 * (cap >= 32); returns the length. */
int cf_format_double(double v, char *out, int cap);
/* The snapshot CSV of cf_snapshot_cells' output (copied to HOST), x/y/z the
 * cell centres ((i+0.5)h ...): byte-identical to write_snapshot
 * (src/snapshots.py:82-108) for any `threads`. */
int cf_snapshot_write(const char *path, const double *cells_host, int nx, int ny, int nz, double h, int threads);
/* The same CSV from seven HOST columns (a prebuilt Snapshot). */
int cf_csv_write_columns(const char *path, const double *x, const double *y, const double *z, const double *u,
                         const double *v, const double *w, const double *p, int64_t nrows, int threads);

#ifdef __cplusplus
}
#endif

#endif /* CFGPU_H */
