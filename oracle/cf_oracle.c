/*
 * cf_oracle.c -- CPU restatement of the cavityflow reference kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path (and the CPU baseline timed by bench.py); nothing in the product
 * package links or calls it.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Every routine restates one reference loop with the same per-element
 * operation order.  Build with -ffp-contract=off (see oracle/Makefile): the
 * reference's numba kernels are compiled without fastmath, so no FMA
 * contraction happens there either, and the restatement is bit-identical
 * for a fixed chunking (pinned by tests/test_oracle.py against
 * the tests/golden fixtures, which were produced by the reference itself).
 *
 * Parallelism mirrors the reference WorkerPool (src/parallel.py:24-44):
 * the caller passes chunk bounds computed exactly like
 * np.linspace(0, n, chunks + 1).astype(int64); each chunk runs on its own
 * OpenMP thread and reductions are returned per chunk so the caller sums
 * them in chunk order, as src/sparse.py:281 does.
 */
#include <stdint.h>
#include <math.h>

typedef int64_t i64;

#define CHUNK_LOOP(nch) _Pragma("omp parallel for schedule(static, 1) num_threads(nch > 0 ? nch : 1)") \
    for (int c_ = 0; c_ < (nch); ++c_)

/* src/sparse.py:194-201 (_spmv_range): ascending CSR row sum. */
static void spmv_rows(const i64 *rp, const i64 *ci, const double *val,
                      const double *x, double *y, i64 lo, i64 hi)
{
    for (i64 i = lo; i < hi; ++i) {
        double s = 0.0;
        for (i64 p = rp[i]; p < rp[i + 1]; ++p)
            s += val[p] * x[ci[p]];
        y[i] = s;
    }
}

void orc_spmv_csr(const i64 *rp, const i64 *ci, const double *val,
                  const double *x, double *y, const i64 *bounds, int nch)
{
    CHUNK_LOOP(nch) spmv_rows(rp, ci, val, x, y, bounds[c_], bounds[c_ + 1]);
}

/* src/sparse.py:204-213 (_spmv_sym_range): diagonal, upper, then the
 * lower triangle gathered through the cached transpose (t_perm). */
static void spmv_sym_rows(const double *diag, const i64 *rp, const i64 *ci,
                          const double *val, const i64 *trp, const i64 *tci,
                          const i64 *tperm, const double *x, double *y,
                          i64 lo, i64 hi)
{
    for (i64 i = lo; i < hi; ++i) {
        double s = diag[i] * x[i];
        for (i64 p = rp[i]; p < rp[i + 1]; ++p)
            s += val[p] * x[ci[p]];
        for (i64 p = trp[i]; p < trp[i + 1]; ++p)
            s += val[tperm[p]] * x[tci[p]];
        y[i] = s;
    }
}

void orc_spmv_sym(const double *diag, const i64 *rp, const i64 *ci,
                  const double *val, const i64 *trp, const i64 *tci,
                  const i64 *tperm, const double *x, double *y,
                  const i64 *bounds, int nch)
{
    CHUNK_LOOP(nch) spmv_sym_rows(diag, rp, ci, val, trp, tci, tperm, x, y,
                                  bounds[c_], bounds[c_ + 1]);
}

/* src/sparse.py:216-221 (_dot_range): one serial partial per chunk. */
void orc_dot(const double *x, const double *y, const i64 *bounds, int nch,
             double *partials)
{
    CHUNK_LOOP(nch) {
        double s = 0.0;
        for (i64 i = bounds[c_]; i < bounds[c_ + 1]; ++i)
            s += x[i] * y[i];
        partials[c_] = s;
    }
}

/* src/sparse.py:224-228 (_maxpy_range): y += alpha * x, unfused. */
void orc_maxpy(double *y, double alpha, const double *x, const i64 *bounds,
               int nch)
{
    CHUNK_LOOP(nch) {
        for (i64 i = bounds[c_]; i < bounds[c_ + 1]; ++i)
            y[i] += alpha * x[i];
    }
}

/* src/precond.py:24-34: modified DIC diagonal; returns first bad row or -1. */
i64 orc_dic_diag(const i64 *lp, const i64 *lc, const double *lv,
                 const double *diag, double *out, i64 n)
{
    for (i64 i = 0; i < n; ++i) {
        double s = diag[i];
        for (i64 p = lp[i]; p < lp[i + 1]; ++p) {
            double v = lv[p];
            s -= v * v / out[lc[p]];
        }
        out[i] = s;
        if (s <= 0.0)
            return i;
    }
    return -1;
}

/* src/precond.py:37-54: forward solve (L + D) w = r, then backward
 * (D + L^T) z = D w, both strictly sequential. */
void orc_dic_apply(const i64 *lp, const i64 *lc, const double *lv,
                   const i64 *up, const i64 *uc, const double *uv,
                   const double *d, const double *r, double *w, double *z,
                   i64 n)
{
    for (i64 i = 0; i < n; ++i) {
        double s = r[i];
        for (i64 p = lp[i]; p < lp[i + 1]; ++p)
            s -= lv[p] * w[lc[p]];
        w[i] = s / d[i];
    }
    for (i64 i = n - 1; i >= 0; --i) {
        double s = 0.0;
        for (i64 p = up[i]; p < up[i + 1]; ++p)
            s += uv[p] * z[uc[p]];
        z[i] = w[i] - s / d[i];
    }
}

/* ---- semi-Lagrangian advection, reference layout (C order, k fastest) ---- */

static inline double clampd(double a, double hi)
{
    if (a < 0.0)
        return 0.0;
    if (a > hi)
        return hi;
    return a;
}

static inline i64 base_index(double a, i64 na)
{
    i64 i0 = (i64)a;
    if (i0 > na - 2)
        i0 = na > 1 ? na - 2 : 0;
    return i0;
}

/* src/sim.py:156-190 (_tri): clamped trilinear sample at lattice coords. */
static double trilerp(const double *arr, i64 na, i64 nb, i64 nc,
                      double a, double b, double c)
{
    a = clampd(a, na - 1.0);
    b = clampd(b, nb - 1.0);
    c = clampd(c, nc - 1.0);
    i64 i0 = base_index(a, na), j0 = base_index(b, nb), k0 = base_index(c, nc);
    i64 i1 = i0 + 1 < na - 1 ? i0 + 1 : na - 1;
    i64 j1 = j0 + 1 < nb - 1 ? j0 + 1 : nb - 1;
    i64 k1 = k0 + 1 < nc - 1 ? k0 + 1 : nc - 1;
    double fa = a - (double)i0, fb = b - (double)j0, fc = c - (double)k0;
#define AT(i, j, k) arr[((i) * nb + (j)) * nc + (k)]
    double c00 = AT(i0, j0, k0) * (1.0 - fa) + AT(i1, j0, k0) * fa;
    double c10 = AT(i0, j1, k0) * (1.0 - fa) + AT(i1, j1, k0) * fa;
    double c01 = AT(i0, j0, k1) * (1.0 - fa) + AT(i1, j0, k1) * fa;
    double c11 = AT(i0, j1, k1) * (1.0 - fa) + AT(i1, j1, k1) * fa;
#undef AT
    return (c00 * (1.0 - fb) + c10 * fb) * (1.0 - fc) + (c01 * (1.0 - fb) + c11 * fb) * fc;
}

/* src/sim.py:193-229 (_advect_face) and :232-240 (_advect_range). */
void orc_advect(const double *u, const double *v, const double *w,
                double *out, int comp, i64 nx, i64 ny, i64 nz, double h, double dt,
                const i64 *bounds, int nch)
{
    /* the reference's cube has nx = ny = nz = n and one side length n*h
     * (src/grid.py:35-37); a box (extension) clamps each axis to its own */
    const double lx = nx * h, ly = ny * h, lz = nz * h;
    i64 na = nx + (comp == 0), nb = ny + (comp == 1), nc = nz + (comp == 2);
    CHUNK_LOOP(nch) {
        for (i64 idx = bounds[c_]; idx < bounds[c_ + 1]; ++idx) {
            i64 i = idx % na, j = (idx / na) % nb, k = idx / (na * nb);
            double x, y, z;
            if (comp == 0) {
                x = i * h; y = (j + 0.5) * h; z = (k + 0.5) * h;
            } else if (comp == 1) {
                x = (i + 0.5) * h; y = j * h; z = (k + 0.5) * h;
            } else {
                x = (i + 0.5) * h; y = (j + 0.5) * h; z = k * h;
            }
            double su = trilerp(u, nx + 1, ny, nz, x / h, y / h - 0.5, z / h - 0.5);
            double sv = trilerp(v, nx, ny + 1, nz, x / h - 0.5, y / h, z / h - 0.5);
            double sw = trilerp(w, nx, ny, nz + 1, x / h - 0.5, y / h - 0.5, z / h);
            double xb = clampd(x - dt * su, lx);
            double yb = clampd(y - dt * sv, ly);
            double zb = clampd(z - dt * sw, lz);
            double r;
            if (comp == 0)
                r = trilerp(u, nx + 1, ny, nz, xb / h, yb / h - 0.5, zb / h - 0.5);
            else if (comp == 1)
                r = trilerp(v, nx, ny + 1, nz, xb / h - 0.5, yb / h, zb / h - 0.5);
            else
                r = trilerp(w, nx, ny, nz + 1, xb / h - 0.5, yb / h - 0.5, zb / h);
            out[(i * nb + j) * nc + k] = r;
        }
    }
}

/* src/grid.py:145-154 (divergence): numpy evaluates the six-term flux
 * expression left to right, then divides by h; output flat, i fastest. */
void orc_divergence(const double *u, const double *v, const double *w,
                    i64 nx, i64 ny, i64 nz, double h, double *out, int nthreads)
{
    /* C-order arrays: u (nx+1, ny, nz), v (nx, ny+1, nz), w (nx, ny, nz+1) */
#pragma omp parallel for num_threads(nthreads > 0 ? nthreads : 1)
    for (i64 k = 0; k < nz; ++k)
        for (i64 j = 0; j < ny; ++j)
            for (i64 i = 0; i < nx; ++i) {
                double t = u[((i + 1) * ny + j) * nz + k] - u[(i * ny + j) * nz + k];
                t = t + v[(i * (ny + 1) + j + 1) * nz + k];
                t = t - v[(i * (ny + 1) + j) * nz + k];
                t = t + w[(i * ny + j) * (nz + 1) + k + 1];
                t = t - w[(i * ny + j) * (nz + 1) + k];
                out[i + nx * (j + ny * k)] = t / h;
            }
}
