// cf_cg_common.cuh -- device state shared by the single-domain CG
// (cf_cg.cu) and the z-slab CG (cf_dist.cu).
#pragma once

#include "cf_common.cuh"

namespace cf {

enum PrecKind { PK_NONE = 0, PK_JCONST = 1, PK_JVEC = 2, PK_ZVEC = 3 };

struct CgScalars {
    double rz, alpha, beta, pap, rr, norm_b, res, tol;
    double alpha_prev;  // alpha of the previous iteration (deferred x update, XM_DOUBLE)
    long long it, max_iter;
    int done, status;  // status: 0 running, 1 converged, 2 max_iter, 3 breakdown
    unsigned long long phase;  // collective phases completed (peer-memory z-slab CG, cf_p2p.cu)
};

enum { ST_RUNNING = 0, ST_CONVERGED = 1, ST_MAXITER = 2, ST_BREAKDOWN = 3 };

// x-update modes of the update kernels.  The solution is only read at the
// end, so the loop body (two iterations, p buffers swapped) updates x once:
// the first iteration skips it, the second applies both steps in order,
//   x = (x + alpha_prev * p_prev) + alpha * p,
// the same two roundings as two separate updates (src/solver.py:155), saving
// 16 N of the 128 N a pair of iterations moves (+8 N for reading p_prev).
// A solve that stops after a skipping iteration is finished by
// cg_x_fixup (x += alpha * p_prev when the iteration count is odd).
enum { XM_EACH = 0, XM_SKIP = 1, XM_DOUBLE = 2 };

struct CgTickets {
    unsigned int init, dir, upd, pad;
};

template <int PK>
__device__ __forceinline__ double zval(double r, const double *__restrict__ jd, long long i, double zc)
{
    // z = M^-1 r: src/solver.py:71-76 (none) and src/precond.py:94 (Jacobi)
    if (PK == PK_NONE) return r;
    if (PK == PK_JCONST) return r * zc;
    return r * __ldg(jd + i);
}

// The scalar recurrences of src/solver.py, shared by the last block of the
// single-domain kernels and by the z-slab scalar kernel (after the
// all-reduce).
__device__ __forceinline__ void scalar_after_dir(CgScalars *sc, double pap)
{
    sc->pap = pap;
    if (pap <= 0.0) {  // src/solver.py:151-152
        sc->status = ST_BREAKDOWN;
        sc->done = 1;
    } else {
        sc->alpha_prev = sc->alpha;
        sc->alpha = sc->rz / pap;  // :153
    }
}

// returns true when the solve has stopped
template <bool HAS_RZ>
__device__ __forceinline__ bool scalar_after_update(CgScalars *sc, double rr, double rz)
{
    sc->rr = rr;
    sc->it += 1;                          // :158
    sc->res = sqrt(rr) / sc->norm_b;      // :159
    if (sc->res <= sc->tol) {             // :160-162
        sc->status = ST_CONVERGED;
        sc->done = 1;
    } else if (sc->it >= sc->max_iter) {  // :147
        sc->status = ST_MAXITER;
        sc->done = 1;
    } else if (HAS_RZ) {
        sc->beta = rz / sc->rz;  // :165-166
        sc->rz = rz;
    }
    return sc->done != 0;
}

__device__ __forceinline__ void scalar_after_init(CgScalars *sc, double bb, double rz)
{
    sc->norm_b = sqrt(bb);  // src/solver.py:60-61
    sc->rz = rz;            // :143
    sc->beta = 0.0;
    sc->it = 0;
    sc->res = INFINITY;
    if (sc->norm_b == 0.0) {  // :62-64
        sc->done = 1;
        sc->status = ST_CONVERGED;
        sc->res = 0.0;
    }
}

// The single-reduction (Chronopoulos-Gear) scalars of the pass forms
// (cf_cg_pass.cuh, cf_cg_lpass.cuh, cf_cg_spass.cuh; z-slab: cf_p2p.cu).
// After the pass's reduction: stop test on r_{k+1} (src/solver.py:158-162),
// then the next pass's beta and alpha by the single-reduction identity.
__device__ __forceinline__ void scalar_after_pass(CgScalars *sc, double rr, double gam, double dlt)
{
    sc->rr = rr;
    sc->it += 1;
    sc->res = sqrt(rr) / sc->norm_b;
    if (sc->res <= sc->tol) {
        sc->status = ST_CONVERGED;
        sc->done = 1;
        return;
    }
    if (sc->it >= sc->max_iter) {
        sc->status = ST_MAXITER;
        sc->done = 1;
        return;
    }
    const double beta = gam / sc->rz;                 // src/solver.py:165
    const double pap = dlt - beta * gam / sc->alpha;  // p_{k+1}.A p_{k+1}
    sc->pap = pap;
    if (pap <= 0.0) {  // src/solver.py:151-152
        sc->status = ST_BREAKDOWN;
        sc->done = 1;
        return;
    }
    sc->alpha_prev = sc->alpha;
    sc->alpha = gam / pap;  // :153
    sc->beta = beta;
    sc->rz = gam;
}

// After the init pass: |b|, gamma_0, delta_0 -> alpha_0 = gamma_0 / delta_0.
__device__ __forceinline__ void scalar_after_pass_init(CgScalars *sc, double bb, double gam, double dlt)
{
    scalar_after_init(sc, bb, gam);
    if (sc->done) return;
    sc->pap = dlt;
    if (dlt <= 0.0) {
        sc->status = ST_BREAKDOWN;
        sc->done = 1;
        return;
    }
    sc->alpha = gam / dlt;
}

}  // namespace cf
