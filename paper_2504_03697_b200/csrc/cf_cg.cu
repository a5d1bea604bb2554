// cf_cg.cu -- fused, device-resident conjugate gradient for the pressure
// system (src/solver.py:33-171 with the matrix-free operator of
// src/sim.py:296-333).
//
// Per iteration the reference does 1 SpMV, 3 dots, 3 axpys and a
// preconditioner apply with 3 host syncs -- 88 B/cell of
// HBM traffic at best.  Here an iteration is two kernels and no host sync:
//
//   dir:    p_k = z_k + beta*p_{k-1}  (z = M^-1 r formed on the fly from r,
//           so p is built tile-by-tile with its halo) then A p_k by the
//           z-march stencil, partial p.Ap; the last block forms alpha.
//           HBM: read r, p_{k-1}; write p_k                    = 24 B/cell
//   update: A p_k recomputed from p_k (cheaper than storing Ap: 8 B vs 16 B),
//           x += alpha p, r -= alpha Ap, partials r.r and r.z; the last block
//           checks sqrt(r.r)/|b| <= tol, forms beta.
//           HBM: read p, r, x; write r, x                       = 40 B/cell
//
// 64 B/cell instead of 88, with every per-element operation identical to
// the reference's (same rounding, -fmad=false); only the dot-product
// summation order differs (a fixed two-level tree, deterministic).
// The iteration loop is a CUDA graph with a conditional WHILE node whose
// condition is cleared on the device when the solve stops.
#include <algorithm>
#include <type_traits>
#include <cstring>
#include <mutex>
#include <vector>

#include "cf_cg_common.cuh"
#include "cf_dic.cuh"
#include "cf_stencil.cuh"
#include "cf_tma_march.cuh"

namespace cf {

// ---------------------------------------------------------------- init
// r = b, x = 0, |b|^2 and r.z (src/solver.py:60-61, :130-143).
template <int PK>
__global__ void __launch_bounds__(kMarchThreads) cg_init_flat(long long n, const double *__restrict__ b,
                                                              double *__restrict__ r, double *__restrict__ x,
                                                              const double *__restrict__ jd, double zc,
                                                              CgScalars *sc, double *partials,
                                                              CgTickets *tk)
{
    __shared__ double red[32];
    __shared__ int is_last;
    double bb = 0.0, rz = 0.0;
    const long long stride = (long long)gridDim.x * kMarchThreads;
    for (long long i = (long long)blockIdx.x * kMarchThreads + threadIdx.x; i < n; i += stride) {
        const double bi = b[i];
        r[i] = bi;
        x[i] = 0.0;
        bb = bb + bi * bi;
        rz = rz + bi * zval<PK>(bi, jd, i, zc);
    }
    bb = block_sum<kMarchThreads>(bb, red);
    rz = block_sum<kMarchThreads>(rz, red);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = bb;
        partials[2 * blockIdx.x + 1] = rz;
    }
    if (last_block(&tk->init, &is_last)) {
        bb = reduce_partials<kMarchThreads>(partials, gridDim.x, 2, red);
        rz = reduce_partials<kMarchThreads>(partials + 1, gridDim.x, 2, red);
        if (threadIdx.x == 0) {
            sc->norm_b = sqrt(bb);
            sc->rz = rz;
            sc->beta = 0.0;
            sc->it = 0;
            sc->res = INFINITY;
            if (sc->norm_b == 0.0) {  // src/solver.py:62-64
                sc->done = 1;
                sc->status = ST_CONVERGED;
                sc->res = 0.0;
            }
        }
    }
}

// r = b - A x0, x = x0 (src/solver.py:134-139).
template <int ORDER, int PK>
__global__ void __launch_bounds__(kMarchThreads) cg_init_x0(Box bx, double off, double diag,
                                                            const double *__restrict__ b,
                                                            const double *__restrict__ x0,
                                                            double *__restrict__ r, double *__restrict__ x,
                                                            const double *__restrict__ jd, double zc,
                                                            CgScalars *sc, double *partials,
                                                            CgTickets *tk)
{
    __shared__ double red[32];
    __shared__ int is_last;
    double bb = 0.0, rz = 0.0;
    auto load = [&](long long i) { return __ldg(x0 + i); };
    auto epi = [&](long long i, double c, double ax) {
        const double bi = b[i];
        const double rn = bi + -1.0 * ax;
        r[i] = rn;
        x[i] = c;
        bb = bb + bi * bi;
        rz = rz + rn * zval<PK>(rn, jd, i, zc);
    };
    march<ORDER>(bx, off, diag, load, epi);
    bb = block_sum<kMarchThreads>(bb, red);
    rz = block_sum<kMarchThreads>(rz, red);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = bb;
        partials[2 * blockIdx.x + 1] = rz;
    }
    if (last_block(&tk->init, &is_last)) {
        bb = reduce_partials<kMarchThreads>(partials, gridDim.x, 2, red);
        rz = reduce_partials<kMarchThreads>(partials + 1, gridDim.x, 2, red);
        if (threadIdx.x == 0) {
            sc->norm_b = sqrt(bb);
            sc->rz = rz;
            sc->beta = 0.0;
            sc->it = 0;
            sc->res = INFINITY;
            if (sc->norm_b == 0.0) {
                sc->done = 1;
                sc->status = ST_CONVERGED;
                sc->res = 0.0;
            }
        }
    }
}

// ---------------------------------------------------------------- direction
template <int ORDER, int PK>
__global__ void __launch_bounds__(kMarchThreads) cg_dir_kernel(Box bx, double off, double diag,
                                                               const double *__restrict__ r,
                                                               const double *__restrict__ jd,
                                                               const double *__restrict__ zbuf,
                                                               const double *__restrict__ p_old,
                                                               double *__restrict__ p_new, double zc,
                                                               CgScalars *sc, double *partials,
                                                               CgTickets *tk)
{
    __shared__ double red[32];
    __shared__ int is_last;
    if (sc->done) return;
    const bool first = sc->it == 0;
    const double beta = sc->beta;
    double pap = 0.0;
    // p = z + beta*p_old (src/solver.py:167-170); the first direction is z
    // itself (:142).
    auto load = [&](long long i) {
        const double z = PK == PK_ZVEC ? __ldg(zbuf + i) : zval<PK>(__ldg(r + i), jd, i, zc);
        return first ? z : z + beta * __ldg(p_old + i);
    };
    auto epi = [&](long long i, double c, double ax) {
        p_new[i] = c;
        pap = pap + c * ax;
    };
    march<ORDER>(bx, off, diag, load, epi);
    pap = block_sum<kMarchThreads>(pap, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = pap;
    if (last_block(&tk->dir, &is_last)) {
        pap = reduce_partials<kMarchThreads>(partials, gridDim.x, 1, red);
        if (threadIdx.x == 0) {
            sc->pap = pap;
            if (pap <= 0.0) {  // src/solver.py:151-152
                sc->status = ST_BREAKDOWN;
                sc->done = 1;
            } else {
                sc->alpha = sc->rz / pap;
            }
        }
    }
}

// ---------------------------------------------------------------- update
template <int ORDER, int PK>
__global__ void __launch_bounds__(kMarchThreads) cg_update_kernel(Box bx, double off, double diag,
                                                                  const double *__restrict__ p,
                                                                  double *__restrict__ r,
                                                                  double *__restrict__ x,
                                                                  const double *__restrict__ jd,
                                                                  double zc, CgScalars *sc,
                                                                  double *partials, CgTickets *tk,
                                                                  int use_cond,
                                                                  cudaGraphConditionalHandle cond)
{
    __shared__ double red[32];
    __shared__ int is_last;
    if (sc->done) {
        if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    const double alpha = sc->alpha, malpha = -alpha;
    double rr = 0.0, rz = 0.0;
    auto load = [&](long long i) { return __ldg(p + i); };
    auto epi = [&](long long i, double c, double ax) {
        x[i] = x[i] + alpha * c;             // src/solver.py:155
        const double rn = r[i] + malpha * ax;  // :157
        r[i] = rn;
        rr = rr + rn * rn;                     // :159
        if (PK != PK_ZVEC) rz = rz + rn * zval<PK>(rn, jd, i, zc);  // :163-164
    };
    march<ORDER>(bx, off, diag, load, epi);
    rr = block_sum<kMarchThreads>(rr, red);
    if (PK != PK_ZVEC) rz = block_sum<kMarchThreads>(rz, red);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = rr;
        partials[2 * blockIdx.x + 1] = rz;
    }
    if (last_block(&tk->upd, &is_last)) {
        rr = reduce_partials<kMarchThreads>(partials, gridDim.x, 2, red);
        if (PK != PK_ZVEC) rz = reduce_partials<kMarchThreads>(partials + 1, gridDim.x, 2, red);
        if (threadIdx.x == 0) {
            sc->rr = rr;
            sc->it += 1;
            sc->res = sqrt(rr) / sc->norm_b;
            if (sc->res <= sc->tol) {  // :160-162
                sc->status = ST_CONVERGED;
                sc->done = 1;
            } else if (sc->it >= sc->max_iter) {  // :147
                sc->status = ST_MAXITER;
                sc->done = 1;
            } else if (PK != PK_ZVEC) {
                sc->beta = rz / sc->rz;  // :165-166
                sc->rz = rz;
            }
            if (sc->done && use_cond) cudaGraphSetConditional(cond, 0);
        }
    }
}

// r.z after a DIC apply (src/solver.py:143 for mode 0, :164-166 for mode 1).
__global__ void __launch_bounds__(kMarchThreads) cg_rz_kernel(long long n, const double *__restrict__ r,
                                                              const double *__restrict__ z, CgScalars *sc,
                                                              double *partials, CgTickets *tk, int mode)
{
    __shared__ double red[32];
    __shared__ int is_last;
    if (sc->done) return;
    double rz = 0.0;
    const long long stride = (long long)gridDim.x * kMarchThreads;
    for (long long i = (long long)blockIdx.x * kMarchThreads + threadIdx.x; i < n; i += stride)
        rz = rz + r[i] * z[i];
    rz = block_sum<kMarchThreads>(rz, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = rz;
    if (last_block(&tk->pad, &is_last)) {
        rz = reduce_partials<kMarchThreads>(partials, gridDim.x, 1, red);
        if (threadIdx.x == 0) {
            if (mode == 1) sc->beta = rz / sc->rz;
            sc->rz = rz;
        }
    }
}

// Deferred-x epilogue: a solve that stopped after a skipping iteration (odd
// iteration count) still owes x += alpha * p of that iteration; p is the
// buffer the skipping half read as its new direction (p[1]).
__global__ void __launch_bounds__(kMarchThreads) cg_x_fixup(long long n, double *__restrict__ x,
                                                           const double *__restrict__ p, const CgScalars *sc)
{
    if ((sc->it & 1) == 0) return;
    const double alpha = sc->alpha;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        x[i] = x[i] + alpha * p[i];  // src/solver.py:155
}

#include "cf_cg_tma.cuh"
#include "cf_cg_pair.cuh"
#include "cf_cg_pass.cuh"
#include "cf_cg_lean.cuh"
#include "cf_cg_lpass.cuh"
#include "cf_cg_spass.cuh"
#include "cf_cg_persist.cuh"

// Host: single-reduction pass geometry (32 x 16 tiles; chunks of ~32 planes,
// the 4-plane pipeline prologue amortised; CF_PASS_CHUNKS overrides).
PassGeom pass_geom(int nx, int ny, int nz)
{
    PassGeom g{nx, ny, nz, (nx + kPassTX - 1) / kPassTX, (ny + kPassTY - 1) / kPassTY, 1};
    int c = (nz + 31) / 32;
    const int tiles = g.ntx * g.nty;
    const int by_ctas = (num_sms() * 4 + tiles - 1) / tiles;
    c = std::max(c, std::min(by_ctas, std::max(1, nz / 8)));
    if (const char *e = getenv("CF_PASS_CHUNKS")) {
        const int v = atoi(e);
        if (v >= 1) c = v;
    }
    g.nchunk = std::min(std::max(c, 1), nz);
    return g;
}

// Host: geometry of the pair-march kernels -- 64 x kPairRows tiles, z cut into
// chunks by wave_chunks (8 resident 128-thread CTAs per SM, >= 4 planes per
// chunk; measured 256^3: 9 chunks 2304 CTAs = 0.97 of two waves, vs 8 chunks
// 207 -> 203 us per CG iteration; 5 chunks = 1280 CTAs, 1.08 waves, 240 us).
// env_name overrides the chunk count.
PairGeom pair_geom(int nx, int ny, int nz, int lo_halo, int hi_halo, const char *env_name)
{
    PairGeom g{nx, ny, nz, lo_halo, hi_halo, (nx + kPairX - 1) / kPairX, (ny + kPairRows - 1) / kPairRows, 1};
    const int tiles = g.ntx * g.nty;
    int c = wave_chunks(tiles, nz, (long long)num_sms() * 8, 4);
    if (const char *e = env_name ? getenv(env_name) : nullptr) {
        const int v = atoi(e);
        if (v >= 1) c = v;
    }
    g.nchunk = c < 1 ? 1 : (c > nz ? nz : c);
    return g;
}

// Host: geometry of the lean kernels -- 64 x rows tiles (rows warps per CTA),
// z chunks by wave_chunks over the resident CTAs (ctas4: resident 4-row CTAs
// per SM; the register budget is per thread, so CTAs scale as 4 / rows).
PairGeom lean_geom(int nx, int ny, int nz, int rows, int ctas4)
{
    PairGeom g{nx, ny, nz, 0, 0, (nx + kPairX - 1) / kPairX, (ny + rows - 1) / rows, 1};
    const long long slots = (long long)num_sms() * std::max(1, ctas4 * kPairRows / rows);
    g.nchunk = wave_chunks((long long)g.ntx * g.nty, nz, slots, 4);
    if (const char *e = getenv("CF_LEAN_CHUNKS")) {
        const int v = atoi(e);
        if (v >= 1 && v <= nz) g.nchunk = v;
    }
    return g;
}

// Which form runs each CG kernel: the lean register march (cf_cg_lean.cuh),
// the pair march, the TMA pipeline, or the scalar LDG march (odd nx).
// Defaults (measured, tools/gpu_lean.sh, 256^3 / 512^3): direction = lean
// march run top-down (8-row CTAs), update = TMA -- 193 / 1425 us per
// iteration against 207 / 1525 with the pair-march direction kernel and
// 198 / 1460 with the lean update kernel.
// CF_CG_DIR / CF_CG_UPD = "lean" | "pair" | "tma" | "ldg" override.
enum KernKind { KK_LDG = 0, KK_TMA = 1, KK_PAIR = 2, KK_LEAN = 3 };
int kern_kind(const char *env_name, int deflt, bool tma_ok, bool pair_ok)
{
    int k = deflt;
    if (const char *e = getenv(env_name)) {
        if (!strcmp(e, "pair")) k = KK_PAIR;
        else if (!strcmp(e, "tma")) k = KK_TMA;
        else if (!strcmp(e, "ldg")) k = KK_LDG;
        else if (!strcmp(e, "lean")) k = KK_LEAN;
    }
    if (k == KK_LEAN && !pair_ok) k = KK_LDG;
    if (k == KK_TMA && !tma_ok) k = pair_ok ? KK_PAIR : KK_LDG;
    if (k == KK_PAIR && !pair_ok) k = KK_LDG;
    return k;
}

// ---------------------------------------------------------------- small grids
// Whole solve in ONE block: r, p, x live in shared memory (16^3: 96 KB), the
// two grid-wide reductions per iteration become block reductions, and a
// solve is a single launch -- the latency-bound regime of BASELINE config 1,
// where the grid kernels cost ~19 us per iteration in launch/sync overhead.
// Same per-element arithmetic and stop rule as the fused grid kernels.
constexpr int kSmallThreads = 1024;
constexpr long long kSmallMaxCells = 5120;  // 3 vectors <= 120 KB of shared memory

template <int ORDER>
__device__ __forceinline__ double small_ap(const double *v, int c, const Box &bx, double off, double diag)
{
    const int nx = bx.nx, ny = bx.ny;
    const int i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
    const int pl = nx * ny;
    const bool hxm = i > 0, hxp = i < nx - 1, hym = j > 0, hyp = j < ny - 1, hzm = k > 0, hzp = k < bx.nz - 1;
    return stencil7<ORDER>(v[c], hxm ? v[c - 1] : 0.0, hxp ? v[c + 1] : 0.0, hym ? v[c - nx] : 0.0,
                           hyp ? v[c + nx] : 0.0, hzm ? v[c - pl] : 0.0, hzp ? v[c + pl] : 0.0, hxm, hxp, hym, hyp,
                           hzm, hzp, off, diag);
}

// block_sum (cf_common.cuh) whose result every thread receives, in ONE
// barrier: every warp repeats warp 0's final tree over the per-warp partials
// (the same operations in the same order, so the same bits), then broadcasts
// lane 0.  buf must not be reused before every thread has passed the next
// barrier (the callers rotate buffers).
template <int NT>
__device__ __forceinline__ double block_sum_all(double v, double *buf)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = NT / 32;
    if (lane == 0) buf[wid] = v;
    __syncthreads();
    v = lane < NW ? buf[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return __shfl_sync(0xffffffffu, v, 0);
}

// a cell's existing-neighbour mask (bit 0..5: x-, x+, y-, y+, z-, z+)
__device__ __forceinline__ int small_mask(int c, const Box &bx)
{
    const int nx = bx.nx, ny = bx.ny;
    const int i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
    return (i > 0) | (i < nx - 1) << 1 | (j > 0) << 2 | (j < ny - 1) << 3 | (k > 0) << 4 | (k < bx.nz - 1) << 5;
}

template <int ORDER>
__device__ __forceinline__ double small_ap_m(const double *v, int c, int m, int nx, int pl, double off, double diag)
{
    const bool hxm = m & 1, hxp = m & 2, hym = m & 4, hyp = m & 8, hzm = m & 16, hzp = m & 32;
    return stencil7<ORDER>(v[c], hxm ? v[c - 1] : 0.0, hxp ? v[c + 1] : 0.0, hym ? v[c - nx] : 0.0,
                           hyp ? v[c + nx] : 0.0, hzm ? v[c - pl] : 0.0, hzp ? v[c + pl] : 0.0, hxm, hxp, hym, hyp,
                           hzm, hzp, off, diag);
}

// Per iteration: p update | barrier | A p kept in registers, p.Ap (one
// barrier) | r, x from the kept A p, r.r and r.z (one barrier) -- three
// barriers instead of nine, each cell's neighbour mask computed once per
// solve and A p evaluated once (the same values: bit-identical).
constexpr int kSmallPer = (int)((kSmallMaxCells + kSmallThreads - 1) / kSmallThreads);

template <int ORDER, int PK>
__global__ void __launch_bounds__(kSmallThreads) cg_small_kernel(Box bx, double off, double diag,
                                                                 const double *__restrict__ b,
                                                                 const double *__restrict__ x0, double *__restrict__ xout,
                                                                 const double *__restrict__ jd, double zc, CgScalars *sc)
{
    extern __shared__ double sm[];
    __shared__ double red[32];
    __shared__ double rbuf[3][32];  // rotating broadcast-reduction buffers
    __shared__ double bc[2];
    const int n = (int)bx.cells();
    double *r = sm, *p = sm + n, *x = sm + 2 * n;
    const int t = threadIdx.x;
    const int nx = bx.nx, pl = bx.nx * bx.ny;
    // r = b (or b - A x0), x = 0 (or x0); |b|^2 and r.z  (src/solver.py:60-61, :130-143)
    for (int c = t; c < n; c += kSmallThreads) x[c] = x0 ? x0[c] : 0.0;
    __syncthreads();
    double bb = 0.0, rz = 0.0;
    for (int c = t; c < n; c += kSmallThreads) {
        const double bi = b[c];
        const double rn = x0 ? bi + -1.0 * small_ap<ORDER>(x, c, bx, off, diag) : bi;
        r[c] = rn;
        bb = bb + bi * bi;
        rz = rz + rn * zval<PK>(rn, jd, c, zc);
    }
    bb = block_sum<kSmallThreads>(bb, red);
    rz = block_sum<kSmallThreads>(rz, red);
    if (t == 0) {
        bc[0] = bb;
        bc[1] = rz;
    }
    __syncthreads();
    CgScalars s = *sc;  // tol, max_iter from the host
    scalar_after_init(&s, bc[0], bc[1]);
    int mask[kSmallPer];
    double ap[kSmallPer];
#pragma unroll
    for (int q = 0; q < kSmallPer; ++q) {
        const int c = t + q * kSmallThreads;
        mask[q] = c < n ? small_mask(c, bx) : 0;
    }
    while (!s.done) {
        // p = z + beta p (in place: each element depends on itself only)
#pragma unroll
        for (int q = 0; q < kSmallPer; ++q) {
            const int c = t + q * kSmallThreads;
            if (c < n) {
                const double z = zval<PK>(r[c], jd, c, zc);
                p[c] = s.it == 0 ? z : z + s.beta * p[c];
            }
        }
        __syncthreads();
        double pap = 0.0;
#pragma unroll
        for (int q = 0; q < kSmallPer; ++q) {
            const int c = t + q * kSmallThreads;
            if (c < n) {
                ap[q] = small_ap_m<ORDER>(p, c, mask[q], nx, pl, off, diag);
                pap = pap + p[c] * ap[q];
            }
        }
        pap = block_sum_all<kSmallThreads>(pap, rbuf[0]);
        scalar_after_dir(&s, pap);
        if (s.done) break;
        const double alpha = s.alpha, malpha = -alpha;
        double rr = 0.0;
        rz = 0.0;
#pragma unroll
        for (int q = 0; q < kSmallPer; ++q) {
            const int c = t + q * kSmallThreads;
            if (c < n) {
                const double pc = p[c];
                x[c] = x[c] + alpha * pc;
                const double rn = r[c] + malpha * ap[q];
                r[c] = rn;
                rr = rr + rn * rn;
                rz = rz + rn * zval<PK>(rn, jd, c, zc);
            }
        }
        rr = block_sum_all<kSmallThreads>(rr, rbuf[1]);
        rz = block_sum_all<kSmallThreads>(rz, rbuf[2]);
        scalar_after_update<true>(&s, rr, rz);
    }
    __syncthreads();
    for (int c = t; c < n; c += kSmallThreads) xout[c] = x[c];
    if (t == 0) *sc = s;
}

// Small grids with the simplified-DIC preconditioner (the reference's
// default, src/sim.py:65): the whole solve in one block as above, the DIC
// sweeps (src/precond.py:38-54) level by level (i+j+k = const) between block
// barriers -- on the 7-point pattern verified at attach (one lower and one
// upper value), every row in the reference's operand order.
constexpr long long kSmallDicMaxCells = 5120;  // r, p, x, w, z: 200 KB of shared memory

__device__ __forceinline__ void small_dic_apply(const double *r, double *w, double *z, const double *__restrict__ d,
                                                const int32_t *__restrict__ rows,
                                                const long long *__restrict__ lptr, int nlev, const Box &bx,
                                                double lval, double uval)
{
    const int nx = bx.nx, ny = bx.ny, nz = bx.nz, pl = nx * ny;
    for (int L = 0; L < nlev; ++L) {  // (L + D~) w = r
        for (long long q = lptr[L] + threadIdx.x; q < lptr[L + 1]; q += kSmallThreads) {
            const int c = rows[q];
            const int i = c % nx, j = (c / nx) % ny, k = c / pl;
            double acc = r[c];
            if (k > 0) acc = acc - lval * w[c - pl];
            if (j > 0) acc = acc - lval * w[c - nx];
            if (i > 0) acc = acc - lval * w[c - 1];
            w[c] = acc / d[c];
        }
        __syncthreads();
    }
    for (int L = nlev - 1; L >= 0; --L) {  // (D~ + L^T) z = D~ w
        for (long long q = lptr[L] + threadIdx.x; q < lptr[L + 1]; q += kSmallThreads) {
            const int c = rows[q];
            const int i = c % nx, j = (c / nx) % ny, k = c / pl;
            double acc = 0.0;
            if (i < nx - 1) acc = acc + uval * z[c + 1];
            if (j < ny - 1) acc = acc + uval * z[c + nx];
            if (k < nz - 1) acc = acc + uval * z[c + pl];
            z[c] = w[c] - acc / d[c];
        }
        __syncthreads();
    }
}

template <int ORDER>
__global__ void __launch_bounds__(kSmallThreads) cg_small_dic_kernel(Box bx, double off, double diag,
                                                                     const double *__restrict__ b,
                                                                     double *__restrict__ xout,
                                                                     const double *__restrict__ d,
                                                                     const int32_t *__restrict__ rows,
                                                                     const long long *__restrict__ lptr, int nlev,
                                                                     double lval, double uval, CgScalars *sc)
{
    extern __shared__ double sm[];
    __shared__ double red[32];
    __shared__ double bc[2];
    const int n = (int)bx.cells();
    double *r = sm, *p = sm + n, *x = sm + 2 * n, *w = sm + 3 * n, *z = sm + 4 * n;
    const int t = threadIdx.x;
    double bb = 0.0;
    for (int c = t; c < n; c += kSmallThreads) {  // r = b, x = 0 (src/solver.py:130-140)
        const double bi = b[c];
        r[c] = bi;
        x[c] = 0.0;
        bb = bb + bi * bi;
    }
    __syncthreads();
    small_dic_apply(r, w, z, d, rows, lptr, nlev, bx, lval, uval);  // z = M^-1 r (:141)
    double rz = 0.0;
    for (int c = t; c < n; c += kSmallThreads) rz = rz + r[c] * z[c];
    bb = block_sum<kSmallThreads>(bb, red);
    rz = block_sum<kSmallThreads>(rz, red);
    if (t == 0) {
        bc[0] = bb;
        bc[1] = rz;
    }
    __syncthreads();
    CgScalars s = *sc;
    scalar_after_init(&s, bc[0], bc[1]);
    while (!s.done) {
        for (int c = t; c < n; c += kSmallThreads) p[c] = s.it == 0 ? z[c] : z[c] + s.beta * p[c];
        __syncthreads();
        double pap = 0.0;
        for (int c = t; c < n; c += kSmallThreads) pap = pap + p[c] * small_ap<ORDER>(p, c, bx, off, diag);
        pap = block_sum<kSmallThreads>(pap, red);
        if (t == 0) bc[0] = pap;
        __syncthreads();
        scalar_after_dir(&s, bc[0]);
        if (s.done) break;
        const double alpha = s.alpha, malpha = -alpha;
        double rr = 0.0;
        for (int c = t; c < n; c += kSmallThreads) {
            const double pc = p[c];
            x[c] = x[c] + alpha * pc;
            const double rn = r[c] + malpha * small_ap<ORDER>(p, c, bx, off, diag);
            r[c] = rn;
            rr = rr + rn * rn;
        }
        __syncthreads();
        // z = M^-1 r and r.z before the stop test's beta (src/solver.py:163-166)
        small_dic_apply(r, w, z, d, rows, lptr, nlev, bx, lval, uval);
        rz = 0.0;
        for (int c = t; c < n; c += kSmallThreads) rz = rz + r[c] * z[c];
        rr = block_sum<kSmallThreads>(rr, red);
        rz = block_sum<kSmallThreads>(rz, red);
        if (t == 0) {
            bc[0] = rr;
            bc[1] = rz;
        }
        __syncthreads();
        scalar_after_update<true>(&s, bc[0], bc[1]);
    }
    for (int c = t; c < n; c += kSmallThreads) xout[c] = x[c];
    if (t == 0) *sc = s;
}

}  // namespace cf

// ---------------------------------------------------------------- workspace
struct cf_cg {
    cf::Box bx;
    double h, off, diag;
    int order;
    long long n;
    double *r = nullptr, *x = nullptr, *p[2] = {nullptr, nullptr}, *jd = nullptr;
    double *partials = nullptr;
    cf::CgScalars *sc = nullptr;
    cf::CgScalars *sc_host = nullptr;
    cf::CgTickets *tk = nullptr;
    int grid_init = 1, grid_init_x0 = 1, grid_dir = 1, grid_upd = 1;
    // DIC (CF_PRECOND_DIC): level-scheduled factor attached by cf_cg_set_dic
    bool has_dic = false;
    cf::DicData dic;
    long long *dic_lptr = nullptr;  // device copy of the level pointers (small-grid DIC kernel)
    double *zbuf = nullptr, *wbuf = nullptr;
    // CF_CG_DIRECT=<batch> in the environment: host-driven loop instead of
    // the conditional graph (ncu cannot profile conditional-graph kernels)
    int direct = 0, direct_batch = 8;
    // TMA-staged kernels (even nx >= 32; CF_NO_TMA=1 forces the LDG march)
    bool tma = false;
    // kernel form per CG kernel (cf::KernKind) and the pair-march geometry
    int kind_dir = 0, kind_upd = 0, kind_upd_skip = -1;
    // pair-march direction kernel with the next plane's loads issued one
    // iteration early (cf_cg_pair.cuh PF); CF_PAIR_PF=0/1 overrides
    int pair_pf = 0;
    // lean kernels (cf_cg_lean.cuh): warps (tile rows) per CTA, CF_LEAN_ROWS
    int lean_rows = 16;  // with lean2: 8 warps x 2 rows (measured +0.4 % over 8-row tiles in the sustained bench)
    // TMA ring depth of the skip-x update kernel (3 = the shared layout; CF_SKIP_STAGES=4/6)
    int double_stages = 4;  // double-x update ring depth: 4 (70 KB, 3 CTAs/SM, own geometry; within noise of 3 in the sustained bench; CF_DOUBLE_STAGES=3)
    int skip_stages = 4;
    // persistent single-launch solve for L2-resident grids (cf_cg_persist.cuh; CF_PERSIST=0/1)
    bool persist = false;
    cf::PairGeom per_g{};
    int per_blocks = 0;
    double *per_part = nullptr;
    cf::GridBar *per_bar = nullptr;  // measured 3 / 4 / 6: 192.6 / 191.7 / 192.3 us (256^3), 1403 / 1389 / 1396 (512^3)
    // programmatic dependent launch between the loop kernels (CF_PDL)
    bool pdl = false;
    bool lean2 = true;  // two-rows-per-warp direction march (CF_LEAN2=0: one row per warp); +0.5 % in the sustained bench
    cf::PairGeom lg_dir{}, lg_upd{};
    cf::PairGeom pg_dir{}, pg_upd{};
    cf::TmaGeom geom_dir{}, geom_upd{}, geom_dbl{};  // geom_dbl: the 4-deep double-x update (3 CTAs/SM)
    CUtensorMap m_r{}, m_z{}, m_p[2]{}, m_ri{}, m_xi{}, m_pi[2]{};
    // x updated once per two iterations (XM_SKIP / XM_DOUBLE, cf_cg_common.cuh)
    bool defer_x = false;
    // single-reduction CG (cf_cg_pass.cuh): one kernel per iteration; r ping-pongs
    bool pass = false;
    cf::PassGeom pass_g{};
    // lean pass kernel (cf_cg_lpass.cuh; CF_PASS_FORM=old selects cg_pass_kernel)
    int pass_form = 1;  // 0 cg_pass_kernel, 1 / 2 cg_lpass_kernel with 8 / 16-row tiles (CF_PASS_FORM=old|lean|lean16)
    cf::PairGeom lpass_g{};
    double *r2 = nullptr;
    // TMA-fed single-reduction pass (cf_cg_spass.cuh): one kernel per
    // iteration, 40 N; r ping-pongs with r2, x updated every second pass
    bool spass = false;
    int sp_ty = 16;  // tile height: 16 (one CTA per SM) or 8 (two; form 1 only)
    int sp_form = 2;  // 2: two rows per warp, SoA planes; 1: one row per warp (CF_SPASS_FORM=1)
    int *sp_perm = nullptr;  // device tile permutation of the phase-aligned schedule
    cf::SpGeom sp_g{};
    int sp_ctas = 0;
    CUtensorMap m_spr[2]{}, m_spp[2]{}, m_spx{};
    cudaGraphExec_t exec_pass[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaGraph_t graph_pass[4] = {nullptr, nullptr, nullptr, nullptr};
    double zc_pass[4] = {0, 0, 0, 0};
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    float last_loop_ms = 0.f;
    // the form the last solve ran (CF_CG_FORM_*) and its kernel launches
    int last_form = 0;
    long long last_launches = 0;
    bool last_x0 = false;
    // one instantiated while-graph per (preconditioner kind)
    cudaGraphExec_t exec[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaGraph_t graph[4] = {nullptr, nullptr, nullptr, nullptr};
    double zc_graph[4] = {0, 0, 0, 0};
    std::mutex mu;
};

namespace cf {

// Launch with the PDL attribute when the workspace enables it (the kernels call
// griddep_enter() first, so they are correct either way).
template <typename... K, typename... A>
static void launch_k(const cf_cg *ws, void (*kern)(K...), int grid, int block, size_t smem, cudaStream_t s,
                     A &&...args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = ws->pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}

template <int ORDER, int PK, int PF, int ROWS>
static void dir_lean_go(cf_cg *ws, cudaStream_t s, const double *zs, const double *po, double *pn, double zc)
{
    launch_k(ws, cg_dir_lean<ORDER, PK, PF, ROWS>, ws->lg_dir.ctas(), 32 * ROWS, 0, s, ws->lg_dir, ws->off, ws->diag,
             zs, po, pn, zc, ws->sc, ws->partials, ws->tk);
}

template <int ORDER, int PK>
static void dir_lean_launch(cf_cg *ws, cudaStream_t s, const double *zs, const double *po, double *pn, double zc)
{
    // the geometry (lg_dir) is built for lean_rows; PF variants exist for 4 / 8 rows
    if (ws->lean2 && ws->lean_rows == 8) {  // two rows per warp: 4 warps cover the 8-row tile
        launch_k(ws, cg_dir_lean2<ORDER, PK, 4>, ws->lg_dir.ctas(), 128, 0, s, ws->lg_dir, ws->off, ws->diag, zs, po,
                 pn, zc, ws->sc, ws->partials, ws->tk);
        return;
    }
    if (ws->lean2 && ws->lean_rows == 16) {  // 8 warps x 2 rows
        launch_k(ws, cg_dir_lean2<ORDER, PK, 8>, ws->lg_dir.ctas(), 256, 0, s, ws->lg_dir, ws->off, ws->diag, zs, po,
                 pn, zc, ws->sc, ws->partials, ws->tk);
        return;
    }
    const int pf = ws->lean_rows == 16 ? 0 : ws->pair_pf;
    if (ws->lean_rows == 16) dir_lean_go<ORDER, PK, 0, 16>(ws, s, zs, po, pn, zc);
    else if (ws->lean_rows == 8 && pf == 1) dir_lean_go<ORDER, PK, 1, 8>(ws, s, zs, po, pn, zc);
    else if (ws->lean_rows == 8 && pf == 2) dir_lean_go<ORDER, PK, 2, 8>(ws, s, zs, po, pn, zc);
    else if (ws->lean_rows == 8) dir_lean_go<ORDER, PK, 0, 8>(ws, s, zs, po, pn, zc);
    else if (pf == 1) dir_lean_go<ORDER, PK, 1, 4>(ws, s, zs, po, pn, zc);
    else if (pf == 2) dir_lean_go<ORDER, PK, 2, 4>(ws, s, zs, po, pn, zc);
    else dir_lean_go<ORDER, PK, 0, 4>(ws, s, zs, po, pn, zc);
}

template <int ORDER, int PK, int XM, int ROWS>
static void upd_lean_go(cf_cg *ws, cudaStream_t s, const double *p, const double *q, double zc, int use_cond,
                        cudaGraphConditionalHandle cond)
{
    launch_k(ws, cg_update_lean<ORDER, PK, XM, ROWS>, ws->lg_upd.ctas(), 32 * ROWS, 0, s, ws->lg_upd, ws->off,
             ws->diag, p, q, ws->r, ws->x, zc, ws->sc, ws->partials, ws->tk, use_cond, cond);
}

template <int ORDER, int PK, int XM>
static void upd_lean_launch(cf_cg *ws, cudaStream_t s, const double *p, const double *q, double zc, int use_cond,
                            cudaGraphConditionalHandle cond)
{
    if (ws->lean_rows == 8) upd_lean_go<ORDER, PK, XM, 8>(ws, s, p, q, zc, use_cond, cond);
    else if (ws->lean_rows == 16) upd_lean_go<ORDER, PK, XM, 16>(ws, s, p, q, zc, use_cond, cond);
    else upd_lean_go<ORDER, PK, XM, 4>(ws, s, p, q, zc, use_cond, cond);
}

template <int ORDER, int PK>
static int capture_body(cf_cg *ws, cudaStream_t s, double zc, cudaGraphConditionalHandle cond, int use_cond = 1)
{
    for (int half = 0; half < 2; ++half) {
        const double *p_old = ws->p[half];
        double *p_new = ws->p[half ^ 1];
        // the TMA forms have no per-cell Jacobi vector
        // the TMA and lean forms have no per-cell Jacobi vector
        const int kd = (PK == PK_JVEC && (ws->kind_dir == KK_TMA || ws->kind_dir == KK_LEAN)) ? KK_PAIR : ws->kind_dir;
        int ku = (PK == PK_JVEC && (ws->kind_upd == KK_TMA || ws->kind_upd == KK_LEAN)) ? KK_PAIR : ws->kind_upd;
        if (half == 0 && ws->defer_x && ws->kind_upd_skip >= 0)  // tuning override (no per-cell Jacobi in TMA / lean forms)
            ku = (PK == PK_JVEC && ws->kind_upd_skip != KK_PAIR && ws->kind_upd_skip != KK_LDG) ? KK_PAIR : ws->kind_upd_skip;
        if (kd == KK_TMA) {
            const TmaGeom &gd = ws->geom_dir;
            cg_dir_tma<ORDER, PK><<<gd.ntx * gd.nty * gd.nchunk, kWSThreads, kDirSmem, s>>>(
                PK == PK_ZVEC ? ws->m_z : ws->m_r, ws->m_p[half], gd, ws->off, ws->diag, p_new, zc, ws->sc,
                ws->partials, ws->tk, nullptr);
            CF_CHECK_LAUNCH("cg_dir_tma");
        } else if (kd == KK_LEAN) {
            dir_lean_launch<ORDER, PK>(ws, s, PK == PK_ZVEC ? ws->zbuf : ws->r, p_old, p_new, zc);
            CF_CHECK_LAUNCH("cg_dir_lean");
        } else if (kd == KK_PAIR) {
            if (ws->pair_pf)
                cg_dir_pair<ORDER, PK, true><<<ws->pg_dir.ctas(), kPairThreads, 0, s>>>(
                    ws->pg_dir, ws->off, ws->diag, PK == PK_ZVEC ? ws->zbuf : ws->r, ws->jd, p_old, p_new, zc, ws->sc,
                    ws->partials, ws->tk, nullptr);
            else
                cg_dir_pair<ORDER, PK><<<ws->pg_dir.ctas(), kPairThreads, 0, s>>>(
                    ws->pg_dir, ws->off, ws->diag, PK == PK_ZVEC ? ws->zbuf : ws->r, ws->jd, p_old, p_new, zc, ws->sc,
                    ws->partials, ws->tk, nullptr);
            CF_CHECK_LAUNCH("cg_dir_pair");
        } else {
            cg_dir_kernel<ORDER, PK><<<ws->grid_dir, kMarchThreads, 0, s>>>(
                ws->bx, ws->off, ws->diag, ws->r, ws->jd, ws->zbuf, p_old, p_new, zc, ws->sc, ws->partials,
                ws->tk);
            CF_CHECK_LAUNCH("cg_dir_kernel");
        }
        if (ku == KK_TMA) {
            const TmaGeom &gu = ws->geom_upd;
            const int nb = gu.ntx * gu.nty * gu.nchunk;
            if (!ws->defer_x)
                launch_k(ws, cg_update_tma<ORDER, PK, XM_EACH>, nb, kWSThreads, kUpdSmem, s, ws->m_p[half ^ 1], ws->m_ri,
                         ws->m_xi, ws->m_pi[half], gu, ws->off, ws->diag, ws->r, ws->x, zc, ws->sc, ws->partials,
                         ws->tk, use_cond, cond, (double *)nullptr);
            else if (half == 0 && ws->skip_stages == 4)
                launch_k(ws, cg_update_tma<ORDER, PK, XM_SKIP, 4>, nb, kWSThreads, upd_skip_smem<4>(), s,
                         ws->m_p[half ^ 1], ws->m_ri, ws->m_xi, ws->m_pi[half], gu, ws->off, ws->diag, ws->r, ws->x,
                         zc, ws->sc, ws->partials, ws->tk, use_cond, cond, (double *)nullptr);
            else if (half == 0 && ws->skip_stages == 6)
                launch_k(ws, cg_update_tma<ORDER, PK, XM_SKIP, 6>, nb, kWSThreads, upd_skip_smem<6>(), s,
                         ws->m_p[half ^ 1], ws->m_ri, ws->m_xi, ws->m_pi[half], gu, ws->off, ws->diag, ws->r, ws->x,
                         zc, ws->sc, ws->partials, ws->tk, use_cond, cond, (double *)nullptr);
            else if (half == 0)
                launch_k(ws, cg_update_tma<ORDER, PK, XM_SKIP>, nb, kWSThreads, kUpdSmem, s, ws->m_p[half ^ 1], ws->m_ri,
                         ws->m_xi, ws->m_pi[half], gu, ws->off, ws->diag, ws->r, ws->x, zc, ws->sc, ws->partials,
                         ws->tk, use_cond, cond, (double *)nullptr);
            else if (ws->double_stages == 4)
                launch_k(ws, cg_update_tma<ORDER, PK, XM_DOUBLE, 4>, ws->geom_dbl.ntx * ws->geom_dbl.nty * ws->geom_dbl.nchunk,
                         kWSThreads, upd_full_smem<4>(), s, ws->m_p[half ^ 1], ws->m_ri, ws->m_xi, ws->m_pi[half],
                         ws->geom_dbl, ws->off, ws->diag, ws->r, ws->x, zc, ws->sc, ws->partials, ws->tk, use_cond,
                         cond, (double *)nullptr);
            else
                launch_k(ws, cg_update_tma<ORDER, PK, XM_DOUBLE>, nb, kWSThreads, kUpdSmem, s, ws->m_p[half ^ 1], ws->m_ri,
                         ws->m_xi, ws->m_pi[half], gu, ws->off, ws->diag, ws->r, ws->x, zc, ws->sc, ws->partials,
                         ws->tk, use_cond, cond, (double *)nullptr);
            CF_CHECK_LAUNCH("cg_update_tma");
        } else if (ku == KK_LEAN) {
            if (!ws->defer_x) upd_lean_launch<ORDER, PK, XM_EACH>(ws, s, p_new, p_old, zc, use_cond, cond);
            else if (half == 0) upd_lean_launch<ORDER, PK, XM_SKIP>(ws, s, p_new, p_old, zc, use_cond, cond);
            else upd_lean_launch<ORDER, PK, XM_DOUBLE>(ws, s, p_new, p_old, zc, use_cond, cond);
            CF_CHECK_LAUNCH("cg_update_lean");
        } else if (ku == KK_PAIR) {
            const int nb = ws->pg_upd.ctas();
            if (!ws->defer_x)
                cg_update_pair<ORDER, PK, XM_EACH><<<nb, kPairThreads, 0, s>>>(
                    ws->pg_upd, ws->off, ws->diag, p_new, p_old, ws->r, ws->x, ws->jd, zc, ws->sc, ws->partials,
                    ws->tk, use_cond, cond, nullptr);
            else if (half == 0)
                cg_update_pair<ORDER, PK, XM_SKIP><<<nb, kPairThreads, 0, s>>>(
                    ws->pg_upd, ws->off, ws->diag, p_new, p_old, ws->r, ws->x, ws->jd, zc, ws->sc, ws->partials,
                    ws->tk, use_cond, cond, nullptr);
            else
                cg_update_pair<ORDER, PK, XM_DOUBLE><<<nb, kPairThreads, 0, s>>>(
                    ws->pg_upd, ws->off, ws->diag, p_new, p_old, ws->r, ws->x, ws->jd, zc, ws->sc, ws->partials,
                    ws->tk, use_cond, cond, nullptr);
            CF_CHECK_LAUNCH("cg_update_pair");
        } else {
            cg_update_kernel<ORDER, PK><<<ws->grid_upd, kMarchThreads, 0, s>>>(
                ws->bx, ws->off, ws->diag, p_new, ws->r, ws->x, ws->jd, zc, ws->sc, ws->partials, ws->tk, use_cond,
                cond);
            CF_CHECK_LAUNCH("cg_update_kernel");
        }
        if (PK == PK_ZVEC) {
            // z = M^-1 r by the level sweeps, then r.z and beta (src/solver.py:163-166)
            int rc = ws->dic.wave.ok ? dic_wave_apply(ws->dic, ws->r, ws->wbuf, ws->zbuf, &ws->sc->done, s)
                                     : dic_apply_launch(ws->dic, ws->r, ws->wbuf, ws->zbuf, &ws->sc->done, s);
            if (rc != CF_OK) return rc;
            cg_rz_kernel<<<ws->grid_init, kMarchThreads, 0, s>>>(ws->n, ws->r, ws->zbuf, ws->sc, ws->partials,
                                                                 ws->tk, 1);
            CF_CHECK_LAUNCH("cg_rz_kernel");
        }
    }
    return CF_OK;
}

template <int ORDER, int PK>
static int build_graph(cf_cg *ws, cudaStream_t s, double zc)
{
    cudaGraph_t g;
    CF_CUDA(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle cond;
    CF_CUDA(cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CF_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    // capture the body on a private stream (capture-to-graph)
    cudaStream_t cs;
    CF_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CF_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    int rc = capture_body<ORDER, PK>(ws, cs, zc, cond);
    cudaGraph_t captured;
    cudaError_t e = cudaStreamEndCapture(cs, &captured);
    cudaStreamDestroy(cs);
    if (rc != CF_OK) return rc;
    CF_CUDA(e);
    if (ws->defer_x) {  // x += alpha * p owed by a final skipping iteration
        cudaKernelNodeParams kp = {};
        void *args[] = {&ws->n, &ws->x, &ws->p[1], &ws->sc};
        kp.func = (void *)cg_x_fixup;
        kp.gridDim = dim3(ws->grid_init);
        kp.blockDim = dim3(kMarchThreads);
        kp.kernelParams = args;
        cudaGraphNode_t fix;
        CF_CUDA(cudaGraphAddKernelNode(&fix, g, &node, 1, &kp));
    }
    cudaGraphExec_t exec;
    CF_CUDA(cudaGraphInstantiate(&exec, g, 0));
    ws->graph[PK] = g;
    ws->exec[PK] = exec;
    ws->zc_graph[PK] = zc;
    (void)s;
    return CF_OK;
}

template <int ORDER, int PK>
static int launch_init(cf_cg *ws, const double *b, const double *x0, double zc, cudaStream_t s)
{
    // for DIC the init pass computes r and |b| (its r.z is replaced below)
    constexpr int IPK = PK == PK_ZVEC ? PK_NONE : PK;
    if (x0) {
        cg_init_x0<ORDER, IPK><<<ws->grid_init_x0, kMarchThreads, 0, s>>>(
            ws->bx, ws->off, ws->diag, b, x0, ws->r, ws->x, ws->jd, zc, ws->sc, ws->partials, ws->tk);
    } else {
        cg_init_flat<IPK><<<ws->grid_init, kMarchThreads, 0, s>>>(ws->n, b, ws->r, ws->x, ws->jd, zc,
                                                                  ws->sc, ws->partials, ws->tk);
    }
    CF_CHECK_LAUNCH("cg_init");
    if (PK == PK_ZVEC) {  // z = M^-1 r, rz = r.z (src/solver.py:141-143)
        int rc = ws->dic.wave.ok ? dic_wave_apply(ws->dic, ws->r, ws->wbuf, ws->zbuf, &ws->sc->done, s)
                                 : dic_apply_launch(ws->dic, ws->r, ws->wbuf, ws->zbuf, &ws->sc->done, s);
        if (rc != CF_OK) return rc;
        cg_rz_kernel<<<ws->grid_init, kMarchThreads, 0, s>>>(ws->n, ws->r, ws->zbuf, ws->sc, ws->partials, ws->tk,
                                                             0);
        CF_CHECK_LAUNCH("cg_rz_kernel");
    }
    return CF_OK;
}

template <int ORDER, int PK>
static int pass_body(cf_cg *ws, cudaStream_t s, double zc, cudaGraphConditionalHandle cond, int use_cond)
{
    const PassGeom &g = ws->pass_g;
    for (int half = 0; half < 2; ++half) {
        const double *r_in = half ? ws->r2 : ws->r;
        double *r_out = half ? ws->r : ws->r2;
        if (ws->pass_form == 2) {
            cg_lpass_kernel<ORDER, PK, 16><<<ws->lpass_g.ctas(), Lp<16>::Threads, Lp<16>::Smem, s>>>(
                ws->lpass_g, ws->off, ws->diag, zc, r_in, r_out, ws->p[half], ws->p[half ^ 1], ws->x, ws->sc,
                ws->partials, ws->tk, use_cond, cond);
            CF_CHECK_LAUNCH("cg_lpass_kernel");
            continue;
        }
        if (ws->pass_form == 1) {
            cg_lpass_kernel<ORDER, PK, 8><<<ws->lpass_g.ctas(), Lp<8>::Threads, Lp<8>::Smem, s>>>(
                ws->lpass_g, ws->off, ws->diag, zc, r_in, r_out, ws->p[half], ws->p[half ^ 1], ws->x, ws->sc,
                ws->partials, ws->tk, use_cond, cond);
            CF_CHECK_LAUNCH("cg_lpass_kernel");
            continue;
        }
        cg_pass_kernel<ORDER, PK><<<g.ctas(), kPassThreads, kPassSmem, s>>>(
            g, ws->off, ws->diag, zc, r_in, r_out, ws->p[half], ws->p[half ^ 1], ws->x, ws->sc, ws->partials, ws->tk,
            use_cond, cond);
        CF_CHECK_LAUNCH("cg_pass_kernel");
    }
    return CF_OK;
}

template <int ORDER, int PK>
static int pass_build_graph(cf_cg *ws, double zc)
{
    cudaGraph_t g;
    CF_CUDA(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle cond;
    CF_CUDA(cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CF_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &np));
    cudaStream_t cs;
    CF_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CF_CUDA(cudaStreamBeginCaptureToGraph(cs, np.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                          cudaStreamCaptureModeRelaxed));
    int rc = pass_body<ORDER, PK>(ws, cs, zc, cond, 1);
    cudaGraph_t captured;
    cudaError_t e = cudaStreamEndCapture(cs, &captured);
    cudaStreamDestroy(cs);
    if (rc != CF_OK) return rc;
    CF_CUDA(e);
    cudaGraphExec_t exec;
    CF_CUDA(cudaGraphInstantiate(&exec, g, 0));
    ws->graph_pass[PK] = g;
    ws->exec_pass[PK] = exec;
    ws->zc_pass[PK] = zc;
    return CF_OK;
}

template <int ORDER, int PK>
static int pass_solve(cf_cg *ws, const double *b, double zc, cudaStream_t s)
{
    cg_pass_init<ORDER, PK><<<ws->pg_upd.ctas(), kPairThreads, 0, s>>>(ws->pg_upd, ws->off, ws->diag, zc, b, ws->r,
                                                                       ws->x, ws->sc, ws->partials, ws->tk);
    CF_CHECK_LAUNCH("cg_pass_init");
    if (ws->direct) {
        CF_CUDA(cudaEventRecord(ws->ev0, s));
        for (;;) {
            for (int b2 = 0; b2 < ws->direct_batch; ++b2) {
                int rc = pass_body<ORDER, PK>(ws, s, zc, 0, 0);
                if (rc != CF_OK) return rc;
            }
            CF_CUDA(cudaMemcpyAsync(&ws->sc_host->done, &ws->sc->done, sizeof(int), cudaMemcpyDeviceToHost, s));
            CF_CUDA(cudaStreamSynchronize(s));
            if (ws->sc_host->done) break;
        }
        CF_CUDA(cudaEventRecord(ws->ev1, s));
        return CF_OK;
    }
    if (!ws->exec_pass[PK] || ws->zc_pass[PK] != zc) {
        if (ws->exec_pass[PK]) {
            cudaGraphExecDestroy(ws->exec_pass[PK]);
            cudaGraphDestroy(ws->graph_pass[PK]);
            ws->exec_pass[PK] = nullptr;
        }
        int rc = pass_build_graph<ORDER, PK>(ws, zc);
        if (rc != CF_OK) return rc;
    }
    CF_CUDA(cudaEventRecord(ws->ev0, s));
    CF_CUDA(cudaGraphLaunch(ws->exec_pass[PK], s));
    CF_CUDA(cudaEventRecord(ws->ev1, s));
    return CF_OK;
}

// ---------------------------------------------------------------- TMA-fed single pass
// tile height / ring depth variants: 16-row tiles, one CTA per SM (default);
// 8-row tiles, two CTAs per SM (CF_SPASS_TY=8)
template <int PK, int TY, int S, int FORM>
static void spass_launch(cf_cg *ws, cudaStream_t s, double zc, cudaGraphConditionalHandle cond, int use_cond)
{
    using G = Sp<TY, S, FORM>;
    for (int half = 0; half < 2; ++half) {
        // half 0: r, p[0] -> r2, p[1], x skipped; half 1: r2, p[1] -> r, p[0], x for both passes
        double *r_out = half ? ws->r : ws->r2;
        if (half == 0)
            cg_spass_kernel<PK, TY, S, false, FORM><<<ws->sp_ctas, G::Threads, G::Smem, s>>>(
                ws->m_spr[0], ws->m_spp[0], ws->m_spx, ws->sp_g, ws->off, ws->diag, zc, r_out, ws->p[1], ws->x,
                ws->sc, ws->partials, ws->tk, use_cond, cond);
        else
            cg_spass_kernel<PK, TY, S, true, FORM><<<ws->sp_ctas, G::Threads, G::Smem, s>>>(
                ws->m_spr[1], ws->m_spp[1], ws->m_spx, ws->sp_g, ws->off, ws->diag, zc, r_out, ws->p[0], ws->x,
                ws->sc, ws->partials, ws->tk, use_cond, cond);
    }
}

template <int PK>
static int spass_body_launch(cf_cg *ws, cudaStream_t s, double zc, cudaGraphConditionalHandle cond, int use_cond)
{
    if (ws->sp_form == 1 && ws->sp_ty == 8) spass_launch<PK, 8, 5, 1>(ws, s, zc, cond, use_cond);
    else if (ws->sp_form == 1) spass_launch<PK, 16, 6, 1>(ws, s, zc, cond, use_cond);
    else if (ws->sp_ty == 8) spass_launch<PK, 8, 5, 2>(ws, s, zc, cond, use_cond);
    else spass_launch<PK, 16, 6, 2>(ws, s, zc, cond, use_cond);
    CF_CHECK_LAUNCH("cg_spass_kernel");
    return CF_OK;
}

// host setup of one variant: smem opt-in, (tile, chunk) geometry, resident CTAs
template <int TY, int S, int FORM>
static void spass_setup(cf_cg *ws)
{
    using G = Sp<TY, S, FORM>;
    cudaFuncSetAttribute(cg_spass_kernel<PK_NONE, TY, S, false, FORM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::Smem);
    cudaFuncSetAttribute(cg_spass_kernel<PK_NONE, TY, S, true, FORM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::Smem);
    cudaFuncSetAttribute(cg_spass_kernel<PK_JCONST, TY, S, false, FORM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::Smem);
    cudaFuncSetAttribute(cg_spass_kernel<PK_JCONST, TY, S, true, FORM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::Smem);
    SpGeom g{ws->bx.nx, ws->bx.ny, ws->bx.nz, (ws->bx.nx + kSpTX - 1) / kSpTX, (ws->bx.ny + TY - 1) / TY, 1, nullptr};
    const int bps = blocks_per_sm((const void *)cg_spass_kernel<PK_JCONST, TY, S, true, FORM>, G::Threads, G::Smem);
    const long long slots = (long long)num_sms() * (bps > 0 ? bps : 1), tiles = (long long)g.ntx * g.nty;
    // z-chunks: as many as fill the resident slots in one round, each >= 8 planes
    long long c = std::max(1LL, std::min(slots / std::max(1LL, tiles), (long long)g.nz / 8));
    if (const char *e = getenv("CF_SPASS_CHUNKS")) c = std::max(1, std::min(atoi(e), g.nz));
    g.nchunk = (int)c;
    const long long items = tiles * c, rounds = (items + slots - 1) / slots;
    ws->sp_ctas = (int)((items + rounds - 1) / rounds);  // equal rounds for every CTA
    // CF_SPASS_SCHED=phase: every resident slot busy on equal contiguous
    // ranges, tiles permuted so that neighbours keep their phase (SpGeom)
    const char *sched = getenv("CF_SPASS_SCHED");
    if (sched && !strcmp(sched, "phase")) {
        const long long G2 = std::max(1LL, std::min(slots, tiles * g.nz / 8));
        // position p starts at unit p * nz; its phase within a range of
        // tiles * nz / G2 units, scaled by G2 to stay integral
        std::vector<std::pair<long long, int>> ph((size_t)tiles);
        for (long long p = 0; p < tiles; ++p) ph[(size_t)p] = {(long long)g.nz * p * G2 % (tiles * g.nz), (int)p};
        std::stable_sort(ph.begin(), ph.end());
        std::vector<int> perm((size_t)tiles);
        for (long long i = 0; i < tiles; ++i) perm[(size_t)ph[(size_t)i].second] = (int)i;  // y-major tiles by phase
        if (!ws->sp_perm) cudaMalloc(&ws->sp_perm, (size_t)tiles * sizeof(int));
        if (ws->sp_perm) {
            cudaMemcpy(ws->sp_perm, perm.data(), (size_t)tiles * sizeof(int), cudaMemcpyHostToDevice);
            g.perm = ws->sp_perm;
            ws->sp_ctas = (int)G2;
        }
    }
    ws->sp_g = g;
    ws->spass = bps >= 1;
}

template <int ORDER, int PK>
static int spass_build_graph(cf_cg *ws, double zc)
{
    cudaGraph_t g;
    CF_CUDA(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle cond;
    CF_CUDA(cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CF_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &np));
    cudaStream_t cs;
    CF_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CF_CUDA(cudaStreamBeginCaptureToGraph(cs, np.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                          cudaStreamCaptureModeRelaxed));
    int rc = spass_body_launch<PK>(ws, cs, zc, cond, 1);
    cudaGraph_t captured;
    cudaError_t e = cudaStreamEndCapture(cs, &captured);
    cudaStreamDestroy(cs);
    if (rc != CF_OK) return rc;
    CF_CUDA(e);
    {  // x += alpha p_k owed by a final skipping pass (odd iteration count), p_k in p[1]
        cudaKernelNodeParams kp = {};
        void *args[] = {&ws->n, &ws->x, &ws->p[1], &ws->sc};
        kp.func = (void *)cg_x_fixup;
        kp.gridDim = dim3(ws->grid_init);
        kp.blockDim = dim3(kMarchThreads);
        kp.kernelParams = args;
        cudaGraphNode_t fix;
        CF_CUDA(cudaGraphAddKernelNode(&fix, g, &node, 1, &kp));
    }
    cudaGraphExec_t exec;
    CF_CUDA(cudaGraphInstantiate(&exec, g, 0));
    ws->graph_pass[PK] = g;
    ws->exec_pass[PK] = exec;
    ws->zc_pass[PK] = zc;
    return CF_OK;
}

template <int ORDER, int PK>
static int spass_solve(cf_cg *ws, const double *b, double zc, cudaStream_t s)
{
    // r = b, x = 0, |b|^2, gamma_0 = r.z, delta_0 = z.A z -> alpha_0 (cf_cg_pass.cuh)
    cg_pass_init<ORDER, PK><<<ws->pg_upd.ctas(), kPairThreads, 0, s>>>(ws->pg_upd, ws->off, ws->diag, zc, b, ws->r,
                                                                       ws->x, ws->sc, ws->partials, ws->tk);
    CF_CHECK_LAUNCH("cg_pass_init");
    if (ws->direct) {
        CF_CUDA(cudaEventRecord(ws->ev0, s));
        for (;;) {
            for (int b2 = 0; b2 < ws->direct_batch; ++b2) {
                int rc = spass_body_launch<PK>(ws, s, zc, 0, 0);
                if (rc != CF_OK) return rc;
            }
            CF_CUDA(cudaMemcpyAsync(&ws->sc_host->done, &ws->sc->done, sizeof(int), cudaMemcpyDeviceToHost, s));
            CF_CUDA(cudaStreamSynchronize(s));
            if (ws->sc_host->done) break;
        }
        cg_x_fixup<<<ws->grid_init, kMarchThreads, 0, s>>>(ws->n, ws->x, ws->p[1], ws->sc);
        CF_CHECK_LAUNCH("cg_x_fixup");
        CF_CUDA(cudaEventRecord(ws->ev1, s));
        return CF_OK;
    }
    if (!ws->exec_pass[PK] || ws->zc_pass[PK] != zc) {
        if (ws->exec_pass[PK]) {
            cudaGraphExecDestroy(ws->exec_pass[PK]);
            cudaGraphDestroy(ws->graph_pass[PK]);
            ws->exec_pass[PK] = nullptr;
        }
        int rc = spass_build_graph<ORDER, PK>(ws, zc);
        if (rc != CF_OK) return rc;
    }
    CF_CUDA(cudaEventRecord(ws->ev0, s));
    CF_CUDA(cudaGraphLaunch(ws->exec_pass[PK], s));
    CF_CUDA(cudaEventRecord(ws->ev1, s));
    return CF_OK;
}

template <int ORDER, int PK>
static int solve_impl(cf_cg *ws, const double *b, const double *x0, double zc, cudaStream_t s)
{
    const char *ns = getenv("CF_NO_SMALL");
    if (PK == PK_ZVEC && ws->n <= kSmallDicMaxCells && ws->dic.wave.ok && ws->dic_lptr && !x0 &&
        !(ns && atoi(ns) > 0)) {
        const size_t smem = 5 * (size_t)ws->n * sizeof(double);
        CF_CUDA(cudaFuncSetAttribute(cg_small_dic_kernel<ORDER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        CF_CUDA(cudaEventRecord(ws->ev0, s));
        const int nlev = (int)ws->dic.level_ptr.size() - 1;
        ws->last_form = CF_CG_FORM_SMALL;
        cg_small_dic_kernel<ORDER><<<1, kSmallThreads, smem, s>>>(ws->bx, ws->off, ws->diag, b, ws->x, ws->dic.d,
                                                                  ws->dic.rows, ws->dic_lptr, nlev,
                                                                  ws->dic.wave.lval, ws->dic.wave.uval, ws->sc);
        CF_CHECK_LAUNCH("cg_small_dic_kernel");
        CF_CUDA(cudaEventRecord(ws->ev1, s));
        return CF_OK;
    }
    if (PK != PK_ZVEC && ws->n <= kSmallMaxCells && !(ns && atoi(ns) > 0)) {
        const size_t smem = 3 * (size_t)ws->n * sizeof(double);
        CF_CUDA(cudaFuncSetAttribute(cg_small_kernel<ORDER, PK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CF_CUDA(cudaEventRecord(ws->ev0, s));
        ws->last_form = CF_CG_FORM_SMALL;
        cg_small_kernel<ORDER, PK><<<1, kSmallThreads, smem, s>>>(ws->bx, ws->off, ws->diag, b, x0, ws->x, ws->jd, zc,
                                                                  ws->sc);
        CF_CHECK_LAUNCH("cg_small_kernel");
        CF_CUDA(cudaEventRecord(ws->ev1, s));
        return CF_OK;
    }
    if ((PK == PK_NONE || PK == PK_JCONST) && ws->spass && !x0) {
        ws->last_form = CF_CG_FORM_SPASS;
        if constexpr (PK == PK_NONE || PK == PK_JCONST) return spass_solve<ORDER, PK>(ws, b, zc, s);
    }
    if ((PK == PK_NONE || PK == PK_JCONST) && ws->pass && !x0) {
        ws->last_form = CF_CG_FORM_PASS;
        if constexpr (PK == PK_NONE || PK == PK_JCONST) return pass_solve<ORDER, PK>(ws, b, zc, s);
    }
    if ((PK == PK_NONE || PK == PK_JCONST) && ws->persist && !x0 && !ws->direct) {
        if constexpr (PK == PK_NONE || PK == PK_JCONST) {
            ws->last_form = CF_CG_FORM_PERSIST;
            int rc0 = launch_init<ORDER, PK>(ws, b, x0, zc, s);
            if (rc0 != CF_OK) return rc0;
            CF_CUDA(cudaEventRecord(ws->ev0, s));
            cg_persist_kernel<ORDER, PK><<<ws->per_blocks, kPersistThreads, 0, s>>>(
                ws->per_g, ws->off, ws->diag, zc, ws->r, ws->x, ws->p[0], ws->p[1], ws->sc, ws->per_part,
                ws->per_part + ws->per_blocks, ws->per_bar);
            CF_CHECK_LAUNCH("cg_persist_kernel");
            CF_CUDA(cudaEventRecord(ws->ev1, s));
            return CF_OK;
        }
    }
    ws->last_form = PK == PK_ZVEC ? CF_CG_FORM_TWO_DIC : CF_CG_FORM_TWO;
    int rc = launch_init<ORDER, PK>(ws, b, x0, zc, s);
    if (rc != CF_OK) return rc;
    if (ws->direct) {
        // Host-driven loop (profilers cannot see kernels inside conditional
        // graphs; also the multi-rank path): batches of iterations, kernels
        // early-exit on sc->done, one 4-byte poll per batch.
        CF_CUDA(cudaEventRecord(ws->ev0, s));
        for (;;) {
            for (int b2 = 0; b2 < ws->direct_batch; ++b2) {
                rc = capture_body<ORDER, PK>(ws, s, zc, 0, 0);
                if (rc != CF_OK) return rc;
            }
            CF_CUDA(cudaMemcpyAsync(&ws->sc_host->done, &ws->sc->done, sizeof(int), cudaMemcpyDeviceToHost, s));
            CF_CUDA(cudaStreamSynchronize(s));
            if (ws->sc_host->done) break;
        }
        if (ws->defer_x) {
            cg_x_fixup<<<ws->grid_init, kMarchThreads, 0, s>>>(ws->n, ws->x, ws->p[1], ws->sc);
            CF_CHECK_LAUNCH("cg_x_fixup");
        }
        CF_CUDA(cudaEventRecord(ws->ev1, s));
        return CF_OK;
    }
    if (!ws->exec[PK] || ws->zc_graph[PK] != zc) {
        if (ws->exec[PK]) {
            cudaGraphExecDestroy(ws->exec[PK]);
            cudaGraphDestroy(ws->graph[PK]);
            ws->exec[PK] = nullptr;
        }
        rc = build_graph<ORDER, PK>(ws, s, zc);
        if (rc != CF_OK) return rc;
    }
    CF_CUDA(cudaEventRecord(ws->ev0, s));
    CF_CUDA(cudaGraphLaunch(ws->exec[PK], s));
    CF_CUDA(cudaEventRecord(ws->ev1, s));
    return CF_OK;
}

template <int ORDER>
static int solve_dispatch(cf_cg *ws, int pk, const double *b, const double *x0, double zc,
                          cudaStream_t s)
{
    switch (pk) {
    case PK_NONE: return solve_impl<ORDER, PK_NONE>(ws, b, x0, zc, s);
    case PK_JCONST: return solve_impl<ORDER, PK_JCONST>(ws, b, x0, zc, s);
    case PK_JVEC: return solve_impl<ORDER, PK_JVEC>(ws, b, x0, zc, s);
    case PK_ZVEC: return solve_impl<ORDER, PK_ZVEC>(ws, b, x0, zc, s);
    default: set_error("unsupported preconditioner kind"); return CF_EINVAL;
    }
}

template <int ORDER, int XM>
static void set_upd_smem()
{
    cudaFuncSetAttribute(cg_update_tma<ORDER, PK_NONE, XM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUpdSmem);
    cudaFuncSetAttribute(cg_update_tma<ORDER, PK_JCONST, XM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kUpdSmem);
    cudaFuncSetAttribute(cg_update_tma<ORDER, PK_ZVEC, XM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUpdSmem);
}

template <int ORDER>
static void set_grids(cf_cg *ws)
{
    ws->grid_dir = march_grid((const void *)cg_dir_kernel<ORDER, PK_JCONST>, ws->bx);
    ws->grid_upd = march_grid((const void *)cg_update_kernel<ORDER, PK_JCONST>, ws->bx);
    ws->grid_init_x0 = march_grid((const void *)cg_init_x0<ORDER, PK_JCONST>, ws->bx);
    long long want = (ws->n + kMarchThreads - 1) / kMarchThreads;
    long long cap = (long long)num_sms() * blocks_per_sm((const void *)cg_init_flat<PK_JCONST>, kMarchThreads, 0);
    ws->grid_init = (int)(want < cap ? (want > 0 ? want : 1) : cap);
    const char *no_tma = getenv("CF_NO_TMA");
    ws->tma = ws->bx.nx >= 32 && ws->bx.nx % 2 == 0 && !(no_tma && atoi(no_tma) > 0);
    if (ws->tma) {
        int bd = 0, bu = 0;
        // every instantiation the workspace may launch needs the dynamic smem opt-in
        cudaFuncSetAttribute(cg_dir_tma<ORDER, PK_NONE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDirSmem);
        cudaFuncSetAttribute(cg_dir_tma<ORDER, PK_JCONST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDirSmem);
        cudaFuncSetAttribute(cg_dir_tma<ORDER, PK_ZVEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDirSmem);
        set_upd_smem<ORDER, XM_EACH>();
        set_upd_smem<ORDER, XM_SKIP>();
        set_upd_smem<ORDER, XM_DOUBLE>();
        cudaFuncSetAttribute(cg_update_tma<ORDER, PK_NONE, XM_DOUBLE, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_full_smem<4>());
        cudaFuncSetAttribute(cg_update_tma<ORDER, PK_JCONST, XM_DOUBLE, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_full_smem<4>());
        cudaFuncSetAttribute(cg_update_tma<ORDER, PK_ZVEC, XM_DOUBLE, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_full_smem<4>());
        cudaFuncSetAttribute(cg_update_tma<ORDER, PK_NONE, XM_SKIP, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_skip_smem<4>());
        cudaFuncSetAttribute(cg_update_tma<ORDER, PK_JCONST, XM_SKIP, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_skip_smem<4>());
        cudaFuncSetAttribute(cg_update_tma<ORDER, PK_ZVEC, XM_SKIP, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_skip_smem<4>());
        cudaFuncSetAttribute(cg_update_tma<ORDER, PK_NONE, XM_SKIP, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_skip_smem<6>());
        cudaFuncSetAttribute(cg_update_tma<ORDER, PK_JCONST, XM_SKIP, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_skip_smem<6>());
        cudaFuncSetAttribute(cg_update_tma<ORDER, PK_ZVEC, XM_SKIP, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_skip_smem<6>());
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bd, cg_dir_tma<ORDER, PK_JCONST>, kWSThreads, kDirSmem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bu, cg_update_tma<ORDER, PK_JCONST>, kWSThreads, kUpdSmem);
        ws->geom_dir = tma_geom(ws->bx.nx, ws->bx.ny, ws->bx.nz, 0, 0, bd > 0 ? bd : 1);
        ws->geom_upd = tma_geom(ws->bx.nx, ws->bx.ny, ws->bx.nz, 0, 0, bu > 0 ? bu : 1);
        if (const char *e = getenv("CF_TMA_CHUNKS_DIR")) ws->geom_dir.nchunk = atoi(e) > 0 ? atoi(e) : 1;
        if (const char *e = getenv("CF_TMA_CHUNKS_UPD")) ws->geom_upd.nchunk = atoi(e) > 0 ? atoi(e) : 1;
        int bdb = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bdb, cg_update_tma<ORDER, PK_JCONST, XM_DOUBLE, 4>, kWSThreads,
                                                      upd_full_smem<4>());
        ws->geom_dbl = tma_geom(ws->bx.nx, ws->bx.ny, ws->bx.nz, 0, 0, bdb > 0 ? bdb : 1);
    }
    const bool pair_ok = ws->bx.nx % 2 == 0 && !(no_tma && atoi(no_tma) > 0);
    ws->pg_dir = pair_geom(ws->bx.nx, ws->bx.ny, ws->bx.nz, 0, 0, "CF_PAIR_CHUNKS_DIR");
    ws->pg_upd = pair_geom(ws->bx.nx, ws->bx.ny, ws->bx.nz, 0, 0, "CF_PAIR_CHUNKS_UPD");
    ws->kind_dir = kern_kind("CF_CG_DIR", KK_LEAN, ws->tma, pair_ok);
    ws->kind_upd = kern_kind("CF_CG_UPD", KK_TMA, ws->tma, pair_ok);
    if (const char *e = getenv("CF_PAIR_PF")) ws->pair_pf = atoi(e);
    // 32-bit cell indices in the lean kernel
    if (ws->kind_dir == KK_LEAN && ws->n + kLeanPad >= (1LL << 32)) ws->kind_dir = KK_PAIR;
    if (ws->kind_upd == KK_LEAN && ws->n + kLeanPad >= (1LL << 32)) ws->kind_upd = KK_PAIR;
    if (const char *e = getenv("CF_PDL")) ws->pdl = atoi(e) != 0;
    if (const char *e = getenv("CF_LEAN2")) ws->lean2 = atoi(e) != 0;
    if (const char *e = getenv("CF_DOUBLE_STAGES")) ws->double_stages = atoi(e) == 3 ? 3 : 4;
    if (const char *e = getenv("CF_SKIP_STAGES")) ws->skip_stages = atoi(e) == 3 ? 3 : (atoi(e) == 6 ? 6 : 4);
    if (const char *e = getenv("CF_LEAN_ROWS")) ws->lean_rows = atoi(e) == 4 ? 4 : (atoi(e) == 8 ? 8 : 16);
    ws->lg_dir = lean_geom(ws->bx.nx, ws->bx.ny, ws->bx.nz, ws->lean_rows,
                           ws->lean2 && ws->lean_rows == 8 ? 12 : (ws->lean2 && ws->lean_rows == 16 ? 12 : 8));
    // the direction kernel takes its z chunks top-down: its last wave (the low
    // chunks, bottom planes last) is where the update kernel's first wave
    // starts, and the update's last wave (high chunks, top planes last) is
    // where the next direction kernel starts -- both hand-overs in L2
    // (measured: +2 % in the sustained bench, 190 -> 186 us per 256^3 iteration)
    ws->lg_dir.chunk_rev = 1;
    if (const char *e = getenv("CF_CHUNK_REV")) ws->lg_dir.chunk_rev = atoi(e) != 0;
    ws->lg_upd = lean_geom(ws->bx.nx, ws->bx.ny, ws->bx.nz, ws->lean_rows, 8);
    // persistent solve: the four CG vectors fit in L2 with room to spare
    // (<= 96 MB), above the single-block range; all CTAs co-resident
    {
        const long long vec_bytes = ws->n * 8;
        bool on = pair_ok && 4 * vec_bytes <= 96ll * 1024 * 1024 && ws->n > kSmallMaxCells &&
                  ws->n + kLeanPad < (1LL << 32);
        // opt-in (CF_PERSIST=1): measured 64^3 14.4 vs 19.9 us/iteration, 128^3 31.9 vs 32.9,
        // but 96^3 50 vs 24 and 144^3 108 vs 45 -- one short march per CTA per phase is
        // L2-latency bound and the two grid barriers per iteration cost ~25 % (ncu)
        const char *pe = getenv("CF_PERSIST");
        on = on && pe && atoi(pe) != 0;
        const int bps = blocks_per_sm((const void *)cg_persist_kernel<ORDER, PK_JCONST>, kPersistThreads, 0);
        ws->per_blocks = num_sms() * (bps > 0 ? bps : 1);
        ws->per_g = lean_geom(ws->bx.nx, ws->bx.ny, ws->bx.nz, kPersistRows, 8);
        ws->per_g.nchunk = wave_chunks((long long)ws->per_g.ntx * ws->per_g.nty, ws->bx.nz, ws->per_blocks, 4);
        if (ws->per_g.ctas() < ws->per_blocks) ws->per_blocks = ws->per_g.ctas();
        ws->persist = on && bps >= 1;
    }
    // single-reduction CG (one kernel per iteration, cf_cg_pass.cuh): opt-in.
    // Measured at 256^3 it runs 215 us/iteration against 205 for the
    // two-kernel form (instruction-bound: ~64 % issue slots), so the default
    // stays the two-kernel form, which is also the reference's recurrence.
    const char *algo = getenv("CF_CG_ALGO");
    ws->pass = pair_ok && algo && !strcmp(algo, "pass");
    if (ws->pass) {
        ws->pass_g = pass_geom(ws->bx.nx, ws->bx.ny, ws->bx.nz);
        cudaFuncSetAttribute(cg_pass_kernel<ORDER, PK_NONE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kPassSmem);
        cudaFuncSetAttribute(cg_pass_kernel<ORDER, PK_JCONST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kPassSmem);
        const char *pf = getenv("CF_PASS_FORM");
        ws->pass_form = pf && !strcmp(pf, "old") ? 0 : (pf && !strcmp(pf, "lean16") ? 2 : 1);
        if (ws->n + kLeanPad >= (1LL << 32)) ws->pass_form = 0;
        cudaFuncSetAttribute(cg_lpass_kernel<ORDER, PK_NONE, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)Lp<8>::Smem);
        cudaFuncSetAttribute(cg_lpass_kernel<ORDER, PK_JCONST, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)Lp<8>::Smem);
        cudaFuncSetAttribute(cg_lpass_kernel<ORDER, PK_NONE, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)Lp<16>::Smem);
        cudaFuncSetAttribute(cg_lpass_kernel<ORDER, PK_JCONST, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)Lp<16>::Smem);
        const int rows = ws->pass_form == 2 ? 16 : 8;
        PairGeom lg{ws->bx.nx, ws->bx.ny, ws->bx.nz, 0, 0, (ws->bx.nx + kPairX - 1) / kPairX,
                    (ws->bx.ny + rows - 1) / rows, 1};
        const int bps = ws->pass_form == 2
                            ? blocks_per_sm((const void *)cg_lpass_kernel<ORDER, PK_JCONST, 16>, Lp<16>::Threads,
                                            Lp<16>::Smem)
                            : blocks_per_sm((const void *)cg_lpass_kernel<ORDER, PK_JCONST, 8>, Lp<8>::Threads,
                                            Lp<8>::Smem);
        lg.nchunk = wave_chunks((long long)lg.ntx * lg.nty, lg.nz, (long long)num_sms() * bps, 8);
        if (const char *e = getenv("CF_PASS_CHUNKS")) {
            const int v = atoi(e);
            if (v >= 1 && v <= lg.nz) lg.nchunk = v;
        }
        ws->lpass_g = lg;
    }
    // TMA-fed single-reduction pass (cf_cg_spass.cuh): the default for Jacobi /
    // no preconditioner without a start vector (measured 256^3: 125 us per
    // iteration against 181 for the two-kernel loop); CF_CG_ALGO=two (or pass)
    // selects the two-kernel form, which is the reference's own recurrence
    ws->spass = ws->tma && ws->bx.nx % 2 == 0 && ws->n + kLeanPad < (1LL << 32) && !(algo && strcmp(algo, "spass"));
    if (ws->spass) {
        if (const char *e = getenv("CF_SPASS_FORM")) ws->sp_form = atoi(e) == 1 ? 1 : 2;
        if (const char *e = getenv("CF_SPASS_TY")) ws->sp_ty = atoi(e) == 8 ? 8 : 16;
        if (ws->sp_form == 1 && ws->sp_ty == 8) spass_setup<8, 5, 1>(ws);
        else if (ws->sp_form == 1) spass_setup<16, 6, 1>(ws);
        else if (ws->sp_ty == 8) spass_setup<8, 5, 2>(ws);
        else spass_setup<16, 6, 2>(ws);
    }
    if (const char *e = getenv("CF_CG_UPD_SKIP")) ws->kind_upd_skip = kern_kind("CF_CG_UPD_SKIP", ws->kind_upd, ws->tma, pair_ok);
    const char *dx = getenv("CF_CG_DEFER_X");
    ws->defer_x = ws->kind_upd != KK_LDG && !(dx && atoi(dx) == 0);
}

static bool build_maps(cf_cg *ws)
{
    const int nx = ws->bx.nx, ny = ws->bx.ny, nz = ws->bx.nz;
    bool ok = make_map(&ws->m_r, ws->r, nx, ny, nz, kHX, kHY) && make_map(&ws->m_p[0], ws->p[0], nx, ny, nz, kHX, kHY) &&
              make_map(&ws->m_p[1], ws->p[1], nx, ny, nz, kHX, kHY) &&
              make_map(&ws->m_ri, ws->r, nx, ny, nz, kTTX, kTTY) && make_map(&ws->m_xi, ws->x, nx, ny, nz, kTTX, kTTY) &&
              make_map(&ws->m_pi[0], ws->p[0], nx, ny, nz, kTTX, kTTY) &&
              make_map(&ws->m_pi[1], ws->p[1], nx, ny, nz, kTTX, kTTY);
    return ok;
}

}  // namespace cf

extern "C" {

int cf_cg_create(cf_cg **out, int nx, int ny, int nz, double h, int order, void *stream)
{
    CF_REQUIRE(out && nx >= 1 && ny >= 1 && nz >= 1 && h > 0, "cf_cg_create: bad grid");
    CF_REQUIRE(order == CF_ORDER_CSR || order == CF_ORDER_SYM, "cf_cg_create: bad order");
    cf_cg *ws = new cf_cg();
    ws->bx = cf::Box{nx, ny, nz, 0, 0};
    ws->h = h;
    ws->off = -1.0 / (h * h);
    ws->diag = 6.0 / (h * h);
    ws->order = order;
    ws->n = (long long)nx * ny * nz;
    if (const char *d = getenv("CF_CG_DIRECT")) {
        int b = atoi(d);
        if (b > 0) {
            ws->direct = 1;
            ws->direct_batch = b;
        }
    }
    if (order == CF_ORDER_CSR) cf::set_grids<CF_ORDER_CSR>(ws);
    else cf::set_grids<CF_ORDER_SYM>(ws);
    int maxg = ws->grid_dir > ws->grid_upd ? ws->grid_dir : ws->grid_upd;
    if (ws->grid_init > maxg) maxg = ws->grid_init;
    if (ws->grid_init_x0 > maxg) maxg = ws->grid_init_x0;
    if (ws->tma) {
        const cf::TmaGeom &gd = ws->geom_dir, &gu = ws->geom_upd, &gb = ws->geom_dbl;
        maxg = std::max(maxg, gb.ntx * gb.nty * gb.nchunk);
        int g1 = gd.ntx * gd.nty * gd.nchunk, g2 = gu.ntx * gu.nty * gu.nchunk;
        if (g1 > maxg) maxg = g1;
        if (g2 > maxg) maxg = g2;
    }
    maxg = std::max(maxg, std::max(ws->pg_dir.ctas(), ws->pg_upd.ctas()));
    maxg = std::max(maxg, std::max(ws->lg_dir.ctas(), ws->lg_upd.ctas()));
    if (ws->pass) maxg = std::max(maxg, std::max(ws->pass_g.ctas(), ws->lpass_g.ctas()));
    if (ws->spass) maxg = std::max(maxg, ws->sp_ctas);
    size_t vec = (size_t)ws->n * sizeof(double);
    cudaError_t e = cudaSuccess;
    // every CG vector carries kLeanPad zeroed doubles after its n cells (the
    // lean direction kernel reads out-of-domain neighbours there)
    const size_t pad = cf::kLeanPad * sizeof(double);
    for (double **b : {&ws->r, &ws->x, &ws->p[0], &ws->p[1]}) {
        if (e == cudaSuccess) e = cudaMalloc(b, vec + pad);
        if (e == cudaSuccess) e = cudaMemsetAsync(reinterpret_cast<char *>(*b) + vec, 0, pad, cf::as_stream(stream));
    }
    if (e == cudaSuccess) e = cudaMalloc(&ws->partials, sizeof(double) * 3 * (size_t)maxg);
    if (e == cudaSuccess && (ws->pass || ws->spass)) e = cudaMalloc(&ws->r2, vec + pad);
    if (e == cudaSuccess && (ws->pass || ws->spass))
        e = cudaMemsetAsync(reinterpret_cast<char *>(ws->r2) + vec, 0, pad, cf::as_stream(stream));
    if (e == cudaSuccess) e = cudaMalloc(&ws->sc, sizeof(cf::CgScalars));
    if (e == cudaSuccess) e = cudaMalloc(&ws->tk, sizeof(cf::CgTickets));
    if (e == cudaSuccess) e = cudaMemsetAsync(ws->tk, 0, sizeof(cf::CgTickets), cf::as_stream(stream));
    if (e == cudaSuccess) e = cudaMallocHost(&ws->sc_host, sizeof(cf::CgScalars));
    if (e == cudaSuccess && ws->persist) e = cudaMalloc(&ws->per_part, 3 * (size_t)ws->per_blocks * sizeof(double));
    if (e == cudaSuccess && ws->persist) e = cudaMalloc(&ws->per_bar, sizeof(cf::GridBar));
    if (e == cudaSuccess && ws->persist) e = cudaMemsetAsync(ws->per_bar, 0, sizeof(cf::GridBar), cf::as_stream(stream));
    if (e == cudaSuccess) e = cudaEventCreate(&ws->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&ws->ev1);
    if (e != cudaSuccess) {
        int rc = cf::cuda_fail(e, "cf_cg_create");
        cf_cg_destroy(ws);
        return rc;
    }
    if (ws->spass) {  // boxes of the single pass: 68 x (TY+4) halo boxes of r / p, 64 x TY interior box of x
        const int nx = ws->bx.nx, ny = ws->bx.ny, nz = ws->bx.nz;
        const int hy = ws->sp_ty + 4;
        int pr = 256;
        if (const char *e = getenv("CF_SPASS_PROMO")) pr = atoi(e);
        auto mk = [&](CUtensorMap *m, const double *b, int bx, int by) {
            return cf::make_map_promo(m, b, nx, ny, nz, bx, by, pr);
        };
        ws->spass = mk(&ws->m_spr[0], ws->r, cf::kSpBX, hy) && mk(&ws->m_spr[1], ws->r2, cf::kSpBX, hy) &&
                    mk(&ws->m_spp[0], ws->p[0], cf::kSpBX, hy) && mk(&ws->m_spp[1], ws->p[1], cf::kSpBX, hy) &&
                    mk(&ws->m_spx, ws->x, cf::kSpTX, ws->sp_ty);
    }
    if (ws->tma && !cf::build_maps(ws)) {  // TMA cannot describe the arrays: pair / LDG forms
        ws->tma = false;
        if (ws->kind_dir == cf::KK_TMA) ws->kind_dir = ws->bx.nx % 2 == 0 ? cf::KK_PAIR : cf::KK_LDG;
        if (ws->kind_upd == cf::KK_TMA) ws->kind_upd = ws->bx.nx % 2 == 0 ? cf::KK_PAIR : cf::KK_LDG;
        if (ws->kind_upd == cf::KK_LDG) ws->defer_x = false;
    }
    *out = ws;
    return CF_OK;
}

int cf_cg_destroy(cf_cg *ws)
{
    if (!ws) return CF_OK;
    for (int k = 0; k < 4; ++k) {
        if (ws->exec[k]) cudaGraphExecDestroy(ws->exec[k]);
        if (ws->graph[k]) cudaGraphDestroy(ws->graph[k]);
    }
    for (int k = 0; k < 4; ++k) {
        if (ws->exec_pass[k]) cudaGraphExecDestroy(ws->exec_pass[k]);
        if (ws->graph_pass[k]) cudaGraphDestroy(ws->graph_pass[k]);
    }
    for (double *b : {ws->r, ws->x, ws->p[0], ws->p[1], ws->jd, ws->partials, ws->zbuf, ws->wbuf, ws->r2, ws->per_part})
        if (b) cudaFree(b);
    if (ws->per_bar) cudaFree(ws->per_bar);
    if (ws->dic_lptr) cudaFree(ws->dic_lptr);
    if (ws->sp_perm) cudaFree(ws->sp_perm);
    if (ws->dic.wave.prog_f) cudaFree(ws->dic.wave.prog_f);
    if (ws->dic.wave.ex_f) cudaFree(ws->dic.wave.ex_f);
    if (ws->dic.wave.ey_f) cudaFree(ws->dic.wave.ey_f);
    cf::dic_skew_free(ws->dic.skew);
    if (ws->sc) cudaFree(ws->sc);
    if (ws->tk) cudaFree(ws->tk);
    if (ws->sc_host) cudaFreeHost(ws->sc_host);
    if (ws->ev0) cudaEventDestroy(ws->ev0);
    if (ws->ev1) cudaEventDestroy(ws->ev1);
    delete ws;
    return CF_OK;
}

int cf_cg_solve(cf_cg *ws, const double *b, double *x, const double *x0, double tol, int64_t max_iter,
                int precond, const double *inv_diag, int64_t *iters_host, double *res_host, void *stream)
{
    CF_REQUIRE(ws && b && x, "cf_cg_solve: null argument");
    CF_REQUIRE(tol > 0, "tol must be positive");
    CF_REQUIRE(max_iter >= 1, "max_iter must be >= 1");
    std::lock_guard<std::mutex> lk(ws->mu);
    cudaStream_t s = cf::as_stream(stream);
    int pk;
    double zc = 0.0;
    if (precond == CF_PRECOND_NONE) {
        pk = cf::PK_NONE;
    } else if (precond == CF_PRECOND_JACOBI) {
        if (inv_diag == nullptr) {
            pk = cf::PK_JCONST;
            zc = 1.0 / ws->diag;  // jacobi_from: 1.0 / diag (src/precond.py:138)
        } else {
            pk = cf::PK_JVEC;
            if (!ws->jd) CF_CUDA(cudaMalloc(&ws->jd, (size_t)ws->n * sizeof(double)));
            CF_CUDA(cudaMemcpyAsync(ws->jd, inv_diag, (size_t)ws->n * sizeof(double),
                                    cudaMemcpyDeviceToDevice, s));
        }
    } else if (precond == CF_PRECOND_DIC) {
        CF_REQUIRE(ws->has_dic, "cf_cg_solve: CF_PRECOND_DIC needs cf_cg_set_dic first");
        pk = cf::PK_ZVEC;
    } else {
        cf::set_error("cf_cg_solve: preconditioner kind not supported by the fused path");
        return CF_EINVAL;
    }
    cf::CgScalars *h = ws->sc_host;
    *h = cf::CgScalars{};
    h->tol = tol;
    h->max_iter = max_iter;
    CF_CUDA(cudaMemcpyAsync(ws->sc, h, sizeof(*h), cudaMemcpyHostToDevice, s));
    int rc = ws->order == CF_ORDER_CSR ? cf::solve_dispatch<CF_ORDER_CSR>(ws, pk, b, x0, zc, s)
                                       : cf::solve_dispatch<CF_ORDER_SYM>(ws, pk, b, x0, zc, s);
    if (rc != CF_OK) return rc;
    CF_CUDA(cudaMemcpyAsync(h, ws->sc, sizeof(*h), cudaMemcpyDeviceToHost, s));
    CF_CUDA(cudaStreamSynchronize(s));
    CF_CUDA(cudaEventElapsedTime(&ws->last_loop_ms, ws->ev0, ws->ev1));
    if (h->norm_b == 0.0) {
        CF_CUDA(cudaMemsetAsync(x, 0, (size_t)ws->n * sizeof(double), s));  // exact solution of A x = 0
    } else {
        CF_CUDA(cudaMemcpyAsync(x, ws->x, (size_t)ws->n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    if (iters_host) *iters_host = h->it;
    if (res_host) *res_host = h->res;
    {  // kernel launches of this solve (the while body holds two iterations)
        const long long batch = ws->direct ? ws->direct_batch : 1;
        long long bodies = std::max(1LL, (h->it + 1) / 2);
        bodies = (bodies + batch - 1) / batch * batch;
        switch (ws->last_form) {
        case CF_CG_FORM_SMALL: ws->last_launches = 1; break;
        case CF_CG_FORM_SPASS: ws->last_launches = 1 + 2 * bodies + 1; break;  // init, passes, x fix-up
        case CF_CG_FORM_PASS: ws->last_launches = 1 + 2 * bodies; break;
        case CF_CG_FORM_PERSIST: ws->last_launches = 2; break;
        case CF_CG_FORM_TWO_DIC:  // init, z = M^-1 r (2 sweeps), r.z; per iteration dir, update, 2 sweeps
            ws->last_launches = (x0 ? 2 : 1) + 3 + 8 * bodies + (ws->defer_x ? 1 : 0);
            break;
        default: ws->last_launches = (x0 ? 2 : 1) + 4 * bodies + (ws->defer_x ? 1 : 0);
        }
    }
    if (h->status == cf::ST_BREAKDOWN) {
        cf::set_error("p^T A p = " + std::to_string(h->pap) + " at iteration " +
                      std::to_string(h->it + 1));
        return CF_BREAKDOWN;
    }
    return h->status == cf::ST_CONVERGED ? CF_OK : CF_NOT_CONVERGED;
}

int cf_cg_set_dic(cf_cg *ws, const int32_t *lp, const int32_t *lc, const double *lv, const int32_t *up,
                  const int32_t *uc, const double *uv, const double *d, const int32_t *level_rows,
                  const int64_t *level_ptr_host, int nlevels)
{
    CF_REQUIRE(ws && lp && lc && lv && up && uc && uv && d && level_rows && level_ptr_host && nlevels >= 0,
               "cf_cg_set_dic: null argument");
    CF_REQUIRE(level_ptr_host[nlevels] == ws->n, "cf_cg_set_dic: level schedule does not cover the grid");
    std::lock_guard<std::mutex> lk(ws->mu);
    if (!ws->zbuf) {
        CF_CUDA(cudaMalloc(&ws->zbuf, (size_t)(ws->n + cf::kLeanPad) * sizeof(double)));
        CF_CUDA(cudaMemset(ws->zbuf + ws->n, 0, cf::kLeanPad * sizeof(double)));
    }
    if (!ws->wbuf) CF_CUDA(cudaMalloc(&ws->wbuf, (size_t)ws->n * sizeof(double)));
    if (ws->tma && !cf::make_map(&ws->m_z, ws->zbuf, ws->bx.nx, ws->bx.ny, ws->bx.nz, cf::kHX, cf::kHY))
        ws->tma = false;
    cf::DicData &dd = ws->dic;
    dd.n = ws->n;
    dd.lp = lp; dd.lc = lc; dd.lv = lv;
    dd.up = up; dd.uc = uc; dd.uv = uv;
    dd.d = d;
    dd.rows = level_rows;
    dd.level_ptr.assign(level_ptr_host, level_ptr_host + nlevels + 1);
    // the tiled-wavefront sweeps when the triangles are the grid's 7-point pattern
    int rcw = cf::dic_wave_setup(dd, ws->bx.nx, ws->bx.ny, ws->bx.nz, nullptr);
    if (rcw != CF_OK) return rcw;
    if (ws->dic_lptr) cudaFree(ws->dic_lptr);
    ws->dic_lptr = nullptr;
    if (ws->n <= cf::kSmallDicMaxCells) {
        CF_CUDA(cudaMalloc(&ws->dic_lptr, (size_t)(nlevels + 1) * sizeof(long long)));
        CF_CUDA(cudaMemcpy(ws->dic_lptr, level_ptr_host, (size_t)(nlevels + 1) * sizeof(long long),
                           cudaMemcpyHostToDevice));
    }
    ws->has_dic = true;
    if (ws->exec[cf::PK_ZVEC]) {  // pointers changed: rebuild on the next solve
        cudaGraphExecDestroy(ws->exec[cf::PK_ZVEC]);
        cudaGraphDestroy(ws->graph[cf::PK_ZVEC]);
        ws->exec[cf::PK_ZVEC] = nullptr;
        ws->graph[cf::PK_ZVEC] = nullptr;
    }
    return CF_OK;
}

int cf_cg_last_form(cf_cg *ws, int *form_host, int64_t *launches_host)
{
    CF_REQUIRE(ws && form_host, "cf_cg_last_form: null argument");
    *form_host = ws->last_form;
    if (launches_host) *launches_host = ws->last_launches;
    return CF_OK;
}

int cf_cg_last_loop_ms(cf_cg *ws, float *ms_host)
{
    CF_REQUIRE(ws && ms_host, "cf_cg_last_loop_ms: null argument");
    *ms_host = ws->last_loop_ms;
    return CF_OK;
}

}  // extern "C"
