// cf_dic_wave.cu -- the simplified-DIC sweeps (src/precond.py:38-54) as a
// tiled 3-D wavefront, for the 7-point pattern of the structured grid.
//
// The level-scheduled form (cf_dic.cu) runs one launch per hyperplane
// i+j+k = const: 3n-2 dependent launches per sweep, ~5 us each inside a
// graph, so a 128^3 DIC apply costs ~3.9 ms of launch latency.  Here ONE
// launch does a sweep: a CTA owns a 16 x 8 column of cells (its tile) over
// all z and walks it along the diagonals s = ti + tj + k -- every cell's
// lower neighbours (i-1, j-1, k-1) are on diagonal s-1, so one __syncthreads
// per diagonal orders the whole tile.  Neighbours inside the tile come from
// shared memory (left, below) or the thread's own register (k-1); across
// tiles from global memory once the neighbouring tile has published that it
// is far enough (a per-tile progress counter, release/acquire at GPU scope):
// the left tile's cell (x0-1, j, k) is written at its step s + 16 - 1, the
// lower tile's (i, y0-1, k) at s + 8 - 1.  The critical path is the DAG depth
// (3n-2 diagonals) -- the same as the level schedule, without the launches.
//
// Every cell does the reference's operations in the reference's order
// (forward: s = r_i; s -= L*w for the lower columns in ascending order
// k-1, j-1, i-1; w_i = s / d_i; backward: s = 0; s += U*z for i+1, j+1, k+1;
// z_i = w_i - s / d_i), so the result is bit-identical to the sequential
// sweeps.  Used when the factor's triangles are exactly the 7-point pattern
// of the CG workspace's grid with one off-diagonal value each (verified on
// the device at attach time); anything else keeps the level schedule.
#include <algorithm>
#include <cstdlib>

#include "cf_common.cuh"
#include "cf_dic.cuh"
#include "cf_tma.cuh"

namespace cf {

// one-warp tiles synchronise with __syncwarp instead of a block barrier
template <int NT>
__device__ __forceinline__ void tile_sync()
{
    if (NT == 32) __syncwarp();
    else __syncthreads();
}

__device__ __forceinline__ int ld_acquire_gpu(const int *p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ int ld_relaxed_gpu(const int *p)
{
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void st_release_gpu(int *p, int v)
{
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Tile numbers come from an atomic ticket taken at CTA start, not from
// blockIdx: a CTA only waits on lower tickets, whose owners have already
// started (are resident), whatever order the hardware dispatches CTAs in.
// Each sweep re-arms the other sweep's counter (they alternate on one stream).
__device__ __forceinline__ int wave_ticket(int *mine, int *other)
{
    __shared__ int tk;
    if (threadIdx.x == 0) {
        tk = atomicAdd(mine, 1);
        *other = 0;
    }
    __syncthreads();
    return tk;
}

// Forward sweep (L + D~) w = r.  Tickets -> tiles in increasing (a, b), so a
// CTA only ever waits for lower-numbered (earlier-started) CTAs.
template <int kWTX, int kWTY>
__global__ void __launch_bounds__(kWTX *kWTY) dic_wave_fwd(DicWave dw, const double *__restrict__ d,
                                                          const double *__restrict__ r, double *__restrict__ w,
                                                          const int *done)
{
    __shared__ double sm[2][kWTY][kWTX];
    if (done && *done) return;
    const int ntx = dw.ntx;
    const int t = wave_ticket(dw.ticket, dw.ticket + 1), a = t % ntx, b = t / ntx;
    const int ti = threadIdx.x % kWTX, tj = threadIdx.x / kWTX;
    const int i = a * kWTX + ti, j = b * kWTY + tj;
    const bool col_ok = i < dw.nx && j < dw.ny;
    const long long pl = (long long)dw.nx * dw.ny;
    const long long base = (long long)i + (long long)dw.nx * j;
    if (threadIdx.x == 0) dw.prog_b[t] = 0;  // re-arm the backward sweep's counters (it runs after this launch)
    const int *left = a > 0 ? dw.prog_f + (t - 1) : nullptr;
    const int *below = b > 0 ? dw.prog_f + (t - ntx) : nullptr;
    int seen_l = 0, seen_b = 0, peek_l = 0, peek_b = 0;
    double wk = 0.0;  // w at (i, j, k-1)
    const int nsteps = dw.nz + kWTX + kWTY - 2;
    // r and d of this thread's next cell (independent of the sweep: prefetched a step ahead)
    auto ld_rd = [&](int k, double &rv, double &dv) {
        if (col_ok && k >= 0 && k < dw.nz) {
            const long long o = base + pl * k;
            rv = __ldg(r + o);
            dv = __ldg(d + o);
        }
    };
    double r_nx = 0.0, d_nx = 1.0;
    ld_rd(-ti - tj, r_nx, d_nx);  // k at step 0
    // edge values from the neighbouring tiles, prefetched a step ahead; the
    // wait below keeps `slack` steps between the tiles so that both the
    // progress peek and these loads are normally satisfied a step early
    const int slack = dw.slack;
    auto ld_edge = [&](int k, double &xl, double &yl) {
        if (col_ok && k >= 0 && k < dw.nz) {
            const long long o = base + pl * k;
            if (ti == 0 && i > 0) xl = __ldcg(w + o - 1);
            if (tj == 0 && j > 0) yl = __ldcg(w + o - dw.nx);
        }
    };
    double xl_nx = 0.0, yl_nx = 0.0;
    bool edge_loaded = false;
    for (int s = 0; s < nsteps; ++s) {
        // wait until the left / lower tiles have produced what this diagonal
        // reads (a neighbour's counter ends at nsteps); the relaxed peeks were
        // issued a step earlier, a fence makes an accepted value an acquire
        if (threadIdx.x == 0) {
            // A peek's value is only waited on when the cached counter no
            // longer covers the diagonal; otherwise it stays in flight (with
            // progress published every `pub` steps, one in ~pub steps is used)
            const int need_l = min(s + kWTX + slack, nsteps), need_b = min(s + kWTY + slack, nsteps);
            bool fresh = false;
            if (left && seen_l < need_l) {
                seen_l = max(seen_l, peek_l);
                while (seen_l < need_l) seen_l = ld_relaxed_gpu(left);
                fresh = true;
                peek_l = ld_relaxed_gpu(left);
            }
            if (below && seen_b < need_b) {
                seen_b = max(seen_b, peek_b);
                while (seen_b < need_b) seen_b = ld_relaxed_gpu(below);
                fresh = true;
                peek_b = ld_relaxed_gpu(below);
            }
            if (fresh) fence_acq_rel_gpu();  // an accepted counter value acts as an acquire
        }
        tile_sync<kWTX * kWTY>();
        const int k = s - ti - tj;
        if (!edge_loaded) {  // first step: nothing prefetched yet
            ld_edge(k, xl_nx, yl_nx);
            edge_loaded = true;
        }
        const double rv = r_nx, dv = d_nx, xl = xl_nx, yl = yl_nx;
        ld_rd(k + 1, r_nx, d_nx);
        ld_edge(k + 1, xl_nx, yl_nx);  // the neighbours are >= slack steps past what this needs
        double wv = 0.0;
        if (col_ok && k >= 0 && k < dw.nz) {
            const long long o = base + pl * k;
            double acc = rv;
            if (k > 0) acc = acc - dw.lval * wk;                                       // column i - pl
            if (j > 0) acc = acc - dw.lval * (tj > 0 ? sm[s & 1][tj - 1][ti] : yl);  // i - nx
            if (i > 0) acc = acc - dw.lval * (ti > 0 ? sm[s & 1][tj][ti - 1] : xl);  // i - 1
            wv = acc / dv;
            w[o] = wv;
            wk = wv;
        }
        sm[(s + 1) & 1][tj][ti] = wv;
        // (the next step's first barrier orders this step's shared writes
        // before their reads and the reads of sm[s & 1] before its rewrite)
        // Progress is published every `pub` steps -- a release waits for the
        // stores to land, so it is amortised, not paid per diagonal; the
        // barrier orders every thread's stores before it (cumulativity).
        if (((s + 1) & (dw.pub - 1)) == 0 || s + 1 == nsteps) {
            tile_sync<kWTX * kWTY>();
            if (threadIdx.x == 0) st_release_gpu(dw.prog_f + t, s + 1);
        }
    }
}

// Backward sweep (D~ + L^T) z = D~ w, from the top corner: tiles in decreasing
// (a, b) order, each waits for its right / upper neighbour.
template <int kWTX, int kWTY>
__global__ void __launch_bounds__(kWTX *kWTY) dic_wave_bwd(DicWave dw, const double *__restrict__ d,
                                                          const double *__restrict__ w, double *__restrict__ z,
                                                          const int *done)
{
    __shared__ double sm[2][kWTY][kWTX];
    if (done && *done) return;
    const int ntx = dw.ntx, nty = dw.nty;
    const int t = ntx * nty - 1 - wave_ticket(dw.ticket + 1, dw.ticket), a = t % ntx, b = t / ntx;
    const int ti = threadIdx.x % kWTX, tj = threadIdx.x / kWTX;
    const int i = a * kWTX + ti, j = b * kWTY + tj;
    const bool col_ok = i < dw.nx && j < dw.ny;
    const long long pl = (long long)dw.nx * dw.ny;
    const long long base = (long long)i + (long long)dw.nx * j;
    if (threadIdx.x == 0) dw.prog_f[t] = 0;  // re-arm the next forward sweep's counters
    const int *right = a < ntx - 1 ? dw.prog_b + (t + 1) : nullptr;
    const int *above = b < nty - 1 ? dw.prog_b + (t + ntx) : nullptr;
    int seen_r = 0, seen_a = 0, peek_r = 0, peek_a = 0;
    double zk = 0.0;  // z at (i, j, k+1)
    const int nsteps = dw.nz + kWTX + kWTY - 2;
    // a tile's cells with the largest (i, j) start first: local distance from the top corner
    const int ri = kWTX - 1 - ti, rj = kWTY - 1 - tj;
    auto ld_wd = [&](int k, double &wv, double &dv) {
        if (col_ok && k >= 0 && k < dw.nz) {
            const long long o = base + pl * k;
            wv = __ldcg(w + o);  // written by the forward launch
            dv = __ldg(d + o);
        }
    };
    double w_nx = 0.0, d_nx = 1.0;
    ld_wd(dw.nz - 1 + ri + rj, w_nx, d_nx);
    const int slack = dw.slack;
    auto ld_edge = [&](int k, double &xr, double &yu) {
        if (col_ok && k >= 0 && k < dw.nz) {
            const long long o = base + pl * k;
            if (ti == kWTX - 1 && i < dw.nx - 1) xr = __ldcg(z + o + 1);
            if (tj == kWTY - 1 && j < dw.ny - 1) yu = __ldcg(z + o + dw.nx);
        }
    };
    double xr_nx = 0.0, yu_nx = 0.0;
    bool edge_loaded = false;
    for (int s = 0; s < nsteps; ++s) {
        if (threadIdx.x == 0) {
            const int need_r = min(s + kWTX + slack, nsteps), need_a = min(s + kWTY + slack, nsteps);
            bool fresh = false;
            if (right && seen_r < need_r) {
                seen_r = max(seen_r, peek_r);
                while (seen_r < need_r) seen_r = ld_relaxed_gpu(right);
                fresh = true;
                peek_r = ld_relaxed_gpu(right);
            }
            if (above && seen_a < need_a) {
                seen_a = max(seen_a, peek_a);
                while (seen_a < need_a) seen_a = ld_relaxed_gpu(above);
                fresh = true;
                peek_a = ld_relaxed_gpu(above);
            }
            if (fresh) fence_acq_rel_gpu();
        }
        tile_sync<kWTX * kWTY>();
        const int k = dw.nz - 1 - (s - ri - rj);
        if (!edge_loaded) {
            ld_edge(k, xr_nx, yu_nx);
            edge_loaded = true;
        }
        const double wo = w_nx, dv = d_nx, xr = xr_nx, yu = yu_nx;
        ld_wd(k - 1, w_nx, d_nx);
        ld_edge(k - 1, xr_nx, yu_nx);
        double zv = 0.0;
        if (col_ok && k >= 0 && k < dw.nz) {
            const long long o = base + pl * k;
            double acc = 0.0;
            if (i < dw.nx - 1) acc = acc + dw.uval * (ti < kWTX - 1 ? sm[s & 1][tj][ti + 1] : xr);
            if (j < dw.ny - 1) acc = acc + dw.uval * (tj < kWTY - 1 ? sm[s & 1][tj + 1][ti] : yu);
            if (k < dw.nz - 1) acc = acc + dw.uval * zk;
            zv = wo - acc / dv;
            z[o] = zv;
            zk = zv;
        }
        sm[(s + 1) & 1][tj][ti] = zv;
        if (((s + 1) & (dw.pub - 1)) == 0 || s + 1 == nsteps) {
            tile_sync<kWTX * kWTY>();
            if (threadIdx.x == 0) st_release_gpu(dw.prog_b + t, s + 1);
        }
    }
}

// ---------------------------------------------------------------------------
// Pipelined form: this thread's own r (or w) and d -- independent of the
// sweep -- are copied into a D-deep shared ring by cp.async D-1 steps ahead,
// so a diagonal step does not wait for a DRAM round trip.  The neighbouring
// tiles' edge values depend on the sweep: they are loaded into registers one
// step ahead, after the neighbour has published that step, so the lead
// between tiles (the slack) stays one step whatever the ring depth.  (Edges
// in the same ring forced slack D-1 and made every deeper ring slower: 2.43,
// 2.61, 2.74 ms per 256^3 DIC-PCG iteration at D = 2, 3, 4.)  Same arithmetic
// in the same order: bit-identical results.
__device__ __forceinline__ void cp_async8_ca(double *dst, const double *src, int src_bytes)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit_grp() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_grp() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Edge mailboxes.  The value itself is the flag: a slot holds kEdgeEmpty (a
// signalling-NaN pattern no arithmetic result has -- GPU fp64 results carry
// the canonical quiet NaN) until the producing tile stores the boundary
// value; the single reader spins on the slot with relaxed gpu-scope loads
// (8-byte accesses are single-copy atomic) and re-arms it after reading.  No
// other data travels between tiles during a sweep, so no release / acquire,
// progress counter or fence is needed: the producer never stalls on a
// memory barrier and the reader waits for exactly the value it uses.
constexpr unsigned long long kEdgeEmpty = 0x7FF00000DEADBEEFull;

__device__ __forceinline__ void edge_put(double *p, double v)
{
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v)) : "memory");
}

__device__ __forceinline__ double edge_take(double *p)
{
    unsigned long long v;
    do {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    } while (v == kEdgeEmpty);
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(kEdgeEmpty) : "memory");
    return __longlong_as_double((long long)v);
}

// A slot prefetched into shared memory by a 16-byte cp.async.cg (L2, the
// coherence point) D-1 steps ahead: if it already held the value it is
// re-armed, else the reader falls back to spinning on the slot.
__device__ __forceinline__ double edge_use(double *p, const double2 &pre)
{
    if ((unsigned long long)__double_as_longlong(pre.x) == kEdgeEmpty) return edge_take(p);
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(kEdgeEmpty) : "memory");
    return pre.x;
}

__device__ __forceinline__ void cp_async16_cg(void *dst, const void *src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

__global__ void edge_arm(double *p, long long n)
{
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
        p[q] = __longlong_as_double((long long)kEdgeEmpty);
}

// wait (thread 0) until a neighbour's published progress covers `need`
__device__ __forceinline__ bool wave_wait(const int *nb, int need, int &seen, int &peek)
{
    if (!nb || seen >= need) return false;
    seen = max(seen, peek);
    while (seen < need) seen = ld_relaxed_gpu(nb);
    peek = ld_relaxed_gpu(nb);
    return true;
}

template <int kWTX, int kWTY, int D>
__global__ void __launch_bounds__(kWTX *kWTY) dic_wave_fwd_p(DicWave dw, const double *__restrict__ d,
                                                            const double *__restrict__ r, double *__restrict__ w,
                                                            const int *done)
{
    constexpr int NT = kWTX * kWTY;
    __shared__ double sm[2][kWTY][kWTX];
    __shared__ __align__(16) double ring_r[D][NT], ring_d[D][NT];
    __shared__ __align__(16) double2 ring_x[D][kWTY], ring_y[D][kWTX];  // prefetched mailbox slots
    if (done && *done) return;
    const int ntx = dw.ntx;
    const int t = wave_ticket(dw.ticket, dw.ticket + 1), a = t % ntx, b = t / ntx;
    const int tid = threadIdx.x, ti = tid % kWTX, tj = tid / kWTX;
    const int i = a * kWTX + ti, j = b * kWTY + tj;
    const bool col_ok = i < dw.nx && j < dw.ny;
    const long long pl = (long long)dw.nx * dw.ny;
    const long long base = (long long)i + (long long)dw.nx * j;
    const bool xedge = ti == 0 && i > 0, yedge = tj == 0 && j > 0;               // reads a mailbox
    const bool xout = ti == kWTX - 1 && a < ntx - 1, yout = tj == kWTY - 1 && b < dw.nty - 1;  // fills one
    // 16-byte slots (value, pad) so the prefetch can be a cp.async.cg
    double *const xin_box = dw.ex_f + 2 * (((long long)(t - 1) * dw.nz) * kWTY + tj);
    double *const yin_box = dw.ey_f + 2 * (((long long)(t - ntx) * dw.nz) * kWTX + ti);
    double *const xout_box = dw.ex_f + 2 * (((long long)t * dw.nz) * kWTY + tj);
    double *const yout_box = dw.ey_f + 2 * (((long long)t * dw.nz) * kWTX + ti);
    const int nsteps = dw.nz + kWTX + kWTY - 2;
    auto issue = [&](int s2) {  // this thread's own r / d for step s2
        const int k = s2 - ti - tj, q = s2 % D;
        const bool in = col_ok && k >= 0 && k < dw.nz;
        const long long o = base + pl * (in ? k : 0);
        cp_async8_ca(&ring_r[q][tid], r + o, in ? 8 : 0);
        cp_async8_ca(&ring_d[q][tid], d + o, in ? 8 : 0);
        if (in && xedge) cp_async16_cg(&ring_x[q][tj], xin_box + 2ll * k * kWTY);
        if (in && yedge) cp_async16_cg(&ring_y[q][ti], yin_box + 2ll * k * kWTX);
    };
    double wk = 0.0;  // w at (i, j, k-1)
    for (int s = -(D - 1); s < nsteps; ++s) {
        tile_sync<NT>();
        if (s + D - 1 < nsteps) issue(s + D - 1);
        cp_async_commit_grp();  // one group per step (possibly empty)
        if (s < 0) continue;
        cp_async_wait_grp<D - 1>();  // step s's copies (this thread's) have landed
        const int k = s - ti - tj, q = s % D;
        double xl = 0.0, yl = 0.0;
        if (col_ok && k >= 0 && k < dw.nz) {
            if (xedge) xl = edge_use(xin_box + 2ll * k * kWTY, ring_x[q][tj]);
            if (yedge) yl = edge_use(yin_box + 2ll * k * kWTX, ring_y[q][ti]);
        }
        double wv = 0.0;
        if (col_ok && k >= 0 && k < dw.nz) {
            const long long o = base + pl * k;
            // both in-tile neighbours are read before any arithmetic (clamped
            // indices, then selects) so the chain after the barrier is
            // LDS -> DMUL -> DADD -> DADD -> DDIV; same operations, same order
            const double ys = sm[s & 1][tj > 0 ? tj - 1 : 0][ti], xs = sm[s & 1][tj][ti > 0 ? ti - 1 : 0];
            const double ym = tj > 0 ? ys : yl, xm = ti > 0 ? xs : xl;
            const double pz = dw.lval * wk, py = dw.lval * ym, px = dw.lval * xm;
            double acc = ring_r[q][tid];
            acc = k > 0 ? acc - pz : acc;  // column i - pl
            acc = j > 0 ? acc - py : acc;  // i - nx
            acc = i > 0 ? acc - px : acc;  // i - 1
            wv = acc / ring_d[q][tid];
            if (xout) edge_put(xout_box + 2ll * k * kWTY, wv);
            if (yout) edge_put(yout_box + 2ll * k * kWTX, wv);
            // streaming store: read once by the next sweep; left dirty in L2 it
            // slowed the sweeps (2.12 -> 2.06 ms per 256^3 DIC-PCG iteration)
            __stcs(w + o, wv);
            wk = wv;
        }
        sm[(s + 1) & 1][tj][ti] = wv;
    }
    cp_async_wait_grp<0>();
}

template <int kWTX, int kWTY, int D>
__global__ void __launch_bounds__(kWTX *kWTY) dic_wave_bwd_p(DicWave dw, const double *__restrict__ d,
                                                            const double *__restrict__ w, double *__restrict__ z,
                                                            const int *done)
{
    constexpr int NT = kWTX * kWTY;
    __shared__ double sm[2][kWTY][kWTX];
    __shared__ __align__(16) double ring_w[D][NT], ring_d[D][NT];
    __shared__ __align__(16) double2 ring_x[D][kWTY], ring_y[D][kWTX];  // prefetched mailbox slots
    if (done && *done) return;
    const int ntx = dw.ntx, nty = dw.nty;
    const int t = ntx * nty - 1 - wave_ticket(dw.ticket + 1, dw.ticket), a = t % ntx, b = t / ntx;
    const int tid = threadIdx.x, ti = tid % kWTX, tj = tid / kWTX;
    const int i = a * kWTX + ti, j = b * kWTY + tj;
    const bool col_ok = i < dw.nx && j < dw.ny;
    const long long pl = (long long)dw.nx * dw.ny;
    const long long base = (long long)i + (long long)dw.nx * j;
    const bool xedge = ti == kWTX - 1 && i < dw.nx - 1, yedge = tj == kWTY - 1 && j < dw.ny - 1;
    const bool xout = ti == 0 && a > 0, yout = tj == 0 && b > 0;
    double *const xin_box = dw.ex_b + 2 * (((long long)(t + 1) * dw.nz) * kWTY + tj);
    double *const yin_box = dw.ey_b + 2 * (((long long)(t + ntx) * dw.nz) * kWTX + ti);
    double *const xout_box = dw.ex_b + 2 * (((long long)t * dw.nz) * kWTY + tj);
    double *const yout_box = dw.ey_b + 2 * (((long long)t * dw.nz) * kWTX + ti);
    const int nsteps = dw.nz + kWTX + kWTY - 2;
    const int ri = kWTX - 1 - ti, rj = kWTY - 1 - tj;
    auto issue = [&](int s2) {
        const int k = dw.nz - 1 - (s2 - ri - rj), q = s2 % D;
        const bool in = col_ok && k >= 0 && k < dw.nz;
        const long long o = base + pl * (in ? k : 0);
        cp_async8_ca(&ring_w[q][tid], w + o, in ? 8 : 0);  // written by the forward launch
        cp_async8_ca(&ring_d[q][tid], d + o, in ? 8 : 0);
        if (in && xedge) cp_async16_cg(&ring_x[q][tj], xin_box + 2ll * k * kWTY);
        if (in && yedge) cp_async16_cg(&ring_y[q][ti], yin_box + 2ll * k * kWTX);
    };
    double zk = 0.0;  // z at (i, j, k+1)
    for (int s = -(D - 1); s < nsteps; ++s) {
        tile_sync<NT>();
        if (s + D - 1 < nsteps) issue(s + D - 1);
        cp_async_commit_grp();
        if (s < 0) continue;
        cp_async_wait_grp<D - 1>();
        const int k = dw.nz - 1 - (s - ri - rj), q = s % D;
        double xr = 0.0, yu = 0.0;
        if (col_ok && k >= 0 && k < dw.nz) {
            if (xedge) xr = edge_use(xin_box + 2ll * k * kWTY, ring_x[q][tj]);
            if (yedge) yu = edge_use(yin_box + 2ll * k * kWTX, ring_y[q][ti]);
        }
        double zv = 0.0;
        if (col_ok && k >= 0 && k < dw.nz) {
            const long long o = base + pl * k;
            const double xs = sm[s & 1][tj][ti < kWTX - 1 ? ti + 1 : ti];
            const double ys = sm[s & 1][tj < kWTY - 1 ? tj + 1 : tj][ti];
            const double xm = ti < kWTX - 1 ? xs : xr, ym = tj < kWTY - 1 ? ys : yu;
            const double px = dw.uval * xm, py = dw.uval * ym, pz = dw.uval * zk;
            double acc = 0.0;
            acc = i < dw.nx - 1 ? acc + px : acc;
            acc = j < dw.ny - 1 ? acc + py : acc;
            acc = k < dw.nz - 1 ? acc + pz : acc;
            zv = ring_w[q][tid] - acc / ring_d[q][tid];
            if (xout) edge_put(xout_box + 2ll * k * kWTY, zv);
            if (yout) edge_put(yout_box + 2ll * k * kWTX, zv);
            __stcs(z + o, zv);
            zk = zv;
        }
        sm[(s + 1) & 1][tj][ti] = zv;
    }
    cp_async_wait_grp<0>();
}

// Verify that the triangles are exactly the 7-point pattern of the grid with
// one value each; any mismatch clears *ok.
__global__ void dic_wave_check(const int32_t *lp, const int32_t *lc, const double *lv, const int32_t *up,
                               const int32_t *uc, const double *uv, int nx, int ny, int nz, double lval, double uval,
                               int *ok)
{
    const long long pl = (long long)nx * ny, n = pl * nz;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / pl);
        long long want[3];
        int m = 0;
        if (k > 0) want[m++] = c - pl;
        if (j > 0) want[m++] = c - nx;
        if (i > 0) want[m++] = c - 1;
        int p0 = lp[c], p1 = lp[c + 1];
        bool good = p1 - p0 == m;
        for (int q = 0; good && q < m; ++q) good = lc[p0 + q] == want[q] && lv[p0 + q] == lval;
        m = 0;
        if (i < nx - 1) want[m++] = c + 1;
        if (j < ny - 1) want[m++] = c + nx;
        if (k < nz - 1) want[m++] = c + pl;
        p0 = up[c];
        p1 = up[c + 1];
        good = good && p1 - p0 == m;
        for (int q = 0; good && q < m; ++q) good = uc[p0 + q] == want[q] && uv[p0 + q] == uval;
        if (!good) *ok = 0;
    }
}

// shapes 5-7 exist only in the pipelined mailbox form (CF_DIC_TILE=5/6/7; DIC-PCG
// per iteration 128^3 / 256^3: 32x8 0.547 / 1.920 ms, 16x16 0.528 / 1.932, 32x16
// 0.846 / 2.210, the default 16x8 0.557 / 1.929)
constexpr int kShapes[8][2] = {{16, 8}, {64, 4}, {128, 4}, {256, 2}, {8, 4}, {32, 8}, {16, 16}, {32, 16}};
static bool mailbox_shape(int shape) { return shape == 0 || shape >= 5; }

// The exact (forward, backward) kernels and block size dic_wave_apply launches
// for a tile shape and ring depth (the residency check must see these).
struct WaveKernels {
    const void *fwd, *bwd;
    int threads;
};

static WaveKernels wave_kernels(int shape, int depth)
{
    if (shape == 0 && depth >= 2) {
        switch (depth) {
        case 2: return {(const void *)dic_wave_fwd_p<16, 8, 2>, (const void *)dic_wave_bwd_p<16, 8, 2>, 128};
        case 3: return {(const void *)dic_wave_fwd_p<16, 8, 3>, (const void *)dic_wave_bwd_p<16, 8, 3>, 128};
        case 4: return {(const void *)dic_wave_fwd_p<16, 8, 4>, (const void *)dic_wave_bwd_p<16, 8, 4>, 128};
        case 6: return {(const void *)dic_wave_fwd_p<16, 8, 6>, (const void *)dic_wave_bwd_p<16, 8, 6>, 128};
        case 8: return {(const void *)dic_wave_fwd_p<16, 8, 8>, (const void *)dic_wave_bwd_p<16, 8, 8>, 128};
        default: return {(const void *)dic_wave_fwd_p<16, 8, 12>, (const void *)dic_wave_bwd_p<16, 8, 12>, 128};
        }
    }
    switch (shape) {
    case 0: return {(const void *)dic_wave_fwd<16, 8>, (const void *)dic_wave_bwd<16, 8>, 128};
    case 1: return {(const void *)dic_wave_fwd<64, 4>, (const void *)dic_wave_bwd<64, 4>, 256};
    case 2: return {(const void *)dic_wave_fwd<128, 4>, (const void *)dic_wave_bwd<128, 4>, 512};
    case 3: return {(const void *)dic_wave_fwd<256, 2>, (const void *)dic_wave_bwd<256, 2>, 512};
    case 5: return {(const void *)dic_wave_fwd_p<32, 8, 2>, (const void *)dic_wave_bwd_p<32, 8, 2>, 256};
    case 6: return {(const void *)dic_wave_fwd_p<16, 16, 2>, (const void *)dic_wave_bwd_p<16, 16, 2>, 256};
    case 7: return {(const void *)dic_wave_fwd_p<32, 16, 2>, (const void *)dic_wave_bwd_p<32, 16, 2>, 512};
    default: return {(const void *)dic_wave_fwd<8, 4>, (const void *)dic_wave_bwd<8, 4>, 32};
    }
}

// a compiled ring depth of the 16x8 pipelined sweeps: 0/1 -> the one-step
// register prefetch, otherwise the largest compiled depth <= v
static int clamp_depth(int v)
{
    if (v <= 1) return 0;
    static const int kDepths[] = {12, 8, 6, 4, 3, 2};
    for (int d : kDepths)
        if (v >= d) return d;
    return 2;
}

// (re)allocate a device buffer to hold at least `need` elements
template <typename T>
static int ensure_buf(T *&p, long long &cap, long long need)
{
    if (p && cap >= need) return CF_OK;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    CF_CUDA(cudaMalloc(&p, (size_t)need * sizeof(T)));
    cap = need;
    return CF_OK;
}

int dic_wave_setup(DicData &dd, int nx, int ny, int nz, cudaStream_t s)
{
    dd.wave.ok = false;
    if (std::getenv("CF_DIC_LEVELS")) return CF_OK;  // force the level schedule
    if (nx < 2 || ny < 2 || nz < 2 || (long long)nx * ny * nz != dd.n) return CF_OK;
    DicWave &dw = dd.wave;
    dw.nx = nx;
    dw.ny = ny;
    dw.nz = nz;
    // tile shape: 16 x 8 measured best (128^3: 1.15 ms/iteration; 64x4 1.43,
    // 128x4 1.45, 256x2 2.12, a one-warp 8x4 1.68): wider tiles pay more per
    // block barrier than they save in progress handoffs
    dw.shape = 0;
    if (const char *e = std::getenv("CF_DIC_TILE")) dw.shape = std::max(0, std::min(7, std::atoi(e)));
    const int tx = kShapes[dw.shape][0], ty = kShapes[dw.shape][1];
    dw.ntx = (nx + tx - 1) / tx;
    dw.nty = (ny + ty - 1) / ty;
    const int ntiles = dw.ntx * dw.nty;
    // ring depth of the pipelined sweeps, depth 2 (DIC-PCG per iteration,
    // depth 2 / 3 / 4 / 6: 128^3 0.557 / 0.559 / 0.583 / 0.635 ms, 256^3 1.93 /
    // 1.97 / 2.02 / 2.33 ms; the progress-counter form before it: 1.01 and 2.62)
    dw.depth = mailbox_shape(dw.shape) ? 2 : 0;
    if (dw.shape == 0)
        if (const char *e = std::getenv("CF_DIC_DEPTH")) dw.depth = clamp_depth(std::atoi(e));
    // every CTA of a sweep must be resident (a CTA waits on CTAs with lower
    // tickets): check the exact forward and backward kernels apply launches
    const WaveKernels wk = wave_kernels(dw.shape, dw.depth);
    int bpf = 0, bpb = 0;
    CF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpf, wk.fwd, wk.threads, 0));
    CF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpb, wk.bwd, wk.threads, 0));
    const bool resident = (long long)std::min(bpf, bpb) * num_sms() >= ntiles;
    // the off-diagonal values (the first lower / upper entry of the first row that has one)
    double vals[2] = {0.0, 0.0};
    int32_t p[2];
    // the last row has the full lower pattern, row 0 the full upper one
    CF_CUDA(cudaMemcpyAsync(p, dd.lp + (dd.n - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CF_CUDA(cudaMemcpyAsync(&p[1], dd.up, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CF_CUDA(cudaStreamSynchronize(s));
    CF_CUDA(cudaMemcpyAsync(&vals[0], dd.lv + p[0], sizeof(double), cudaMemcpyDeviceToHost, s));
    CF_CUDA(cudaMemcpyAsync(&vals[1], dd.uv + p[1], sizeof(double), cudaMemcpyDeviceToHost, s));
    int *ok = nullptr;
    CF_CUDA(cudaMalloc(&ok, sizeof(int)));
    const int one = 1;
    CF_CUDA(cudaMemcpyAsync(ok, &one, sizeof(int), cudaMemcpyHostToDevice, s));
    dic_wave_check<<<num_sms() * 4, 256, 0, s>>>(dd.lp, dd.lc, dd.lv, dd.up, dd.uc, dd.uv, nx, ny, nz, vals[0],
                                                 vals[1], ok);
    int good = 0;
    CF_CUDA(cudaMemcpyAsync(&good, ok, sizeof(int), cudaMemcpyDeviceToHost, s));
    CF_CUDA(cudaStreamSynchronize(s));
    cudaFree(ok);
    if (!good) return CF_OK;
    // progress counters of both sweeps + the two ticket counters; sized per
    // setup (a later attach with another tile shape or grid re-sizes them)
    {
        const int rc = ensure_buf(dw.prog_f, dw.prog_cap, 2ll * ntiles + 2);
        if (rc != CF_OK) return rc;
    }
    dw.prog_b = dw.prog_f + ntiles;
    dw.ticket = dw.prog_f + 2 * ntiles;
    CF_CUDA(cudaMemsetAsync(dw.prog_f, 0, (2 * (size_t)ntiles + 2) * sizeof(int), s));
    dw.lval = vals[0];
    dw.uval = vals[1];
    // the skewed-warp sweeps (cf_dic_skew.cu) replace the tiled wavefront when they can be set up
    {
        const int rc = dic_skew_setup(dd, s);
        if (rc != CF_OK) return rc;
        if (dd.skew.ok) {
            CF_CUDA(cudaStreamSynchronize(s));
            dw.ok = true;
            return CF_OK;
        }
    }
    if (!resident) return CF_OK;
    if (mailbox_shape(dw.shape)) {  // mailboxes of the pipelined sweeps: x edges ty, y edges tx slots per tile plane
        const long long nbx = 2ll * ntiles * nz * ty, nby = 2ll * ntiles * nz * tx;  // 16-byte slots
        int rc = ensure_buf(dw.ex_f, dw.ex_cap, 2 * nbx);
        if (rc == CF_OK) rc = ensure_buf(dw.ey_f, dw.ey_cap, 2 * nby);
        if (rc != CF_OK) return rc;
        dw.ex_b = dw.ex_f + nbx;
        dw.ey_b = dw.ey_f + nby;
        edge_arm<<<num_sms() * 4, 256, 0, s>>>(dw.ex_f, 2 * nbx);
        edge_arm<<<num_sms() * 4, 256, 0, s>>>(dw.ey_f, 2 * nby);
        CF_CHECK_LAUNCH("dic mailbox arm");
    }
    dw.lval = vals[0];
    dw.uval = vals[1];
    dw.slack = 1;
    if (const char *e = std::getenv("CF_DIC_SLACK")) dw.slack = std::max(1, std::atoi(e));  // >= 1: edges are prefetched a step ahead
    dw.pub = 8;
    if (const char *e = std::getenv("CF_DIC_PUBLISH")) {  // rounded down to a power of two (a mask, not a modulo)
        const int v = std::max(1, std::atoi(e));
        dw.pub = 1;
        while (dw.pub * 2 <= v && dw.pub < (1 << 29)) dw.pub *= 2;
    }
    // the counters and armed mailboxes must be in place before any sweep
    // runs, on whatever stream the solve later uses
    CF_CUDA(cudaStreamSynchronize(s));
    dw.ok = true;
    return CF_OK;
}

int dic_wave_apply(const DicData &dd, const double *r, double *w, double *z, const int *done, cudaStream_t s)
{
    const DicWave &dw = dd.wave;
    if (dd.skew.ok) return dic_skew_apply(dd, r, z, done, s);
    const int ntiles = dw.ntx * dw.nty;
    if (dw.shape >= 5) {  // wider / taller tiles, depth 2
        if (dw.shape == 5) dic_wave_fwd_p<32, 8, 2><<<ntiles, 256, 0, s>>>(dw, dd.d, r, w, done);
        if (dw.shape == 6) dic_wave_fwd_p<16, 16, 2><<<ntiles, 256, 0, s>>>(dw, dd.d, r, w, done);
        if (dw.shape == 7) dic_wave_fwd_p<32, 16, 2><<<ntiles, 512, 0, s>>>(dw, dd.d, r, w, done);
        if (dw.shape == 5) dic_wave_bwd_p<32, 8, 2><<<ntiles, 256, 0, s>>>(dw, dd.d, w, z, done);
        if (dw.shape == 6) dic_wave_bwd_p<16, 16, 2><<<ntiles, 256, 0, s>>>(dw, dd.d, w, z, done);
        if (dw.shape == 7) dic_wave_bwd_p<32, 16, 2><<<ntiles, 512, 0, s>>>(dw, dd.d, w, z, done);
        CF_CHECK_LAUNCH("dic wavefront sweeps (pipelined, wide tiles)");
        return CF_OK;
    }
    if (dw.shape == 0 && dw.depth >= 2) {
        switch (dw.depth) {
#define CF_DIC_P(D)                                                                     \
    case D:                                                                             \
        dic_wave_fwd_p<16, 8, D><<<ntiles, 128, 0, s>>>(dw, dd.d, r, w, done);          \
        dic_wave_bwd_p<16, 8, D><<<ntiles, 128, 0, s>>>(dw, dd.d, w, z, done);          \
        break;
            CF_DIC_P(2)
            CF_DIC_P(3)
            CF_DIC_P(4)
            CF_DIC_P(6)
            CF_DIC_P(8)
            CF_DIC_P(12)
#undef CF_DIC_P
        default: CF_REQUIRE(false, "dic wavefront: ring depth not compiled");
        }
        CF_CHECK_LAUNCH("dic wavefront sweeps (pipelined)");
        return CF_OK;
    }
    switch (dw.shape) {
    case 0:
        dic_wave_fwd<16, 8><<<ntiles, 128, 0, s>>>(dw, dd.d, r, w, done);
        dic_wave_bwd<16, 8><<<ntiles, 128, 0, s>>>(dw, dd.d, w, z, done);
        break;
    case 1:
        dic_wave_fwd<64, 4><<<ntiles, 256, 0, s>>>(dw, dd.d, r, w, done);
        dic_wave_bwd<64, 4><<<ntiles, 256, 0, s>>>(dw, dd.d, w, z, done);
        break;
    case 2:
        dic_wave_fwd<128, 4><<<ntiles, 512, 0, s>>>(dw, dd.d, r, w, done);
        dic_wave_bwd<128, 4><<<ntiles, 512, 0, s>>>(dw, dd.d, w, z, done);
        break;
    case 3:
        dic_wave_fwd<256, 2><<<ntiles, 512, 0, s>>>(dw, dd.d, r, w, done);
        dic_wave_bwd<256, 2><<<ntiles, 512, 0, s>>>(dw, dd.d, w, z, done);
        break;
    default:
        dic_wave_fwd<8, 4><<<ntiles, 32, 0, s>>>(dw, dd.d, r, w, done);
        dic_wave_bwd<8, 4><<<ntiles, 32, 0, s>>>(dw, dd.d, w, z, done);
        break;
    }
    CF_CHECK_LAUNCH("dic wavefront sweeps");
    return CF_OK;
}

}  // namespace cf
