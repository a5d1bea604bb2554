// cf_tma_march.cuh -- the staged z-march device loops (see cf_tma.cuh).
//
// Tile 32 x 16 cells, 256 threads: a thread owns the x-adjacent cell pair
// (i, i+1) of one tile row, so shared-memory operands move as 16-byte
// LDS.128/STS.128 and results as 16-byte global stores, and the per-plane
// control overhead is paid once per two cells.  Pairs never straddle the
// x walls because the TMA path requires an even nx.
#pragma once

#include "cf_stencil.cuh"
#include "cf_tma.cuh"

namespace cf {

constexpr int kPairs = kTTX / 2;              // pair-columns per tile row
constexpr int kPThreads = kPairs * kTTY;      // 256
constexpr int kBox = kHX * kHY;               // halo box, doubles (648)
constexpr int kBoxStride = 656;               // padded to a 128-byte multiple
constexpr int kInt = kTTX * kTTY;             // interior box, doubles (512)
constexpr uint32_t kBoxBytes = kBox * 8;
constexpr uint32_t kIntBytes = kInt * 8;

// (Offset arithmetic on the shared array itself, so the compiler keeps the
// pointer in the shared window and emits LDS/STS, not generic LD/ST.)
__device__ __forceinline__ double *aligned_smem(unsigned char *raw)
{
    return reinterpret_cast<double *>(raw + ((128u - (smem_u32(raw) & 127u)) & 127u));
}

__device__ __forceinline__ double2 ld2(const double *p) { return *reinterpret_cast<const double2 *>(p); }
__device__ __forceinline__ void st2(double *p, double a, double b) { *reinterpret_cast<double2 *>(p) = make_double2(a, b); }

// Block coordinates of the staged march: blockIdx.x = chunk * ntiles + tile.
struct MarchCoords {
    int tx2, ty;        // pair column, tile row
    int x0, y0, z0, z1; // tile origin and owned planes [z0, z1)
    int zlo, zhi;       // lowest / highest plane present in memory
    int zs, nplanes;    // staged planes zs .. zs+nplanes-1
    int bx0, by0;       // halo-box origin (x 16-byte aligned, clamped at 0)
    int i, j;           // first cell of the pair
    bool valid;
    int o;              // smem offset of cell (i, j) in a halo box
};

__device__ __forceinline__ MarchCoords march_coords(const TmaGeom &g, int bid)
{
    MarchCoords m;
    const int tid = threadIdx.x;
    m.tx2 = tid % kPairs;
    m.ty = tid / kPairs;
    const int ntiles = g.ntx * g.nty;
    const int tile = bid % ntiles, chunk = bid / ntiles;
    m.x0 = (tile % g.ntx) * kTTX;
    m.y0 = (tile / g.ntx) * kTTY;
    m.z0 = (int)((long long)g.nz * chunk / g.nchunk);
    m.z1 = (int)((long long)g.nz * (chunk + 1) / g.nchunk);
    m.zlo = g.lo_halo ? -1 : 0;
    m.zhi = g.hi_halo ? g.nz : g.nz - 1;
    m.zs = max(m.z0 - 1, m.zlo);
    m.nplanes = min(m.z1, m.zhi) - m.zs + 1;
    m.bx0 = max(m.x0 - 2, 0);
    m.by0 = max(m.y0 - 1, 0);
    m.i = m.x0 + 2 * m.tx2;
    m.j = m.y0 + m.ty;
    m.valid = m.i < g.nx && m.j < g.ny;
    m.o = (m.j - m.by0) * kHX + (m.i - m.bx0);
    return m;
}

__device__ __forceinline__ MarchCoords march_coords(const TmaGeom &g) { return march_coords(g, blockIdx.x); }

__device__ __forceinline__ void init_bars(uint64_t *bars)
{
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
}

// A(pair) for one plane: centre pair c, x-outer neighbours xl (of cell i) and
// xr (of cell i+1), y pairs ym/yp, z pairs zm/zp.  FAST: every neighbour
// exists (no masking); otherwise the existence flags drop missing terms.
template <int ORDER, bool FAST>
__device__ __forceinline__ void stencil_pair(double2 c, double xl, double xr, double2 ym, double2 yp, double2 zm,
                                             double2 zp, bool hxl, bool hxr, bool hym, bool hyp, bool hzm, bool hzp,
                                             double off, double diag, double &a0, double &a1)
{
    if (FAST) {
        a0 = stencil7<ORDER>(c.x, xl, c.y, ym.x, yp.x, zm.x, zp.x, true, true, true, true, true, true, off, diag);
        a1 = stencil7<ORDER>(c.y, c.x, xr, ym.y, yp.y, zm.y, zp.y, true, true, true, true, true, true, off, diag);
    } else {
        a0 = stencil7<ORDER>(c.x, xl, c.y, ym.x, yp.x, zm.x, zp.x, hxl, true, hym, hyp, hzm, hzp, off, diag);
        a1 = stencil7<ORDER>(c.y, c.x, xr, ym.y, yp.y, zm.y, zp.y, true, hxr, hym, hyp, hzm, hzp, off, diag);
    }
}

// Operand staged as-is (update / apply).  Pol: issue(slot, m, z, bar) on
// thread 0; epi(slot, m, z, c, a0, a1) for each owned pair.  The pair's own
// column at z-1, z, z+1 lives in registers; in-plane neighbours come from the
// slot of plane z; slot z is recycled once every thread has used it.
template <int ORDER, class Pol>
__device__ __forceinline__ void staged_pair_march(const TmaGeom &g, double off, double diag, Pol &pol,
                                                  uint64_t *bars)
{
    const MarchCoords m = march_coords(g);
    init_bars(bars);
    if (threadIdx.x == 0) {
        pol.prefetch();
        for (int q = 0; q < min(kStages, m.nplanes); ++q) pol.issue(q % kStages, m, m.zs + q, &bars[q % kStages]);
    }
    const bool hxl = m.i > 0, hxr = m.i + 2 < g.nx, hym = m.j > 0, hyp = m.j < g.ny - 1;
    const bool inplane_fast = hxl && hxr && hym && hyp;
    auto wait = [&](int q) { mbar_wait(&bars[q % kStages], (uint32_t)((q / kStages) & 1)); };
    auto release = [&](int q) {
        fence_proxy_async_smem();  // my reads of slot q before its TMA refill
        __syncthreads();
        if (threadIdx.x == 0 && q + kStages < m.nplanes)
            pol.issue(q % kStages, m, m.zs + q + kStages, &bars[q % kStages]);
    };
    int q = 0;
    double2 cprev = make_double2(0.0, 0.0);
    wait(0);
    if (m.zs < m.z0) {
        cprev = ld2(pol.box(0) + m.o);
        release(0);
        q = 1;
        wait(1);
    }
    double2 ccur = ld2(pol.box(q % kStages) + m.o);
    for (int z = m.z0; z < m.z1; ++z, ++q) {
        const bool hzm = z - 1 >= m.zlo, hzp = z + 1 <= m.zhi;
        double2 cnext = make_double2(0.0, 0.0);
        if (hzp) {
            wait(q + 1);
            cnext = ld2(pol.box((q + 1) % kStages) + m.o);
        }
        const int s = q % kStages;
        if (m.valid) {
            const double *b = pol.box(s) + m.o;
            // (wall-side neighbours are not read: at x0 = 0 / y0 = 0 they would
            // fall before the box)
            const double xl = hxl ? b[-1] : 0.0, xr = hxr ? b[2] : 0.0;
            const double2 zero = make_double2(0.0, 0.0);
            const double2 ym = hym ? ld2(b - kHX) : zero, yp = hyp ? ld2(b + kHX) : zero;
            double a0, a1;
            if (inplane_fast && hzm && hzp)
                stencil_pair<ORDER, true>(ccur, xl, xr, ym, yp, cprev, cnext, true, true, true, true, true, true, off,
                                          diag, a0, a1);
            else
                stencil_pair<ORDER, false>(ccur, xl, xr, ym, yp, cprev, cnext, hxl, hxr, hym, hyp, hzm, hzp, off,
                                           diag, a0, a1);
            pol.epi(s, m, z, ccur, a0, a1);
        }
        release(q);
        cprev = ccur;
        ccur = cnext;
    }
}

// ---------------------------------------------------------------------------
// Warp-specialised form: warps 0..7 consume (one cell pair per thread as
// above), warp 8 is the TMA producer.  Each stage slot has a `full` barrier
// (TMA transaction bytes) and an `empty` barrier (one arrival per consumer
// warp, after a proxy fence), so consumer warps never wait for each other --
// there is no block-wide barrier inside the plane loop.
constexpr int kConsumerWarps = kPThreads / 32;
constexpr int kWSThreads = kPThreads + 32;

template <int S = kStages>
__device__ __forceinline__ void init_ws_bars(uint64_t *full, uint64_t *empty)
{
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        fence_barrier_init();
    }
    __syncthreads();
}

// Producer loop (run by one elected lane of warp 8).
template <class Issue, int S = kStages>
__device__ __forceinline__ void ws_produce(int nplanes, uint64_t *full, uint64_t *empty, Issue issue)
{
    for (int q = 0; q < nplanes; ++q) {
        const int s = q % S;
        if (q >= S) mbar_wait(&empty[s], (uint32_t)(((q / S) - 1) & 1));
        issue(q, s, &full[s]);
    }
}

// Consumer: this warp is done with slot q.
template <int S = kStages>
__device__ __forceinline__ void ws_release(uint64_t *empty, int q)
{
    fence_proxy_async_smem();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[q % S]);
}

// Consumer march over the block's planes.  Pol: value(slot, offset) ->
// operand at a box offset (may compute it), box geometry as in
// staged_pair_march; epi(slot, m, z, centre pair, a0, a1).
template <int ORDER, class Pol, int S = kStages>
__device__ __forceinline__ void ws_consume(const TmaGeom &g, const MarchCoords &m, double off, double diag, Pol &pol,
                                           uint64_t *full, uint64_t *empty)
{
    const bool hxl = m.i > 0, hxr = m.i + 2 < g.nx, hym = m.j > 0, hyp = m.j < g.ny - 1;
    const bool inplane_fast = hxl && hxr && hym && hyp;
    auto wait = [&](int q) { mbar_wait(&full[q % S], (uint32_t)((q / S) & 1)); };
    int q = 0;
    double2 cprev = make_double2(0.0, 0.0);
    wait(0);
    if (m.zs < m.z0) {
        cprev = pol.value2(0, m.o);
        pol.halo(m, m.zs, cprev);
        ws_release<S>(empty, 0);
        q = 1;
        wait(1);
    }
    double2 ccur = pol.value2(q % S, m.o);
    const double2 zero = make_double2(0.0, 0.0);
    for (int z = m.z0; z < m.z1; ++z, ++q) {
        const bool hzm = z - 1 >= m.zlo, hzp = z + 1 <= m.zhi;
        double2 cnext = zero;
        if (hzp) {
            wait(q + 1);
            cnext = pol.value2((q + 1) % S, m.o);
            if (z + 1 == m.z1) pol.halo(m, z + 1, cnext);
        }
        const int s = q % S;
        if (m.valid) {
            double a0, a1;
            if (inplane_fast && hzm && hzp) {
                stencil_pair<ORDER, true>(ccur, pol.value(s, m.o - 1), pol.value(s, m.o + 2),
                                          pol.value2(s, m.o - kHX), pol.value2(s, m.o + kHX), cprev, cnext, true,
                                          true, true, true, true, true, off, diag, a0, a1);
            } else {
                stencil_pair<ORDER, false>(ccur, hxl ? pol.value(s, m.o - 1) : 0.0,
                                           hxr ? pol.value(s, m.o + 2) : 0.0,
                                           hym ? pol.value2(s, m.o - kHX) : zero,
                                           hyp ? pol.value2(s, m.o + kHX) : zero, cprev, cnext, hxl, hxr, hym, hyp,
                                           hzm, hzp, off, diag, a0, a1);
            }
            pol.epi(s, m, z, ccur, a0, a1);
        }
        ws_release<S>(empty, q);
        cprev = ccur;
        ccur = cnext;
    }
    // the last staged plane (z1, read as cnext) is released too
    if (q < m.nplanes) ws_release<S>(empty, q);
}

}  // namespace cf
