// cf_p2p.cu -- z-slab conjugate gradient with the collectives fused into the
// compute kernels over peer memory (SURVEY.md §5.8, §8 e).
//
// The NCCL form (cf_dist.cu) runs, per CG iteration, the two compute kernels
// plus a sum kernel, an ncclAllReduce and a scalar kernel per reduction, and
// ncclSend/Recv for the r halo.  Here each iteration is TWO kernels per GPU and
// nothing else:
//
//   direction  p = z + beta p_old (owned + halo planes), A p, local p.Ap;
//              the last block posts the slab's partial into EVERY rank's
//              mailbox (NVLink stores to the peers' device memory), waits
//              for all ranks' partials of this phase in its own mailbox, sums
//              them in rank order (identical on every rank) and sets alpha.
//   update     r -= alpha A p, x every second iteration (XM_SKIP/XM_DOUBLE),
//              local r.r; each block stores its boundary r planes straight
//              into the neighbours' halo planes (peer stores), and the last
//              block does the same post / wait / sum for r.r, r.z -> beta,
//              convergence, and the graph's loop condition.
//
// The exchange therefore overlaps the compute tile by tile (halo planes are
// written as they are produced), and a reduction costs one NVLink round trip
// instead of three launches and an NCCL call.  Mailbox slots are
// double-buffered by phase parity: a rank can run at most one phase ahead of
// any other (it cannot pass a phase's wait before every rank has posted it).
//
// Memory ordering: blocks that stored peer memory execute fence.sc.sys before
// their last-block ticket; the last block publishes its sequence number with
// st.release.sys after its values; readers poll with ld.acquire.sys.  Every
// rank sums the same values in the same order, so alpha, beta and the stop
// decision are bit-identical everywhere and all ranks leave the loop together.
//
// Ranks: one slab per process (GPU), peers' mailboxes and r arrays opened
// through CUDA IPC handles exchanged by the host (cf_pcg_export/import).
// Verification on one GPU: several slabs in ONE process are launched as ONE
// kernel over all slabs' data (blocks partitioned by slab); the "peer" pointers
// are the other slabs' arrays, so the exact protocol -- stores, fences, polls
// -- runs, with the waiting blocks of one launch (never separate launches
// waiting on each other).  At most one block per slab waits, so the other
// blocks of the launch always find SM slots.
#include <algorithm>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "cf_cg_common.cuh"
#include "cf_tma_march.cuh"

namespace cf {

#include "cf_cg_tma.cuh"
#include "cf_cg_pair.cuh"
#include "cf_cg_lean.cuh"
#include "cf_cg_spass.cuh"

constexpr int kMaxRanks = 8;

struct Mailbox {
    double val[2][kMaxRanks][3];           // [phase parity][sender][component] (3: the single pass)
    unsigned long long seq[2][kMaxRanks];  // phase number posted by each sender
};

struct P2PSlab {
    CUtensorMap m_p[2], m_ri, m_xi, m_pi[2];  // TMA update form (halo box of p; interior r, x, p_prev)
    TmaGeom gt;                              // its geometry
    int blk_updt;                            // first block of this slab in the TMA update launch
    PairGeom gd, gu;
    int blk_dir, blk_upd, blk_init;  // first block of this slab in each launch
    double *r, *x, *p0, *p1;         // owned plane 0 (halo planes at -1 / nzl)
    double *partials;
    CgTickets *tk;
    CgScalars *sc;
    double *lo_r, *hi_r;  // where this slab's bottom / top r plane goes: the lower neighbour's hi halo plane,
                          // the upper neighbour's lo halo plane (peer or local), or null
    const double *b;      // right-hand side (owned planes), for the init launch
    int rank;             // global rank of this slab
};

struct P2PSet {
    int nslab, nranks;
    Mailbox *mail[kMaxRanks];  // every rank's mailbox, by global rank
    P2PSlab s[kMaxRanks];
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// release/acquire fence at system scope (lighter than __threadfence_system's fence.sc.sys)
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ double ld_relaxed_sys(const double *p)
{
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_sys(double *p, double v)
{
    asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// Slab of this block: blocks [off_k, off_{k+1}) belong to slab k.
template <int WHICH>  // 0 init, 1 dir, 2 update (pair form), 3 update (TMA form)
__device__ __forceinline__ int slab_of(const P2PSet &ps, int &bid, int &nblk)
{
    auto off = [&](int k) {
        return WHICH == 0 ? ps.s[k].blk_init
                          : (WHICH == 1 ? ps.s[k].blk_dir : (WHICH == 2 ? ps.s[k].blk_upd : ps.s[k].blk_updt));
    };
    int k = 0;
    for (int q = 1; q < ps.nslab; ++q)
        if ((int)blockIdx.x >= off(q)) k = q;
    const int end = k + 1 < ps.nslab ? off(k + 1) : (int)gridDim.x;
    bid = blockIdx.x - off(k);
    nblk = end - off(k);
    return k;
}

// Last-block ticket over this slab's blocks.  SYS: this block stored into
// peer memory (boundary r planes), so its stores are made visible system-wide
// (fence.sc.sys) before the ticket; other blocks need only the device-scope
// fence (their data is read on this GPU only).
__device__ __forceinline__ bool last_block_sys(unsigned int *ticket, int *flag_smem, int nblk, bool sys)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        if (sys) fence_acq_rel_sys();
        else __threadfence();
        const unsigned int t = atomicAdd(ticket, 1u);
        *flag_smem = (t == (unsigned int)nblk - 1);
        if (*flag_smem) *ticket = 0u;
    }
    __syncthreads();
    const bool last = *flag_smem;
    if (last) fence_acq_rel_sys();
    return last;
}

__device__ __forceinline__ unsigned long long globaltimer_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// A peer that never posts (a crashed or diverged rank) must not hang the GPU:
// the wait gives up after kPeerTimeoutNs, stops the solve (done, status
// ST_PEER_TIMEOUT) and the host reports an error.
constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;
constexpr int ST_PEER_TIMEOUT = 4;

// Thread 0 of a slab's last block: post `v` (ncomp values) to every rank,
// wait for every rank's post of this phase, return the rank-ordered sums.
__device__ __forceinline__ void allreduce_core(int nranks, Mailbox *const *mail, CgScalars *sc, int me, int ncomp,
                                               const double *v, double *out)
{
    if (nranks == 1) {  // one rank (single-slab run): nothing to exchange
        for (int c = 0; c < ncomp; ++c) out[c] = 0.0 + v[c];
        return;
    }
    const unsigned long long ph = ++sc->phase;
    const int par = (int)(ph & 1ull);
    for (int q = 0; q < nranks; ++q)
        for (int c = 0; c < ncomp; ++c) st_relaxed_sys(&mail[q]->val[par][me][c], v[c]);
    for (int q = 0; q < nranks; ++q) st_release_sys(&mail[q]->seq[par][me], ph);
    Mailbox *mine = mail[me];
    const unsigned long long t0 = globaltimer_ns();
    for (int q = 0; q < nranks; ++q) {
        while (ld_acquire_sys(&mine->seq[par][q]) < ph) {
            __nanosleep(64);
            if (globaltimer_ns() - t0 > kPeerTimeoutNs) {
                sc->status = ST_PEER_TIMEOUT;
                sc->done = 1;
                for (int c = 0; c < ncomp; ++c) out[c] = __longlong_as_double(0x7ff8000000000000ll);
                return;
            }
        }
    }
    for (int c = 0; c < ncomp; ++c) {
        double sum = 0.0;
        for (int q = 0; q < nranks; ++q) sum = sum + ld_relaxed_sys(&mine->val[par][q][c]);
        out[c] = sum;
    }
}

__device__ __forceinline__ void p2p_allreduce(const P2PSet &ps, const P2PSlab &sl, int ncomp, const double *v,
                                              double *out)
{
    allreduce_core(ps.nranks, ps.mail, sl.sc, sl.rank, ncomp, v, out);
}

// ---------------------------------------------------------------- init
// r = b and x = 0 on the owned planes, boundary r planes into the
// neighbours' halos, |b|^2 and r.z all-reduced -> scalar_after_init.
template <int PK>
__global__ void __launch_bounds__(256) p2p_init(const P2PSet *__restrict__ psp, double zc)
{
    const P2PSet &ps = *psp;
    __shared__ double red[32];
    __shared__ int is_last;
    int bid, nblk;
    const P2PSlab &sl = ps.s[slab_of<0>(ps, bid, nblk)];
    const long long pl = (long long)sl.gd.nx * sl.gd.ny, n = pl * sl.gd.nz;
    double bb = 0.0, rz = 0.0;
    for (long long i = (long long)bid * 256 + threadIdx.x; i < n; i += (long long)nblk * 256) {
        const double bi = sl.b[i];
        sl.r[i] = bi;
        sl.x[i] = 0.0;
        if (i < pl && sl.lo_r) sl.lo_r[i] = bi;
        if (i >= n - pl && sl.hi_r) sl.hi_r[i - (n - pl)] = bi;
        bb = bb + bi * bi;
        rz = rz + bi * zval<PK>(bi, nullptr, 0, zc);
    }
    bb = block_sum<256>(bb, red);
    rz = block_sum<256>(rz, red);
    if (threadIdx.x == 0) {
        sl.partials[2 * bid] = bb;
        sl.partials[2 * bid + 1] = rz;
    }
    if (last_block_sys(&sl.tk->init, &is_last, nblk, sl.lo_r || sl.hi_r)) {
        bb = reduce_partials<256>(sl.partials, nblk, 2, red);
        rz = reduce_partials<256>(sl.partials + 1, nblk, 2, red);
        if (threadIdx.x == 0) {
            const double v[2] = {bb, rz};
            double tot[2];
            p2p_allreduce(ps, sl, 2, v, tot);
            scalar_after_init(sl.sc, tot[0], tot[1]);
        }
    }
}

// ---------------------------------------------------------------- direction
// SINGLE (one slab per GPU, the multi-GPU case): geometry and arrays also
// come as kernel parameters, so the compiler sees constant-bank geometry and
// __restrict__ pointers exactly as in the single-domain kernels; the
// multi-slab emulation reads them from the descriptor.
// direction CTAs: 4 warps x 2 rows (dir_lean2_march), 8-row tiles
constexpr int kP2PDirRows = 8;
template <int ORDER, int PK, bool SINGLE>
__global__ void __launch_bounds__(kPairThreads, 6) p2p_dir(const P2PSet *__restrict__ psp, int half, double off,
                                                          double diag, double zc, PairGeom g1,
                                                          const double *__restrict__ r1, double *__restrict__ p0_1,
                                                          double *__restrict__ p1_1)
{
    const P2PSet &ps = *psp;
    __shared__ double red[32];
    __shared__ int is_last;
    int bid, nblk;
    const P2PSlab &sl = ps.s[SINGLE ? 0 : slab_of<1>(ps, bid, nblk)];
    if (SINGLE) {
        bid = blockIdx.x;
        nblk = gridDim.x;
    }
    CgScalars *sc = sl.sc;
    if (sc->done) return;
    double pap;
    // the lean march (cf_cg_lean.cuh) at the pair geometry's 4-row tiles: the
    // same values and block partials as dir_pair_body, ~half the instructions.
    // SINGLE: r1 / p0_1 / p1_1 point at the slab's lowest plane in memory.
    if constexpr (SINGLE) {
        const double *po = half ? p1_1 : p0_1;
        double *pn = half ? p0_1 : p1_1;
        pap = sc->it == 0 ? dir_lean2_march<ORDER, PK, true, 4, true>(g1, bid, off, diag, r1, po, pn, zc, 0.0)
                          : dir_lean2_march<ORDER, PK, false, 4, true>(g1, bid, off, diag, r1, po, pn, zc, sc->beta);
    } else {
        const PairGeom g = sl.gd;
        const size_t sh = g.lo_halo ? (size_t)g.nx * g.ny : 0;
        const double *po = (half ? sl.p1 : sl.p0) - sh;
        double *pn = (half ? sl.p0 : sl.p1) - sh;
        pap = sc->it == 0
                  ? dir_lean2_march<ORDER, PK, true, 4, true>(g, bid, off, diag, sl.r - sh, po, pn, zc, 0.0)
                  : dir_lean2_march<ORDER, PK, false, 4, true>(g, bid, off, diag, sl.r - sh, po, pn, zc, sc->beta);
    }
    pap = block_sum<kPairThreads>(pap, red);
    if (threadIdx.x == 0) sl.partials[bid] = pap;
    if (last_block_sys(&sl.tk->dir, &is_last, nblk, false)) {
        pap = reduce_partials<kPairThreads>(sl.partials, nblk, 1, red);
        if (threadIdx.x == 0) {
            double tot;
            p2p_allreduce(ps, sl, 1, &pap, &tot);
            scalar_after_dir(sc, tot);
        }
    }
}

// ---------------------------------------------------------------- update
template <int ORDER, int PK, int XM>
__global__ void __launch_bounds__(kPairThreads, 8) p2p_update(const P2PSet *__restrict__ psp, int half, double off,
                                                             double diag, double zc, int use_cond,
                                                             cudaGraphConditionalHandle cond)
{
    const P2PSet &ps = *psp;
    __shared__ double red[32];
    __shared__ int is_last;
    int bid, nblk;
    const P2PSlab &sl = ps.s[slab_of<2>(ps, bid, nblk)];
    CgScalars *sc = sl.sc;
    if (sc->done) {
        if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    const PairGeom g = sl.gu;
    const PairCoords c = pair_coords(g, bid);
    const long long pl = (long long)g.nx * g.ny;
    struct Epi {
        double *r, *x, *lo_r, *hi_r;
        const double *q;
        double alpha, malpha, zc, alpha_prev;
        long long pl, top;
        double rr, rz;
        __device__ __forceinline__ void cell(long long o, double2 cc, double a0, double a1)
        {
            const double2 ro = *reinterpret_cast<const double2 *>(r + o);
            if (XM == XM_EACH) {
                const double2 xo = *reinterpret_cast<const double2 *>(x + o);
                *reinterpret_cast<double2 *>(x + o) = make_double2(xo.x + alpha * cc.x, xo.y + alpha * cc.y);
            } else if (XM == XM_DOUBLE) {  // the skipped step first, then this one
                const double2 xo = *reinterpret_cast<const double2 *>(x + o);
                const double2 qo = *reinterpret_cast<const double2 *>(q + o);
                const double x0 = xo.x + alpha_prev * qo.x, x1 = xo.y + alpha_prev * qo.y;
                *reinterpret_cast<double2 *>(x + o) = make_double2(x0 + alpha * cc.x, x1 + alpha * cc.y);
            }
            const double r0 = ro.x + malpha * a0, r1 = ro.y + malpha * a1;  // src/solver.py:155-157
            const double2 rn = make_double2(r0, r1);
            *reinterpret_cast<double2 *>(r + o) = rn;
            // boundary planes straight into the neighbours' halo planes (NVLink stores)
            if (lo_r && o < pl) *reinterpret_cast<double2 *>(lo_r + o) = rn;
            if (hi_r && o >= top) *reinterpret_cast<double2 *>(hi_r + (o - top)) = rn;
            rr = rr + r0 * r0;
            rr = rr + r1 * r1;
            if (PK != PK_ZVEC) {
                rz = rz + r0 * zval<PK>(r0, nullptr, 0, zc);
                rz = rz + r1 * zval<PK>(r1, nullptr, 0, zc);
            }
        }
        __device__ __forceinline__ void halo(long long, double2) {}
    } epi{sl.r, sl.x, sl.lo_r, sl.hi_r, half ? sl.p1 : sl.p0, sc->alpha, -sc->alpha, zc, sc->alpha_prev, pl,
          pl * (g.nz - 1), 0.0, 0.0};
    const double *p = half ? sl.p0 : sl.p1;  // this iteration's direction (written by p2p_dir)
    if (c.row_ok) pair_march<ORDER, false>(c, g, off, diag, UpdSrc{p}, epi);
    double rr = block_sum<kPairThreads>(epi.rr, red);
    double rz = block_sum<kPairThreads>(epi.rz, red);
    if (threadIdx.x == 0) {
        sl.partials[2 * bid] = rr;
        sl.partials[2 * bid + 1] = rz;
    }
    if (last_block_sys(&sl.tk->upd, &is_last, nblk,
                       (sl.lo_r && c.z0 == 0) || (sl.hi_r && c.z1 == g.nz))) {
        rr = reduce_partials<kPairThreads>(sl.partials, nblk, 2, red);
        rz = reduce_partials<kPairThreads>(sl.partials + 1, nblk, 2, red);
        if (threadIdx.x == 0) {
            const double v[2] = {rr, rz};
            double tot[2];
            p2p_allreduce(ps, sl, 2, v, tot);
            if (scalar_after_update<PK != PK_ZVEC>(sc, tot[0], tot[1]) && use_cond) cudaGraphSetConditional(cond, 0);
        }
    }
}

// update, TMA form: the single-domain pipeline (update_tma_body) with the
// boundary r planes also stored into the neighbours' halo planes
// (S: TMA ring depth; the skip-x form stages only p and r, 4 deep as in the
// single-domain loop)
template <int ORDER, int PK, int XM, bool SINGLE, int S = (XM == XM_SKIP ? 4 : kStages)>
__global__ void __launch_bounds__(kWSThreads, 4) p2p_update_tma(
    const P2PSet *__restrict__ psp, int half, double off, double diag, double zc, int use_cond,
    cudaGraphConditionalHandle cond, const __grid_constant__ CUtensorMap mp0, const __grid_constant__ CUtensorMap mp1,
    const __grid_constant__ CUtensorMap mr, const __grid_constant__ CUtensorMap mx,
    const __grid_constant__ CUtensorMap mq0, const __grid_constant__ CUtensorMap mq1, TmaGeom g1,
    double *__restrict__ r1, double *__restrict__ x1, double *__restrict__ lo1, double *__restrict__ hi1)
{
    const P2PSet &ps = *psp;
    __shared__ double red[32];
    __shared__ int is_last;
    int bid, nblk;
    const P2PSlab &sl = ps.s[SINGLE ? 0 : slab_of<3>(ps, bid, nblk)];
    if (SINGLE) {
        bid = blockIdx.x;
        nblk = gridDim.x;
    }
    CgScalars *sc = sl.sc;
    if (sc->done) {
        if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    double rr, rz;
    int nchunk, ntiles;
    if constexpr (SINGLE) {
        update_tma_body<ORDER, PK, XM, S>(half ? &mp0 : &mp1, &mr, &mx, half ? &mq1 : &mq0, g1, bid, off, diag, r1, x1,
                                       zc, sc->alpha, sc->alpha_prev, lo1, hi1, red, rr, rz);
        nchunk = g1.nchunk;
        ntiles = g1.ntx * g1.nty;
    } else {
        const TmaGeom g = sl.gt;
        update_tma_body<ORDER, PK, XM, S>(&sl.m_p[half ^ 1], &sl.m_ri, &sl.m_xi, &sl.m_pi[half], g, bid, off, diag, sl.r,
                                       sl.x, zc, sc->alpha, sc->alpha_prev, sl.lo_r, sl.hi_r, red, rr, rz);
        nchunk = g.nchunk;
        ntiles = g.ntx * g.nty;
    }
    if (threadIdx.x == 0) {
        sl.partials[2 * bid] = rr;
        sl.partials[2 * bid + 1] = rz;
    }
    const int chunk = bid / ntiles;
    const bool peer = (sl.lo_r && chunk == 0) || (sl.hi_r && chunk == nchunk - 1);
    if (last_block_sys(&sl.tk->upd, &is_last, nblk, peer)) {
        rr = reduce_partials<kWSThreads>(sl.partials, nblk, 2, red);
        rz = reduce_partials<kWSThreads>(sl.partials + 1, nblk, 2, red);
        if (threadIdx.x == 0) {
            const double v[2] = {rr, rz};
            double tot[2];
            p2p_allreduce(ps, sl, 2, v, tot);
            if (scalar_after_update<PK != PK_ZVEC>(sc, tot[0], tot[1]) && use_cond) cudaGraphSetConditional(cond, 0);
        }
    }
}

// x += alpha * p owed by a final skipping iteration (odd iteration count)
__global__ void __launch_bounds__(256) p2p_x_fixup(const P2PSet *__restrict__ psp)
{
    const P2PSet &ps = *psp;
    int bid, nblk;
    const P2PSlab &sl = ps.s[slab_of<0>(ps, bid, nblk)];
    if ((sl.sc->it & 1) == 0) return;
    const double alpha = sl.sc->alpha;
    const long long n = (long long)sl.gd.nx * sl.gd.ny * sl.gd.nz;
    for (long long i = (long long)bid * 256 + threadIdx.x; i < n; i += (long long)nblk * 256)
        sl.x[i] = sl.x[i] + alpha * sl.p1[i];  // src/solver.py:155
}


// ================================================================ single pass over z-slabs
// The default single-domain CG form (cf_cg_spass.cuh: one TMA-fed
// Chronopoulos-Gear pass per iteration, 40 N) on z-slabs.  Each slab array
// carries TWO halo planes below and above its owned planes (the pass reads
// r_k and p_{k-1} on planes z0-2 .. z1+1); the pass stores its boundary planes
// 0, 1 / nz-2, nz-1 of r_{k+1} and p_k also into the neighbours' halo planes
// (peer stores as they are produced), and the slab's last block all-reduces
// (r.r, gamma, delta) over the mailboxes -- one collective per iteration
// instead of two.  A missing neighbour's halo planes stay zero (the Dirichlet
// ghost), exactly as the single domain's out-of-range TMA boxes.
constexpr int kSpSlabTY = 16, kSpSlabS = 6;
using SpSlabCfg = Sp<kSpSlabTY, kSpSlabS, 2>;

struct SpSlab {
    CUtensorMap m_r[2], m_p[2], m_x;  // maps over the slab arrays (nz + 4 planes, the lowest halo plane first)
    SpGeom g;                         // nz = owned planes
    int blk, blk_init;                // first block of this slab in the pass / init launches
    double *r[2], *p[2], *x;          // owned plane 0 (two halo planes below it in memory)
    const double *b;
    double *lo[2][2], *hi[2][2];      // [r | p][buffer]: the neighbours' planes matching ours (null: none)
    int lo_ghost, hi_ghost;
    double *partials;
    CgTickets *tk;
    CgScalars *sc;
    int rank;
};

struct SpSet {
    int nslab, nranks;
    Mailbox *mail[kMaxRanks];
    SpSlab s[kMaxRanks];
};

template <int WHICH>  // 0 init, 1 pass
__device__ __forceinline__ int sp_slab_of(const SpSet &ps, int &bid, int &nblk)
{
    auto off = [&](int k) { return WHICH == 0 ? ps.s[k].blk_init : ps.s[k].blk; };
    int k = 0;
    for (int q = 1; q < ps.nslab; ++q)
        if ((int)blockIdx.x >= off(q)) k = q;
    const int end = k + 1 < ps.nslab ? off(k + 1) : (int)gridDim.x;
    bid = blockIdx.x - off(k);
    nblk = end - off(k);
    return k;
}

// the p2p_allreduce protocol over the single-pass descriptors
__device__ __forceinline__ void sp_allreduce(const SpSet &ps, const SpSlab &sl, int ncomp, const double *v,
                                             double *out)
{
    allreduce_core(ps.nranks, ps.mail, sl.sc, sl.rank, ncomp, v, out);
}

// init 1: r = b on the owned planes (and the boundary planes into the
// neighbours' halos), x = 0; |b|^2 all-reduced (also the point after which
// every rank's halo planes are written)
__global__ void __launch_bounds__(256) sp_init_copy(const SpSet *__restrict__ psp)
{
    const SpSet &ps = *psp;
    __shared__ double red[32];
    __shared__ int is_last;
    int bid, nblk;
    const SpSlab &sl = ps.s[sp_slab_of<0>(ps, bid, nblk)];
    const long long pl = (long long)sl.g.nx * sl.g.ny, n = pl * sl.g.nz, top = pl * (sl.g.nz - 2);
    double bb = 0.0;
    for (long long i = (long long)bid * 256 + threadIdx.x; i < n; i += (long long)nblk * 256) {
        const double bi = sl.b[i];
        sl.r[0][i] = bi;
        sl.x[i] = 0.0;
        if (i < 2 * pl && sl.lo[0][0]) sl.lo[0][0][i] = bi;
        if (i >= top && sl.hi[0][0]) sl.hi[0][0][i - top] = bi;
        bb = bb + bi * bi;
    }
    bb = block_sum<256>(bb, red);
    if (threadIdx.x == 0) sl.partials[bid] = bb;
    if (last_block_sys(&sl.tk->init, &is_last, nblk, sl.lo[0][0] || sl.hi[0][0])) {
        bb = reduce_partials<256>(sl.partials, nblk, 1, red);
        if (threadIdx.x == 0) {
            double tot;
            sp_allreduce(ps, sl, 1, &bb, &tot);
            sl.sc->rr = tot;  // |b|^2 until init 2
        }
    }
}

// init 2: gamma_0 = r.z, delta_0 = z.A z (z = M^-1 r, the halo planes of r
// from the neighbours), all-reduced -> alpha_0 (scalar_after_pass_init)
template <int PK>
__global__ void __launch_bounds__(256) sp_init_dots(const SpSet *__restrict__ psp, double off, double diag, double zc)
{
    const SpSet &ps = *psp;
    __shared__ double red[32];
    __shared__ int is_last;
    int bid, nblk;
    const SpSlab &sl = ps.s[sp_slab_of<0>(ps, bid, nblk)];
    const int nx = sl.g.nx, ny = sl.g.ny, nz = sl.g.nz;
    const long long pl = (long long)nx * ny, n = pl * nz;
    const double *r = sl.r[0];
    double gam = 0.0, dlt = 0.0;
    for (long long i = (long long)bid * 256 + threadIdx.x; i < n; i += (long long)nblk * 256) {
        const int ix = (int)(i % nx), iy = (int)((i / nx) % ny);
        const double c = sp_z<PK>(r[i], zc);
        double nb = sp_z<PK>(r[i - pl], zc) + sp_z<PK>(r[i + pl], zc);  // halo planes exist (zero at ghosts)
        if (ix > 0) nb = nb + sp_z<PK>(r[i - 1], zc);
        if (ix + 1 < nx) nb = nb + sp_z<PK>(r[i + 1], zc);
        if (iy > 0) nb = nb + sp_z<PK>(r[i - nx], zc);
        if (iy + 1 < ny) nb = nb + sp_z<PK>(r[i + nx], zc);
        const double az = __fma_rn(off, nb, diag * c);
        gam = __fma_rn(r[i], c, gam);
        dlt = __fma_rn(c, az, dlt);
    }
    gam = block_sum<256>(gam, red);
    dlt = block_sum<256>(dlt, red);
    if (threadIdx.x == 0) {
        sl.partials[2 * bid] = gam;
        sl.partials[2 * bid + 1] = dlt;
    }
    if (last_block_sys(&sl.tk->dir, &is_last, nblk, false)) {
        gam = reduce_partials<256>(sl.partials, nblk, 2, red);
        dlt = reduce_partials<256>(sl.partials + 1, nblk, 2, red);
        if (threadIdx.x == 0) {
            const double v[2] = {gam, dlt};
            double tot[2];
            sp_allreduce(ps, sl, 2, v, tot);
            scalar_after_pass_init(sl.sc, sl.sc->rr, tot[0], tot[1]);
        }
    }
}

// one pass over every slab: half 0 reads r[0], p[0] and writes r[1], p[1]
// (x skipped); half 1 the other way round, x for both passes
// SINGLE (one slab per GPU, the multi-GPU case): the slab's descriptor --
// maps, geometry, pointers -- comes as a __grid_constant__ kernel parameter,
// so the loop reads constant-bank values as the single-domain kernel does;
// the multi-slab emulation reads it from the device copy of the set.
template <int PK, bool XDBL, bool SINGLE>
__global__ void __launch_bounds__(SpSlabCfg::Threads, 1)
    sp_slab_pass(const SpSet *__restrict__ psp, const __grid_constant__ SpSlab one, double off, double diag,
                 double zc, int use_cond, cudaGraphConditionalHandle cond)
{
    using G = SpSlabCfg;
    const SpSet &ps = *psp;
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[kSpSlabS], empty[kSpSlabS];
    __shared__ double red[32];
    __shared__ int is_last;
    int bid, nblk;
    if (SINGLE) {
        bid = blockIdx.x;
        nblk = gridDim.x;
    }
    const SpSlab &sl = SINGLE ? one : ps.s[sp_slab_of<1>(ps, bid, nblk)];
    CgScalars *sc = sl.sc;
    if (sc->done) {
        if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    double *const ring = aligned_smem(smem_raw);
    if (threadIdx.x == 0) {
        for (int i = 0; i < kSpSlabS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], G::CWarps);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const int in = XDBL ? 1 : 0, out = in ^ 1;
    const SpSlabIO io{2, sl.lo_ghost, sl.hi_ghost, sl.lo[0][out], sl.lo[1][out], sl.hi[0][out], sl.hi[1][out]};
    double rr = 0.0, gam = 0.0, dlt = 0.0;
    const double alpha = sc->alpha, alpha_prev = sc->alpha_prev;
    if (!XDBL && sc->it == 0)
        spass2_body<PK, kSpSlabTY, kSpSlabS, true, false, true>(&sl.m_r[in], &sl.m_p[in], &sl.m_x, sl.g, off, diag,
                                                                zc, sl.r[out], sl.p[out], sl.x, alpha, alpha_prev,
                                                                0.0, ring, full, empty, rr, gam, dlt, bid, nblk, io);
    else
        spass2_body<PK, kSpSlabTY, kSpSlabS, false, XDBL, true>(&sl.m_r[in], &sl.m_p[in], &sl.m_x, sl.g, off, diag,
                                                                 zc, sl.r[out], sl.p[out], sl.x, alpha, alpha_prev,
                                                                 sc->beta, ring, full, empty, rr, gam, dlt, bid, nblk,
                                                                 io);
    rr = block_sum<G::Threads>(rr, red);
    gam = block_sum<G::Threads>(gam, red);
    dlt = block_sum<G::Threads>(dlt, red);
    if (threadIdx.x == 0) {
        sl.partials[3 * bid] = rr;
        sl.partials[3 * bid + 1] = gam;
        sl.partials[3 * bid + 2] = dlt;
    }
    if (last_block_sys(&sl.tk->upd, &is_last, nblk, sl.lo[0][0] || sl.hi[0][0])) {
        rr = reduce_partials<G::Threads>(sl.partials, nblk, 3, red);
        gam = reduce_partials<G::Threads>(sl.partials + 1, nblk, 3, red);
        dlt = reduce_partials<G::Threads>(sl.partials + 2, nblk, 3, red);
        if (threadIdx.x == 0) {
            const double v[3] = {rr, gam, dlt};
            double tot[3];
            sp_allreduce(ps, sl, 3, v, tot);
            scalar_after_pass(sc, tot[0], tot[1], tot[2]);
            if (sc->done && use_cond) cudaGraphSetConditional(cond, 0);
        }
    }
}

// x += alpha p_k owed by a final skipping pass (odd iteration count; p_k in p[1])
__global__ void __launch_bounds__(256) sp_slab_fixup(const SpSet *__restrict__ psp)
{
    const SpSet &ps = *psp;
    int bid, nblk;
    const SpSlab &sl = ps.s[sp_slab_of<0>(ps, bid, nblk)];
    if ((sl.sc->it & 1) == 0) return;
    const double alpha = sl.sc->alpha;
    const long long n = (long long)sl.g.nx * sl.g.ny * sl.g.nz;
    for (long long i = (long long)bid * 256 + threadIdx.x; i < n; i += (long long)nblk * 256)
        sl.x[i] = sl.x[i] + alpha * sl.p[1][i];
}

template <int ORDER, bool SINGLE>
static void p2p_tma_attrs1()
{
    cudaFuncSetAttribute(p2p_update_tma<ORDER, PK_NONE, XM_SKIP, SINGLE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)upd_skip_smem<4>());
    cudaFuncSetAttribute(p2p_update_tma<ORDER, PK_NONE, XM_DOUBLE, SINGLE>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUpdSmem);
    cudaFuncSetAttribute(p2p_update_tma<ORDER, PK_JCONST, XM_SKIP, SINGLE>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_skip_smem<4>());
    cudaFuncSetAttribute(p2p_update_tma<ORDER, PK_JCONST, XM_DOUBLE, SINGLE>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUpdSmem);
}

template <int ORDER>
static void p2p_tma_attrs()
{
    p2p_tma_attrs1<ORDER, true>();
    p2p_tma_attrs1<ORDER, false>();
}

}  // namespace cf

// ---------------------------------------------------------------- host
namespace {

struct PSlab {
    int z0 = 0, z1 = 0, nzl = 0, lo = 0, hi = 0;
    double *alloc[4] = {nullptr, nullptr, nullptr, nullptr};  // r, x, p0, p1 incl. halo planes
    double *partials = nullptr;
    cf::CgTickets *tk = nullptr;
    cf::CgScalars *sc = nullptr;
    cf::Mailbox *mail = nullptr;
};

struct ExportBlob {  // what one rank publishes to the others
    cudaIpcMemHandle_t mail, r;
    unsigned long long mail_off, r_off;  // byte offsets of the arrays inside the exported allocations
    int nzl, lo, hi, rank;
    // the single-pass arrays (one allocation: r0, r1, p0, p1, x, each nzl + 4 planes)
    cudaIpcMemHandle_t sp;
    unsigned long long sp_off;
    int has_sp;
};

// cudaMalloc may sub-allocate small requests from a larger driver allocation;
// an IPC handle names that allocation and the importer maps its base, so the
// exporter publishes each array's offset within it (cuMemGetAddressRange).
typedef int (*AddressRangeFn)(unsigned long long *base, size_t *size, unsigned long long ptr);
static AddressRangeFn address_range_fn()
{
    static AddressRangeFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<AddressRangeFn>(p);
    }
    return fn;
}

static bool alloc_offset(const void *ptr, unsigned long long *off)
{
    AddressRangeFn fn = address_range_fn();
    if (!fn) return false;
    unsigned long long base = 0;
    size_t size = 0;
    if (fn(&base, &size, reinterpret_cast<unsigned long long>(ptr)) != 0) return false;
    *off = reinterpret_cast<unsigned long long>(ptr) - base;
    return true;
}

}  // namespace

struct cf_pcg {
    int nx = 0, ny = 0, nz = 0, order = 1;
    double h = 1, off = 0, diag = 0;
    int nranks = 1, rank = 0;
    std::vector<PSlab> slabs;  // local slabs (1 per rank; all of them in the emulation)
    cf::P2PSet set{};            // host copy of the slab descriptors
    cf::P2PSet *d_set = nullptr;  // device copy the kernels read
    std::vector<void *> opened;  // IPC-opened peer allocations
    bool linked = false;
    cf::CgScalars *sc_host = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    float last_ms = 0.f;
    int grid_init = 0, grid_dir = 0, grid_upd = 0, grid_updt = 0;
    bool tma = false;  // TMA update form (even nx >= 32, maps encodable)
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    int exec_key = -1;
    int direct = 0;  // CF_PCG_DIRECT=1: host-driven loop (profilers)
    // single pass over the slabs (the default; CF_PCG_ALGO=two selects the two-kernel form)
    bool spass = false;
    std::vector<double *> sp_alloc;  // per slab: r0 | r1 | p0 | p1 | x, each sp_stride doubles
    std::vector<double *> sp_part;   // per slab partials
    size_t sp_stride = 0;            // doubles per array (nzl + 4 planes + pad, 256-byte multiple)
    cf::SpSet sset{};
    cf::SpSet *d_sset = nullptr;
    int sp_grid = 0, sp_grid_init = 0;
};

namespace cf {

template <int ORDER, int PK, bool SINGLE>
static int p2p_body_t(cf_pcg *ws, cudaStream_t s, double zc, cudaGraphConditionalHandle cond, int use_cond)
{
    const P2PSlab &d = ws->set.s[0];
    for (int half = 0; half < 2; ++half) {
        const size_t sh = d.gd.lo_halo ? (size_t)d.gd.nx * d.gd.ny : 0;  // lowest plane in memory
        p2p_dir<ORDER, PK, SINGLE><<<ws->grid_dir, kPairThreads, 0, s>>>(ws->d_set, half, ws->off, ws->diag, zc, d.gd,
                                                                        d.r - sh, d.p0 - sh, d.p1 - sh);
        CF_CHECK_LAUNCH("p2p_dir");
        if (ws->tma) {
            if (half == 0)
                p2p_update_tma<ORDER, PK, XM_SKIP, SINGLE><<<ws->grid_updt, kWSThreads, upd_skip_smem<4>(), s>>>(
                    ws->d_set, half, ws->off, ws->diag, zc, use_cond, cond, d.m_p[0], d.m_p[1], d.m_ri, d.m_xi,
                    d.m_pi[0], d.m_pi[1], d.gt, d.r, d.x, d.lo_r, d.hi_r);
            else
                p2p_update_tma<ORDER, PK, XM_DOUBLE, SINGLE><<<ws->grid_updt, kWSThreads, kUpdSmem, s>>>(
                    ws->d_set, half, ws->off, ws->diag, zc, use_cond, cond, d.m_p[0], d.m_p[1], d.m_ri, d.m_xi,
                    d.m_pi[0], d.m_pi[1], d.gt, d.r, d.x, d.lo_r, d.hi_r);
        } else if (half == 0) {
            p2p_update<ORDER, PK, XM_SKIP><<<ws->grid_upd, kPairThreads, 0, s>>>(ws->d_set, half, ws->off, ws->diag, zc,
                                                                               use_cond, cond);
        } else {
            p2p_update<ORDER, PK, XM_DOUBLE><<<ws->grid_upd, kPairThreads, 0, s>>>(ws->d_set, half, ws->off, ws->diag,
                                                                                 zc, use_cond, cond);
        }
        CF_CHECK_LAUNCH("p2p_update");
    }
    return CF_OK;
}

template <int ORDER, int PK>
static int p2p_body(cf_pcg *ws, cudaStream_t s, double zc, cudaGraphConditionalHandle cond, int use_cond)
{
    return ws->slabs.size() == 1 ? p2p_body_t<ORDER, PK, true>(ws, s, zc, cond, use_cond)
                                 : p2p_body_t<ORDER, PK, false>(ws, s, zc, cond, use_cond);
}

template <int ORDER, int PK>
static int p2p_build_graph(cf_pcg *ws, double zc)
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
    cudaStream_t cs;
    CF_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CF_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    int rc = p2p_body<ORDER, PK>(ws, cs, zc, cond, 1);
    cudaGraph_t captured;
    cudaError_t e = cudaStreamEndCapture(cs, &captured);
    cudaStreamDestroy(cs);
    if (rc != CF_OK) return rc;
    CF_CUDA(e);
    cudaKernelNodeParams kp = {};
    void *args[] = {&ws->d_set};
    kp.func = (void *)p2p_x_fixup;
    kp.gridDim = dim3(ws->grid_init);
    kp.blockDim = dim3(256);
    kp.kernelParams = args;
    cudaGraphNode_t fix;
    CF_CUDA(cudaGraphAddKernelNode(&fix, g, &node, 1, &kp));
    if (ws->exec) {
        cudaGraphExecDestroy(ws->exec);
        cudaGraphDestroy(ws->graph);
        ws->exec = nullptr;
    }
    CF_CUDA(cudaGraphInstantiate(&ws->exec, g, 0));
    ws->graph = g;
    return CF_OK;
}

template <int ORDER, int PK>
static int p2p_solve(cf_pcg *ws, double zc, cudaStream_t s)
{
    p2p_init<PK><<<ws->grid_init, 256, 0, s>>>(ws->d_set, zc);
    CF_CHECK_LAUNCH("p2p_init");
    if (ws->direct) {
        CF_CUDA(cudaEventRecord(ws->ev0, s));
        for (;;) {
            for (int b = 0; b < 4; ++b) {
                int rc = p2p_body<ORDER, PK>(ws, s, zc, 0, 0);
                if (rc != CF_OK) return rc;
            }
            CF_CUDA(cudaMemcpyAsync(&ws->sc_host->done, &ws->slabs[0].sc->done, sizeof(int), cudaMemcpyDeviceToHost,
                                    s));
            CF_CUDA(cudaStreamSynchronize(s));
            if (ws->sc_host->done) break;
        }
        p2p_x_fixup<<<ws->grid_init, 256, 0, s>>>(ws->d_set);
        CF_CHECK_LAUNCH("p2p_x_fixup");
        CF_CUDA(cudaEventRecord(ws->ev1, s));
        return CF_OK;
    }
    const int key = ORDER * 4 + PK;
    if (!ws->exec || ws->exec_key != key) {
        int rc = p2p_build_graph<ORDER, PK>(ws, zc);
        if (rc != CF_OK) return rc;
        ws->exec_key = key;
    }
    CF_CUDA(cudaEventRecord(ws->ev0, s));
    CF_CUDA(cudaGraphLaunch(ws->exec, s));
    CF_CUDA(cudaEventRecord(ws->ev1, s));
    return CF_OK;
}

// ---- single pass over the slabs
template <int PK, bool SINGLE>
static void sp_body_t(cf_pcg *ws, cudaStream_t s, double zc, cudaGraphConditionalHandle cond, int use_cond)
{
    sp_slab_pass<PK, false, SINGLE><<<ws->sp_grid, SpSlabCfg::Threads, SpSlabCfg::Smem, s>>>(
        ws->d_sset, ws->sset.s[0], ws->off, ws->diag, zc, use_cond, cond);
    sp_slab_pass<PK, true, SINGLE><<<ws->sp_grid, SpSlabCfg::Threads, SpSlabCfg::Smem, s>>>(
        ws->d_sset, ws->sset.s[0], ws->off, ws->diag, zc, use_cond, cond);
}

template <int PK>
static int sp_body(cf_pcg *ws, cudaStream_t s, double zc, cudaGraphConditionalHandle cond, int use_cond)
{
    if (ws->slabs.size() == 1) sp_body_t<PK, true>(ws, s, zc, cond, use_cond);
    else sp_body_t<PK, false>(ws, s, zc, cond, use_cond);
    CF_CHECK_LAUNCH("sp_slab_pass");
    return CF_OK;
}

template <int PK>
static int sp_solve(cf_pcg *ws, double zc, cudaStream_t s)
{
    sp_init_copy<<<ws->sp_grid_init, 256, 0, s>>>(ws->d_sset);
    CF_CHECK_LAUNCH("sp_init_copy");
    sp_init_dots<PK><<<ws->sp_grid_init, 256, 0, s>>>(ws->d_sset, ws->off, ws->diag, zc);
    CF_CHECK_LAUNCH("sp_init_dots");
    if (ws->direct) {
        CF_CUDA(cudaEventRecord(ws->ev0, s));
        for (;;) {
            for (int b = 0; b < 4; ++b) {
                int rc = sp_body<PK>(ws, s, zc, 0, 0);
                if (rc != CF_OK) return rc;
            }
            CF_CUDA(cudaMemcpyAsync(&ws->sc_host->done, &ws->slabs[0].sc->done, sizeof(int), cudaMemcpyDeviceToHost,
                                    s));
            CF_CUDA(cudaStreamSynchronize(s));
            if (ws->sc_host->done) break;
        }
        sp_slab_fixup<<<ws->sp_grid_init, 256, 0, s>>>(ws->d_sset);
        CF_CHECK_LAUNCH("sp_slab_fixup");
        CF_CUDA(cudaEventRecord(ws->ev1, s));
        return CF_OK;
    }
    const int key = 100 + PK;
    if (!ws->exec || ws->exec_key != key) {
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
        int rc = sp_body<PK>(ws, cs, zc, cond, 1);
        cudaGraph_t captured;
        cudaError_t e = cudaStreamEndCapture(cs, &captured);
        cudaStreamDestroy(cs);
        if (rc != CF_OK) return rc;
        CF_CUDA(e);
        cudaKernelNodeParams kp = {};
        void *args[] = {&ws->d_sset};
        kp.func = (void *)sp_slab_fixup;
        kp.gridDim = dim3(ws->sp_grid_init);
        kp.blockDim = dim3(256);
        kp.kernelParams = args;
        cudaGraphNode_t fix;
        CF_CUDA(cudaGraphAddKernelNode(&fix, g, &node, 1, &kp));
        if (ws->exec) {
            cudaGraphExecDestroy(ws->exec);
            cudaGraphDestroy(ws->graph);
            ws->exec = nullptr;
        }
        CF_CUDA(cudaGraphInstantiate(&ws->exec, g, 0));
        ws->graph = g;
        ws->exec_key = key;
    }
    CF_CUDA(cudaEventRecord(ws->ev0, s));
    CF_CUDA(cudaGraphLaunch(ws->exec, s));
    CF_CUDA(cudaEventRecord(ws->ev1, s));
    return CF_OK;
}

// the single-pass arrays of slab k: 0 r0, 1 r1, 2 p0, 3 p1, 4 x (each starting at its lowest halo plane)
static double *sp_array(const cf_pcg *ws, size_t k, int a) { return ws->sp_alloc[k] + (size_t)a * ws->sp_stride; }

// neighbours' planes matching ours, for local slabs in one process: the lower
// neighbour's hi halo planes (its local planes nzl, nzl+1 = array planes
// nzl+2, nzl+3), the upper neighbour's lo halo planes (array planes 0, 1)
static void sp_link_local(cf_pcg *ws)
{
    const size_t pl = (size_t)ws->nx * ws->ny;
    for (size_t k = 0; k < ws->slabs.size(); ++k) {
        SpSlab &d = ws->sset.s[k];
        for (int a = 0; a < 4; ++a) {  // a = 2 * (r | p) + buffer
            if (k > 0) d.lo[a / 2][a % 2] = sp_array(ws, k - 1, a) + (size_t)(ws->slabs[k - 1].nzl + 2) * pl;
            if (k + 1 < ws->slabs.size()) d.hi[a / 2][a % 2] = sp_array(ws, k + 1, a);
        }
    }
}

// halo-plane targets of local slab k: the lower neighbour's hi halo plane and
// the upper neighbour's lo halo plane, when both live in this process
static void link_local(cf_pcg *ws)
{
    const size_t pl = (size_t)ws->nx * ws->ny;
    for (size_t k = 0; k < ws->slabs.size(); ++k) {
        PSlab &a = ws->slabs[k];
        P2PSlab &d = ws->set.s[k];
        if (k > 0) {
            PSlab &lo = ws->slabs[k - 1];
            d.lo_r = lo.alloc[0] + (size_t)(lo.lo + lo.nzl) * pl;
        }
        if (k + 1 < ws->slabs.size()) d.hi_r = ws->slabs[k + 1].alloc[0];
        (void)a;
    }
}

}  // namespace cf

extern "C" {

int cf_pcg_create(cf_pcg **out, int nx, int ny, int nz, double h, int order, int nranks, int rank, int nslabs,
                  const int *slab_bounds, void *stream)
{
    CF_REQUIRE(out && nx >= 2 && nx % 2 == 0 && ny >= 1 && nz >= 1 && h > 0, "cf_pcg_create: bad grid (nx even)");
    CF_REQUIRE(order == CF_ORDER_CSR || order == CF_ORDER_SYM, "cf_pcg_create: bad order");
    CF_REQUIRE(nranks >= 1 && nranks <= cf::kMaxRanks && rank >= 0 && rank < nranks,
               "cf_pcg_create: 1..8 ranks and 0 <= rank < nranks");
    CF_REQUIRE(nslabs == 1 || (nslabs == nranks && rank == 0),
               "cf_pcg_create: one slab per rank, or every slab in one process (emulation)");
    CF_REQUIRE(slab_bounds, "cf_pcg_create: slab bounds required");
    for (int k = 0; k < nslabs; ++k)
        CF_REQUIRE(slab_bounds[k] >= 0 && slab_bounds[k] < slab_bounds[k + 1] && slab_bounds[k + 1] <= nz,
                   "cf_pcg_create: slab bounds must increase within [0, nz]");
    cf_pcg *ws = new cf_pcg();
    ws->nx = nx;
    ws->ny = ny;
    ws->nz = nz;
    ws->h = h;
    ws->off = -1.0 / (h * h);
    ws->diag = 6.0 / (h * h);
    ws->order = order;
    ws->nranks = nranks;
    ws->rank = rank;
    if (const char *d = getenv("CF_PCG_DIRECT")) ws->direct = atoi(d) > 0;
    const size_t pl = (size_t)nx * ny;
    cudaStream_t s = cf::as_stream(stream);
    cudaError_t e = cudaSuccess;
    ws->slabs.resize(nslabs);
    ws->set.nslab = nslabs;
    ws->set.nranks = nranks;
    int bd = 0, bu = 0, bi = 0, bt = 0;
    const char *no_tma = getenv("CF_NO_TMA");
    ws->tma = nx >= 32 && nx % 2 == 0 && !(no_tma && atoi(no_tma) > 0);
    int tma_bpsm = 1;
    if (ws->tma) {
        if (order == CF_ORDER_CSR) cf::p2p_tma_attrs<CF_ORDER_CSR>();
        else cf::p2p_tma_attrs<CF_ORDER_SYM>();
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tma_bpsm, cf::p2p_update_tma<CF_ORDER_SYM, cf::PK_JCONST,
                                                                                    cf::XM_DOUBLE, true>,
                                                      cf::kWSThreads, cf::kUpdSmem);
        if (tma_bpsm < 1) tma_bpsm = 1;
    }
    for (int k = 0; k < nslabs && e == cudaSuccess; ++k) {
        PSlab &sb = ws->slabs[k];
        const int grank = nslabs == 1 ? rank : k;
        sb.z0 = slab_bounds[k];
        sb.z1 = slab_bounds[k + 1];
        sb.nzl = sb.z1 - sb.z0;
        sb.lo = grank > 0 ? 1 : 0;
        sb.hi = grank < nranks - 1 ? 1 : 0;
        const size_t planes = (size_t)sb.nzl + sb.lo + sb.hi;
        for (int a = 0; a < 4 && e == cudaSuccess; ++a) {
            // + kLeanPad zeroed doubles: the lean direction march reads out-of-domain
            // neighbours there (cf_cg_lean.cuh)
            const size_t bytes = (planes * pl + cf::kLeanPad) * sizeof(double);
            e = cudaMalloc(&sb.alloc[a], bytes);
            if (e == cudaSuccess) e = cudaMemsetAsync(sb.alloc[a], 0, bytes, s);
        }
        cf::P2PSlab &d = ws->set.s[k];
        d.gd = cf::lean_geom(nx, ny, sb.nzl, cf::kP2PDirRows, 12);  // 6 resident 128-thread CTAs per SM
        d.gd.lo_halo = sb.lo;
        d.gd.hi_halo = sb.hi;
        d.gd.chunk_rev = 1;  // top-down chunk order: L2 hand-over to / from the update kernel (cf_cg.cu)
        d.gu = cf::pair_geom(nx, ny, sb.nzl, sb.lo, sb.hi, "CF_PAIR_CHUNKS_UPD");
        d.blk_dir = bd;
        d.blk_upd = bu;
        d.blk_init = bi;
        const int ni = (int)std::min<long long>(((long long)pl * sb.nzl + 255) / 256, (long long)cf::num_sms() * 4);
        bd += d.gd.ctas();
        bu += d.gu.ctas();
        bi += ni;
        int nt = 0;
        if (ws->tma) {
            d.gt = cf::tma_geom(nx, ny, sb.nzl, sb.lo, sb.hi, tma_bpsm);
            d.blk_updt = bt;
            nt = d.gt.ntx * d.gt.nty * d.gt.nchunk;
            bt += nt;
        }
        const int maxg = std::max(std::max(std::max(d.gd.ctas(), d.gu.ctas()), ni), nt);
        if (e == cudaSuccess) e = cudaMalloc(&sb.partials, 2 * (size_t)maxg * sizeof(double));
        if (e == cudaSuccess) e = cudaMalloc(&sb.tk, sizeof(cf::CgTickets));
        if (e == cudaSuccess) e = cudaMemsetAsync(sb.tk, 0, sizeof(cf::CgTickets), s);
        if (e == cudaSuccess) e = cudaMalloc(&sb.sc, sizeof(cf::CgScalars));
        if (e == cudaSuccess) e = cudaMemsetAsync(sb.sc, 0, sizeof(cf::CgScalars), s);
        if (e == cudaSuccess) e = cudaMalloc(&sb.mail, sizeof(cf::Mailbox));
        if (e == cudaSuccess) e = cudaMemsetAsync(sb.mail, 0, sizeof(cf::Mailbox), s);
        if (e != cudaSuccess) break;
        d.r = sb.alloc[0] + sb.lo * pl;
        d.x = sb.alloc[1] + sb.lo * pl;
        d.p0 = sb.alloc[2] + sb.lo * pl;
        d.p1 = sb.alloc[3] + sb.lo * pl;
        d.partials = sb.partials;
        d.tk = sb.tk;
        d.sc = sb.sc;
        d.rank = grank;
        ws->set.mail[grank] = sb.mail;
        if (ws->tma) {
            const int hp = (int)planes;
            const bool ok = cf::make_map(&d.m_p[0], sb.alloc[2], nx, ny, hp, cf::kHX, cf::kHY) &&
                            cf::make_map(&d.m_p[1], sb.alloc[3], nx, ny, hp, cf::kHX, cf::kHY) &&
                            cf::make_map(&d.m_ri, sb.alloc[0], nx, ny, hp, cf::kTTX, cf::kTTY) &&
                            cf::make_map(&d.m_xi, sb.alloc[1], nx, ny, hp, cf::kTTX, cf::kTTY) &&
                            cf::make_map(&d.m_pi[0], sb.alloc[2], nx, ny, hp, cf::kTTX, cf::kTTY) &&
                            cf::make_map(&d.m_pi[1], sb.alloc[3], nx, ny, hp, cf::kTTX, cf::kTTY);
            if (!ok) ws->tma = false;  // the pair form needs no descriptors
        }
    }
    ws->grid_dir = bd;
    ws->grid_upd = bu;
    ws->grid_updt = bt;
    ws->grid_init = bi;
    // ---- the single pass (default): 2-halo-plane arrays, TMA maps, lockstep items per slab
    {
        const char *algo = getenv("CF_PCG_ALGO");
        bool want = !(algo && strcmp(algo, "spass")) && nx % 2 == 0;
        for (const PSlab &sb : ws->slabs) want = want && sb.nzl >= 4;
        if (want && e == cudaSuccess) {
            const void *kerns[] = {(const void *)cf::sp_slab_pass<cf::PK_NONE, false, false>,
                                   (const void *)cf::sp_slab_pass<cf::PK_NONE, true, false>,
                                   (const void *)cf::sp_slab_pass<cf::PK_JCONST, false, false>,
                                   (const void *)cf::sp_slab_pass<cf::PK_JCONST, true, false>,
                                   (const void *)cf::sp_slab_pass<cf::PK_NONE, false, true>,
                                   (const void *)cf::sp_slab_pass<cf::PK_NONE, true, true>,
                                   (const void *)cf::sp_slab_pass<cf::PK_JCONST, false, true>,
                                   (const void *)cf::sp_slab_pass<cf::PK_JCONST, true, true>};
            for (const void *kf : kerns)
                cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cf::SpSlabCfg::Smem);
            const int bps = cf::blocks_per_sm((const void *)cf::sp_slab_pass<cf::PK_JCONST, true, true>,
                                              cf::SpSlabCfg::Threads, cf::SpSlabCfg::Smem);
            const long long slots = std::max(1LL, (long long)cf::num_sms() * std::max(bps, 1) / nslabs);
            int maxz = 0;
            for (const PSlab &sb : ws->slabs) maxz = std::max(maxz, sb.nzl);
            ws->sp_stride = ((size_t)(maxz + 4) * pl + cf::kLeanPad + 31) / 32 * 32;
            int blk = 0, blki = 0;
            for (int k = 0; k < nslabs && e == cudaSuccess; ++k) {
                PSlab &sb = ws->slabs[k];
                const int grank = nslabs == 1 ? rank : k;
                double *a = nullptr;
                const size_t bytes = 5 * ws->sp_stride * sizeof(double);
                e = cudaMalloc(&a, bytes);
                if (e == cudaSuccess) e = cudaMemsetAsync(a, 0, bytes, s);
                if (e != cudaSuccess) break;
                ws->sp_alloc.push_back(a);
                cf::SpSlab &d = ws->sset.s[k];
                d = cf::SpSlab{};
                cf::SpGeom g{nx, ny, sb.nzl, (nx + cf::kSpTX - 1) / cf::kSpTX, (ny + cf::kSpSlabTY - 1) / cf::kSpSlabTY,
                             1, nullptr};
                const long long tiles = (long long)g.ntx * g.nty;
                g.nchunk = (int)std::max(1LL, std::min(slots / std::max(1LL, tiles), (long long)sb.nzl / 8));
                const long long items = tiles * g.nchunk, rounds = (items + slots - 1) / slots;
                const int nblk = (int)((items + rounds - 1) / rounds);
                d.g = g;
                d.blk = blk;
                d.blk_init = blki;
                blk += nblk;
                const int ni = (int)std::min<long long>(((long long)pl * sb.nzl + 255) / 256, slots * 4);
                blki += ni;
                const size_t off2 = 2 * pl;  // owned plane 0 behind two halo planes
                d.r[0] = a + off2;
                d.r[1] = a + ws->sp_stride + off2;
                d.p[0] = a + 2 * ws->sp_stride + off2;
                d.p[1] = a + 3 * ws->sp_stride + off2;
                d.x = a + 4 * ws->sp_stride + off2;
                d.lo_ghost = grank == 0;
                d.hi_ghost = grank == nranks - 1;
                d.tk = sb.tk;
                d.sc = sb.sc;
                d.rank = grank;
                double *part = nullptr;
                e = cudaMalloc(&part, (size_t)std::max(3 * nblk, 2 * ni) * sizeof(double));
                if (e != cudaSuccess) break;
                ws->sp_part.push_back(part);
                d.partials = part;
                const int planes = sb.nzl + 4, hy = cf::kSpSlabTY + 4;
                bool ok = true;
                for (int q = 0; q < 2; ++q) {
                    ok = ok && cf::make_map_promo(&d.m_r[q], a + q * ws->sp_stride, nx, ny, planes, cf::kSpBX, hy, 256);
                    ok = ok && cf::make_map_promo(&d.m_p[q], a + (2 + q) * ws->sp_stride, nx, ny, planes, cf::kSpBX, hy,
                                                  256);
                }
                ok = ok && cf::make_map_promo(&d.m_x, a + 4 * ws->sp_stride, nx, ny, planes, cf::kSpTX, cf::kSpSlabTY, 256);
                if (!ok) want = false;
            }
            ws->sset.nslab = nslabs;
            ws->sset.nranks = nranks;
            ws->sp_grid = blk;
            ws->sp_grid_init = blki;
            ws->spass = want && e == cudaSuccess;
        }
    }
    if (e == cudaSuccess) e = cudaMalloc(&ws->d_sset, sizeof(cf::SpSet));
    if (e == cudaSuccess) e = cudaMallocHost(&ws->sc_host, sizeof(cf::CgScalars));
    if (e == cudaSuccess) e = cudaMalloc(&ws->d_set, sizeof(cf::P2PSet));
    if (e == cudaSuccess) e = cudaEventCreate(&ws->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&ws->ev1);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        int rc = cf::cuda_fail(e, "cf_pcg_create");
        cf_pcg_destroy(ws);
        return rc;
    }
    for (int k = 0; k < nslabs; ++k) ws->sset.mail[ws->sset.s[k].rank] = ws->slabs[k].mail;
    if (nslabs == nranks) {  // every slab here: link directly
        cf::link_local(ws);
        if (ws->spass) cf::sp_link_local(ws);
        ws->linked = true;
    }
    *out = ws;
    return CF_OK;
}

int cf_pcg_export_size(void) { return (int)sizeof(ExportBlob); }

int cf_pcg_export(cf_pcg *ws, void *out, int cap)
{
    CF_REQUIRE(ws && out && cap >= (int)sizeof(ExportBlob) && ws->slabs.size() == 1,
               "cf_pcg_export: one local slab and a cf_pcg_export_size() buffer");
    ExportBlob b{};
    const PSlab &sb = ws->slabs[0];
    CF_CUDA(cudaIpcGetMemHandle(&b.mail, sb.mail));
    CF_CUDA(cudaIpcGetMemHandle(&b.r, sb.alloc[0]));
    CF_REQUIRE(alloc_offset(sb.mail, &b.mail_off) && alloc_offset(sb.alloc[0], &b.r_off),
               "cf_pcg_export: cuMemGetAddressRange unavailable");
    b.nzl = sb.nzl;
    b.lo = sb.lo;
    b.hi = sb.hi;
    b.rank = ws->rank;
    b.has_sp = ws->spass ? 1 : 0;
    if (ws->spass) {
        CF_CUDA(cudaIpcGetMemHandle(&b.sp, ws->sp_alloc[0]));
        CF_REQUIRE(alloc_offset(ws->sp_alloc[0], &b.sp_off), "cf_pcg_export: cuMemGetAddressRange unavailable");
    }
    std::memcpy(out, &b, sizeof(b));
    return CF_OK;
}

// all: nranks blobs in rank order (the allgather of cf_pcg_export)
int cf_pcg_import(cf_pcg *ws, const void *all, int nranks)
{
    CF_REQUIRE(ws && all && nranks == ws->nranks && ws->slabs.size() == 1, "cf_pcg_import: bad arguments");
    const ExportBlob *blobs = static_cast<const ExportBlob *>(all);
    const size_t pl = (size_t)ws->nx * ws->ny;
    cf::P2PSlab &d = ws->set.s[0];
    for (int q = 0; q < nranks; ++q) {
        CF_REQUIRE(blobs[q].rank == q, "cf_pcg_import: blobs must be in rank order");
        if (q == ws->rank) continue;
        void *m = nullptr;
        CF_CUDA(cudaIpcOpenMemHandle(&m, blobs[q].mail, cudaIpcMemLazyEnablePeerAccess));
        ws->opened.push_back(m);
        ws->set.mail[q] = reinterpret_cast<cf::Mailbox *>(static_cast<char *>(m) + blobs[q].mail_off);
        ws->sset.mail[q] = ws->set.mail[q];
        if (q == ws->rank - 1 || q == ws->rank + 1) {
            void *r = nullptr;
            CF_CUDA(cudaIpcOpenMemHandle(&r, blobs[q].r, cudaIpcMemLazyEnablePeerAccess));
            ws->opened.push_back(r);
            double *base = reinterpret_cast<double *>(static_cast<char *>(r) + blobs[q].r_off);
            if (q == ws->rank - 1) d.lo_r = base + (size_t)(blobs[q].lo + blobs[q].nzl) * pl;  // its hi halo plane
            else d.hi_r = base;                                                                // its lo halo plane
            if (ws->spass) {
                CF_REQUIRE(blobs[q].has_sp, "cf_pcg_import: a neighbour runs without the single-pass arrays");
                void *sp = nullptr;
                CF_CUDA(cudaIpcOpenMemHandle(&sp, blobs[q].sp, cudaIpcMemLazyEnablePeerAccess));
                ws->opened.push_back(sp);
                double *sbase = reinterpret_cast<double *>(static_cast<char *>(sp) + blobs[q].sp_off);
                cf::SpSlab &e2 = ws->sset.s[0];
                for (int a = 0; a < 4; ++a) {  // same stride on every rank (equal slab heights +-1: see create)
                    double *arr = sbase + (size_t)a * ws->sp_stride;
                    if (q == ws->rank - 1) e2.lo[a / 2][a % 2] = arr + (size_t)(blobs[q].nzl + 2) * pl;
                    else e2.hi[a / 2][a % 2] = arr;
                }
            }
        }
    }
    if (ws->spass) {  // every rank must agree on the form
        for (int q = 0; q < nranks; ++q)
            CF_REQUIRE(blobs[q].has_sp, "cf_pcg_import: ranks disagree on the single-pass form");
    }
    ws->linked = true;
    return CF_OK;
}

int cf_pcg_destroy(cf_pcg *ws)
{
    if (!ws) return CF_OK;
    if (ws->exec) cudaGraphExecDestroy(ws->exec);
    if (ws->graph) cudaGraphDestroy(ws->graph);
    for (void *p : ws->opened) cudaIpcCloseMemHandle(p);
    for (PSlab &sb : ws->slabs) {
        for (double *a : sb.alloc)
            if (a) cudaFree(a);
        if (sb.partials) cudaFree(sb.partials);
        if (sb.tk) cudaFree(sb.tk);
        if (sb.sc) cudaFree(sb.sc);
        if (sb.mail) cudaFree(sb.mail);
    }
    for (double *a : ws->sp_alloc) cudaFree(a);
    for (double *a : ws->sp_part) cudaFree(a);
    if (ws->d_sset) cudaFree(ws->d_sset);
    if (ws->sc_host) cudaFreeHost(ws->sc_host);
    if (ws->d_set) cudaFree(ws->d_set);
    if (ws->ev0) cudaEventDestroy(ws->ev0);
    if (ws->ev1) cudaEventDestroy(ws->ev1);
    delete ws;
    return CF_OK;
}

int cf_pcg_solve(cf_pcg *ws, const double *const *b_slabs, double *const *x_slabs, double tol, int64_t max_iter,
                 int precond, int64_t *iters_host, double *res_host, void *stream)
{
    CF_REQUIRE(ws && b_slabs && x_slabs, "cf_pcg_solve: null argument");
    CF_REQUIRE(ws->linked, "cf_pcg_solve: ranks not linked (cf_pcg_export / cf_pcg_import first)");
    CF_REQUIRE(tol > 0, "tol must be positive");
    CF_REQUIRE(max_iter >= 1, "max_iter must be >= 1");
    CF_REQUIRE(precond == CF_PRECOND_NONE || precond == CF_PRECOND_JACOBI,
               "the z-slab solver shards Jacobi-PCG / CG only (DIC's sweeps do not shard)");
    cudaStream_t s = cf::as_stream(stream);
    for (size_t k = 0; k < ws->slabs.size(); ++k) {
        CF_REQUIRE(b_slabs[k] && x_slabs[k], "cf_pcg_solve: null slab pointer");
        ws->set.s[k].b = b_slabs[k];
        ws->sset.s[k].b = b_slabs[k];
    }
    cf::CgScalars *h = ws->sc_host;
    *h = cf::CgScalars{};
    h->tol = tol;
    h->max_iter = max_iter;
    for (size_t k = 0; k < ws->slabs.size(); ++k) {
        // keep the phase counter (the mailboxes hold the last phase numbers)
        CF_CUDA(cudaMemcpyAsync(ws->sc_host, ws->slabs[k].sc, sizeof(cf::CgScalars), cudaMemcpyDeviceToHost, s));
        CF_CUDA(cudaStreamSynchronize(s));
        const unsigned long long ph = ws->sc_host->phase;
        *h = cf::CgScalars{};
        h->tol = tol;
        h->max_iter = max_iter;
        h->phase = ph;
        CF_CUDA(cudaMemcpyAsync(ws->slabs[k].sc, h, sizeof(*h), cudaMemcpyHostToDevice, s));
        CF_CUDA(cudaStreamSynchronize(s));
    }
    CF_CUDA(cudaMemcpyAsync(ws->d_set, &ws->set, sizeof(cf::P2PSet), cudaMemcpyHostToDevice, s));
    if (ws->spass) CF_CUDA(cudaMemcpyAsync(ws->d_sset, &ws->sset, sizeof(cf::SpSet), cudaMemcpyHostToDevice, s));
    CF_CUDA(cudaStreamSynchronize(s));
    const double zc = 1.0 / ws->diag;
    const int pk = precond == CF_PRECOND_JACOBI ? cf::PK_JCONST : cf::PK_NONE;
    int rc;
    if (ws->spass)  // the single pass (its stencil order is the CSR column order, both orders)
        rc = pk == cf::PK_JCONST ? cf::sp_solve<cf::PK_JCONST>(ws, zc, s) : cf::sp_solve<cf::PK_NONE>(ws, zc, s);
    else if (ws->order == CF_ORDER_CSR)
        rc = pk == cf::PK_JCONST ? cf::p2p_solve<CF_ORDER_CSR, cf::PK_JCONST>(ws, zc, s)
                                 : cf::p2p_solve<CF_ORDER_CSR, cf::PK_NONE>(ws, zc, s);
    else
        rc = pk == cf::PK_JCONST ? cf::p2p_solve<CF_ORDER_SYM, cf::PK_JCONST>(ws, zc, s)
                                 : cf::p2p_solve<CF_ORDER_SYM, cf::PK_NONE>(ws, zc, s);
    if (rc != CF_OK) return rc;
    CF_CUDA(cudaMemcpyAsync(h, ws->slabs[0].sc, sizeof(*h), cudaMemcpyDeviceToHost, s));
    CF_CUDA(cudaStreamSynchronize(s));
    CF_CUDA(cudaEventElapsedTime(&ws->last_ms, ws->ev0, ws->ev1));
    const size_t pl = (size_t)ws->nx * ws->ny;
    for (size_t k = 0; k < ws->slabs.size(); ++k) {
        const size_t bytes = pl * ws->slabs[k].nzl * sizeof(double);
        if (h->norm_b == 0.0) CF_CUDA(cudaMemsetAsync(x_slabs[k], 0, bytes, s));
        else
            CF_CUDA(cudaMemcpyAsync(x_slabs[k], ws->spass ? ws->sset.s[k].x : ws->set.s[k].x, bytes,
                                    cudaMemcpyDeviceToDevice, s));
    }
    CF_CUDA(cudaStreamSynchronize(s));
    if (iters_host) *iters_host = h->it;
    if (res_host) *res_host = h->res;
    if (h->status == cf::ST_PEER_TIMEOUT) {
        cf::set_error("cf_pcg_solve: a peer rank did not post its partial sums within 20 s (rank failed or "
                      "ranks diverged)");
        return CF_ECUDA;
    }
    if (h->status == cf::ST_BREAKDOWN) {
        cf::set_error("p^T A p = " + std::to_string(h->pap) + " at iteration " + std::to_string(h->it + 1));
        return CF_BREAKDOWN;
    }
    return h->status == cf::ST_CONVERGED ? CF_OK : CF_NOT_CONVERGED;
}

int cf_pcg_debug_io(cf_pcg *ws, int which, int write, double *host, int64_t n)
{
    CF_REQUIRE(ws && host && n >= 0 && ws->slabs.size() == 1 && which >= 0 && which <= 5,
               "cf_pcg_debug_io: bad arguments");
    const size_t pl = (size_t)ws->nx * ws->ny;
    const PSlab &sb = ws->slabs[0];
    double *dev = nullptr;
    size_t cap = 0;
    if (which >= 3) {  // the single pass's r0: own array (nzl + 4 planes), the neighbours' matching planes
        CF_REQUIRE(ws->spass, "cf_pcg_debug_io: no single-pass arrays");
        if (which == 3) {
            dev = ws->sp_alloc[0];
            cap = pl * (size_t)(sb.nzl + 4);
        } else {
            dev = which == 4 ? ws->sset.s[0].lo[0][0] : ws->sset.s[0].hi[0][0];
            cap = 2 * pl;
            CF_REQUIRE(!write, "cf_pcg_debug_io: peer planes are read-only here");
        }
    } else if (which == 0) {
        dev = sb.alloc[0];
        cap = pl * (size_t)(sb.nzl + sb.lo + sb.hi);
    } else {
        dev = which == 1 ? ws->set.s[0].lo_r : ws->set.s[0].hi_r;
        cap = pl;
        CF_REQUIRE(!write, "cf_pcg_debug_io: peer planes are read-only here");
    }
    CF_REQUIRE(dev != nullptr, "cf_pcg_debug_io: no such plane (no neighbour / not linked)");
    CF_REQUIRE((size_t)n <= cap, "cf_pcg_debug_io: n exceeds the region");
    // (a pageable H2D cudaMemcpy may return before the DMA lands: synchronise
    // so a peer reading right after the caller's barrier sees the data)
    if (write) CF_CUDA(cudaMemcpy(dev, host, (size_t)n * sizeof(double), cudaMemcpyHostToDevice));
    else CF_CUDA(cudaMemcpy(host, dev, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost));
    CF_CUDA(cudaDeviceSynchronize());
    return CF_OK;
}

int cf_pcg_form(cf_pcg *ws, int *form_host)
{
    CF_REQUIRE(ws && form_host, "cf_pcg_form: null argument");
    *form_host = ws->spass ? CF_CG_FORM_SPASS : CF_CG_FORM_TWO;
    return CF_OK;
}

int cf_pcg_last_loop_ms(cf_pcg *ws, float *ms_host)
{
    CF_REQUIRE(ws && ms_host, "cf_pcg_last_loop_ms: null argument");
    *ms_host = ws->last_ms;
    return CF_OK;
}

}  // extern "C"
