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
#include <vector>

#include "cf_cg_common.cuh"
#include "cf_tma_march.cuh"

namespace cf {

#include "cf_cg_tma.cuh"
#include "cf_cg_pair.cuh"
#include "cf_cg_lean.cuh"

constexpr int kMaxRanks = 8;

struct Mailbox {
    double val[2][kMaxRanks][2];           // [phase parity][sender][component]
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
__device__ __forceinline__ void p2p_allreduce(const P2PSet &ps, const P2PSlab &sl, int ncomp, const double *v,
                                              double *out)
{
    if (ps.nranks == 1) {  // one rank (single-slab run): nothing to exchange
        for (int c = 0; c < ncomp; ++c) out[c] = 0.0 + v[c];
        return;
    }
    const unsigned long long ph = ++sl.sc->phase;
    const int par = (int)(ph & 1ull), me = sl.rank;
    for (int q = 0; q < ps.nranks; ++q)
        for (int c = 0; c < ncomp; ++c) st_relaxed_sys(&ps.mail[q]->val[par][me][c], v[c]);
    for (int q = 0; q < ps.nranks; ++q) st_release_sys(&ps.mail[q]->seq[par][me], ph);
    Mailbox *mine = ps.mail[me];
    const unsigned long long t0 = globaltimer_ns();
    for (int q = 0; q < ps.nranks; ++q) {
        while (ld_acquire_sys(&mine->seq[par][q]) < ph) {
            __nanosleep(64);
            if (globaltimer_ns() - t0 > kPeerTimeoutNs) {
                sl.sc->status = ST_PEER_TIMEOUT;
                sl.sc->done = 1;
                for (int c = 0; c < ncomp; ++c) out[c] = __longlong_as_double(0x7ff8000000000000ll);
                return;
            }
        }
    }
    for (int c = 0; c < ncomp; ++c) {
        double sum = 0.0;
        for (int q = 0; q < ps.nranks; ++q) sum = sum + ld_relaxed_sys(&mine->val[par][q][c]);
        out[c] = sum;
    }
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
    if (nslabs == nranks) {  // every slab here: link directly
        cf::link_local(ws);
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
        if (q == ws->rank - 1 || q == ws->rank + 1) {
            void *r = nullptr;
            CF_CUDA(cudaIpcOpenMemHandle(&r, blobs[q].r, cudaIpcMemLazyEnablePeerAccess));
            ws->opened.push_back(r);
            double *base = reinterpret_cast<double *>(static_cast<char *>(r) + blobs[q].r_off);
            if (q == ws->rank - 1) d.lo_r = base + (size_t)(blobs[q].lo + blobs[q].nzl) * pl;  // its hi halo plane
            else d.hi_r = base;                                                                // its lo halo plane
        }
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
    CF_CUDA(cudaStreamSynchronize(s));
    const double zc = 1.0 / ws->diag;
    const int pk = precond == CF_PRECOND_JACOBI ? cf::PK_JCONST : cf::PK_NONE;
    int rc;
    if (ws->order == CF_ORDER_CSR)
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
        else CF_CUDA(cudaMemcpyAsync(x_slabs[k], ws->set.s[k].x, bytes, cudaMemcpyDeviceToDevice, s));
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
    CF_REQUIRE(ws && host && n >= 0 && ws->slabs.size() == 1 && which >= 0 && which <= 2,
               "cf_pcg_debug_io: bad arguments");
    const size_t pl = (size_t)ws->nx * ws->ny;
    const PSlab &sb = ws->slabs[0];
    double *dev = nullptr;
    size_t cap = 0;
    if (which == 0) {
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

int cf_pcg_last_loop_ms(cf_pcg *ws, float *ms_host)
{
    CF_REQUIRE(ws && ms_host, "cf_pcg_last_loop_ms: null argument");
    *ms_host = ws->last_ms;
    return CF_OK;
}

}  // extern "C"
