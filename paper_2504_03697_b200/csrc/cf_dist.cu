// cf_dist.cu -- conjugate gradient over z-slabs (SURVEY.md §5.8, §8 e).
//
// The cube is cut into contiguous z-slabs; each slab lives in HBM as an
// x-fastest block with one halo plane towards each existing neighbour.  A
// process owns one or more consecutive slabs (one per GPU in the multi-rank
// NCCL run; several on one device for the single-process emulation that lets
// the decomposed kernels be parity-tested on one GPU without ranks waiting on
// each other).  Per CG iteration:
//
//   dir    (per slab)  p = z + beta p_old on owned AND halo planes (the halo
//                      p is recomputed from the exchanged r halo and the
//                      slab's own p_old halo, bit-identical to the owner's),
//                      stencil, local p.Ap
//   sum    local slab partials in slab order  -> ncclAllReduce(sum)  -> alpha
//   update (per slab)  x, r; local r.r, r.z
//   sum    -> ncclAllReduce(sum) -> convergence, beta
//   halo   r boundary planes: D2D copies between local slabs, ncclSend/Recv
//          with the neighbouring ranks
//
// The halo overlaps the reduction: the neighbour send/recv pairs go into the
// same NCCL group as the (r.r, r.z) all-reduce, so one NCCL launch moves both
// concurrently, and the D2D copies between local slabs run on a side stream
// forked after the update kernels and joined before the next dir kernels.
// (Nothing of the next iteration can start earlier: every plane of the dir
// kernel needs beta, the all-reduce's result.)
//
// Every rank applies the same all-reduced scalars, so convergence decisions
// are identical everywhere; kernels early-exit once `done` is set, and the
// host polls `done` once per batch of iterations.
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "cf_cg_common.cuh"
#include "cf_tma_march.cuh"

namespace cf {

#include "cf_cg_tma.cuh"

// r = b, x = 0 on the owned planes; local |b|^2 and r.z
template <int PK>
__global__ void __launch_bounds__(256) dcg_init_kernel(long long n, const double *__restrict__ b, double *__restrict__ r,
                                                       double *__restrict__ x, double zc, double *partials,
                                                       CgTickets *tk, double *red_out)
{
    __shared__ double red[32];
    __shared__ int is_last;
    double bb = 0.0, rz = 0.0;
    const long long stride = (long long)gridDim.x * 256;
    for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < n; i += stride) {
        const double bi = b[i];
        r[i] = bi;
        x[i] = 0.0;
        bb = bb + bi * bi;
        rz = rz + bi * zval<PK>(bi, nullptr, 0, zc);
    }
    bb = block_sum<256>(bb, red);
    rz = block_sum<256>(rz, red);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = bb;
        partials[2 * blockIdx.x + 1] = rz;
    }
    if (last_block(&tk->init, &is_last)) {
        bb = reduce_partials<256>(partials, gridDim.x, 2, red);
        rz = reduce_partials<256>(partials + 1, gridDim.x, 2, red);
        if (threadIdx.x == 0) {
            red_out[0] = bb;
            red_out[1] = rz;
        }
    }
}

// Sum the local slabs' partials (slab order), written to red_sum.
__global__ void dcg_sum_kernel(const double *red, int nslabs, int ncomp, double *red_sum, const CgScalars *sc)
{
    (void)sc;
    if (threadIdx.x < ncomp) {
        double s = 0.0;
        for (int k = 0; k < nslabs; ++k) s = s + red[2 * k + threadIdx.x];
        red_sum[threadIdx.x] = s;
    }
}

enum { PH_INIT = 0, PH_DIR = 1, PH_UPD = 2 };

__global__ void dcg_scalar_kernel(CgScalars *sc, const double *red_sum, int phase)
{
    if (threadIdx.x != 0) return;
    if (phase == PH_INIT) {
        scalar_after_init(sc, red_sum[0], red_sum[1]);
        return;
    }
    if (sc->done) return;
    if (phase == PH_DIR) scalar_after_dir(sc, red_sum[0]);
    else scalar_after_update<true>(sc, red_sum[0], red_sum[1]);
}

struct Slab {
    int z0 = 0, z1 = 0, nzl = 0, lo = 0, hi = 0;
    double *alloc[4] = {nullptr, nullptr, nullptr, nullptr};  // r, x, p0, p1 (with halo planes)
    double *r = nullptr, *x = nullptr, *p[2] = {nullptr, nullptr};  // owned plane 0
    TmaGeom gd{}, gu{};
    CUtensorMap m_r{}, m_p[2]{}, m_ri{}, m_xi{};
    double *partials = nullptr;
    CgTickets *tk = nullptr;
};

}  // namespace cf

struct cf_dcg {
    int nx = 0, ny = 0, nz = 0, order = 1;
    double h = 1, off = 0, diag = 0;
    int nranks = 1, rank = 0, lo_rank = -1, hi_rank = -1;
    ncclComm_t comm = nullptr;
    std::vector<cf::Slab> slabs;
    cf::CgScalars *sc = nullptr, *sc_host = nullptr;
    double *red = nullptr, *red_sum = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaStream_t side = nullptr;                      // local halo copies
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    float last_ms = 0.f;
    int batch = 8;
    cudaGraphExec_t exec = nullptr;  // two captured iterations
    int exec_key = -1;
};

namespace cf {

static int nccl_fail(ncclResult_t r, const char *where)
{
    set_error(std::string(where) + ": " + ncclGetErrorString(r));
    return CF_ECUDA;
}

#define CF_NCCL(call)                                              \
    do {                                                           \
        ncclResult_t r_ = (call);                                  \
        if (r_ != ncclSuccess) return ::cf::nccl_fail(r_, #call);  \
    } while (0)

static int all_reduce(cf_dcg *ws, int ncomp, cudaStream_t s)
{
    if (ws->comm) CF_NCCL(ncclAllReduce(ws->red_sum, ws->red_sum, ncomp, ncclDouble, ncclSum, ws->comm, s));
    return CF_OK;
}

static int reduce_phase(cf_dcg *ws, int ncomp, int phase, cudaStream_t s)
{
    dcg_sum_kernel<<<1, 32, 0, s>>>(ws->red, (int)ws->slabs.size(), ncomp, ws->red_sum, ws->sc);
    CF_CHECK_LAUNCH("dcg_sum_kernel");
    int rc = all_reduce(ws, ncomp, s);
    if (rc != CF_OK) return rc;
    dcg_scalar_kernel<<<1, 32, 0, s>>>(ws->sc, ws->red_sum, phase);
    CF_CHECK_LAUNCH("dcg_scalar_kernel");
    return CF_OK;
}

// The neighbour-rank half of the r halo: this rank's boundary planes out, the
// neighbours' into the halo planes (enqueued inside the caller's NCCL group).
static int halo_p2p(cf_dcg *ws, cudaStream_t s)
{
    const size_t pl = (size_t)ws->nx * ws->ny;
    Slab &f = ws->slabs.front(), &l = ws->slabs.back();
    if (ws->lo_rank >= 0) {
        CF_NCCL(ncclSend(f.r, pl, ncclDouble, ws->lo_rank, ws->comm, s));
        CF_NCCL(ncclRecv(f.r - pl, pl, ncclDouble, ws->lo_rank, ws->comm, s));
    }
    if (ws->hi_rank >= 0) {
        CF_NCCL(ncclSend(l.r + pl * (l.nzl - 1), pl, ncclDouble, ws->hi_rank, ws->comm, s));
        CF_NCCL(ncclRecv(l.r + pl * l.nzl, pl, ncclDouble, ws->hi_rank, ws->comm, s));
    }
    return CF_OK;
}

// The local half: slab k's top plane -> slab k+1's lo halo, slab k+1's bottom
// plane -> slab k's hi halo.
static int halo_local(cf_dcg *ws, cudaStream_t s)
{
    const size_t pl = (size_t)ws->nx * ws->ny;
    const size_t bytes = pl * sizeof(double);
    auto &sl = ws->slabs;
    for (size_t k = 0; k + 1 < sl.size(); ++k) {
        CF_CUDA(cudaMemcpyAsync(sl[k + 1].r - pl, sl[k].r + pl * (sl[k].nzl - 1), bytes, cudaMemcpyDeviceToDevice, s));
        CF_CUDA(cudaMemcpyAsync(sl[k].r + pl * sl[k].nzl, sl[k + 1].r, bytes, cudaMemcpyDeviceToDevice, s));
    }
    return CF_OK;
}

// After the update kernels: the (r.r, r.z) reduction and the r halo
// exchange, overlapped (see the header).  `overlap` false (the init) runs
// them one after the other.
static int reduce_and_exchange(cf_dcg *ws, int phase, bool overlap, cudaStream_t s)
{
    const bool local = ws->slabs.size() > 1;
    const bool peers = ws->comm && (ws->lo_rank >= 0 || ws->hi_rank >= 0);
    if (!overlap) {
        int rc = reduce_phase(ws, 2, phase, s);
        if (rc == CF_OK && local) rc = halo_local(ws, s);
        if (rc == CF_OK && peers) {
            CF_NCCL(ncclGroupStart());
            rc = halo_p2p(ws, s);
            CF_NCCL(ncclGroupEnd());
        }
        return rc;
    }
    if (local) {
        CF_CUDA(cudaEventRecord(ws->ev_fork, s));
        CF_CUDA(cudaStreamWaitEvent(ws->side, ws->ev_fork, 0));
        int rc = halo_local(ws, ws->side);
        if (rc != CF_OK) return rc;
        CF_CUDA(cudaEventRecord(ws->ev_join, ws->side));
    }
    dcg_sum_kernel<<<1, 32, 0, s>>>(ws->red, (int)ws->slabs.size(), 2, ws->red_sum, ws->sc);
    CF_CHECK_LAUNCH("dcg_sum_kernel");
    if (ws->comm) {
        CF_NCCL(ncclGroupStart());
        ncclResult_t r = ncclAllReduce(ws->red_sum, ws->red_sum, 2, ncclDouble, ncclSum, ws->comm, s);
        int rc = r == ncclSuccess ? (peers ? halo_p2p(ws, s) : CF_OK) : nccl_fail(r, "ncclAllReduce");
        CF_NCCL(ncclGroupEnd());
        if (rc != CF_OK) return rc;
    }
    dcg_scalar_kernel<<<1, 32, 0, s>>>(ws->sc, ws->red_sum, phase);
    CF_CHECK_LAUNCH("dcg_scalar_kernel");
    if (local) CF_CUDA(cudaStreamWaitEvent(s, ws->ev_join, 0));
    return CF_OK;
}

template <int ORDER, int PK>
static int iteration(cf_dcg *ws, int half, double zc, cudaStream_t s)
{
    for (size_t k = 0; k < ws->slabs.size(); ++k) {
        Slab &sb = ws->slabs[k];
        const TmaGeom &g = sb.gd;
        cg_dir_tma<ORDER, PK><<<g.ntx * g.nty * g.nchunk, kWSThreads, kDirSmem, s>>>(
            sb.m_r, sb.m_p[half], g, ws->off, ws->diag, sb.p[half ^ 1], zc, ws->sc, sb.partials, sb.tk,
            ws->red + 2 * k);
        CF_CHECK_LAUNCH("cg_dir_tma (slab)");
    }
    int rc = reduce_phase(ws, 1, PH_DIR, s);
    if (rc != CF_OK) return rc;
    for (size_t k = 0; k < ws->slabs.size(); ++k) {
        Slab &sb = ws->slabs[k];
        const TmaGeom &g = sb.gu;
        cg_update_tma<ORDER, PK><<<g.ntx * g.nty * g.nchunk, kWSThreads, kUpdSmem, s>>>(
            sb.m_p[half ^ 1], sb.m_ri, sb.m_xi, sb.m_xi, g, ws->off, ws->diag, sb.r, sb.x, zc, ws->sc, sb.partials,
            sb.tk, 0, 0, ws->red + 2 * k);
        CF_CHECK_LAUNCH("cg_update_tma (slab)");
    }
    return reduce_and_exchange(ws, PH_UPD, true, s);
}

// Two iterations (p buffers back to their original roles) captured once into
// a CUDA graph -- kernels, D2D halo copies and the NCCL collectives alike --
// then replayed; CF_DCG_GRAPH=0 launches them directly.
template <int ORDER, int PK>
static int solve_loop(cf_dcg *ws, double zc, cudaStream_t s)
{
    const char *ge = getenv("CF_DCG_GRAPH");
    const bool use_graph = !(ge && atoi(ge) == 0);
    const int key = ORDER * 4 + PK;
    if (use_graph && (!ws->exec || ws->exec_key != key)) {
        if (ws->exec) {
            cudaGraphExecDestroy(ws->exec);
            ws->exec = nullptr;
        }
        // capture on a private stream (the caller's may be the legacy default
        // stream, which cannot be captured); the graph is launched on `s`
        cudaGraph_t g;
        cudaStream_t cs;
        CF_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        CF_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
        int rc = iteration<ORDER, PK>(ws, 0, zc, cs);
        if (rc == CF_OK) rc = iteration<ORDER, PK>(ws, 1, zc, cs);
        cudaError_t e = cudaStreamEndCapture(cs, &g);
        cudaStreamDestroy(cs);
        if (rc != CF_OK) return rc;
        CF_CUDA(e);
        e = cudaGraphInstantiate(&ws->exec, g, 0);
        cudaGraphDestroy(g);
        CF_CUDA(e);
        ws->exec_key = key;
    }
    int half = 0;
    for (;;) {
        for (int b = 0; b < ws->batch; b += 2) {
            if (use_graph) {
                CF_CUDA(cudaGraphLaunch(ws->exec, s));
            } else {
                int rc = iteration<ORDER, PK>(ws, half, zc, s);
                if (rc == CF_OK) rc = iteration<ORDER, PK>(ws, half ^ 1, zc, s);
                if (rc != CF_OK) return rc;
            }
        }
        CF_CUDA(cudaMemcpyAsync(&ws->sc_host->done, &ws->sc->done, sizeof(int), cudaMemcpyDeviceToHost, s));
        CF_CUDA(cudaStreamSynchronize(s));
        if (ws->sc_host->done) break;
    }
    return CF_OK;
}

template <int ORDER>
static void set_smem_attrs()
{
    cudaFuncSetAttribute(cg_dir_tma<ORDER, PK_NONE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDirSmem);
    cudaFuncSetAttribute(cg_dir_tma<ORDER, PK_JCONST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDirSmem);
    cudaFuncSetAttribute(cg_update_tma<ORDER, PK_NONE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUpdSmem);
    cudaFuncSetAttribute(cg_update_tma<ORDER, PK_JCONST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kUpdSmem);
}

template <int ORDER>
static void occupancy(int *bd, int *bu)
{
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(bd, cg_dir_tma<ORDER, PK_JCONST>, kWSThreads, kDirSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(bu, cg_update_tma<ORDER, PK_JCONST>, kWSThreads, kUpdSmem);
}

}  // namespace cf

extern "C" {

int cf_nccl_unique_id(void *out128)
{
    CF_REQUIRE(out128, "cf_nccl_unique_id: null output");
    ncclUniqueId id;
    CF_NCCL(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    memcpy(out128, &id, sizeof(id));
    return CF_OK;
}

int cf_dcg_destroy(cf_dcg *ws)
{
    if (!ws) return CF_OK;
    for (auto &sb : ws->slabs) {
        for (double *a : sb.alloc)
            if (a) cudaFree(a);
        if (sb.partials) cudaFree(sb.partials);
        if (sb.tk) cudaFree(sb.tk);
    }
    if (ws->sc) cudaFree(ws->sc);
    if (ws->sc_host) cudaFreeHost(ws->sc_host);
    if (ws->red) cudaFree(ws->red);
    if (ws->red_sum) cudaFree(ws->red_sum);
    if (ws->ev0) cudaEventDestroy(ws->ev0);
    if (ws->ev1) cudaEventDestroy(ws->ev1);
    if (ws->ev_fork) cudaEventDestroy(ws->ev_fork);
    if (ws->ev_join) cudaEventDestroy(ws->ev_join);
    if (ws->exec) cudaGraphExecDestroy(ws->exec);
    if (ws->side) cudaStreamDestroy(ws->side);
    if (ws->comm) ncclCommDestroy(ws->comm);
    delete ws;
    return CF_OK;
}

int cf_dcg_create(cf_dcg **out, int nx, int ny, int nz, double h, int order, int nranks, int rank,
                  const void *nccl_id, int nslabs, const int *slab_bounds, int lo_rank, int hi_rank, void *stream)
{
    CF_REQUIRE(out && nx >= 32 && nx % 2 == 0 && ny >= 1 && nz >= 1 && h > 0,
               "cf_dcg_create: the z-slab solver needs an even nx >= 32 (TMA rows)");
    CF_REQUIRE(order == CF_ORDER_CSR || order == CF_ORDER_SYM, "cf_dcg_create: bad order");
    CF_REQUIRE(nslabs >= 1 && slab_bounds && nranks >= 1 && rank >= 0 && rank < nranks, "cf_dcg_create: bad slabs");
    for (int k = 0; k < nslabs; ++k)
        CF_REQUIRE(slab_bounds[k] < slab_bounds[k + 1] && slab_bounds[k] >= 0 && slab_bounds[k + 1] <= nz,
                   "cf_dcg_create: slab bounds must be increasing within [0, nz]");
    cf_dcg *ws = new cf_dcg();
    ws->nx = nx;
    ws->ny = ny;
    ws->nz = nz;
    ws->h = h;
    ws->off = -1.0 / (h * h);
    ws->diag = 6.0 / (h * h);
    ws->order = order;
    ws->nranks = nranks;
    ws->rank = rank;
    ws->lo_rank = lo_rank;
    ws->hi_rank = hi_rank;
    if (const char *b = getenv("CF_DCG_BATCH")) ws->batch = atoi(b) > 0 ? atoi(b) : ws->batch;
    int bd = 1, bu = 1;
    if (order == CF_ORDER_CSR) {
        cf::set_smem_attrs<CF_ORDER_CSR>();
        cf::occupancy<CF_ORDER_CSR>(&bd, &bu);
    } else {
        cf::set_smem_attrs<CF_ORDER_SYM>();
        cf::occupancy<CF_ORDER_SYM>(&bd, &bu);
    }
    const size_t pl = (size_t)nx * ny;
    cudaError_t e = cudaSuccess;
    ws->slabs.resize(nslabs);
    for (int k = 0; k < nslabs && e == cudaSuccess; ++k) {
        cf::Slab &sb = ws->slabs[k];
        sb.z0 = slab_bounds[k];
        sb.z1 = slab_bounds[k + 1];
        sb.nzl = sb.z1 - sb.z0;
        sb.lo = (k > 0 || lo_rank >= 0) ? 1 : 0;
        sb.hi = (k < nslabs - 1 || hi_rank >= 0) ? 1 : 0;
        const size_t planes = (size_t)sb.nzl + sb.lo + sb.hi;
        for (int a = 0; a < 4 && e == cudaSuccess; ++a) {
            e = cudaMalloc(&sb.alloc[a], planes * pl * sizeof(double));
            if (e == cudaSuccess) e = cudaMemsetAsync(sb.alloc[a], 0, planes * pl * sizeof(double), cf::as_stream(stream));
        }
        if (e != cudaSuccess) break;
        sb.r = sb.alloc[0] + sb.lo * pl;
        sb.x = sb.alloc[1] + sb.lo * pl;
        sb.p[0] = sb.alloc[2] + sb.lo * pl;
        sb.p[1] = sb.alloc[3] + sb.lo * pl;
        sb.gd = cf::tma_geom(nx, ny, sb.nzl, sb.lo, sb.hi, bd > 0 ? bd : 1);
        sb.gu = cf::tma_geom(nx, ny, sb.nzl, sb.lo, sb.hi, bu > 0 ? bu : 1);
        const int hp = (int)planes;
        bool ok = cf::make_map(&sb.m_r, sb.alloc[0], nx, ny, hp, cf::kHX, cf::kHY) &&
                  cf::make_map(&sb.m_p[0], sb.alloc[2], nx, ny, hp, cf::kHX, cf::kHY) &&
                  cf::make_map(&sb.m_p[1], sb.alloc[3], nx, ny, hp, cf::kHX, cf::kHY) &&
                  cf::make_map(&sb.m_ri, sb.alloc[0], nx, ny, hp, cf::kTTX, cf::kTTY) &&
                  cf::make_map(&sb.m_xi, sb.alloc[1], nx, ny, hp, cf::kTTX, cf::kTTY);
        if (!ok) {
            cf_dcg_destroy(ws);
            cf::set_error("cf_dcg_create: tensor map encoding failed");
            return CF_EINVAL;
        }
        int g = std::max(sb.gd.ntx * sb.gd.nty * sb.gd.nchunk, sb.gu.ntx * sb.gu.nty * sb.gu.nchunk);
        g = std::max(g, cf::num_sms() * 8);
        e = cudaMalloc(&sb.partials, 2 * (size_t)g * sizeof(double));
        if (e == cudaSuccess) e = cudaMalloc(&sb.tk, sizeof(cf::CgTickets));
        if (e == cudaSuccess) e = cudaMemsetAsync(sb.tk, 0, sizeof(cf::CgTickets), cf::as_stream(stream));
    }
    if (e == cudaSuccess) e = cudaMalloc(&ws->sc, sizeof(cf::CgScalars));
    if (e == cudaSuccess) e = cudaMallocHost(&ws->sc_host, sizeof(cf::CgScalars));
    if (e == cudaSuccess) e = cudaMalloc(&ws->red, 2 * (size_t)nslabs * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&ws->red_sum, 2 * sizeof(double));
    if (e == cudaSuccess) e = cudaEventCreate(&ws->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&ws->ev1);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ws->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ws->ev_join, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ws->side, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        int rc = cf::cuda_fail(e, "cf_dcg_create");
        cf_dcg_destroy(ws);
        return rc;
    }
    if (nccl_id && nranks > 1) {
        ncclUniqueId id;
        memcpy(&id, nccl_id, sizeof(id));
        ncclResult_t r = ncclCommInitRank(&ws->comm, nranks, id, rank);
        if (r != ncclSuccess) {
            ws->comm = nullptr;
            int rc = cf::nccl_fail(r, "ncclCommInitRank");
            cf_dcg_destroy(ws);
            return rc;
        }
    }
    *out = ws;
    return CF_OK;
}

int cf_dcg_solve(cf_dcg *ws, const double *const *b_slabs, double *const *x_slabs, double tol, int64_t max_iter,
                 int precond, int64_t *iters_host, double *res_host, void *stream)
{
    CF_REQUIRE(ws && b_slabs && x_slabs, "cf_dcg_solve: null argument");
    CF_REQUIRE(tol > 0 && max_iter >= 1, "cf_dcg_solve: bad tol / max_iter");
    CF_REQUIRE(precond == CF_PRECOND_NONE || precond == CF_PRECOND_JACOBI,
               "cf_dcg_solve: the z-slab solver supports none / Jacobi (DIC does not shard)");
    cudaStream_t s = cf::as_stream(stream);
    const size_t pl = (size_t)ws->nx * ws->ny;
    const double zc = 1.0 / ws->diag;
    cf::CgScalars *h = ws->sc_host;
    *h = cf::CgScalars{};
    h->tol = tol;
    h->max_iter = max_iter;
    CF_CUDA(cudaMemcpyAsync(ws->sc, h, sizeof(*h), cudaMemcpyHostToDevice, s));
    for (size_t k = 0; k < ws->slabs.size(); ++k) {
        cf::Slab &sb = ws->slabs[k];
        const long long n = (long long)pl * sb.nzl;
        int grid = (int)std::min<long long>((n + 255) / 256, (long long)cf::num_sms() * 8);
        if (precond == CF_PRECOND_JACOBI)
            cf::dcg_init_kernel<cf::PK_JCONST><<<grid, 256, 0, s>>>(n, b_slabs[k], sb.r, sb.x, zc, sb.partials, sb.tk,
                                                                    ws->red + 2 * k);
        else
            cf::dcg_init_kernel<cf::PK_NONE><<<grid, 256, 0, s>>>(n, b_slabs[k], sb.r, sb.x, zc, sb.partials, sb.tk,
                                                                  ws->red + 2 * k);
        CF_CHECK_LAUNCH("dcg_init_kernel");
    }
    int rc = cf::reduce_and_exchange(ws, cf::PH_INIT, false, s);
    if (rc != CF_OK) return rc;
    CF_CUDA(cudaEventRecord(ws->ev0, s));
    if (ws->order == CF_ORDER_CSR)
        rc = precond == CF_PRECOND_JACOBI ? cf::solve_loop<CF_ORDER_CSR, cf::PK_JCONST>(ws, zc, s)
                                          : cf::solve_loop<CF_ORDER_CSR, cf::PK_NONE>(ws, zc, s);
    else
        rc = precond == CF_PRECOND_JACOBI ? cf::solve_loop<CF_ORDER_SYM, cf::PK_JCONST>(ws, zc, s)
                                          : cf::solve_loop<CF_ORDER_SYM, cf::PK_NONE>(ws, zc, s);
    if (rc != CF_OK) return rc;
    CF_CUDA(cudaEventRecord(ws->ev1, s));
    CF_CUDA(cudaMemcpyAsync(h, ws->sc, sizeof(*h), cudaMemcpyDeviceToHost, s));
    CF_CUDA(cudaStreamSynchronize(s));
    CF_CUDA(cudaEventElapsedTime(&ws->last_ms, ws->ev0, ws->ev1));
    for (size_t k = 0; k < ws->slabs.size(); ++k) {
        cf::Slab &sb = ws->slabs[k];
        const size_t bytes = pl * sb.nzl * sizeof(double);
        if (h->norm_b == 0.0) CF_CUDA(cudaMemsetAsync(x_slabs[k], 0, bytes, s));
        else CF_CUDA(cudaMemcpyAsync(x_slabs[k], sb.x, bytes, cudaMemcpyDeviceToDevice, s));
    }
    CF_CUDA(cudaStreamSynchronize(s));
    if (iters_host) *iters_host = h->it;
    if (res_host) *res_host = h->res;
    if (h->status == cf::ST_BREAKDOWN) {
        cf::set_error("p^T A p = " + std::to_string(h->pap) + " at iteration " + std::to_string(h->it + 1));
        return CF_BREAKDOWN;
    }
    return h->status == cf::ST_CONVERGED ? CF_OK : CF_NOT_CONVERGED;
}

int cf_dcg_last_loop_ms(cf_dcg *ws, float *ms_host)
{
    CF_REQUIRE(ws && ms_host, "cf_dcg_last_loop_ms: null argument");
    *ms_host = ws->last_ms;
    return CF_OK;
}

}  // extern "C"
