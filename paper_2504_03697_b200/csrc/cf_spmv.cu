// cf_spmv.cu -- the two ways of applying the pressure operator:
//   * CSR SpMV (src/sparse.py:236-247) and symmetric-storage SpMV
//     (src/sparse.py:250-267), int32 indices, one thread per row summing in
//     the reference's per-row order (bit-identical results);
//   * the matrix-free 7-point stencil (cf_stencil.cuh), 16 B/cell of HBM
//     traffic against 12*nnz/N + 20 B/cell for CSR.
#include <cstdlib>
#include <cstring>

#include "cf_cg_common.cuh"
#include "cf_stencil.cuh"
#include "cf_tma_march.cuh"

namespace cf {

#include "cf_cg_pair.cuh"

// y = A x through the full-occupancy register pair march (cf_cg_pair.cuh):
// warp = one 64-cell tile row of cell pairs, x-neighbours by shuffle.
template <int ORDER>
__global__ void __launch_bounds__(kPairThreads, 8) stencil_apply_pair(PairGeom g, double off, double diag,
                                                                     const double *__restrict__ x,
                                                                     double *__restrict__ y)
{
    const PairCoords c = pair_coords(g, blockIdx.x);
    struct Epi {
        double *y;
        __device__ __forceinline__ void cell(long long o, double2, double a0, double a1)
        {
            *reinterpret_cast<double2 *>(y + o) = make_double2(a0, a1);
        }
        __device__ __forceinline__ void halo(long long, double2) {}
    } epi{y};
    if (c.row_ok) pair_march<ORDER, false>(c, g, off, diag, UpdSrc{x}, epi);
}

// y = A x through the warp-specialised TMA march (halo boxes of x staged by a
// producer warp; the consumer warps' stencil reads shared memory only).
struct ApplyPolicy {
    const double *sx;
    double *y;  // at (i, j) of plane 0
    long long plane;
    __device__ __forceinline__ double2 value2(int s, int o) const { return ld2(sx + s * kBoxStride + o); }
    __device__ __forceinline__ double value(int s, int o) const { return sx[s * kBoxStride + o]; }
    __device__ __forceinline__ void epi(int, const MarchCoords &, int z, double2, double a0, double a1)
    {
        st2(y + plane * z, a0, a1);
    }
    __device__ __forceinline__ void halo(const MarchCoords &, int, double2) {}
};

template <int ORDER>
__global__ void __launch_bounds__(kWSThreads) stencil_apply_tma(const __grid_constant__ CUtensorMap mx, TmaGeom g,
                                                                double off, double diag, double *__restrict__ y)
{
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    double *const sx = aligned_smem(smem_raw);
    const MarchCoords m = march_coords(g);
    const long long plane = (long long)g.nx * g.ny;
    ApplyPolicy pol{sx, y + m.i + (long long)g.nx * m.j, plane};
    init_ws_bars(full, empty);
    if (threadIdx.x >= kPThreads) {
        if (threadIdx.x == kPThreads) {
            prefetch_map(&mx);
            ws_produce(m.nplanes, full, empty, [&](int q, int s, uint64_t *bar) {
                mbar_expect_tx(bar, kBoxBytes);
                tma_load_3d(sx + s * kBoxStride, &mx, m.bx0, m.by0, m.zs + q + g.lo_halo, bar);
            });
        }
    } else {
        ws_consume<ORDER>(g, m, off, diag, pol, full, empty);
    }
}

constexpr size_t kApplySmem = kStages * kBoxStride * sizeof(double) + 128;

template <int ORDER>
static int stencil_apply_tma_launch(int nx, int ny, int nz, double off, double diag, const double *x, double *y,
                                    cudaStream_t s, bool *used)
{
    *used = false;
    if (nx < 32 || nx % 2 != 0) return CF_OK;
    CUtensorMap map;
    if (!make_map(&map, x, nx, ny, nz, kHX, kHY)) return CF_OK;
    static bool attr[2] = {false, false};
    if (!attr[ORDER]) {
        cudaFuncSetAttribute(stencil_apply_tma<ORDER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kApplySmem);
        attr[ORDER] = true;
    }
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, stencil_apply_tma<ORDER>, kWSThreads, kApplySmem);
    TmaGeom g = tma_geom(nx, ny, nz, 0, 0, b > 0 ? b : 1);
    stencil_apply_tma<ORDER><<<g.ntx * g.nty * g.nchunk, kWSThreads, kApplySmem, s>>>(map, g, off, diag, y);
    CF_CHECK_LAUNCH("stencil_apply_tma");
    *used = true;
    return CF_OK;
}

constexpr int kRowThreads = 256;

__global__ void __launch_bounds__(kRowThreads) csr_spmv_kernel(int64_t n_rows,
                                                                const int32_t *__restrict__ rp,
                                                                const int32_t *__restrict__ ci,
                                                                const double *__restrict__ val,
                                                                const double *__restrict__ x,
                                                                double *__restrict__ y)
{
    const int64_t stride = (int64_t)gridDim.x * kRowThreads;
    for (int64_t r = (int64_t)blockIdx.x * kRowThreads + threadIdx.x; r < n_rows; r += stride) {
        double s = 0.0;
        const int32_t e = __ldg(rp + r + 1);
        for (int32_t p = __ldg(rp + r); p < e; ++p) s = s + __ldg(val + p) * __ldg(x + __ldg(ci + p));
        y[r] = s;
    }
}

__global__ void __launch_bounds__(kRowThreads) sym_spmv_kernel(
    int64_t n, const double *__restrict__ diag, const int32_t *__restrict__ rp,
    const int32_t *__restrict__ ci, const double *__restrict__ val, const int32_t *__restrict__ trp,
    const int32_t *__restrict__ tci, const int32_t *__restrict__ tperm, const double *__restrict__ x,
    double *__restrict__ y)
{
    const int64_t stride = (int64_t)gridDim.x * kRowThreads;
    for (int64_t r = (int64_t)blockIdx.x * kRowThreads + threadIdx.x; r < n; r += stride) {
        double s = __ldg(diag + r) * __ldg(x + r);
        for (int32_t p = __ldg(rp + r), e = __ldg(rp + r + 1); p < e; ++p)
            s = s + __ldg(val + p) * __ldg(x + __ldg(ci + p));
        for (int32_t p = __ldg(trp + r), e = __ldg(trp + r + 1); p < e; ++p)
            s = s + __ldg(val + __ldg(tperm + p)) * __ldg(x + __ldg(tci + p));
        y[r] = s;
    }
}

template <int ORDER>
__global__ void __launch_bounds__(kMarchThreads) stencil_apply_kernel(Box bx, double off, double diag,
                                                                      const double *__restrict__ x,
                                                                      double *__restrict__ y)
{
    auto load = [&](long long i) { return __ldg(x + i); };
    auto epi = [&](long long i, double, double ax) { y[i] = ax; };
    march<ORDER>(bx, off, diag, load, epi);
}

static int row_grid(int64_t n)
{
    int64_t want = (n + kRowThreads - 1) / kRowThreads;
    int64_t cap = (int64_t)num_sms() * 8;
    return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

int march_grid(const void *kernel, const Box &bx)
{
    long long units = (long long)((bx.nx + kTX - 1) / kTX) * ((bx.ny + kTY - 1) / kTY) * bx.nz;
    long long cap = (long long)num_sms() * blocks_per_sm(kernel, kMarchThreads, 0);
    return (int)(units < cap ? (units > 0 ? units : 1) : cap);
}

}  // namespace cf

extern "C" {

int cf_csr_spmv(int64_t n_rows, const int32_t *row_ptr, const int32_t *col_idx, const double *values,
                const double *x, double *y, void *stream)
{
    CF_REQUIRE(n_rows >= 0, "cf_csr_spmv: negative row count");
    if (n_rows == 0) return CF_OK;
    cf::csr_spmv_kernel<<<cf::row_grid(n_rows), cf::kRowThreads, 0, cf::as_stream(stream)>>>(
        n_rows, row_ptr, col_idx, values, x, y);
    CF_CHECK_LAUNCH("csr_spmv_kernel");
    return CF_OK;
}

int cf_sym_spmv(int64_t n, const double *diag, const int32_t *row_ptr, const int32_t *col_idx,
                const double *values, const int32_t *t_row_ptr, const int32_t *t_col_idx,
                const int32_t *t_perm, const double *x, double *y, void *stream)
{
    CF_REQUIRE(n >= 0, "cf_sym_spmv: negative dimension");
    if (n == 0) return CF_OK;
    cf::sym_spmv_kernel<<<cf::row_grid(n), cf::kRowThreads, 0, cf::as_stream(stream)>>>(
        n, diag, row_ptr, col_idx, values, t_row_ptr, t_col_idx, t_perm, x, y);
    CF_CHECK_LAUNCH("sym_spmv_kernel");
    return CF_OK;
}

int cf_stencil7_apply(int nx, int ny, int nz, double h, int order, const double *x, double *y,
                      void *stream)
{
    CF_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1 && h > 0, "cf_stencil7_apply: bad grid");
    CF_REQUIRE(order == CF_ORDER_CSR || order == CF_ORDER_SYM, "cf_stencil7_apply: bad order");
    cf::Box bx{nx, ny, nz, 0, 0};
    // the same literals the reference assembles (src/sim.py:303-304)
    const double off = -1.0 / (h * h), diag = 6.0 / (h * h);
    cudaStream_t s = cf::as_stream(stream);
    // default: the pair march (even nx); CF_APPLY=tma selects the TMA pipeline
    const char *form = getenv("CF_APPLY");
    if (nx % 2 == 0 && !(form && !strcmp(form, "tma")) && !(form && !strcmp(form, "ldg"))) {
        const cf::PairGeom g = cf::pair_geom(nx, ny, nz, 0, 0, "CF_APPLY_CHUNKS");
        if (order == CF_ORDER_CSR)
            cf::stencil_apply_pair<CF_ORDER_CSR><<<g.ctas(), cf::kPairThreads, 0, s>>>(g, off, diag, x, y);
        else
            cf::stencil_apply_pair<CF_ORDER_SYM><<<g.ctas(), cf::kPairThreads, 0, s>>>(g, off, diag, x, y);
        CF_CHECK_LAUNCH("stencil_apply_pair");
        return CF_OK;
    }
    bool used = false;
    int rc = (form && !strcmp(form, "ldg")) ? CF_OK
             : order == CF_ORDER_CSR
                 ? cf::stencil_apply_tma_launch<CF_ORDER_CSR>(nx, ny, nz, off, diag, x, y, s, &used)
                 : cf::stencil_apply_tma_launch<CF_ORDER_SYM>(nx, ny, nz, off, diag, x, y, s, &used);
    if (rc != CF_OK || used) return rc;
    if (order == CF_ORDER_CSR) {
        auto k = cf::stencil_apply_kernel<CF_ORDER_CSR>;
        k<<<cf::march_grid((const void *)k, bx), cf::kMarchThreads, 0, s>>>(bx, off, diag, x, y);
    } else {
        auto k = cf::stencil_apply_kernel<CF_ORDER_SYM>;
        k<<<cf::march_grid((const void *)k, bx), cf::kMarchThreads, 0, s>>>(bx, off, diag, x, y);
    }
    CF_CHECK_LAUNCH("stencil_apply_kernel");
    return CF_OK;
}

}  // extern "C"
