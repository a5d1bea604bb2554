// cf_tma.cu -- host helpers of the TMA-staged march (cf_tma.cuh).
#include <mutex>

#include "cf_tma.cuh"

namespace cf {

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn()
{
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

bool make_map(CUtensorMap *map, const double *base, int nx, int ny, int planes, int bx, int by)
{
    return make_map_promo(map, base, nx, ny, planes, bx, by, 256);
}

bool make_map_promo(CUtensorMap *map, const double *base, int nx, int ny, int planes, int bx, int by, int promo)
{
    EncodeTiledFn enc = encode_fn();
    if (!enc || !base) return false;
    const cuuint64_t row = (cuuint64_t)nx * sizeof(double);
    if (row % 16 != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)planes};
    cuuint64_t strides[2] = {row, row * (cuuint64_t)ny};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    // OOB_FILL_NONE: out-of-bounds elements of a box read as zero
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     promo >= 256   ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                     : promo >= 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                     : promo >= 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                    : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_map_pitched(CUtensorMap *map, const double *base, int nx, int ny, int planes, int pitch, int bx, int by)
{
    EncodeTiledFn enc = encode_fn();
    if (!enc || !base || pitch < nx) return false;
    const cuuint64_t row = (cuuint64_t)pitch * sizeof(double);
    if (row % 16 != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)planes};
    cuuint64_t strides[2] = {row, row * (cuuint64_t)ny};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

TmaGeom tma_geom(int nx, int ny, int nz, int lo_halo, int hi_halo, int blocks_per_sm)
{
    TmaGeom g;
    g.nx = nx;
    g.ny = ny;
    g.nz = nz;
    g.lo_halo = lo_halo;
    g.hi_halo = hi_halo;
    g.ntx = (nx + kTTX - 1) / kTTX;
    g.nty = (ny + kTTY - 1) / kTTY;
    const long long tiles = (long long)g.ntx * g.nty;
    const long long cap = (long long)num_sms() * (blocks_per_sm > 0 ? blocks_per_sm : 1);
    long long c = wave_chunks(tiles, nz, cap, 8);
    if (const char *e = getenv("CF_TMA_CHUNKS")) {  // debugging / tuning override
        const int v = atoi(e);
        if (v >= 1 && v <= nz) c = v;
    }
    g.nchunk = (int)c;
    return g;
}

}  // namespace cf
