// Probe: LDG (no TMA, no shared memory) forms of the two fused CG kernels at
// full occupancy -- cell pairs per thread, xy tiles marching z over chunks,
// in-plane neighbours through L1.  Same loads/stores/arithmetic as
// cg_dir_tma / cg_update_tma (minus the last-block scalar epilogue).  Times
// each kernel at n^3 for several tile shapes and chunk counts.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int NT>
__device__ double block_sum(double v, double *red)
{
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < NT / 32 ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    return v;
}

__device__ __forceinline__ double2 ldp(const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); }

template <int TX, int TY>
__global__ void __launch_bounds__(TX / 2 * TY) dir_ldg(const double *__restrict__ r, const double *__restrict__ po,
                                                       double *__restrict__ pn, int n, int nchunk, double zc,
                                                       double beta, double off, double diag, double *partials)
{
    __shared__ double red[32];
    const int ntx = n / TX, nty = n / TY, ntiles = ntx * nty;
    const int tile = blockIdx.x % ntiles, chunk = blockIdx.x / ntiles;
    const int i = (tile % ntx) * TX + 2 * (threadIdx.x % (TX / 2));
    const int j = (tile / ntx) * TY + threadIdx.x / (TX / 2);
    const int z0 = n * chunk / nchunk, z1 = n * (chunk + 1) / nchunk;
    const long long pl = (long long)n * n;
    const long long base = i + (long long)n * j;
    const bool hxl = i > 0, hxr = i + 2 < n, hym = j > 0, hyp = j + 1 < n;
    auto P2 = [&](long long o) {
        double2 a = ldp(r + o), b = ldp(po + o);
        return make_double2(a.x * zc + beta * b.x, a.y * zc + beta * b.y);
    };
    auto P1 = [&](long long o) { return __ldg(r + o) * zc + beta * __ldg(po + o); };
    const double2 zero = make_double2(0, 0);
    double2 cm = z0 > 0 ? P2(base + pl * (z0 - 1)) : zero;
    double2 cc = P2(base + pl * z0);
    double pap = 0.0;
    for (int z = z0; z < z1; ++z) {
        const long long o = base + pl * z;
        double2 cp = z + 1 < n ? P2(o + pl) : zero;
        double xl = hxl ? P1(o - 1) : 0.0, xr = hxr ? P1(o + 2) : 0.0;
        double2 ym = hym ? P2(o - n) : zero, yp = hyp ? P2(o + n) : zero;
        double a0 = diag * cc.x;
        a0 = a0 + off * cc.y;
        a0 = a0 + off * yp.x;
        a0 = a0 + off * cp.x;
        a0 = a0 + off * cm.x;
        a0 = a0 + off * ym.x;
        a0 = a0 + off * xl;
        double a1 = diag * cc.y;
        a1 = a1 + off * xr;
        a1 = a1 + off * yp.y;
        a1 = a1 + off * cp.y;
        a1 = a1 + off * cm.y;
        a1 = a1 + off * ym.y;
        a1 = a1 + off * cc.x;
        *reinterpret_cast<double2 *>(pn + o) = cc;
        pap = pap + cc.x * a0;
        pap = pap + cc.y * a1;
        cm = cc;
        cc = cp;
    }
    pap = block_sum<TX / 2 * TY>(pap, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = pap;
}

template <int TX, int TY>
__global__ void __launch_bounds__(TX / 2 * TY) upd_ldg(const double *__restrict__ p, double *__restrict__ r,
                                                       double *__restrict__ x, int n, int nchunk, double alpha,
                                                       double off, double diag, double *partials)
{
    __shared__ double red[32];
    const int ntx = n / TX, nty = n / TY, ntiles = ntx * nty;
    const int tile = blockIdx.x % ntiles, chunk = blockIdx.x / ntiles;
    const int i = (tile % ntx) * TX + 2 * (threadIdx.x % (TX / 2));
    const int j = (tile / ntx) * TY + threadIdx.x / (TX / 2);
    const int z0 = n * chunk / nchunk, z1 = n * (chunk + 1) / nchunk;
    const long long pl = (long long)n * n;
    const long long base = i + (long long)n * j;
    const bool hxl = i > 0, hxr = i + 2 < n, hym = j > 0, hyp = j + 1 < n;
    const double2 zero = make_double2(0, 0);
    double2 cm = z0 > 0 ? ldp(p + base + pl * (z0 - 1)) : zero;
    double2 cc = ldp(p + base + pl * z0);
    double rr = 0.0;
    for (int z = z0; z < z1; ++z) {
        const long long o = base + pl * z;
        double2 cp = z + 1 < n ? ldp(p + o + pl) : zero;
        double xl = hxl ? __ldg(p + o - 1) : 0.0, xr = hxr ? __ldg(p + o + 2) : 0.0;
        double2 ym = hym ? ldp(p + o - n) : zero, yp = hyp ? ldp(p + o + n) : zero;
        double a0 = diag * cc.x;
        a0 = a0 + off * cc.y;
        a0 = a0 + off * yp.x;
        a0 = a0 + off * cp.x;
        a0 = a0 + off * cm.x;
        a0 = a0 + off * ym.x;
        a0 = a0 + off * xl;
        double a1 = diag * cc.y;
        a1 = a1 + off * xr;
        a1 = a1 + off * yp.y;
        a1 = a1 + off * cp.y;
        a1 = a1 + off * cm.y;
        a1 = a1 + off * ym.y;
        a1 = a1 + off * cc.x;
        double2 xv = __ldcs(reinterpret_cast<const double2 *>(x + o));
        double2 rv = __ldcs(reinterpret_cast<const double2 *>(r + o));
        __stcs(reinterpret_cast<double2 *>(x + o), make_double2(xv.x + alpha * cc.x, xv.y + alpha * cc.y));
        double r0 = rv.x - alpha * a0, r1 = rv.y - alpha * a1;
        __stcs(reinterpret_cast<double2 *>(r + o), make_double2(r0, r1));
        rr = rr + r0 * r0;
        rr = rr + r1 * r1;
        cm = cc;
        cc = cp;
    }
    rr = block_sum<TX / 2 * TY>(rr, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = rr;
}


// x-neighbours by warp shuffle: a warp is one 64-cell tile row (TX == 64),
// lane k's left neighbour is lane k-1's cc.y; only lanes 0 / 31 load.
template <int TY>
__global__ void __launch_bounds__(32 * TY) dir_shfl(const double *__restrict__ r, const double *__restrict__ po,
                                                    double *__restrict__ pn, int n, int nchunk, double zc,
                                                    double beta, double off, double diag, double *partials)
{
    __shared__ double red[32];
    constexpr int TX = 64;
    const int ntx = n / TX, nty = n / TY, ntiles = ntx * nty;
    const int tile = blockIdx.x % ntiles, chunk = blockIdx.x / ntiles;
    const int lane = threadIdx.x & 31;
    const int i = (tile % ntx) * TX + 2 * lane;
    const int j = (tile / ntx) * TY + threadIdx.x / 32;
    const int z0 = n * chunk / nchunk, z1 = n * (chunk + 1) / nchunk;
    const long long pl = (long long)n * n;
    const long long base = i + (long long)n * j;
    const bool hxl = i > 0, hxr = i + 2 < n, hym = j > 0, hyp = j + 1 < n;
    auto P2 = [&](long long o) {
        double2 a = ldp(r + o), b = ldp(po + o);
        return make_double2(a.x * zc + beta * b.x, a.y * zc + beta * b.y);
    };
    auto P1 = [&](long long o) { return __ldg(r + o) * zc + beta * __ldg(po + o); };
    const double2 zero = make_double2(0, 0);
    double2 cm = z0 > 0 ? P2(base + pl * (z0 - 1)) : zero;
    double2 cc = P2(base + pl * z0);
    double pap = 0.0;
    for (int z = z0; z < z1; ++z) {
        const long long o = base + pl * z;
        double2 cp = z + 1 < n ? P2(o + pl) : zero;
        double xl = __shfl_up_sync(0xffffffffu, cc.y, 1), xr = __shfl_down_sync(0xffffffffu, cc.x, 1);
        if (lane == 0) xl = hxl ? P1(o - 1) : 0.0;
        if (lane == 31) xr = hxr ? P1(o + 2) : 0.0;
        double2 ym = hym ? P2(o - n) : zero, yp = hyp ? P2(o + n) : zero;
        double a0 = diag * cc.x;
        a0 = a0 + off * cc.y;
        a0 = a0 + off * yp.x;
        a0 = a0 + off * cp.x;
        a0 = a0 + off * cm.x;
        a0 = a0 + off * ym.x;
        a0 = a0 + off * xl;
        double a1 = diag * cc.y;
        a1 = a1 + off * xr;
        a1 = a1 + off * yp.y;
        a1 = a1 + off * cp.y;
        a1 = a1 + off * cm.y;
        a1 = a1 + off * ym.y;
        a1 = a1 + off * cc.x;
        *reinterpret_cast<double2 *>(pn + o) = cc;
        pap = pap + cc.x * a0;
        pap = pap + cc.y * a1;
        cm = cc;
        cc = cp;
    }
    pap = block_sum<32 * TY>(pap, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = pap;
}

template <int TY>
__global__ void __launch_bounds__(32 * TY) upd_shfl(const double *__restrict__ p, double *__restrict__ r,
                                                    double *__restrict__ x, int n, int nchunk, double alpha,
                                                    double off, double diag, double *partials)
{
    __shared__ double red[32];
    constexpr int TX = 64;
    const int ntx = n / TX, nty = n / TY, ntiles = ntx * nty;
    const int tile = blockIdx.x % ntiles, chunk = blockIdx.x / ntiles;
    const int lane = threadIdx.x & 31;
    const int i = (tile % ntx) * TX + 2 * lane;
    const int j = (tile / ntx) * TY + threadIdx.x / 32;
    const int z0 = n * chunk / nchunk, z1 = n * (chunk + 1) / nchunk;
    const long long pl = (long long)n * n;
    const long long base = i + (long long)n * j;
    const bool hxl = i > 0, hxr = i + 2 < n, hym = j > 0, hyp = j + 1 < n;
    const double2 zero = make_double2(0, 0);
    double2 cm = z0 > 0 ? ldp(p + base + pl * (z0 - 1)) : zero;
    double2 cc = ldp(p + base + pl * z0);
    double rr = 0.0;
    for (int z = z0; z < z1; ++z) {
        const long long o = base + pl * z;
        double2 cp = z + 1 < n ? ldp(p + o + pl) : zero;
        double xl = __shfl_up_sync(0xffffffffu, cc.y, 1), xr = __shfl_down_sync(0xffffffffu, cc.x, 1);
        if (lane == 0) xl = hxl ? __ldg(p + o - 1) : 0.0;
        if (lane == 31) xr = hxr ? __ldg(p + o + 2) : 0.0;
        double2 ym = hym ? ldp(p + o - n) : zero, yp = hyp ? ldp(p + o + n) : zero;
        double a0 = diag * cc.x;
        a0 = a0 + off * cc.y;
        a0 = a0 + off * yp.x;
        a0 = a0 + off * cp.x;
        a0 = a0 + off * cm.x;
        a0 = a0 + off * ym.x;
        a0 = a0 + off * xl;
        double a1 = diag * cc.y;
        a1 = a1 + off * xr;
        a1 = a1 + off * yp.y;
        a1 = a1 + off * cp.y;
        a1 = a1 + off * cm.y;
        a1 = a1 + off * ym.y;
        a1 = a1 + off * cc.x;
        double2 xv = __ldcs(reinterpret_cast<const double2 *>(x + o));
        double2 rv = __ldcs(reinterpret_cast<const double2 *>(r + o));
        __stcs(reinterpret_cast<double2 *>(x + o), make_double2(xv.x + alpha * cc.x, xv.y + alpha * cc.y));
        double r0 = rv.x - alpha * a0, r1 = rv.y - alpha * a1;
        __stcs(reinterpret_cast<double2 *>(r + o), make_double2(r0, r1));
        rr = rr + r0 * r0;
        rr = rr + r1 * r1;
        cm = cc;
        cc = cp;
    }
    rr = block_sum<32 * TY>(rr, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = rr;
}

struct Bufs;
template <int TY>
static void sweep_shfl(Bufs &b);

__global__ void fill_rand(double *a, long long n, unsigned seed)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        unsigned long long h = (unsigned long long)i * 0x9E3779B97F4A7C15ull + seed;
        h ^= h >> 29;
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 32;
        a[i] = (double)(h & 0xFFFFFFFFFFFFull) / 281474976710656.0 - 0.5;
    }
}

struct Bufs {
    double *r, *po, *pn, *x, *part;
    int n;
};

template <int TX, int TY>
static void sweep(Bufs &b)
{
    const int n = b.n;
    const double N = (double)n * n * n;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int nc : {2, 4, 8, 16, 32}) {
        int ntiles = (n / TX) * (n / TY), grid = ntiles * nc;
        float ms_d, ms_u;
        for (int w = 0; w < 3; ++w)
            dir_ldg<TX, TY><<<grid, TX / 2 * TY>>>(b.r, b.po, b.pn, n, nc, 0.5, 0.3, -1.0, 6.0, b.part);
        cudaEventRecord(e0);
        for (int k = 0; k < 20; ++k)
            dir_ldg<TX, TY><<<grid, TX / 2 * TY>>>(b.r, b.po, b.pn, n, nc, 0.5, 0.3, -1.0, 6.0, b.part);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms_d, e0, e1);
        for (int w = 0; w < 3; ++w) upd_ldg<TX, TY><<<grid, TX / 2 * TY>>>(b.pn, b.r, b.x, n, nc, 1e-9, -1.0, 6.0, b.part);
        cudaEventRecord(e0);
        for (int k = 0; k < 20; ++k)
            upd_ldg<TX, TY><<<grid, TX / 2 * TY>>>(b.pn, b.r, b.x, n, nc, 1e-9, -1.0, 6.0, b.part);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms_u, e0, e1);
        ms_d /= 20;
        ms_u /= 20;
        printf("tile %3dx%-2d thr=%3d chunks=%2d ctas=%5d: dir %6.1f us (%4.0f GB/s of 24N) | upd %6.1f us (%4.0f GB/s "
               "of 40N) | sum %6.1f us\n",
               TX, TY, TX / 2 * TY, nc, grid, ms_d * 1e3, 24 * N / (ms_d * 1e-3) / 1e9, ms_u * 1e3,
               40 * N / (ms_u * 1e-3) / 1e9, (ms_d + ms_u) * 1e3);
    }
}

template <int TY>
static void sweep_shfl(Bufs &b)
{
    const int n = b.n;
    const double N = (double)n * n * n;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int nc : {4, 8, 16, 32, 64}) {
        int ntiles = (n / 64) * (n / TY), grid = ntiles * nc;
        float ms_d, ms_u;
        for (int w = 0; w < 3; ++w) dir_shfl<TY><<<grid, 32 * TY>>>(b.r, b.po, b.pn, n, nc, 0.5, 0.3, -1.0, 6.0, b.part);
        cudaEventRecord(e0);
        for (int k = 0; k < 20; ++k) dir_shfl<TY><<<grid, 32 * TY>>>(b.r, b.po, b.pn, n, nc, 0.5, 0.3, -1.0, 6.0, b.part);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms_d, e0, e1);
        for (int w = 0; w < 3; ++w) upd_shfl<TY><<<grid, 32 * TY>>>(b.pn, b.r, b.x, n, nc, 1e-9, -1.0, 6.0, b.part);
        cudaEventRecord(e0);
        for (int k = 0; k < 20; ++k) upd_shfl<TY><<<grid, 32 * TY>>>(b.pn, b.r, b.x, n, nc, 1e-9, -1.0, 6.0, b.part);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms_u, e0, e1);
        ms_d /= 20;
        ms_u /= 20;
        printf("SHFL tile  64x%-2d thr=%3d chunks=%2d ctas=%5d: dir %6.1f us (%4.0f GB/s of 24N) | upd %6.1f us (%4.0f "
               "GB/s of 40N) | sum %6.1f us\n",
               TY, 32 * TY, nc, grid, ms_d * 1e3, 24 * N / (ms_d * 1e-3) / 1e9, ms_u * 1e3,
               40 * N / (ms_u * 1e-3) / 1e9, (ms_d + ms_u) * 1e3);
    }
}

int main(int argc, char **argv)
{
    Bufs b;
    b.n = argc > 1 ? atoi(argv[1]) : 256;
    const long long N = (long long)b.n * b.n * b.n;
    for (double **p : {&b.r, &b.po, &b.pn, &b.x}) {
        cudaMalloc(p, N * 8);
        if (getenv("PROBE_ZERO")) cudaMemset(*p, 0, N * 8);
        else fill_rand<<<1184, 256>>>(*p, N, (unsigned)(size_t)p);
    }
    cudaMalloc(&b.part, 1 << 20);
    const char *which = argc > 2 ? argv[2] : "all";
    if (which[0] == 'o') {  // one config: dir_shfl<4> / upd_shfl<4> with argv[3] chunks, 5 launches each
        int nc = argc > 3 ? atoi(argv[3]) : 8, grid = (b.n / 64) * (b.n / 4) * nc;
        for (int k = 0; k < 5; ++k) {
            dir_shfl<4><<<grid, 128>>>(b.r, b.po, b.pn, b.n, nc, 0.5, 0.3, -1.0, 6.0, b.part);
            upd_shfl<4><<<grid, 128>>>(b.pn, b.r, b.x, b.n, nc, 1e-9, -1.0, 6.0, b.part);
        }
        printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
        return 0;
    }
    if (which[0] == 'a') {
        sweep<32, 8>(b);
        sweep<64, 4>(b);
        sweep<256, 1>(b);
    }
    sweep_shfl<1>(b);
    sweep_shfl<2>(b);
    sweep_shfl<4>(b);
    sweep_shfl<8>(b);
    printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
