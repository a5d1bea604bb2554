// Calibration tool 2: does the xy-tile / z-march ACCESS PATTERN (not the
// stencil arithmetic) cap HBM throughput?  Copies an n^3 fp64 volume with
// (a) a flat grid-stride double2 copy, (b) xy tiles TX x TY marching z over
// nchunk z-chunks (the CG kernels' pattern, no halo, no arithmetic), and
// (c) the same tiles with a register-window 7-point stencil (halo reads via L1/L2).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void copy2(const double2 *__restrict__ a, double2 *__restrict__ b, long long n2)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x)
        b[i] = a[i];
}

template <int TX, int TY>
__global__ void tile_copy(const double *__restrict__ a, double *__restrict__ b, int n, int nchunk)
{
    const int ntx = n / TX, nty = n / TY, ntiles = ntx * nty;
    const int tile = blockIdx.x % ntiles, chunk = blockIdx.x / ntiles;
    const int i = (tile % ntx) * TX + 2 * (threadIdx.x % (TX / 2));
    const int j = (tile / ntx) * TY + threadIdx.x / (TX / 2);
    const int z0 = n * chunk / nchunk, z1 = n * (chunk + 1) / nchunk;
    const long long pl = (long long)n * n;
    const double *src = a + i + (long long)n * j;
    double *dst = b + i + (long long)n * j;
#pragma unroll 4
    for (int z = z0; z < z1; ++z) {
        double2 v = __ldcs(reinterpret_cast<const double2 *>(src + pl * z));
        __stcs(reinterpret_cast<double2 *>(dst + pl * z), v);
    }
}

// streaming mixes with no stencil: R reads + W writes per cell (distinct arrays)
template <int TX, int TY, int R, int W>
__global__ void tile_mix(const double *__restrict__ a, const double *__restrict__ b, const double *__restrict__ c,
                         double *__restrict__ d, double *__restrict__ e, int n, int nchunk)
{
    const int ntx = n / TX, nty = n / TY, ntiles = ntx * nty;
    const int tile = blockIdx.x % ntiles, chunk = blockIdx.x / ntiles;
    const int i = (tile % ntx) * TX + 2 * (threadIdx.x % (TX / 2));
    const int j = (tile / ntx) * TY + threadIdx.x / (TX / 2);
    const int z0 = n * chunk / nchunk, z1 = n * (chunk + 1) / nchunk;
    const long long pl = (long long)n * n;
    const long long base = i + (long long)n * j;
#pragma unroll 2
    for (int z = z0; z < z1; ++z) {
        const long long o = base + pl * z;
        double2 v = __ldg(reinterpret_cast<const double2 *>(a + o));
        if (R > 1) {
            double2 w = __ldg(reinterpret_cast<const double2 *>(b + o));
            v.x += w.x;
            v.y += w.y;
        }
        if (R > 2) {
            double2 w = __ldg(reinterpret_cast<const double2 *>(c + o));
            v.x += w.x;
            v.y += w.y;
        }
        *reinterpret_cast<double2 *>(d + o) = v;
        if (W > 1) *reinterpret_cast<double2 *>(e + o) = make_double2(v.y, v.x);
    }
}

template <int TX, int TY>
__global__ void tile_stencil(const double *__restrict__ a, double *__restrict__ b, int n, int nchunk)
{
    const int ntx = n / TX, nty = n / TY, ntiles = ntx * nty;
    const int tile = blockIdx.x % ntiles, chunk = blockIdx.x / ntiles;
    const int i = (tile % ntx) * TX + 2 * (threadIdx.x % (TX / 2));
    const int j = (tile / ntx) * TY + threadIdx.x / (TX / 2);
    const int z0 = n * chunk / nchunk, z1 = n * (chunk + 1) / nchunk;
    const long long pl = (long long)n * n;
    const double *src = a + i + (long long)n * j;
    double *dst = b + i + (long long)n * j;
    double2 cm = z0 > 0 ? *reinterpret_cast<const double2 *>(src + pl * (z0 - 1)) : make_double2(0, 0);
    double2 cc = *reinterpret_cast<const double2 *>(src + pl * z0);
    for (int z = z0; z < z1; ++z) {
        double2 cp = z + 1 < n ? *reinterpret_cast<const double2 *>(src + pl * (z + 1)) : make_double2(0, 0);
        const double *s = src + pl * z;
        double xl = i > 0 ? __ldg(s - 1) : 0.0, xr = i + 2 < n ? __ldg(s + 2) : 0.0;
        double2 ym = j > 0 ? __ldg(reinterpret_cast<const double2 *>(s - n)) : make_double2(0, 0);
        double2 yp = j + 1 < n ? __ldg(reinterpret_cast<const double2 *>(s + n)) : make_double2(0, 0);
        double r0 = 6.0 * cc.x - xl - cc.y - ym.x - yp.x - cm.x - cp.x;
        double r1 = 6.0 * cc.y - cc.x - xr - ym.y - yp.y - cm.y - cp.y;
        *reinterpret_cast<double2 *>(dst + pl * z) = make_double2(r0, r1);
        cm = cc;
        cc = cp;
    }
}

static float time_it(void (*launch)(void *), void *arg)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) launch(arg);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) launch(arg);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 20;
}

struct Args {
    double *x, *y;
    int n, nchunk, grid;
};

template <int TX, int TY, bool ST>
static void run_tile(void *p)
{
    Args *a = (Args *)p;
    int ntiles = (a->n / TX) * (a->n / TY);
    if (ST) tile_stencil<TX, TY><<<ntiles * a->nchunk, (TX / 2) * TY>>>(a->x, a->y, a->n, a->nchunk);
    else tile_copy<TX, TY><<<ntiles * a->nchunk, (TX / 2) * TY>>>(a->x, a->y, a->n, a->nchunk);
}

static void run_copy(void *p)
{
    Args *a = (Args *)p;
    long long N = (long long)a->n * a->n * a->n;
    copy2<<<a->grid, 256>>>((double2 *)a->x, (double2 *)a->y, N / 2);
}

template <int TX, int TY>
static void sweep(Args &a, double bytes)
{
    for (int nc : {1, 2, 4, 8, 16, 37}) {
        a.nchunk = nc;
        float c = time_it(run_tile<TX, TY, false>, &a);
        float s = time_it(run_tile<TX, TY, true>, &a);
        int ntiles = (a.n / TX) * (a.n / TY);
        printf("tile %3dx%-2d chunks=%2d ctas=%5d: copy %6.1f us %5.0f GB/s | stencil %6.1f us %5.0f GB/s\n", TX, TY,
               nc, ntiles * nc, c * 1e3, bytes / (c * 1e-3) / 1e9, s * 1e3, bytes / (s * 1e-3) / 1e9);
    }
}

template <int R, int W>
static void mix(double *a, double *b, double *c, double *d, double *e, int n)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int nc : {4, 8, 16}) {
        const int grid = (n / 64) * (n / 4) * nc;
        for (int w = 0; w < 3; ++w) tile_mix<64, 4, R, W><<<grid, 128>>>(a, b, c, d, e, n, nc);
        cudaEventRecord(e0);
        for (int k = 0; k < 10; ++k) tile_mix<64, 4, R, W><<<grid, 128>>>(a, b, c, d, e, n, nc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 10;
        const double bytes = 8.0 * (R + W) * n * (double)n * n;
        printf("mix %dR+%dW chunks=%2d: %6.1f us %5.0f GB/s\n", R, W, nc, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    }
}

int main(int argc, char **argv)
{
    const int n = argc > 1 ? atoi(argv[1]) : 256;
    const long long N = (long long)n * n * n;
    Args a;
    cudaMalloc(&a.x, N * 8);
    cudaMalloc(&a.y, N * 8);
    cudaMemset(a.x, 0, N * 8);
    cudaMemset(a.y, 0, N * 8);
    a.n = n;
    const double bytes = 16.0 * N;
    for (int g : {148 * 4, 148 * 16, 148 * 32}) {
        a.grid = g;
        float ms = time_it(run_copy, &a);
        printf("flat copy grid=%d: %.1f us %.0f GB/s\n", g, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    }
    if (argc > 2) {
        double *c, *d, *e;
        cudaMalloc(&c, N * 8);
        cudaMalloc(&d, N * 8);
        cudaMalloc(&e, N * 8);
        cudaMemset(c, 0, N * 8);
        mix<1, 1>(a.x, a.y, c, d, e, n);
        mix<2, 1>(a.x, a.y, c, d, e, n);
        mix<3, 1>(a.x, a.y, c, d, e, n);
        mix<3, 2>(a.x, a.y, c, d, e, n);
        mix<2, 2>(a.x, a.y, c, d, e, n);
        return 0;
    }
    sweep<32, 16>(a, bytes);
    sweep<64, 8>(a, bytes);
    sweep<128, 4>(a, bytes);
    sweep<256, 2>(a, bytes);
    sweep<64, 16>(a, bytes);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
