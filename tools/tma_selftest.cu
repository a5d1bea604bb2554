// Standalone check of the TMA/mbarrier helpers (cf_tma.cuh) -- debug tool.
// usage: tma_selftest <variant>   0: full helper path  1: no prefetch
//        2: non-negative coords  3: no fence_barrier_init
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2504_03697_b200/csrc/cf_tma.cuh"
using namespace cf;

__global__ void k(const __grid_constant__ CUtensorMap m, double *out, int variant)
{
    extern __shared__ unsigned char raw[];
    __shared__ __align__(8) uint64_t bar;
    double *s = reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        if (variant != 3) fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (variant != 1) prefetch_map(&m);
        mbar_expect_tx(&bar, kHX * kHY * 8);
        int x = variant == 2 ? 0 : (variant == 4 ? 46 : (variant == 5 ? 47 : -1)), y = variant == 4 ? 23 : (variant == 5 ? 0 : x);
        tma_load_3d(s, &m, x, y, 1, &bar);
    }
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < kHX * kHY; i += blockDim.x) out[i] = s[i];
}

int main(int argc, char **argv)
{
    int variant = argc > 1 ? atoi(argv[1]) : 0;
    const int nx = 64, ny = 32, nz = 4;
    std::vector<double> h(nx * ny * nz);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *d, *o;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&o, kHX * kHY * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    CUtensorMap m;
    if (!make_map(&m, d, nx, ny, nz, kHX, kHY)) { printf("make_map failed\n"); return 2; }
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    k<<<1, 128, 16384>>>(m, o, variant);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s\n", variant, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<double> r(kHX * kHY);
    cudaMemcpy(r.data(), o, r.size() * 8, cudaMemcpyDeviceToHost);
    int x0 = variant == 2 ? 0 : (variant == 4 ? 46 : (variant == 5 ? 47 : -1)), y0 = variant == 4 ? 23 : (variant == 5 ? 0 : x0), bad = 0;
    for (int y = 0; y < kHY; ++y)
        for (int x = 0; x < kHX; ++x) {
            int gx = x0 + x, gy = y0 + y;
            double want = (gx < 0 || gy < 0 || gx >= nx || gy >= ny) ? 0.0 : h[gx + nx * (gy + ny * 1)];
            if (r[x + kHX * y] != want) ++bad;
        }
    printf("variant %d: %d mismatches\n", variant, bad);
    return bad != 0;
}
