// Standalone check of the TMA/mbarrier helpers (cf_tma.cuh) -- debug tool.
// usage: tma_selftest <variant>   (box origins per variant: see coords())
//        2: non-negative coords  3: no fence_barrier_init
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2504_03697_b200/csrc/cf_tma.cuh"
using namespace cf;

// box origin per variant: 0 (-1,-1,1)  2 (0,0,1)  4 (46,23,1)  5 (47,0,1)
// 6 (-2,-2,1)  7 (-2,0,1)  8 (0,-2,1)  9 (0,0,-1)  10 (-2,-2,-1)  11 (0,0,4)
__host__ __device__ void coords(int v, int &x, int &y, int &z)
{
    z = 1;
    switch (v) {
    case 2: x = 0; y = 0; break;
    case 4: x = 46; y = 23; break;
    case 5: x = 47; y = 0; break;
    case 6: x = -2; y = -2; break;
    case 7: x = -2; y = 0; break;
    case 8: x = 0; y = -2; break;
    case 9: x = 0; y = 0; z = -1; break;
    case 10: x = -2; y = -2; z = -1; break;
    case 11: x = 0; y = 0; z = 4; break;
    default: x = -1; y = -1;
    }
}

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
        int x, y, z;
        coords(variant, x, y, z);
        tma_load_3d(s, &m, x, y, z, &bar);
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
    int x0, y0, z0, bad = 0;
    coords(variant, x0, y0, z0);
    for (int y = 0; y < kHY; ++y)
        for (int x = 0; x < kHX; ++x) {
            int gx = x0 + x, gy = y0 + y;
            double want = (gx < 0 || gy < 0 || gx >= nx || gy >= ny || z0 < 0 || z0 >= nz) ? 0.0 : h[gx + nx * (gy + ny * z0)];
            if (r[x + kHX * y] != want) ++bad;
        }
    printf("variant %d: %d mismatches\n", variant, bad);
    return bad != 0;
}
