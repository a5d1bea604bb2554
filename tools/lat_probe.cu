// Dependent-issue latencies a lone warp sees on this GPU: DFMA, DMUL, DADD, SHFL.UP (64-bit), FSEL, LDS.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double a, double b, long long *out, double *sink)
{
    __shared__ double sm[64];
    sm[threadIdx.x] = a;
    __syncwarp();
    double x = a + threadIdx.x;
    long long t0, t1;
    const int N = 4096;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = __fma_rn(x, b, a);
    t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = __dmul_rn(x, b);
    t1 = clock64();
    if (threadIdx.x == 0) out[1] = t1 - t0;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = __dadd_rn(x, b);
    t1 = clock64();
    if (threadIdx.x == 0) out[2] = t1 - t0;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = __shfl_up_sync(0xffffffffu, x, 1);
    t1 = clock64();
    if (threadIdx.x == 0) out[3] = t1 - t0;
    float f = (float)x;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) f = __fmaf_rn(f, 1.0001f, 0.5f);
    t1 = clock64();
    if (threadIdx.x == 0) out[4] = t1 - t0;
    int idx = threadIdx.x;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) idx = (int)sm[idx & 31] & 31;
    t1 = clock64();
    if (threadIdx.x == 0) out[5] = t1 - t0;
    sink[threadIdx.x] = x + f + idx;
}
int main()
{
    long long *out, h[6];
    double *sink;
    cudaMalloc(&out, sizeof(h));
    cudaMalloc(&sink, 32 * 8);
    for (int rep = 0; rep < 2; ++rep) {
        k<<<1, 32>>>(1.0000001, 0.9999999, out, sink);
        cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    }
    const char *names[6] = {"DFMA", "DMUL", "DADD", "SHFL.UP x2 (64-bit)", "FFMA", "LDS+cvt chain"};
    for (int i = 0; i < 6; ++i) printf("%s: %.1f cycles per dependent op\n", names[i], h[i] / 4096.0);
    return 0;
}
