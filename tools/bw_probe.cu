// Calibration tool: HBM throughput of simple fp64 kernels on this GPU.
//  copy (double2 grid-stride), naive 7-point stencil (one thread per cell).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void copy2(const double2 *__restrict__ a, double2 *__restrict__ b, long long n2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void stencil_naive(const double *__restrict__ x, double *__restrict__ y, int n, double off, double diag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y * blockDim.y + threadIdx.y, k = blockIdx.z;
  if (i >= n || j >= n) return;
  long long c = i + (long long)n * (j + (long long)n * k), pl = (long long)n * n;
  double s = diag * __ldg(x + c);
  if (i < n - 1) s += off * __ldg(x + c + 1);
  if (j < n - 1) s += off * __ldg(x + c + n);
  if (k < n - 1) s += off * __ldg(x + c + pl);
  if (k > 0) s += off * __ldg(x + c - pl);
  if (j > 0) s += off * __ldg(x + c - n);
  if (i > 0) s += off * __ldg(x + c - 1);
  y[c] = s;
}
int main(int argc, char **argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 256; const long long N = (long long)n * n * n;
  double *x, *y; cudaMalloc(&x, N * 8); cudaMalloc(&y, N * 8); cudaMemset(x, 0, N * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  for (int g : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
    for (int w = 0; w < 3; ++w) copy2<<<g, 256>>>((double2 *)x, (double2 *)y, N / 2);
    cudaEventRecord(a); for (int r = 0; r < 20; ++r) copy2<<<g, 256>>>((double2 *)x, (double2 *)y, N / 2); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("copy grid=%d: %.1f us %.0f GB/s\n", g, ms / 20 * 1e3, 16.0 * N / (ms / 20 * 1e-3) / 1e9);
  }
  for (int by : {4, 8}) {
    dim3 blk(64, by), grd((n + 63) / 64, (n + by - 1) / by, n);
    for (int w = 0; w < 3; ++w) stencil_naive<<<grd, blk>>>(x, y, n, -1.0, 6.0);
    cudaEventRecord(a); for (int r = 0; r < 20; ++r) stencil_naive<<<grd, blk>>>(x, y, n, -1.0, 6.0); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("naive stencil 64x%d: %.1f us %.0f GB/s\n", by, ms / 20 * 1e3, 16.0 * N / (ms / 20 * 1e-3) / 1e9);
  }
  return 0;
}
