// cf_common.cuh -- shared device helpers for the cavityflow B200 kernels.
//
// Everything in this library is compiled with -fmad=false: the reference's
// numba kernels never contract a*b+c into an FMA, and keeping the same
// rounding per element is what lets the SpMV/stencil, axpy, advection,
// divergence and correction kernels match the reference bit for bit.  The
// path is HBM-bound, so the lost FMA throughput is free.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/cfgpu.h"

namespace cf {

constexpr int kWarp = 32;

// ---------------------------------------------------------------- errors
void set_error(const std::string &msg);
int cuda_fail(cudaError_t e, const char *where);

#define CF_CUDA(call)                                                  \
    do {                                                               \
        cudaError_t e_ = (call);                                       \
        if (e_ != cudaSuccess) return ::cf::cuda_fail(e_, #call);      \
    } while (0)

#define CF_CHECK_LAUNCH(name)                                          \
    do {                                                               \
        cudaError_t e_ = cudaGetLastError();                           \
        if (e_ != cudaSuccess) return ::cf::cuda_fail(e_, name);       \
    } while (0)

#define CF_REQUIRE(cond, msg)                                          \
    do {                                                               \
        if (!(cond)) { ::cf::set_error(msg); return CF_EINVAL; }       \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

int num_sms();
// Resident blocks per SM for `kernel` at `threads` threads and `smem` bytes.
int blocks_per_sm(const void *kernel, int threads, size_t smem);
// z-chunk count for a z-march over `tiles` xy tiles and nz planes with
// `slots` resident CTAs on the device: wave-quantisation aware (cf_runtime.cu).
int wave_chunks(long long tiles, int nz, long long slots, int min_planes);

// Per-process scratch for one-shot reductions (cf_dot etc.).
constexpr size_t kScratchPartials = 1 << 16;
double *scratch_partials();
double *host_result_slot();

// ---------------------------------------------------------------- reductions
// Deterministic block reduction: fixed shuffle tree, then warp 0 sums the
// warp partials in warp order.  Every thread must call it; the block total
// is returned on thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *smem)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = NT / 32;
    __syncthreads();
    if (lane == 0) smem[wid] = v;
    __syncthreads();
    if (wid == 0) {
        v = lane < NW ? smem[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    return v;
}

// Three sums with one pair of barriers (smem: 96 doubles); the totals on thread 0.
template <int NT>
__device__ __forceinline__ void block_sum3(double &a, double &b, double &c, double *smem)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, o);
        b += __shfl_down_sync(0xffffffffu, b, o);
        c += __shfl_down_sync(0xffffffffu, c, o);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = NT / 32;
    __syncthreads();
    if (lane == 0) {
        smem[wid] = a;
        smem[32 + wid] = b;
        smem[64 + wid] = c;
    }
    __syncthreads();
    if (wid == 0) {
        a = lane < NW ? smem[lane] : 0.0;
        b = lane < NW ? smem[32 + lane] : 0.0;
        c = lane < NW ? smem[64 + lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_down_sync(0xffffffffu, a, o);
            b += __shfl_down_sync(0xffffffffu, b, o);
            c += __shfl_down_sync(0xffffffffu, c, o);
        }
    }
}

// Fixed-order sums of `count` interleaved partial triples by warp 0 (no block
// barrier); the totals on thread 0.
__device__ __forceinline__ void warp_reduce_partials3(const double *p, int count, double &a, double &b, double &c)
{
    const int lane = threadIdx.x & 31;
    a = b = c = 0.0;
    for (int i = lane; i < count; i += 32) {
        a += __ldcg(p + 3 * (size_t)i);
        b += __ldcg(p + 3 * (size_t)i + 1);
        c += __ldcg(p + 3 * (size_t)i + 2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, o);
        b += __shfl_down_sync(0xffffffffu, b, o);
        c += __shfl_down_sync(0xffffffffu, c, o);
    }
}

template <int NT>
__device__ __forceinline__ double block_max(double v, double *smem)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = NT / 32;
    __syncthreads();
    if (lane == 0) smem[wid] = v;
    __syncthreads();
    if (wid == 0) {
        v = lane < NW ? smem[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    }
    return v;
}

// Last-block-done pattern: returns true in exactly one block (the last to
// finish) after all blocks published their partials.  Thread 0 decides;
// the result is broadcast through shared memory.
__device__ __forceinline__ bool last_block(unsigned int *ticket, int *flag_smem)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned int t = atomicAdd(ticket, 1u);
        *flag_smem = (t == gridDim.x - 1);
        if (*flag_smem) *ticket = 0u;  // re-arm for the next launch
    }
    __syncthreads();
    bool last = *flag_smem;
    if (last) __threadfence();
    return last;
}

// Programmatic dependent launch (PDL): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may be scheduled while
// its predecessor's last CTAs still run; it must wait for the predecessor's
// completion (and memory) before reading anything it produced.  Both
// instructions are no-ops for a normal launch.  The loop kernels trigger their
// dependents only after their sweep (griddep_trigger): triggering at entry let
// waiting CTAs of the next kernel take SM slots early and cost 10 % (CF_PDL=1
// measured: 193 -> 212 us per 256^3 iteration; with the late trigger, neutral).
__device__ __forceinline__ void griddep_enter() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Fixed-order sum of `count` partials with stride `stride` by one block.
template <int NT>
__device__ __forceinline__ double reduce_partials(const double *p, int count, int stride, double *smem)
{
    double v = 0.0;
    for (int i = threadIdx.x; i < count; i += NT) v += __ldcg(p + (size_t)i * stride);
    return block_sum<NT>(v, smem);
}

// ---------------------------------------------------------------- grid geometry
// A cell-centred scalar block: x fastest, row pitch nx, plane pitch nx*ny.
// `lo_halo`/`hi_halo` say whether plane -1 / plane nz exist in memory (the
// z-slab halo of a multi-GPU run); a missing neighbour is a Dirichlet-ghost
// zero, i.e. its stencil term is dropped exactly as the reference's
// assembly drops it (src/sim.py:296-317).
struct Box {
    int nx, ny, nz;
    int lo_halo, hi_halo;
    __host__ __device__ long long plane() const { return (long long)nx * ny; }
    __host__ __device__ long long cells() const { return plane() * nz; }
};

}  // namespace cf
