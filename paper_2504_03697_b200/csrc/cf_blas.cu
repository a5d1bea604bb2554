// cf_blas.cu -- vector kernels of src/sparse.py:270-301 and the Jacobi
// apply of src/precond.py:89-95.  Elementwise kernels perform exactly the
// reference's per-element operation (no FMA: -fmad=false), so axpy/add/
// scale/mul are bit-identical to the reference; dot and max use a fixed
// two-level reduction tree (deterministic run to run, not the reference's
// serial order, which is a tolerance-level difference -- src/sparse.py:273-277).
#include <mutex>

#include "cf_common.cuh"

namespace cf {

constexpr int kBlasThreads = 256;

static int reduce_grid(int64_t n)
{
    int64_t want = (n + kBlasThreads * 4 - 1) / (kBlasThreads * 4);
    int64_t cap = (int64_t)num_sms() * 8;
    if (want > cap) want = cap;
    if (want < 1) want = 1;
    return (int)want;
}

// MODE 0: sum x*y   MODE 1: max |x|
template <int MODE>
__global__ void __launch_bounds__(kBlasThreads) reduce_kernel(const double *__restrict__ x,
                                                               const double *__restrict__ y,
                                                               int64_t n, double *partials,
                                                               unsigned int *ticket,
                                                               double *result)
{
    __shared__ double red[32];
    __shared__ int is_last;
    double acc = 0.0;
    const int64_t stride = (int64_t)gridDim.x * kBlasThreads;
    for (int64_t i = (int64_t)blockIdx.x * kBlasThreads + threadIdx.x; i < n; i += stride) {
        if (MODE == 0) acc += x[i] * y[i];
        else acc = fmax(acc, fabs(x[i]));
    }
    double b = MODE == 0 ? block_sum<kBlasThreads>(acc, red) : block_max<kBlasThreads>(acc, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = b;
    if (last_block(ticket, &is_last)) {
        double v = 0.0;
        for (int i = threadIdx.x; i < (int)gridDim.x; i += kBlasThreads) {
            double p = __ldcg(partials + i);
            v = MODE == 0 ? v + p : fmax(v, p);
        }
        v = MODE == 0 ? block_sum<kBlasThreads>(v, red) : block_max<kBlasThreads>(v, red);
        if (threadIdx.x == 0) *result = v;
    }
}

static std::mutex g_reduce_mu;

template <int MODE>
static int reduce_to_host(const double *x, const double *y, int64_t n, double *out, void *stream)
{
    std::lock_guard<std::mutex> lk(g_reduce_mu);
    if (n == 0) { *out = 0.0; return CF_OK; }
    int grid = reduce_grid(n);
    double *scratch = scratch_partials();
    double *slot = host_result_slot();
    if (!scratch || !slot) { set_error("reduction scratch allocation failed"); return CF_ENOMEM; }
    double *result = scratch + kScratchPartials;
    unsigned int *ticket = reinterpret_cast<unsigned int *>(scratch + kScratchPartials + 1);
    cudaStream_t s = as_stream(stream);
    reduce_kernel<MODE><<<grid, kBlasThreads, 0, s>>>(x, y, n, scratch, ticket, result);
    CF_CHECK_LAUNCH("reduce_kernel");
    CF_CUDA(cudaMemcpyAsync(slot, result, sizeof(double), cudaMemcpyDeviceToHost, s));
    CF_CUDA(cudaStreamSynchronize(s));
    *out = *slot;
    return CF_OK;
}

// OP 0: y += a*x   OP 1: out = x + y   OP 2: out = a*x   OP 3: out = x*y
template <int OP>
__global__ void __launch_bounds__(kBlasThreads) elementwise_kernel(double *__restrict__ out,
                                                                    const double *__restrict__ x,
                                                                    const double *__restrict__ y,
                                                                    double a, int64_t n)
{
    const int64_t stride = (int64_t)gridDim.x * kBlasThreads;
    for (int64_t i = (int64_t)blockIdx.x * kBlasThreads + threadIdx.x; i < n; i += stride) {
        if (OP == 0) out[i] = out[i] + a * x[i];
        else if (OP == 1) out[i] = x[i] + y[i];
        else if (OP == 2) out[i] = a * x[i];
        else out[i] = x[i] * y[i];
    }
}

template <int OP>
static int elementwise(double *out, const double *x, const double *y, double a, int64_t n,
                       void *stream)
{
    CF_REQUIRE(n >= 0, "negative vector length");
    if (n == 0) return CF_OK;
    int64_t want = (n + kBlasThreads - 1) / kBlasThreads;
    int64_t cap = (int64_t)num_sms() * 16;
    int grid = (int)(want < cap ? want : cap);
    elementwise_kernel<OP><<<grid, kBlasThreads, 0, as_stream(stream)>>>(out, x, y, a, n);
    CF_CHECK_LAUNCH("elementwise_kernel");
    return CF_OK;
}

}  // namespace cf

extern "C" {

int cf_dot(const double *x, const double *y, int64_t n, double *result_host, void *stream)
{
    CF_REQUIRE(n >= 0 && result_host, "cf_dot: bad arguments");
    return cf::reduce_to_host<0>(x, y, n, result_host, stream);
}

int cf_max_abs(const double *x, int64_t n, double *result_host, void *stream)
{
    CF_REQUIRE(n >= 0 && result_host, "cf_max_abs: bad arguments");
    return cf::reduce_to_host<1>(x, x, n, result_host, stream);
}

int cf_axpy(double *y, double alpha, const double *x, int64_t n, void *stream)
{
    return cf::elementwise<0>(y, x, nullptr, alpha, n, stream);
}

int cf_add(const double *x, const double *y, double *out, int64_t n, void *stream)
{
    return cf::elementwise<1>(out, x, y, 0.0, n, stream);
}

int cf_scale(double alpha, const double *x, double *out, int64_t n, void *stream)
{
    return cf::elementwise<2>(out, x, nullptr, alpha, n, stream);
}

int cf_mul(const double *x, const double *y, double *out, int64_t n, void *stream)
{
    return cf::elementwise<3>(out, x, y, 0.0, n, stream);
}

}  // extern "C"
