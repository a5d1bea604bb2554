// cf_dic.cu -- see cf_dic.cuh.
#include <algorithm>

#include "cf_dic.cuh"

namespace cf {

constexpr int kLevelThreads = 128;

// src/precond.py:24-34: d_i = A_ii - sum_{lower p} v_p^2 / d_{col p}
__global__ void __launch_bounds__(kLevelThreads) dic_factor_level(int count, const int32_t *__restrict__ rows,
                                                                  const int32_t *__restrict__ lp,
                                                                  const int32_t *__restrict__ lc,
                                                                  const double *__restrict__ lv,
                                                                  const double *__restrict__ diag, double *d,
                                                                  unsigned long long *bad)
{
    const int t = blockIdx.x * kLevelThreads + threadIdx.x;
    if (t >= count) return;
    const int i = rows[t];
    double s = diag[i];
    for (int p = lp[i]; p < lp[i + 1]; ++p) {
        const double v = lv[p];
        s = s - v * v / d[lc[p]];
    }
    d[i] = s;
    if (s <= 0.0) atomicMin(bad, (unsigned long long)i);
}

// src/precond.py:37-44: (L + D~) w = r
__global__ void __launch_bounds__(kLevelThreads) dic_fwd_level(int count, const int32_t *__restrict__ rows,
                                                               const int32_t *__restrict__ lp,
                                                               const int32_t *__restrict__ lc,
                                                               const double *__restrict__ lv,
                                                               const double *__restrict__ d,
                                                               const double *__restrict__ r, double *w,
                                                               const int *done)
{
    if (done && *done) return;
    const int t = blockIdx.x * kLevelThreads + threadIdx.x;
    if (t >= count) return;
    const int i = rows[t];
    double s = r[i];
    for (int p = lp[i]; p < lp[i + 1]; ++p) s = s - lv[p] * w[lc[p]];
    w[i] = s / d[i];
}

// src/precond.py:47-54: (D~ + L^T) z = D~ w, rows in reverse level order
__global__ void __launch_bounds__(kLevelThreads) dic_bwd_level(int count, const int32_t *__restrict__ rows,
                                                               const int32_t *__restrict__ up,
                                                               const int32_t *__restrict__ uc,
                                                               const double *__restrict__ uv,
                                                               const double *__restrict__ d,
                                                               const double *__restrict__ w, double *z,
                                                               const int *done)
{
    if (done && *done) return;
    const int t = blockIdx.x * kLevelThreads + threadIdx.x;
    if (t >= count) return;
    const int i = rows[t];
    double s = 0.0;
    for (int p = up[i]; p < up[i + 1]; ++p) s = s + uv[p] * z[uc[p]];
    z[i] = w[i] - s / d[i];
}

static inline int blocks_for(long long count) { return (int)((count + kLevelThreads - 1) / kLevelThreads); }

int dic_apply_launch(const DicData &dd, const double *r, double *w, double *z, const int *done, cudaStream_t s)
{
    const int nl = (int)dd.level_ptr.size() - 1;
    for (int l = 0; l < nl; ++l) {
        const long long b = dd.level_ptr[l], c = dd.level_ptr[l + 1] - b;
        if (c <= 0) continue;
        dic_fwd_level<<<blocks_for(c), kLevelThreads, 0, s>>>((int)c, dd.rows + b, dd.lp, dd.lc, dd.lv, dd.d, r,
                                                              w, done);
    }
    for (int l = nl - 1; l >= 0; --l) {
        const long long b = dd.level_ptr[l], c = dd.level_ptr[l + 1] - b;
        if (c <= 0) continue;
        dic_bwd_level<<<blocks_for(c), kLevelThreads, 0, s>>>((int)c, dd.rows + b, dd.up, dd.uc, dd.uv, dd.d, w,
                                                              z, done);
    }
    CF_CHECK_LAUNCH("dic sweeps");
    return CF_OK;
}

}  // namespace cf

extern "C" {

int cf_level_schedule(int64_t n, const int64_t *lower_ptr, const int64_t *lower_col, int32_t *level_host,
                      int32_t *nlevels_host)
{
    CF_REQUIRE(n >= 0 && level_host && nlevels_host, "cf_level_schedule: bad arguments");
    int32_t top = -1;
    for (int64_t i = 0; i < n; ++i) {
        int32_t lv = 0;
        for (int64_t p = lower_ptr[i]; p < lower_ptr[i + 1]; ++p) {
            const int64_t j = lower_col[p];
            CF_REQUIRE(j >= 0 && j < i, "cf_level_schedule: lower triangle holds col >= row");
            lv = std::max(lv, level_host[j] + 1);
        }
        level_host[i] = lv;
        top = std::max(top, lv);
    }
    *nlevels_host = top + 1;
    return CF_OK;
}

int cf_dic_factor(int64_t n, const int32_t *lp, const int32_t *lc, const double *lv, const double *diag,
                  const int32_t *level_rows, const int64_t *level_ptr_host, int nlevels, double *d,
                  int64_t *bad_row_host, void *stream)
{
    CF_REQUIRE(n >= 0 && nlevels >= 0 && bad_row_host, "cf_dic_factor: bad arguments");
    cudaStream_t s = cf::as_stream(stream);
    double *scratch = cf::scratch_partials();
    if (!scratch) { cf::set_error("scratch allocation failed"); return CF_ENOMEM; }
    unsigned long long *bad = reinterpret_cast<unsigned long long *>(scratch);
    const unsigned long long none = ~0ull;
    CF_CUDA(cudaMemcpyAsync(bad, &none, sizeof(none), cudaMemcpyHostToDevice, s));
    for (int l = 0; l < nlevels; ++l) {
        const long long b = level_ptr_host[l], c = level_ptr_host[l + 1] - b;
        if (c <= 0) continue;
        cf::dic_factor_level<<<cf::blocks_for(c), cf::kLevelThreads, 0, s>>>((int)c, level_rows + b, lp, lc, lv,
                                                                             diag, d, bad);
    }
    CF_CHECK_LAUNCH("dic_factor_level");
    unsigned long long got = 0;
    CF_CUDA(cudaMemcpyAsync(&got, bad, sizeof(got), cudaMemcpyDeviceToHost, s));
    CF_CUDA(cudaStreamSynchronize(s));
    *bad_row_host = got == none ? -1 : (int64_t)got;
    if (got != none) {
        cf::set_error("DIC breakdown at row " + std::to_string((long long)got));
        return CF_EINVAL;
    }
    return CF_OK;
}

int cf_dic_apply(int64_t n, const int32_t *lp, const int32_t *lc, const double *lv, const int32_t *up,
                 const int32_t *uc, const double *uv, const double *d, const int32_t *level_rows,
                 const int64_t *level_ptr_host, int nlevels, const double *r, double *w, double *z,
                 void *stream)
{
    CF_REQUIRE(n >= 0 && nlevels >= 0, "cf_dic_apply: bad arguments");
    cf::DicData dd;
    dd.n = n;
    dd.lp = lp; dd.lc = lc; dd.lv = lv;
    dd.up = up; dd.uc = uc; dd.uv = uv;
    dd.d = d;
    dd.rows = level_rows;
    dd.level_ptr.assign(level_ptr_host, level_ptr_host + nlevels + 1);
    return cf::dic_apply_launch(dd, r, w, z, nullptr, cf::as_stream(stream));
}

}  // extern "C"
