// cf_runtime.cu -- error state, device queries and reduction scratch.
#include <mutex>
#include <string>

#include "cf_common.cuh"

namespace cf {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int cuda_fail(cudaError_t e, const char *where)
{
    set_error(std::string(where) + ": " + cudaGetErrorName(e) + ": " + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? CF_ENOMEM : CF_ECUDA;
}

int num_sms()
{
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

int blocks_per_sm(const void *kernel, int threads, size_t smem)
{
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem) != cudaSuccess || b < 1)
        b = 1;
    return b;
}

int wave_chunks(long long tiles, int nz, long long slots, int min_planes)
{
    // Each SM runs ceil(tiles*c / slots) waves of CTAs, each marching nz/c
    // planes plus ~2 planes of halo / pipeline fill; pick the chunk count c
    // with the least per-SM march length.  (256^3: a partly filled second
    // wave -- e.g. 1280 pair CTAs on 1184 slots -- cost 15 % of the kernel.)
    if (tiles < 1) tiles = 1;
    if (slots < 1) slots = 1;
    const int cmax = nz / (min_planes > 0 ? min_planes : 1) > 1 ? nz / (min_planes > 0 ? min_planes : 1) : 1;
    int best = 1;
    double best_cost = 1e300;
    for (int c = 1; c <= cmax; ++c) {
        const long long waves = (tiles * c + slots - 1) / slots;
        const double cost = (double)waves * ((double)nz / c + 2.0);
        if (cost < best_cost * 0.999) {
            best_cost = cost;
            best = c;
        }
    }
    return best;
}

static std::mutex g_scratch_mu;
static double *g_scratch = nullptr;
static double *g_host_slot = nullptr;

// Fixed layout: kScratchPartials partial slots, then the result slot, then
// the last-block ticket (zeroed once, re-armed by every reduction).
double *scratch_partials()
{
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    if (!g_scratch) {
        size_t bytes = (kScratchPartials + 2) * sizeof(double);
        if (cudaMalloc(&g_scratch, bytes) != cudaSuccess) { g_scratch = nullptr; return nullptr; }
        if (cudaMemset(g_scratch, 0, bytes) != cudaSuccess) return nullptr;
        cudaDeviceSynchronize();
    }
    return g_scratch;
}

double *host_result_slot()
{
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    if (!g_host_slot && cudaMallocHost(&g_host_slot, 8 * sizeof(double)) != cudaSuccess)
        g_host_slot = nullptr;
    return g_host_slot;
}

}  // namespace cf

extern "C" {

const char *cf_last_error(void) { return cf::g_last_error.c_str(); }

int cf_version(void) { return 1; }

int cf_device_sms(void) { return cf::num_sms(); }

}  // extern "C"
