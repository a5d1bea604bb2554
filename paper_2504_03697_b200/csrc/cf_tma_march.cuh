// cf_tma_march.cuh -- the staged z-march device loop (see cf_tma.cuh).
#pragma once

#include "cf_stencil.cuh"
#include "cf_tma.cuh"

namespace cf {

constexpr int kBox = kHX * kHY;        // halo box, doubles (648)
constexpr int kBoxStride = 656;         // padded to a 128-byte multiple
constexpr int kInt = kTTX * kTTY;       // interior box, doubles (512)
constexpr uint32_t kBoxBytes = kBox * 8;
constexpr uint32_t kIntBytes = kInt * 8;

// 128-byte aligned base of the dynamic shared memory (TMA destinations).
__device__ __forceinline__ double *aligned_smem(unsigned char *raw)
{
    return reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
}

// The block's (tile, chunk) is blockIdx.x = chunk * ntiles + tile.  Pol
// provides issue(slot, x0, y0, z, z0, z1, bar) (thread 0 only; TMA loads of
// plane z into `slot`), value(slot, off) (operand at a stage offset) and
// epi(slot, tx, ty, i, j, z, centre, ax) for each owned cell.
template <int ORDER, class Pol>
__device__ __forceinline__ void staged_march(const TmaGeom &g, double off, double diag, Pol &pol, uint64_t *bars)
{
    const int tid = threadIdx.x, tx = tid % kTTX, ty = tid / kTTX;
    const int ntiles = g.ntx * g.nty;
    const int tile = blockIdx.x % ntiles, chunk = blockIdx.x / ntiles;
    const int x0 = (tile % g.ntx) * kTTX, y0 = (tile / g.ntx) * kTTY;
    const int z0 = (int)((long long)g.nz * chunk / g.nchunk);
    const int z1 = (int)((long long)g.nz * (chunk + 1) / g.nchunk);
    const int zlo = g.lo_halo ? -1 : 0, zhi = g.hi_halo ? g.nz : g.nz - 1;
    const int zs = max(z0 - 1, zlo), ze = min(z1, zhi);
    const int nplanes = ze - zs + 1;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    // Halo box origin (see kHX): two cells before the tile in x (keeps the
    // origin 16-byte aligned), one row before in y, clamped at the low walls
    // where the missing neighbour is masked by the existence flags anyway.
    const int bx0 = max(x0 - 2, 0), by0 = max(y0 - 1, 0);
    if (tid == 0) {
        pol.prefetch();
        for (int q = 0; q < min(kStages, nplanes); ++q)
            pol.issue(q % kStages, bx0, by0, x0, y0, zs + q, z0, z1, &bars[q % kStages]);
    }
    const int i = x0 + tx, j = y0 + ty;
    const bool valid = i < g.nx && j < g.ny;
    const bool hxm = i > 0, hxp = i < g.nx - 1, hym = j > 0, hyp = j < g.ny - 1;
    const int o = (j - by0) * kHX + (i - bx0);
    auto wait = [&](int q) { mbar_wait(&bars[q % kStages], (uint32_t)((q / kStages) & 1)); };
    auto release = [&](int q) {
        __syncthreads();  // every thread is done reading this slot
        if (tid == 0 && q + kStages < nplanes)
            pol.issue(q % kStages, bx0, by0, x0, y0, zs + q + kStages, z0, z1, &bars[q % kStages]);
    };
    int q = 0;
    double cprev = 0.0;
    wait(0);
    if (zs < z0) {
        cprev = pol.value(0, o);
        release(0);
        q = 1;
        wait(1);
    }
    double ccur = pol.value(q % kStages, o);
    for (int z = z0; z < z1; ++z, ++q) {
        const bool hzm = z - 1 >= zlo, hzp = z + 1 <= zhi;
        double cnext = 0.0;
        if (hzp) {
            wait(q + 1);
            cnext = pol.value((q + 1) % kStages, o);
        }
        const int s = q % kStages;
        const double xm = hxm ? pol.value(s, o - 1) : 0.0;
        const double xp = hxp ? pol.value(s, o + 1) : 0.0;
        const double ym = hym ? pol.value(s, o - kHX) : 0.0;
        const double yp = hyp ? pol.value(s, o + kHX) : 0.0;
        const double ax = stencil7<ORDER>(ccur, xm, xp, ym, yp, cprev, cnext, hxm, hxp, hym, hyp, hzm, hzp, off, diag);
        if (valid) pol.epi(s, tx, ty, i, j, z, ccur, ax);
        release(q);
        cprev = ccur;
        ccur = cnext;
    }
}

}  // namespace cf
