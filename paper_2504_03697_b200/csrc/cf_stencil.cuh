// cf_stencil.cuh -- the matrix-free 7-point operator and the 2.5-D z-march
// shared by the stencil apply and the fused CG kernels.
//
// Operator (src/sim.py:296-333): (A x)_c = diag*x_c + off*sum(existing
// neighbours), diag = 6/h^2, off = -1/h^2; a neighbour outside the domain is
// a Dirichlet ghost (value 0) whose term is simply absent.  The summation
// order is a template parameter so the result is bit-identical to either
// reference SpMV (see CF_ORDER_* in cfgpu.h).
//
// Work decomposition: the nx*ny plane is cut into TX x TY tiles; a "unit" is
// one tile on one z-plane.  The units are ordered tile-major, z-minor and
// split into gridDim.x contiguous, equal ranges, so every block marches the
// same number of planes (+-1) whatever the grid shape -- no wave tail.  A
// thread owns one (i, j) column of its tile and keeps x at z-1, z, z+1 in
// registers while marching; in-plane neighbours come through L1.
#pragma once

#include "cf_common.cuh"

namespace cf {

constexpr int kTX = 32;
constexpr int kTY = 8;
constexpr int kMarchThreads = kTX * kTY;

// Grid for a march kernel: resident capacity (148 x blocks/SM), capped by
// the number of (tile, plane) units.
int march_grid(const void *kernel, const Box &bx);

template <int ORDER>
__device__ __forceinline__ double stencil7(double c, double xm, double xp, double ym, double yp,
                                           double zm, double zp, bool hxm, bool hxp, bool hym,
                                           bool hyp, bool hzm, bool hzp, double off, double diag)
{
    double s;
    if (ORDER == CF_ORDER_CSR) {
        // src/sparse.py:194-201 over columns k-1, j-1, i-1, i, i+1, j+1, k+1
        s = 0.0;
        if (hzm) s = s + off * zm;
        if (hym) s = s + off * ym;
        if (hxm) s = s + off * xm;
        s = s + diag * c;
        if (hxp) s = s + off * xp;
        if (hyp) s = s + off * yp;
        if (hzp) s = s + off * zp;
    } else {
        // src/sparse.py:204-213: diagonal, upper (i+1, j+1, k+1), then the
        // transposed lower entries in ascending row order (k-1, j-1, i-1)
        s = diag * c;
        if (hxp) s = s + off * xp;
        if (hyp) s = s + off * yp;
        if (hzp) s = s + off * zp;
        if (hzm) s = s + off * zm;
        if (hym) s = s + off * ym;
        if (hxm) s = s + off * xm;
    }
    return s;
}

// Marches this block's share of (tile, plane) units.  `load(idx)` yields the
// operand value at flat index idx (may compute it on the fly); `epi(idx, c,
// ax)` receives the centre value and (A x) at each owned cell.
template <int ORDER, class Load, class Epi>
__device__ __forceinline__ void march(const Box bx, double off, double diag, Load &load, Epi &epi)
{
    const int tx = threadIdx.x % kTX, ty = threadIdx.x / kTX;
    const int ntx = (bx.nx + kTX - 1) / kTX, nty = (bx.ny + kTY - 1) / kTY;
    const long long nz = bx.nz;
    const long long total = (long long)ntx * nty * nz;
    const long long u_begin = total * blockIdx.x / gridDim.x;
    const long long u_end = total * (blockIdx.x + 1) / gridDim.x;
    const long long pl = bx.plane();
    for (long long u = u_begin; u < u_end;) {
        const long long tile = u / nz;
        const int z0 = (int)(u % nz);
        const int z1 = (int)min(nz, (long long)z0 + (u_end - u));
        u += z1 - z0;
        const int i = (int)(tile % ntx) * kTX + tx;
        const int j = (int)(tile / ntx) * kTY + ty;
        if (i >= bx.nx || j >= bx.ny) continue;
        const bool hxm = i > 0, hxp = i < bx.nx - 1, hym = j > 0, hyp = j < bx.ny - 1;
        long long idx = (long long)i + (long long)bx.nx * j + pl * z0;
        double cm = (z0 > 0 || bx.lo_halo) ? load(idx - pl) : 0.0;
        double cc = load(idx);
        for (int z = z0; z < z1; ++z, idx += pl) {
            const bool hzm = z > 0 || bx.lo_halo;
            const bool hzp = z < bx.nz - 1 || bx.hi_halo;
            const double cp = hzp ? load(idx + pl) : 0.0;
            const double xm = hxm ? load(idx - 1) : 0.0;
            const double xp = hxp ? load(idx + 1) : 0.0;
            const double ym = hym ? load(idx - bx.nx) : 0.0;
            const double yp = hyp ? load(idx + bx.nx) : 0.0;
            const double ax = stencil7<ORDER>(cc, xm, xp, ym, yp, cm, cp, hxm, hxp, hym, hyp, hzm,
                                              hzp, off, diag);
            epi(idx, cc, ax);
            cm = cc;
            cc = cp;
        }
    }
}

}  // namespace cf
