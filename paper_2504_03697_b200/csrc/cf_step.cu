// cf_step.cu -- the non-CG kernels of one cavity time step (src/sim.py:
// 134-289, :352-449, src/grid.py:102-154), each the reference's per-element
// arithmetic in the reference's order (-fmad=false), so results are
// bit-identical to the reference.
//
// Geometry: an nx x ny x nz box of cells of edge h (the reference's cube is
// nx = ny = nz = n; other boxes are the SURVEY.md §8 f2 extension).  Velocity
// component c has extents (nx+[c==0], ny+[c==1], nz+[c==2]) stored x-fastest
// with row pitch ld_c (padded to a 32-double multiple by the host so every row
// starts 256-B aligned) and plane pitch ld_c * (ny+[c==1]).  Every kernel also
// runs on a z-slab: the arrays then hold the global planes k_base .. where
// k_base = z0 - H (H halo planes below the slab's first owned plane z0); the
// single-domain entry points are the slab [0, nz) with H = 0.
#include <algorithm>

#include <cmath>
#include <cstring>

#include "cf_common.cuh"
#include "cf_tma.cuh"

namespace cf {

struct Comp {
    const double *a;
    int na, nb, nc, ld;  // global extents, row pitch
    int k_base;          // global plane index of a's first stored plane
    // 32-bit offsets (a stored component stays below 2^32 elements; checked
    // by make_vel): one IMAD.WIDE per address instead of 64-bit arithmetic
    __device__ __forceinline__ unsigned off(int i, int j, int k) const
    {
        return (unsigned)i + (unsigned)ld * ((unsigned)j + (unsigned)nb * (unsigned)(k - k_base));
    }
    __device__ __forceinline__ double at(int i, int j, int k) const { return __ldg(a + off(i, j, k)); }
};

__device__ __forceinline__ double clamp_hi(double a, double hi)
{
    if (a < 0.0) return 0.0;
    if (a > hi) return hi;
    return a;
}

__device__ __forceinline__ int base_index(double a, int na)
{
    int i0 = (int)a;
    if (i0 > na - 2) i0 = na > 1 ? na - 2 : 0;
    return i0;
}

// src/sim.py:156-190 (_tri): clamped trilinear interpolation at lattice
// coordinates (a, b, c); blend order fixed.
__device__ __forceinline__ double trilerp(const Comp &f, double a, double b, double c)
{
    a = clamp_hi(a, f.na - 1.0);
    b = clamp_hi(b, f.nb - 1.0);
    c = clamp_hi(c, f.nc - 1.0);
    const int i0 = base_index(a, f.na), j0 = base_index(b, f.nb), k0 = base_index(c, f.nc);
    const int i1 = min(i0 + 1, f.na - 1), j1 = min(j0 + 1, f.nb - 1), k1 = min(k0 + 1, f.nc - 1);
    const double fa = a - (double)i0, fb = b - (double)j0, fc = c - (double)k0;
    const double c00 = f.at(i0, j0, k0) * (1.0 - fa) + f.at(i1, j0, k0) * fa;
    const double c10 = f.at(i0, j1, k0) * (1.0 - fa) + f.at(i1, j1, k0) * fa;
    const double c01 = f.at(i0, j0, k1) * (1.0 - fa) + f.at(i1, j0, k1) * fa;
    const double c11 = f.at(i0, j1, k1) * (1.0 - fa) + f.at(i1, j1, k1) * fa;
    return (c00 * (1.0 - fb) + c10 * fb) * (1.0 - fc) + (c01 * (1.0 - fb) + c11 * fb) * fc;
}

struct Vel3 {
    Comp c[3];
};

// Slab of the box: owned planes [z0, z1) of nz; H halo planes each side.
struct SlabZ {
    int nx, ny, nz, z0, z1, H;
    __host__ __device__ int k_base() const { return z0 - H; }
    // owned w faces: [z0, z1), plus the top wall face when the slab ends at nz
    __host__ __device__ int w_end() const { return z1 == nz ? nz + 1 : z1; }
    __host__ __device__ int ext(int axis) const { return axis == 0 ? nx : (axis == 1 ? ny : nz); }
};

__host__ __device__ inline Comp make_comp(const double *a, const SlabZ &sz, int comp, int ld)
{
    return Comp{a, sz.nx + (comp == 0), sz.ny + (comp == 1), sz.nz + (comp == 2), ld, sz.k_base()};
}

static Vel3 make_vel(const double *u, const double *v, const double *w, const SlabZ &sz, int ldu, int ldv, int ldw)
{
    return Vel3{{make_comp(u, sz, 0, ldu), make_comp(v, sz, 1, ldv), make_comp(w, sz, 2, ldw)}};
}

constexpr int kFaceThreads = 256;

// src/sim.py:193-240 + :283-288.  blockIdx.y = component; a grid-stride
// loop over the slab's owned faces with i fastest (coalesced stores).
// POW2: h is a power of two, so every q / h the reference evaluates equals
// q * (1/h) exactly (scaling by 2^k is exact) -- the dozen fp64 divisions per
// face, which dominated this kernel, become multiplications, bit-identically.
template <bool POW2>
__device__ __forceinline__ void advect_face(const Vel3 &in, const Comp &me, double *out, const SlabZ &sz, int comp,
                                            unsigned f, double h, double inv_h, double dt, double lx, double ly,
                                            double lz)
{
    auto over_h = [&](double q) { return POW2 ? q * inv_h : q / h; };
    // 32-bit face index (a slab's faces of one component < 2^32, checked on the host)
    const int i = (int)(f % (unsigned)me.na);
    const unsigned rest = f / (unsigned)me.na;
    const int j = (int)(rest % (unsigned)me.nb), k = sz.z0 + (int)(rest / (unsigned)me.nb);
    double *dst = out + me.off(i, j, k);
    const int wall = comp == 0 ? i : (comp == 1 ? j : k);
    if (wall == 0 || wall == sz.ext(comp)) {  // wall-normal planes are zeroed (:283-288)
        *dst = 0.0;
        return;
    }
    double x, y, z;
    if (comp == 0) {
        x = i * h; y = (j + 0.5) * h; z = (k + 0.5) * h;
    } else if (comp == 1) {
        x = (i + 0.5) * h; y = j * h; z = (k + 0.5) * h;
    } else {
        x = (i + 0.5) * h; y = (j + 0.5) * h; z = k * h;
    }
    const double xh = over_h(x), yh = over_h(y), zh = over_h(z);
    const double su = trilerp(in.c[0], xh, yh - 0.5, zh - 0.5);
    const double sv = trilerp(in.c[1], xh - 0.5, yh, zh - 0.5);
    const double sw = trilerp(in.c[2], xh - 0.5, yh - 0.5, zh);
    const double xb = over_h(clamp_hi(x - dt * su, lx));
    const double yb = over_h(clamp_hi(y - dt * sv, ly));
    const double zb = over_h(clamp_hi(z - dt * sw, lz));
    double r;
    if (comp == 0) r = trilerp(me, xb, yb - 0.5, zb - 0.5);
    else if (comp == 1) r = trilerp(me, xb - 0.5, yb, zb - 0.5);
    else r = trilerp(me, xb - 0.5, yb - 0.5, zb);
    *dst = r;
}

// src/sim.py:193-240 + :283-288: a grid-stride loop over face index f with
// i fastest (coalesced stores); each thread advects face f of ALL three
// components, so the three sweeps move through the domain together and the
// velocity planes they sample are read from HBM once (a launch per component
// -- or blockIdx.y = component -- sweeps the whole field three times).
// The gathers are latency-bound: capped at 64 registers (4 CTAs/SM, no
// spills) the kernel runs 2.10 ms per 256^3 step instead of 2.66 at 100-128
// registers (measured; 48 / 40 registers spill and lose again).
// POW2: h is a power of two, so every q / h the reference evaluates equals
// q * (1/h) exactly (scaling by 2^k is exact): the fp64 divisions become
// multiplications, bit-identically.
template <bool POW2>
__global__ void __launch_bounds__(kFaceThreads, 4) advect_kernel(Vel3 in, double *nu, double *nv, double *nw,
                                                              SlabZ sz, double h, double inv_h, double dt)
{
    unsigned total[3];
    for (int c = 0; c < 3; ++c)
        total[c] = (unsigned)in.c[c].na * (unsigned)in.c[c].nb * (unsigned)((c == 2 ? sz.w_end() : sz.z1) - sz.z0);
    const unsigned tmax = max(total[0], max(total[1], total[2]));
    const unsigned stride = gridDim.x * kFaceThreads;
    const double lx = sz.nx * h, ly = sz.ny * h, lz = sz.nz * h;  // side lengths (length = n*h)
    for (unsigned f = blockIdx.x * kFaceThreads + threadIdx.x; f < tmax; f += stride) {
        if (f < total[0]) advect_face<POW2>(in, in.c[0], nu, sz, 0, f, h, inv_h, dt, lx, ly, lz);
        if (f < total[1]) advect_face<POW2>(in, in.c[1], nv, sz, 1, f, h, inv_h, dt, lx, ly, lz);
        if (f < total[2]) advect_face<POW2>(in, in.c[2], nw, sz, 2, f, h, inv_h, dt, lx, ly, lz);
    }
}

#include "cf_advect.cuh"

static bool is_pow2(double h)
{
    int e;
    return h > 0 && std::frexp(h, &e) == 0.5;
}

// src/sim.py:134-149 on the slab.  blockIdx.y selects the task: 0 = lid row
// u[1:nx, ny-1, k] += lid_dv; 1..6 = the six wall-normal planes.
__global__ void forces_bc_kernel(double *u, double *v, double *w, SlabZ sz, int ldu, int ldv, int ldw, double lid_dv,
                                 int apply_lid)
{
    const int task = blockIdx.y;
    const int nx = sz.nx, ny = sz.ny, nz = sz.nz, kb = sz.k_base(), nzl = sz.z1 - sz.z0;
    long long m;  // items of this task
    if (task == 0) m = apply_lid ? (long long)(nx - 1) * nzl : 0;
    else if (task <= 2) m = (long long)ny * nzl;
    else if (task <= 4) m = (long long)nx * nzl;
    else m = ((task == 5 && sz.z0 == 0) || (task == 6 && sz.z1 == nz)) ? (long long)nx * ny : 0;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < m; t += (long long)gridDim.x * blockDim.x) {
        if (task == 0) {  // u[i, ny-1, k], i in [1, nx-1]
            const int i = 1 + (int)(t % (nx - 1)), k = sz.z0 + (int)(t / (nx - 1));
            double *q = u + i + (long long)ldu * ((long long)(ny - 1) + (long long)ny * (k - kb));
            *q = *q + lid_dv;
        } else if (task <= 2) {  // u[0|nx, j, k]
            const int j = (int)(t % ny), k = sz.z0 + (int)(t / ny);
            u[(task == 1 ? 0 : nx) + (long long)ldu * (j + (long long)ny * (k - kb))] = 0.0;
        } else if (task <= 4) {  // v[i, 0|ny, k]
            const int i = (int)(t % nx), k = sz.z0 + (int)(t / nx);
            v[i + (long long)ldv * ((task == 3 ? 0 : ny) + (long long)(ny + 1) * (k - kb))] = 0.0;
        } else {  // w[i, j, 0|nz], owned by the slab holding that wall
            const int i = (int)(t % nx), j = (int)(t / nx);
            const int k = task == 5 ? 0 : nz;
            w[i + (long long)ldw * (j + (long long)ny * (k - kb))] = 0.0;
        }
    }
}

constexpr int kCellThreads = 256;

// src/grid.py:145-154: ((((u1-u0)+v1)-v0)+w1)-w0, then /h, then * scale
// (src/sim.py:360), over the slab's owned cells; out is slab-local (plane
// k - z0).  Partial max|out| per block.
__global__ void __launch_bounds__(kCellThreads) divergence_kernel(Vel3 in, SlabZ sz, double h, double scale,
                                                                  int do_scale, double *out, double *partials,
                                                                  unsigned int *ticket, double *result)
{
    __shared__ double red[32];
    __shared__ int is_last;
    const int nx = sz.nx, ny = sz.ny;
    // 32-bit cell index (a slab's cells < 2^31, checked by pitches_ok)
    const int total = nx * ny * (sz.z1 - sz.z0);
    const int stride = gridDim.x * kCellThreads;
    double mx = 0.0;
    for (int c = blockIdx.x * kCellThreads + threadIdx.x; c < total; c += stride) {
        const int i = c % nx;
        const int rest = c / nx;
        const int j = rest % ny, k = sz.z0 + rest / ny;
        double t = in.c[0].at(i + 1, j, k) - in.c[0].at(i, j, k);
        t = t + in.c[1].at(i, j + 1, k);
        t = t - in.c[1].at(i, j, k);
        t = t + in.c[2].at(i, j, k + 1);
        t = t - in.c[2].at(i, j, k);
        double d = t / h;
        if (do_scale) d = scale * d;
        out[c] = d;
        mx = fmax(mx, fabs(d));
    }
    mx = block_max<kCellThreads>(mx, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = mx;
    if (last_block(ticket, &is_last)) {
        double v = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += kCellThreads) v = fmax(v, __ldcg(partials + b));
        v = block_max<kCellThreads>(v, red);
        if (threadIdx.x == 0) *result = v;
    }
}

// The same as a z-march (round 2): a CTA owns a 32 x 8 column of cells over a
// chunk of planes, a thread one (i, j) column -- no integer division per
// cell, running pointers, w at k kept from the previous plane, and with a
// power-of-two h the reference's "/ h" as an exact multiplication.  Same
// operations in the same order: bit-identical (the flat kernel above stays
// for the parity test and odd pitches).
constexpr int kDivTX = 32, kDivTY = 8;
template <bool POW2>
__global__ void __launch_bounds__(kCellThreads) divergence_march(Vel3 in, SlabZ sz, double h, double inv_h,
                                                                 double scale, int do_scale, int nchunk, double *out,
                                                                 double *partials, unsigned int *ticket,
                                                                 double *result)
{
    __shared__ double red[32];
    __shared__ int is_last;
    const int nx = sz.nx, ny = sz.ny, nzl = sz.z1 - sz.z0;
    const int tx = threadIdx.x % kDivTX, ty = threadIdx.x / kDivTX;
    const int ntx = (nx + kDivTX - 1) / kDivTX;
    int bid = blockIdx.x;
    const int chunk = bid % nchunk;
    bid /= nchunk;
    const int i = (bid % ntx) * kDivTX + tx, j = (bid / ntx) * kDivTY + ty;
    const int k0 = sz.z0 + (int)((long long)chunk * nzl / nchunk), k1 = sz.z0 + (int)((long long)(chunk + 1) * nzl / nchunk);
    double mx = 0.0;
    if (i < nx && j < ny && k0 < k1) {
        const Comp &cu = in.c[0], &cv = in.c[1], &cw = in.c[2];
        const double *pu = cu.a + cu.off(i, j, k0), *pv = cv.a + cv.off(i, j, k0), *pw = cw.a + cw.off(i, j, k0);
        const unsigned su = (unsigned)cu.ld * (unsigned)cu.nb, sv = (unsigned)cv.ld * (unsigned)cv.nb,
                       sw = (unsigned)cw.ld * (unsigned)cw.nb, rv = (unsigned)cv.ld;
        double *po = out + ((long long)(k0 - sz.z0) * ny + j) * nx + i;
        const long long so = (long long)nx * ny;
        double w0 = __ldg(pw);
        for (int k = k0; k < k1; ++k) {
            const double u0 = __ldg(pu), u1 = __ldg(pu + 1), v0 = __ldg(pv), v1 = __ldg(pv + rv), w1 = __ldg(pw + sw);
            // src/grid.py:145-154: ((((u1-u0)+v1)-v0)+w1)-w0, then /h, then * scale (src/sim.py:360)
            double t = u1 - u0;
            t = t + v1;
            t = t - v0;
            t = t + w1;
            t = t - w0;
            double d = POW2 ? t * inv_h : t / h;
            if (do_scale) d = scale * d;
            *po = d;
            mx = fmax(mx, fabs(d));
            w0 = w1;
            pu += su;
            pv += sv;
            pw += sw;
            po += so;
        }
    }
    mx = block_max<kCellThreads>(mx, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = mx;
    if (last_block(ticket, &is_last)) {
        double v = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += kCellThreads) v = fmax(v, __ldcg(partials + b));
        v = block_max<kCellThreads>(v, red);
        if (threadIdx.x == 0) *result = v;
    }
}

// src/sim.py:434-449.  One thread per owned cell: it recomputes the
// corrected values of its six faces from the OLD field (p with a one-plane
// halo in z, ghost p = 0 outside the box), takes the cell divergence of the
// corrected faces for div_post, and writes the faces it owns (its three lower
// faces and, on the high walls, the upper ones) to the output field with the
// wall-normal faces clamped to zero.  p is slab-local (plane k - z0) and
// readable at planes -1 and nzl when the slab has neighbours there.
__global__ void __launch_bounds__(kCellThreads) correct_kernel(Vel3 in, double *nu, double *nv, double *nw,
                                                               const double *__restrict__ p, SlabZ sz, double h,
                                                               double coef, double *partials, unsigned int *ticket,
                                                               double *result)
{
    __shared__ double red[32];
    __shared__ int is_last;
    const int nx = sz.nx, ny = sz.ny, nz = sz.nz;
    // 32-bit (signed: the slab's p halo plane sits at c - pl < 0) cell index
    const int total = nx * ny * (sz.z1 - sz.z0);
    const int stride = gridDim.x * kCellThreads;
    const int pl = nx * ny;
    double mx = 0.0;
    for (int c = blockIdx.x * kCellThreads + threadIdx.x; c < total; c += stride) {
        const int i = c % nx;
        const int rest = c / nx;
        const int j = rest % ny, k = sz.z0 + rest / ny;
        const double pc = __ldg(p + c);
        // lower face: interior -> coef*(p - p_prev); wall -> coef*p
        // upper face: interior -> coef*(p_next - p); wall -> coef*(0.0 - p)
        const double du0 = i > 0 ? pc - __ldg(p + c - 1) : pc;
        const double du1 = i < nx - 1 ? __ldg(p + c + 1) - pc : 0.0 - pc;
        const double dv0 = j > 0 ? pc - __ldg(p + c - nx) : pc;
        const double dv1 = j < ny - 1 ? __ldg(p + c + nx) - pc : 0.0 - pc;
        const double dw0 = k > 0 ? pc - __ldg(p + c - pl) : pc;
        const double dw1 = k < nz - 1 ? __ldg(p + c + pl) - pc : 0.0 - pc;
        const double u0 = in.c[0].at(i, j, k) - coef * du0;
        const double u1 = in.c[0].at(i + 1, j, k) - coef * du1;
        const double v0 = in.c[1].at(i, j, k) - coef * dv0;
        const double v1 = in.c[1].at(i, j + 1, k) - coef * dv1;
        const double w0 = in.c[2].at(i, j, k) - coef * dw0;
        const double w1 = in.c[2].at(i, j, k + 1) - coef * dw1;
        double t = u1 - u0;
        t = t + v1;
        t = t - v0;
        t = t + w1;
        t = t - w0;
        mx = fmax(mx, fabs(t / h));
        const Comp &cu = in.c[0], &cv = in.c[1], &cw = in.c[2];
        nu[cu.off(i, j, k)] = i == 0 ? 0.0 : u0;
        nv[cv.off(i, j, k)] = j == 0 ? 0.0 : v0;
        nw[cw.off(i, j, k)] = k == 0 ? 0.0 : w0;
        if (i == nx - 1) nu[cu.off(nx, j, k)] = 0.0;
        if (j == ny - 1) nv[cv.off(i, ny, k)] = 0.0;
        if (k == nz - 1) nw[cw.off(i, j, nz)] = 0.0;
    }
    mx = block_max<kCellThreads>(mx, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = mx;
    if (last_block(ticket, &is_last)) {
        double v = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += kCellThreads) v = fmax(v, __ldcg(partials + b));
        v = block_max<kCellThreads>(v, red);
        if (threadIdx.x == 0) *result = v;
    }
}

// The correction as a z-march (round 2; see divergence_march): a thread owns an
// (i, j) column of a chunk of planes, keeps p at k and k+1 and the corrected
// upper w face (which is the next cell's lower one: the same operands and
// operations) in registers -- 10 loads per cell instead of 13, no integer
// division, "/ h" as an exact multiplication for a power-of-two h.
// Bit-identical to correct_kernel.  Six CTAs per SM (40 registers, a few
// spilled words) measured best: 186 us per 256^3 call against 211 / 221 / 272
// at five / four (no cap) / eight.
template <bool POW2>
__global__ void __launch_bounds__(kCellThreads, 6) correct_march(Vel3 in, double *nu, double *nv, double *nw,
                                                              const double *__restrict__ p, SlabZ sz, double h,
                                                              double inv_h, double coef, int nchunk, double *partials,
                                                              unsigned int *ticket, double *result)
{
    __shared__ double red[32];
    __shared__ int is_last;
    const int nx = sz.nx, ny = sz.ny, nz = sz.nz, nzl = sz.z1 - sz.z0;
    const int tx = threadIdx.x % kDivTX, ty = threadIdx.x / kDivTX;
    const int ntx = (nx + kDivTX - 1) / kDivTX;
    int bid = blockIdx.x;
    const int chunk = bid % nchunk;
    bid /= nchunk;
    const int i = (bid % ntx) * kDivTX + tx, j = (bid / ntx) * kDivTY + ty;
    const int k0 = sz.z0 + (int)((long long)chunk * nzl / nchunk), k1 = sz.z0 + (int)((long long)(chunk + 1) * nzl / nchunk);
    double mx = 0.0;
    if (i < nx && j < ny && k0 < k1) {
        const Comp &cu = in.c[0], &cv = in.c[1], &cw = in.c[2];
        const bool hxm = i > 0, hxp = i < nx - 1, hym = j > 0, hyp = j < ny - 1;
        const int pl = nx * ny;
        const double *pp = p + ((long long)(k0 - sz.z0) * ny + j) * nx + i;
        unsigned ou = cu.off(i, j, k0), ov = cv.off(i, j, k0), ow = cw.off(i, j, k0);
        const unsigned su = (unsigned)cu.ld * (unsigned)cu.nb, sv = (unsigned)cv.ld * (unsigned)cv.nb,
                       sw = (unsigned)cw.ld * (unsigned)cw.nb, rv = (unsigned)cv.ld;
        double pc = __ldg(pp);
        // lower face: interior -> coef*(p - p_prev); wall -> coef*p
        // upper face: interior -> coef*(p_next - p); wall -> coef*(0.0 - p)
        double w0 = __ldg(cw.a + ow) - coef * (k0 > 0 ? pc - __ldg(pp - pl) : pc);
        for (int k = k0; k < k1; ++k) {
            const bool hzp = k < nz - 1;
            const double pn = hzp ? __ldg(pp + pl) : 0.0;
            const double du0 = hxm ? pc - __ldg(pp - 1) : pc;
            const double du1 = hxp ? __ldg(pp + 1) - pc : 0.0 - pc;
            const double dv0 = hym ? pc - __ldg(pp - nx) : pc;
            const double dv1 = hyp ? __ldg(pp + nx) - pc : 0.0 - pc;
            const double dw1 = hzp ? pn - pc : 0.0 - pc;
            const double u0 = __ldg(cu.a + ou) - coef * du0;
            const double u1 = __ldg(cu.a + ou + 1) - coef * du1;
            const double v0 = __ldg(cv.a + ov) - coef * dv0;
            const double v1 = __ldg(cv.a + ov + rv) - coef * dv1;
            const double w1 = __ldg(cw.a + ow + sw) - coef * dw1;
            double t = u1 - u0;
            t = t + v1;
            t = t - v0;
            t = t + w1;
            t = t - w0;
            mx = fmax(mx, fabs(POW2 ? t * inv_h : t / h));
            nu[ou] = hxm ? u0 : 0.0;
            nv[ov] = hym ? v0 : 0.0;
            nw[ow] = k == 0 ? 0.0 : w0;
            if (!hxp) nu[ou + 1] = 0.0;
            if (!hyp) nv[ov + rv] = 0.0;
            if (!hzp) nw[ow + sw] = 0.0;
            w0 = w1;
            pc = pn;
            pp += pl;
            ou += su;
            ov += sv;
            ow += sw;
        }
    }
    mx = block_max<kCellThreads>(mx, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = mx;
    if (last_block(ticket, &is_last)) {
        double v = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += kCellThreads) v = fmax(v, __ldcg(partials + b));
        v = block_max<kCellThreads>(v, red);
        if (threadIdx.x == 0) *result = v;
    }
}

// Physics extension (the reference is inviscid): explicit
// viscous diffusion of every non-wall-normal face,
//   new = c + kdt * (((((( xm + xp) + ym) + yp) + zm) + zp) - 6*c),  kdt = nu*dt/h^2,
// on the component's own lattice.  Neighbours across a wall are ghosts:
// mirrored (+c, free slip) or antisymmetric (-c, no slip) for tangential
// components; the lid (y = Ly) with a set velocity U is a Dirichlet wall:
// ghost u = 2U - c, ghost w = -c.  Wall-normal faces stay zero.  The oracle
// restates the same order (oracle/physics_ext.py).
struct DiffBC {
    double lid_u;
    int lid_dirichlet, no_slip;
};

__device__ __forceinline__ double ghost(double c, bool anti) { return anti ? -c : c; }

__global__ void __launch_bounds__(kFaceThreads) diffuse_kernel(Vel3 in, double *nu, double *nv, double *nw, SlabZ sz,
                                                               double kdt, DiffBC bc)
{
    const int comp = blockIdx.y;
    const Comp me = in.c[comp];
    double *out = comp == 0 ? nu : (comp == 1 ? nv : nw);
    const int kend = comp == 2 ? sz.w_end() : sz.z1;
    const long long total = (long long)me.na * me.nb * (kend - sz.z0);
    const long long stride = (long long)gridDim.x * kFaceThreads;
    const bool ns = bc.no_slip != 0;
    const int nx = sz.nx, ny = sz.ny, nz = sz.nz, wall_n = sz.ext(comp);
    for (long long f = (long long)blockIdx.x * kFaceThreads + threadIdx.x; f < total; f += stride) {
        const int i = (int)(f % me.na);
        const long long rest = f / me.na;
        const int j = (int)(rest % me.nb), k = sz.z0 + (int)(rest / me.nb);
        double *dst = out + me.off(i, j, k);
        const int wall = comp == 0 ? i : (comp == 1 ? j : k);
        if (wall == 0 || wall == wall_n) {
            *dst = 0.0;
            continue;
        }
        const double c = me.at(i, j, k);
        // neighbours along the component's own axis always exist (walls are 0)
        double xm, xp, ym, yp, zm, zp;
        if (comp == 0) {
            xm = me.at(i - 1, j, k);
            xp = me.at(i + 1, j, k);
        } else {
            xm = i > 0 ? me.at(i - 1, j, k) : ghost(c, ns);
            xp = i < nx - 1 ? me.at(i + 1, j, k) : ghost(c, ns);
        }
        if (comp == 1) {
            ym = me.at(i, j - 1, k);
            yp = me.at(i, j + 1, k);
        } else {
            ym = j > 0 ? me.at(i, j - 1, k) : ghost(c, ns);
            if (j < ny - 1) yp = me.at(i, j + 1, k);
            else if (bc.lid_dirichlet) yp = comp == 0 ? 2.0 * bc.lid_u - c : -c;
            else yp = ghost(c, ns);
        }
        if (comp == 2) {
            zm = me.at(i, j, k - 1);
            zp = me.at(i, j, k + 1);
        } else {
            zm = k > 0 ? me.at(i, j, k - 1) : ghost(c, ns);
            zp = k < nz - 1 ? me.at(i, j, k + 1) : ghost(c, ns);
        }
        double s = xm + xp;
        s = s + ym;
        s = s + yp;
        s = s + zm;
        s = s + zp;
        s = s - 6.0 * c;
        *dst = c + kdt * s;
    }
}

// The same as a z-march (round 2; see divergence_march): blockIdx.y = component,
// a thread owns an (i, j) column of faces over a chunk of planes and keeps the
// component at k-1, k, k+1 in registers (five loads per face instead of
// seven, no 64-bit division).  Bit-identical to diffuse_kernel.
__global__ void __launch_bounds__(kFaceThreads) diffuse_march(Vel3 in, double *nu, double *nv, double *nw, SlabZ sz,
                                                              double kdt, DiffBC bc, int nchunk)
{
    const int comp = blockIdx.y;
    // (selected field by field: indexing the parameter array with blockIdx.y would copy it to local memory)
    const Comp me{comp == 0 ? in.c[0].a : (comp == 1 ? in.c[1].a : in.c[2].a),
                  sz.nx + (comp == 0), sz.ny + (comp == 1), sz.nz + (comp == 2),
                  comp == 0 ? in.c[0].ld : (comp == 1 ? in.c[1].ld : in.c[2].ld), in.c[0].k_base};
    double *out = comp == 0 ? nu : (comp == 1 ? nv : nw);
    const int kend = comp == 2 ? sz.w_end() : sz.z1, nzl = kend - sz.z0;
    const bool ns = bc.no_slip != 0;
    const int nx = sz.nx, ny = sz.ny, nz = sz.nz;
    const int tx = threadIdx.x % kDivTX, ty = threadIdx.x / kDivTX;
    const int ntx = (nx + 1 + kDivTX - 1) / kDivTX;
    int bid = blockIdx.x;
    const int chunk = bid % nchunk;
    bid /= nchunk;
    const int i = (bid % ntx) * kDivTX + tx, j = (bid / ntx) * kDivTY + ty;
    const int k0 = sz.z0 + (int)((long long)chunk * nzl / nchunk), k1 = sz.z0 + (int)((long long)(chunk + 1) * nzl / nchunk);
    if (i >= me.na || j >= me.nb || k0 >= k1) return;
    const bool colwall = (comp == 0 && (i == 0 || i == nx)) || (comp == 1 && (j == 0 || j == ny));
    const unsigned sp = (unsigned)me.ld * (unsigned)me.nb, rw = (unsigned)me.ld;
    unsigned o = me.off(i, j, k0);
    const int last = me.nc - 1;  // last stored plane of this component
    double cm = k0 > 0 ? __ldg(me.a + o - sp) : 0.0, c = __ldg(me.a + o);
    for (int k = k0; k < k1; ++k, o += sp) {
        const double cp = k < last ? __ldg(me.a + o + sp) : 0.0;
        if (colwall || (comp == 2 && (k == 0 || k == nz))) {
            out[o] = 0.0;
        } else {
            // neighbours along the component's own axis always exist (walls are 0)
            double xm, xp, ym, yp, zm, zp;
            if (comp == 0) {
                xm = __ldg(me.a + o - 1);
                xp = __ldg(me.a + o + 1);
            } else {
                xm = i > 0 ? __ldg(me.a + o - 1) : ghost(c, ns);
                xp = i < nx - 1 ? __ldg(me.a + o + 1) : ghost(c, ns);
            }
            if (comp == 1) {
                ym = __ldg(me.a + o - rw);
                yp = __ldg(me.a + o + rw);
            } else {
                ym = j > 0 ? __ldg(me.a + o - rw) : ghost(c, ns);
                if (j < ny - 1) yp = __ldg(me.a + o + rw);
                else if (bc.lid_dirichlet) yp = comp == 0 ? 2.0 * bc.lid_u - c : -c;
                else yp = ghost(c, ns);
            }
            if (comp == 2) {
                zm = cm;
                zp = cp;
            } else {
                zm = k > 0 ? cm : ghost(c, ns);
                zp = k < nz - 1 ? cp : ghost(c, ns);
            }
            double s = xm + xp;
            s = s + ym;
            s = s + yp;
            s = s + zm;
            s = s + zp;
            s = s - 6.0 * c;
            out[o] = c + kdt * s;
        }
        cm = c;
        c = cp;
    }
}

// Implicit (backward-Euler) diffusion of one component: (I - kdt L) u = u*,
// L the same ghost-aware Laplacian as diffuse_kernel.  A mirrored ghost (+c)
// or negated ghost (-c) folds into the diagonal, the lid's Dirichlet ghost
// 2U - c folds +kdt*c into the diagonal and 2U*kdt into the right-hand side.
// Unknowns are the component's physical (padded) array; wall-normal faces and
// row padding are identity rows with a zero right-hand side.
// MODE 0: y = A x   MODE 1: y = diag(A)   MODE 2: y = rhs from x = u*
template <int MODE>
__global__ void __launch_bounds__(kFaceThreads) helmholtz_kernel(const double *__restrict__ xin, double *__restrict__ y,
                                                                 int comp, int nx, int ny, int nz, int ld, double kdt,
                                                                 DiffBC bc)
{
    const int na = nx + (comp == 0), nb = ny + (comp == 1), nc = nz + (comp == 2);
    const long long total = (long long)ld * nb * nc;
    const long long stride = (long long)gridDim.x * kFaceThreads;
    const bool ns = bc.no_slip != 0;
    const long long pj = ld, pk = (long long)ld * nb;
    const int wall_n = comp == 0 ? nx : (comp == 1 ? ny : nz);
    for (long long f = (long long)blockIdx.x * kFaceThreads + threadIdx.x; f < total; f += stride) {
        const int i = (int)(f % ld);
        const long long rest = f / ld;
        const int j = (int)(rest % nb), k = (int)(rest / nb);
        const int wall = comp == 0 ? i : (comp == 1 ? j : k);
        if (i >= na || wall == 0 || wall == wall_n) {  // fixed faces, padding: identity
            y[f] = MODE == 1 ? 1.0 : (MODE == 0 ? xin[f] : 0.0);
            continue;
        }
        // Along the component's own axis a missing neighbour is a fixed wall
        // face (value 0: no term, keeps A symmetric); across the other axes it
        // is a ghost folded into the diagonal (+1 mirror, -1 negate).
        const double g = ns ? -1.0 : 1.0;
        double gsum = 0.0;  // sum of ghost coefficients multiplying c
        double lid = 0.0;   // Dirichlet lid contribution to the rhs
        const bool ex_xm = comp == 0 ? i > 1 : i > 0, ex_xp = i < nx - 1;
        const bool ex_ym = comp == 1 ? j > 1 : j > 0, ex_yp = j < ny - 1;
        const bool ex_zm = comp == 2 ? k > 1 : k > 0, ex_zp = k < nz - 1;
        if (comp != 0 && !ex_xm) gsum += g;
        if (comp != 0 && !ex_xp) gsum += g;
        if (comp != 1 && !ex_ym) gsum += g;
        if (comp != 1 && !ex_yp) {
            if (bc.lid_dirichlet) {
                gsum += -1.0;
                if (comp == 0) lid = 2.0 * bc.lid_u;
            } else {
                gsum += g;
            }
        }
        if (comp != 2 && !ex_zm) gsum += g;
        if (comp != 2 && !ex_zp) gsum += g;
        const double dia = 1.0 + kdt * (6.0 - gsum);
        if (MODE == 1) {
            y[f] = dia;
        } else if (MODE == 2) {
            y[f] = xin[f] + kdt * lid;
        } else {
            double s = 0.0;
            if (ex_xm) s = s + xin[f - 1];
            if (ex_xp) s = s + xin[f + 1];
            if (ex_ym) s = s + xin[f - pj];
            if (ex_yp) s = s + xin[f + pj];
            if (ex_zm) s = s + xin[f - pk];
            if (ex_zp) s = s + xin[f + pk];
            y[f] = dia * xin[f] - kdt * s;
        }
    }
}

__global__ void sample_kernel(Vel3 in, double h, double px, double py, double pz, double *out)
{
    // src/grid.py:124-142 with the lattice offsets of :99
    out[0] = trilerp(in.c[0], px / h - 0.0, py / h - 0.5, pz / h - 0.5);
    out[1] = trilerp(in.c[1], px / h - 0.5, py / h - 0.0, pz / h - 0.5);
    out[2] = trilerp(in.c[2], px / h - 0.5, py / h - 0.5, pz / h - 0.0);
}

static int grid_for(long long work, int threads, int per_sm)
{
    long long want = (work + threads - 1) / threads;
    long long cap = (long long)num_sms() * per_sm;
    return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

static bool pitches_ok(const SlabZ &sz, int ldu, int ldv, int ldw)
{
    // stored planes of the widest component (w: the slab plus its halos and the
    // top face) must stay below 2^31 elements: the kernels index in 32 bits
    const long long planes = (long long)(sz.z1 - sz.z0) + 2LL * sz.H + 1;
    const long long big = (long long)std::max(ldu, std::max(ldv, ldw)) * (sz.ny + 1) * planes;
    return ldu >= sz.nx + 1 && ldv >= sz.nx && ldw >= sz.nx && big < (1LL << 31);
}

static bool slab_ok(const SlabZ &s)
{
    return s.nx >= 1 && s.ny >= 1 && s.nz >= 1 && 0 <= s.z0 && s.z0 < s.z1 && s.z1 <= s.nz && s.H >= 0;
}

// One-shot max reduction through the shared scratch, result to host.
template <class Launch>
static int reduce_max_to_host(Launch launch, double *result_host, cudaStream_t s)
{
    double *scratch = scratch_partials();
    double *slot = host_result_slot();
    if (!scratch || !slot) { set_error("reduction scratch allocation failed"); return CF_ENOMEM; }
    double *result = scratch + kScratchPartials;
    unsigned int *ticket = reinterpret_cast<unsigned int *>(scratch + kScratchPartials + 1);
    launch(scratch, ticket, result);
    CF_CHECK_LAUNCH("reduction kernel");
    if (result_host) {
        CF_CUDA(cudaMemcpyAsync(slot, result, sizeof(double), cudaMemcpyDeviceToHost, s));
        CF_CUDA(cudaStreamSynchronize(s));
        *result_host = *slot;
    }
    return CF_OK;
}

static int forces_bc(double *u, double *v, double *w, SlabZ sz, int ldu, int ldv, int ldw, double lid_dv, int lid,
                     void *stream)
{
    CF_REQUIRE(slab_ok(sz) && pitches_ok(sz, ldu, ldv, ldw), "forces_bc: bad slab/pitch");
    long long m = std::max((long long)(sz.nx + 1) * (sz.ny + 1),
                           (long long)std::max(sz.nx, sz.ny) * (sz.z1 - sz.z0));
    dim3 grid((unsigned)((m + 255) / 256 < 1024 ? (m + 255) / 256 : 1024), 7);
    forces_bc_kernel<<<grid, 256, 0, as_stream(stream)>>>(u, v, w, sz, ldu, ldv, ldw, lid_dv, lid);
    CF_CHECK_LAUNCH("forces_bc_kernel");
    return CF_OK;
}

static int advect(const double *u, const double *v, const double *w, double *nu, double *nv, double *nw, SlabZ sz,
                  int ldu, int ldv, int ldw, double h, double dt, void *stream)
{
    CF_REQUIRE(slab_ok(sz) && h > 0 && pitches_ok(sz, ldu, ldv, ldw), "advect: bad slab/pitch");
    CF_REQUIRE(nu != u && nv != v && nw != w, "advect: output aliases input");
    Vel3 in = make_vel(u, v, w, sz, ldu, ldv, ldw);
    // TMA-fed z-march (cf_advect.cuh) for the single domain; CF_ADVECT=global
    // selects the global-gather kernel (also the z-slab form)
    const char *ae = getenv("CF_ADVECT");
    const bool single = sz.H == 0 && sz.z0 == 0 && sz.z1 == sz.nz;
    if (single && is_pow2(h) && sz.nx >= 2 && sz.ny >= 2 && sz.nz >= 2 && !(ae && !strcmp(ae, "global"))) {
        CUtensorMap mu, mv, mw;
        const bool ok = make_map_pitched(&mu, u, sz.nx + 1, sz.ny, sz.nz, ldu, kAdvBX, kAdvBY) &&
                        make_map_pitched(&mv, v, sz.nx, sz.ny + 1, sz.nz, ldv, kAdvBX, kAdvBY) &&
                        make_map_pitched(&mw, w, sz.nx, sz.ny, sz.nz + 1, ldw, kAdvBX, kAdvBY);
        if (ok) {
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(advect_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kAdvSmem);
                attr = true;
            }
            AdvGeom ag{(sz.nx + kAdvTX - 1) / kAdvTX, (sz.ny + kAdvTY - 1) / kAdvTY, 1};
            const int bps = blocks_per_sm((const void *)advect_tma_kernel<true>, kAdvThreads, kAdvSmem);
            ag.nchunk = wave_chunks((long long)ag.ntx * ag.nty, sz.nz + 1, (long long)num_sms() * (bps > 0 ? bps : 1),
                                    8);
            const int ctas = ag.ntx * ag.nty * ag.nchunk;
            advect_tma_kernel<true><<<ctas, kAdvThreads, kAdvSmem, as_stream(stream)>>>(mu, mv, mw, in, nu, nv, nw, sz,
                                                                                      ag, h, 1.0 / h, dt);
            CF_CHECK_LAUNCH("advect_tma_kernel");
            return CF_OK;
        }
    }
    long long faces = (long long)(sz.nx + 1) * (sz.ny + 1) * (sz.z1 - sz.z0 + 1);
    const int grid = grid_for(faces, kFaceThreads, 8);
    if (is_pow2(h))
        advect_kernel<true><<<grid, kFaceThreads, 0, as_stream(stream)>>>(in, nu, nv, nw, sz, h, 1.0 / h, dt);
    else
        advect_kernel<false><<<grid, kFaceThreads, 0, as_stream(stream)>>>(in, nu, nv, nw, sz, h, 1.0 / h, dt);
    CF_CHECK_LAUNCH("advect_kernel");
    return CF_OK;
}

static int divergence(const double *u, const double *v, const double *w, SlabZ sz, int ldu, int ldv, int ldw,
                      double h, double scale, double *out, double *maxabs_host, void *stream)
{
    CF_REQUIRE(slab_ok(sz) && h > 0 && pitches_ok(sz, ldu, ldv, ldw), "divergence: bad slab/pitch");
    Vel3 in = make_vel(u, v, w, sz, ldu, ldv, ldw);
    cudaStream_t s = as_stream(stream);
    const char *de = std::getenv("CF_DIVERGENCE");
    const long long tiles = (long long)((sz.nx + kDivTX - 1) / kDivTX) * ((sz.ny + kDivTY - 1) / kDivTY);
    const int nchunk = wave_chunks(tiles, sz.z1 - sz.z0, (long long)num_sms() * 8, 4);
    if (!(de && !strcmp(de, "flat")) && tiles * nchunk <= kScratchPartials) {
        const int grid = (int)(tiles * nchunk);
        const bool p2 = is_pow2(h);
        return reduce_max_to_host(
            [&](double *part, unsigned int *tk, double *res) {
                if (p2)
                    divergence_march<true><<<grid, kCellThreads, 0, s>>>(in, sz, h, 1.0 / h, scale, scale != 1.0,
                                                                          nchunk, out, part, tk, res);
                else
                    divergence_march<false><<<grid, kCellThreads, 0, s>>>(in, sz, h, 1.0 / h, scale, scale != 1.0,
                                                                           nchunk, out, part, tk, res);
            },
            maxabs_host, s);
    }
    int grid = grid_for((long long)sz.nx * sz.ny * (sz.z1 - sz.z0), kCellThreads, 8);
    return reduce_max_to_host(
        [&](double *part, unsigned int *tk, double *res) {
            divergence_kernel<<<grid, kCellThreads, 0, s>>>(in, sz, h, scale, scale != 1.0, out, part, tk, res);
        },
        maxabs_host, s);
}

static int correct(const double *u, const double *v, const double *w, double *nu, double *nv, double *nw,
                   const double *p, SlabZ sz, int ldu, int ldv, int ldw, double h, double coef, double *div_post_host,
                   void *stream)
{
    CF_REQUIRE(slab_ok(sz) && h > 0 && pitches_ok(sz, ldu, ldv, ldw), "pressure_correct: bad slab/pitch");
    CF_REQUIRE(nu != u && nv != v && nw != w, "pressure_correct: output aliases input");
    Vel3 in = make_vel(u, v, w, sz, ldu, ldv, ldw);
    cudaStream_t s = as_stream(stream);
    const char *ce = std::getenv("CF_CORRECT");
    const long long tiles = (long long)((sz.nx + kDivTX - 1) / kDivTX) * ((sz.ny + kDivTY - 1) / kDivTY);
    const int nchunk = wave_chunks(tiles, sz.z1 - sz.z0, (long long)num_sms() * 8, 4);
    if (!(ce && !strcmp(ce, "flat")) && tiles * nchunk <= kScratchPartials) {
        const int grid = (int)(tiles * nchunk);
        const bool p2 = is_pow2(h);
        return reduce_max_to_host(
            [&](double *part, unsigned int *tk, double *res) {
                if (p2)
                    correct_march<true><<<grid, kCellThreads, 0, s>>>(in, nu, nv, nw, p, sz, h, 1.0 / h, coef, nchunk,
                                                                       part, tk, res);
                else
                    correct_march<false><<<grid, kCellThreads, 0, s>>>(in, nu, nv, nw, p, sz, h, 1.0 / h, coef, nchunk,
                                                                        part, tk, res);
            },
            div_post_host, s);
    }
    int grid = grid_for((long long)sz.nx * sz.ny * (sz.z1 - sz.z0), kCellThreads, 8);
    return reduce_max_to_host(
        [&](double *part, unsigned int *tk, double *res) {
            correct_kernel<<<grid, kCellThreads, 0, s>>>(in, nu, nv, nw, p, sz, h, coef, part, tk, res);
        },
        div_post_host, s);
}

static int diffuse(const double *u, const double *v, const double *w, double *nu, double *nv, double *nw, SlabZ sz,
                   int ldu, int ldv, int ldw, double kdt, DiffBC bc, void *stream)
{
    CF_REQUIRE(slab_ok(sz) && pitches_ok(sz, ldu, ldv, ldw), "diffuse: bad slab/pitch");
    CF_REQUIRE(nu != u && nv != v && nw != w, "diffuse: output aliases input");
    Vel3 in = make_vel(u, v, w, sz, ldu, ldv, ldw);
    const char *fe = std::getenv("CF_DIFFUSE");
    if (!(fe && !strcmp(fe, "flat"))) {
        const long long tiles = (long long)((sz.nx + 1 + kDivTX - 1) / kDivTX) * ((sz.ny + 1 + kDivTY - 1) / kDivTY);
        const int nchunk = wave_chunks(3 * tiles, sz.z1 - sz.z0 + 1, (long long)num_sms() * 8, 4);
        if (tiles * nchunk < (1LL << 31)) {
            dim3 grid((unsigned)(tiles * nchunk), 3);
            diffuse_march<<<grid, kFaceThreads, 0, as_stream(stream)>>>(in, nu, nv, nw, sz, kdt, bc, nchunk);
            CF_CHECK_LAUNCH("diffuse_march");
            return CF_OK;
        }
    }
    long long faces = (long long)(sz.nx + 1) * (sz.ny + 1) * (sz.z1 - sz.z0 + 1);
    dim3 grid(grid_for(faces, kFaceThreads, 8), 3);
    diffuse_kernel<<<grid, kFaceThreads, 0, as_stream(stream)>>>(in, nu, nv, nw, sz, kdt, bc);
    CF_CHECK_LAUNCH("diffuse_kernel");
    return CF_OK;
}

}  // namespace cf

extern "C" {

// ---- the reference's cube (nx = ny = nz = n) -----------------------------
int cf_forces_bc(double *u, double *v, double *w, int n, int ldu, int ldv, int ldw, double lid_dv, int apply_lid,
                 void *stream)
{
    return cf::forces_bc(u, v, w, cf::SlabZ{n, n, n, 0, n, 0}, ldu, ldv, ldw, lid_dv, apply_lid, stream);
}

int cf_advect(const double *u, const double *v, const double *w, double *nu, double *nv, double *nw, int n, int ldu,
              int ldv, int ldw, double h, double dt, void *stream)
{
    return cf::advect(u, v, w, nu, nv, nw, cf::SlabZ{n, n, n, 0, n, 0}, ldu, ldv, ldw, h, dt, stream);
}

int cf_divergence(const double *u, const double *v, const double *w, int n, int ldu, int ldv, int ldw, double h,
                  double scale, double *out, double *maxabs_host, void *stream)
{
    return cf::divergence(u, v, w, cf::SlabZ{n, n, n, 0, n, 0}, ldu, ldv, ldw, h, scale, out, maxabs_host, stream);
}

int cf_pressure_correct(const double *u, const double *v, const double *w, double *nu, double *nv, double *nw,
                        const double *p, int n, int ldu, int ldv, int ldw, double h, double coef, double *div_post_host,
                        void *stream)
{
    return cf::correct(u, v, w, nu, nv, nw, p, cf::SlabZ{n, n, n, 0, n, 0}, ldu, ldv, ldw, h, coef, div_post_host,
                       stream);
}

int cf_diffuse(const double *u, const double *v, const double *w, double *nu, double *nv, double *nw, int n, int ldu,
               int ldv, int ldw, double kdt, double lid_u, int lid_dirichlet, int no_slip, void *stream)
{
    return cf::diffuse(u, v, w, nu, nv, nw, cf::SlabZ{n, n, n, 0, n, 0}, ldu, ldv, ldw, kdt,
                       cf::DiffBC{lid_u, lid_dirichlet, no_slip}, stream);
}

// ---- boxes and z-slabs (nx x ny x nz; owned planes [z0, z1), halo planes) -
int cf_forces_bc_slab(double *u, double *v, double *w, int nx, int ny, int nz, int z0, int z1, int halo, int ldu,
                      int ldv, int ldw, double lid_dv, int apply_lid, void *stream)
{
    return cf::forces_bc(u, v, w, cf::SlabZ{nx, ny, nz, z0, z1, halo}, ldu, ldv, ldw, lid_dv, apply_lid, stream);
}

int cf_advect_slab(const double *u, const double *v, const double *w, double *nu, double *nv, double *nw, int nx, int ny,
                   int nz, int z0, int z1, int halo, int ldu, int ldv, int ldw, double h, double dt, void *stream)
{
    return cf::advect(u, v, w, nu, nv, nw, cf::SlabZ{nx, ny, nz, z0, z1, halo}, ldu, ldv, ldw, h, dt, stream);
}

int cf_divergence_slab(const double *u, const double *v, const double *w, int nx, int ny, int nz, int z0, int z1,
                       int halo, int ldu, int ldv, int ldw, double h, double scale, double *out, double *maxabs_host,
                       void *stream)
{
    return cf::divergence(u, v, w, cf::SlabZ{nx, ny, nz, z0, z1, halo}, ldu, ldv, ldw, h, scale, out, maxabs_host,
                          stream);
}

int cf_pressure_correct_slab(const double *u, const double *v, const double *w, double *nu, double *nv, double *nw,
                             const double *p, int nx, int ny, int nz, int z0, int z1, int halo, int ldu, int ldv,
                             int ldw, double h, double coef, double *div_post_host, void *stream)
{
    return cf::correct(u, v, w, nu, nv, nw, p, cf::SlabZ{nx, ny, nz, z0, z1, halo}, ldu, ldv, ldw, h, coef,
                       div_post_host, stream);
}

int cf_diffuse_slab(const double *u, const double *v, const double *w, double *nu, double *nv, double *nw, int nx,
                    int ny, int nz, int z0, int z1, int halo, int ldu, int ldv, int ldw, double kdt, double lid_u,
                    int lid_dirichlet, int no_slip, void *stream)
{
    return cf::diffuse(u, v, w, nu, nv, nw, cf::SlabZ{nx, ny, nz, z0, z1, halo}, ldu, ldv, ldw, kdt,
                       cf::DiffBC{lid_u, lid_dirichlet, no_slip}, stream);
}

int cf_helmholtz(int mode, int comp, const double *x, double *y, int nx, int ny, int nz, int ld, double kdt,
                 double lid_u, int lid_dirichlet, int no_slip, void *stream)
{
    CF_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1 && comp >= 0 && comp <= 2 && mode >= 0 && mode <= 2 &&
                   ld >= nx + (comp == 0),
               "cf_helmholtz: bad arguments");
    long long total = (long long)ld * (ny + (comp == 1)) * (nz + (comp == 2));
    int grid = cf::grid_for(total, cf::kFaceThreads, 8);
    cf::DiffBC bc{lid_u, lid_dirichlet, no_slip};
    cudaStream_t s = cf::as_stream(stream);
    if (mode == 0) cf::helmholtz_kernel<0><<<grid, cf::kFaceThreads, 0, s>>>(x, y, comp, nx, ny, nz, ld, kdt, bc);
    else if (mode == 1) cf::helmholtz_kernel<1><<<grid, cf::kFaceThreads, 0, s>>>(x, y, comp, nx, ny, nz, ld, kdt, bc);
    else cf::helmholtz_kernel<2><<<grid, cf::kFaceThreads, 0, s>>>(x, y, comp, nx, ny, nz, ld, kdt, bc);
    CF_CHECK_LAUNCH("helmholtz_kernel");
    return CF_OK;
}

int cf_sample_velocity(const double *u, const double *v, const double *w, int n, int ldu, int ldv, int ldw, double h,
                       double px, double py, double pz, double *out_host, void *stream)
{
    cf::SlabZ sz{n, n, n, 0, n, 0};
    CF_REQUIRE(n >= 1 && h > 0 && out_host && cf::pitches_ok(sz, ldu, ldv, ldw), "cf_sample_velocity: bad args");
    cf::Vel3 in = cf::make_vel(u, v, w, sz, ldu, ldv, ldw);
    cudaStream_t s = cf::as_stream(stream);
    double *scratch = cf::scratch_partials();
    if (!scratch) { cf::set_error("scratch allocation failed"); return CF_ENOMEM; }
    cf::sample_kernel<<<1, 1, 0, s>>>(in, h, px, py, pz, scratch);
    CF_CHECK_LAUNCH("sample_kernel");
    CF_CUDA(cudaMemcpyAsync(out_host, scratch, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CF_CUDA(cudaStreamSynchronize(s));
    return CF_OK;
}

}  // extern "C"
