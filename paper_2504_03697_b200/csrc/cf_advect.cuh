// cf_advect.cuh -- semi-Lagrangian advection as a TMA-fed z-march (included
// by cf_step.cu inside namespace cf, after Comp / Vel3 / SlabZ / trilerp).
//
// Same per-face arithmetic as advect_face (src/sim.py:156-256, blend order
// fixed, -fmad=false), so the result is bit-identical to the reference; what
// changes is where the samples come from.  A CTA owns a 32 x 8 tile of face
// columns (i, j) -- the u, v and w faces with those indices -- and marches
// the z planes k of its chunk.  For output plane k every sample the reference
// takes lies in planes k-1 .. k+2 and columns i-1 .. i+2, rows j-1 .. j+2 of
// each component as long as the backtrace moves at most one cell (CFL <= 1:
// the departure lattice coordinate stays within one of the face's own), so a
// producer warp streams, per plane, one 36 x 11 box (x0-2 .. x0+33,
// y0-1 .. y0+9) of each component into an 8-deep ring by TMA, and the
// trilinear gathers read shared memory.  A sample outside the staged window
// (a faster flow) falls back to a global load, so any dt stays correct.
// With h a power of two (every BASELINE config) the velocity samples at a
// face sit on a lattice point of its own component and on lattice lines of
// the other two, where the trilinear weights are exactly 1, 0 and 0.5: a face
// takes 1 + 4 + 4 staged values for the velocity (avg2) and 8 for the
// departure value instead of 32 gathers.  HBM per step: each component read
// once and written once, 48 F (the global-gather kernel moved 1.7x that).
// Other h run the global-gather kernel.

constexpr int kAdvTX = 32, kAdvTY = 8, kAdvS = 8;
constexpr int kAdvBX = kAdvTX + 4;           // x0-2 .. x0+33 (16-byte aligned x origin)
constexpr int kAdvBY = kAdvTY + 3;           // y0-1 .. y0+TY+1
constexpr int kAdvPD = 400;                  // 36 x 11 = 396 doubles, padded to a 128-byte multiple
constexpr int kAdvStageD = 3 * kAdvPD;       // u | v | w boxes of one plane
constexpr int kAdvThreads = 32 * kAdvTY + 32;  // consumers + the producer warp
constexpr size_t kAdvSmem = (size_t)kAdvS * kAdvStageD * sizeof(double) + 128;

struct AdvGeom {
    int ntx, nty, nchunk;
};

// One component's sample source for output plane k: the staged ring window
// (planes k-1 .. k+2 of the box) or, when a stencil leaves it, global memory.
struct AdvSrc {
    const double *ring;  // this component's box in stage 0 (stages kAdvStageD apart)
    Comp f;
    int bx0, by0, kw0, q0;  // box origin, first plane of the window, its load index
};

// the whole trilerp from global memory (a stencil outside the staged window)
__device__ __noinline__ double trilerp_global(const Comp &f, double a, double b, double c)
{
    return trilerp(f, a, b, c);
}

// trilerp (src/sim.py:156-190) over an AdvSrc: the same corners, the same
// blend order, the corners read from the staged window
__device__ __forceinline__ double trilerp_s(const AdvSrc &s, double a, double b, double c)
{
    const Comp &f = s.f;
    a = clamp_hi(a, f.na - 1.0);
    b = clamp_hi(b, f.nb - 1.0);
    c = clamp_hi(c, f.nc - 1.0);
    const int i0 = base_index(a, f.na), j0 = base_index(b, f.nb), k0 = base_index(c, f.nc);
    const int i1 = min(i0 + 1, f.na - 1), j1 = min(j0 + 1, f.nb - 1), k1 = min(k0 + 1, f.nc - 1);
    const double fa = a - (double)i0, fb = b - (double)j0, fc = c - (double)k0;
    const int di = i0 - s.bx0, dj = j0 - s.by0, dk = k0 - s.kw0;
    if (!((unsigned)di <= (unsigned)(kAdvBX - 2) && (unsigned)dj <= (unsigned)(kAdvBY - 2) && (unsigned)dk <= 2u))
        return trilerp_global(f, a, b, c);
    double v[8];  // corners: bit 0 = i1, bit 1 = j1, bit 2 = k1
    const double *p0 = s.ring + ((s.q0 + dk) & (kAdvS - 1)) * kAdvStageD + dj * kAdvBX + di;
    const double *p1 = s.ring + ((s.q0 + dk + (k1 - k0)) & (kAdvS - 1)) * kAdvStageD + dj * kAdvBX + di;
    const int oi = i1 - i0, oj = (j1 - j0) * kAdvBX;
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = ((q & 4) ? p1 : p0)[((q & 1) ? oi : 0) + ((q & 2) ? oj : 0)];
    const double c00 = v[0] * (1.0 - fa) + v[1] * fa;
    const double c10 = v[2] * (1.0 - fa) + v[3] * fa;
    const double c01 = v[4] * (1.0 - fa) + v[5] * fa;
    const double c11 = v[6] * (1.0 - fa) + v[7] * fa;
    return (c00 * (1.0 - fb) + c10 * fb) * (1.0 - fc) + (c01 * (1.0 - fb) + c11 * fb) * fc;
}

// The velocity sample at a face when h is a power of two and the face is not
// a wall: it sits on a lattice point of its own component and on lattice
// lines of the other two, where trilerp's weights are exactly 1, 0 and 0.5
// (every clamp inactive): the blend reduces to
//   (p*0.5 + q*0.5)*0.5 + (r*0.5 + s*0.5)*0.5
// over the four corners with weight 0.5 x 0.5 -- the same roundings, minus
// terms multiplied by exactly 0.
__device__ __forceinline__ double avg2(double p, double q, double r, double s)
{
    return (p * 0.5 + q * 0.5) * 0.5 + (r * 0.5 + s * 0.5) * 0.5;
}

// the face value of component `comp` at (i, j, k): advect_face's arithmetic.
// pm / p0 / p1: the staged boxes (u | v | w) of planes k-1, k, k+1; ob: the
// face column's offset in a box.
template <bool POW2>
__device__ __forceinline__ double advect_staged(const AdvSrc *src, const double *pm, const double *p0,
                                                const double *p1, int ob, int comp, int i, int j, int k, double h,
                                                double inv_h, double dt, double lx, double ly, double lz)
{
    auto over_h = [&](double q) { return POW2 ? q * inv_h : q / h; };
    double x, y, z;
    if (comp == 0) {
        x = i * h; y = (j + 0.5) * h; z = (k + 0.5) * h;
    } else if (comp == 1) {
        x = (i + 0.5) * h; y = j * h; z = (k + 0.5) * h;
    } else {
        x = (i + 0.5) * h; y = (j + 0.5) * h; z = k * h;
    }
    static_assert(POW2, "the staged kernel runs for power-of-two h only (exact lattice positions)");
    double su, sv, sw;
    {  // exact lattice positions (see avg2): 1 + 4 + 4 staged values
        constexpr int U = 0, V = kAdvPD, W = 2 * kAdvPD, Y = kAdvBX;
        if (comp == 0) {
            su = p0[U + ob];
            sv = avg2(p0[V + ob - 1], p0[V + ob], p0[V + ob - 1 + Y], p0[V + ob + Y]);
            sw = avg2(p0[W + ob - 1], p0[W + ob], p1[W + ob - 1], p1[W + ob]);
        } else if (comp == 1) {
            su = avg2(p0[U + ob - Y], p0[U + ob - Y + 1], p0[U + ob], p0[U + ob + 1]);
            sv = p0[V + ob];
            sw = avg2(p0[W + ob - Y], p0[W + ob], p1[W + ob - Y], p1[W + ob]);
        } else {
            su = avg2(pm[U + ob], pm[U + ob + 1], p0[U + ob], p0[U + ob + 1]);
            sv = avg2(pm[V + ob], pm[V + ob + Y], p0[V + ob], p0[V + ob + Y]);
            sw = p0[W + ob];
        }
    }
    const double xb = over_h(clamp_hi(x - dt * su, lx));
    const double yb = over_h(clamp_hi(y - dt * sv, ly));
    const double zb = over_h(clamp_hi(z - dt * sw, lz));
    if (comp == 0) return trilerp_s(src[0], xb, yb - 0.5, zb - 0.5);
    if (comp == 1) return trilerp_s(src[1], xb - 0.5, yb, zb - 0.5);
    return trilerp_s(src[2], xb - 0.5, yb - 0.5, zb);
}

// maps: the three input components (3-D, planes of the stored slab), box 36 x 11 x 1
template <bool POW2>
__global__ void __launch_bounds__(kAdvThreads, 2)
    advect_tma_kernel(const __grid_constant__ CUtensorMap mu, const __grid_constant__ CUtensorMap mv,
                      const __grid_constant__ CUtensorMap mw, Vel3 in, double *nu, double *nv, double *nw, SlabZ sz,
                      AdvGeom ag, double h, double inv_h, double dt)
{
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[kAdvS], empty[kAdvS];
    double *const ring = reinterpret_cast<double *>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles = ag.ntx * ag.nty;
    const int tile = blockIdx.x % tiles, chunk = blockIdx.x / tiles;
    const int x0 = (tile % ag.ntx) * kAdvTX, y0 = (tile / ag.ntx) * kAdvTY;
    const int nzo = sz.w_end() - sz.z0;  // owned planes, the top w wall plane included
    const int kz0 = sz.z0 + (int)((long long)nzo * chunk / ag.nchunk);
    const int kz1 = sz.z0 + (int)((long long)nzo * (chunk + 1) / ag.nchunk);
    const int kb = sz.k_base();
    if (threadIdx.x == 0) {
        for (int s = 0; s < kAdvS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kAdvTY);
        }
        fence_barrier_init();
    }
    __syncthreads();
    // load q = plane kz0 - 1 + q of every component (stored plane index - k_base)
    const int nload = kz1 - kz0 + 3;
    if (warp == kAdvTY) {  // ---------------- producer
        if (lane == 0) {
            prefetch_map(&mu);
            prefetch_map(&mv);
            prefetch_map(&mw);
            for (int q = 0; q < nload; ++q) {
                const int s = q & (kAdvS - 1);
                if (q >= kAdvS) mbar_wait(&empty[s], (uint32_t)(((q >> 3) - 1) & 1));
                const int kz = kz0 - 1 + q - kb;
                double *st = ring + s * kAdvStageD;
                mbar_expect_tx(&full[s], 3u * kAdvBX * kAdvBY * 8u);
                tma_load_3d(st, &mu, x0 - 2, y0 - 1, kz, &full[s]);
                tma_load_3d(st + kAdvPD, &mv, x0 - 2, y0 - 1, kz, &full[s]);
                tma_load_3d(st + 2 * kAdvPD, &mw, x0 - 2, y0 - 1, kz, &full[s]);
            }
        }
        return;
    }
    // ---------------- consumers: thread (lane, warp) = face column (x0 + lane, y0 + warp)
    const int i = x0 + lane, j = y0 + warp;
    const int ob = (warp + 1) * kAdvBX + lane + 2;  // the column (i, j) in a staged box
    const double lx = sz.nx * h, ly = sz.ny * h, lz = sz.nz * h;
    AdvSrc src[3];
    for (int c = 0; c < 3; ++c) src[c] = AdvSrc{ring + c * kAdvPD, in.c[c], x0 - 2, y0 - 1, 0, 0};
    for (int q = 0; q + 3 < nload; ++q) {
        const int k = kz0 + q;  // output plane; the window is planes k-1 .. k+2 = loads q .. q+3
        if (q == 0) {
            for (int t = 0; t < 3; ++t) mbar_wait(&full[t], 0u);
        }
        mbar_wait(&full[(q + 3) & (kAdvS - 1)], (uint32_t)(((q + 3) >> 3) & 1));
        for (int c = 0; c < 3; ++c) {
            src[c].kw0 = k - 1;
            src[c].q0 = q;
        }
        const bool uv = k < sz.z1;  // u, v planes end at z1; w's top wall plane nz is owned by the top slab
        const double *pm = ring + (q & (kAdvS - 1)) * kAdvStageD;  // plane k-1
        const double *p0 = ring + ((q + 1) & (kAdvS - 1)) * kAdvStageD;
        const double *p1 = ring + ((q + 2) & (kAdvS - 1)) * kAdvStageD;
        // u faces (i, j, k): walls i = 0 and i = nx are zeroed (src/sim.py:283-288)
        if (uv && j < sz.ny && i <= sz.nx) {
            nu[in.c[0].off(i, j, k)] = (i == 0 || i == sz.nx)
                                           ? 0.0
                                           : advect_staged<POW2>(src, pm, p0, p1, ob, 0, i, j, k, h, inv_h, dt, lx,
                                                                 ly, lz);
            if (i == sz.nx - 1) nu[in.c[0].off(sz.nx, j, k)] = 0.0;  // the i = nx wall (past the last tile when 32 | nx)
        }
        if (uv && i < sz.nx && j <= sz.ny) {
            nv[in.c[1].off(i, j, k)] = (j == 0 || j == sz.ny)
                                           ? 0.0
                                           : advect_staged<POW2>(src, pm, p0, p1, ob, 1, i, j, k, h, inv_h, dt, lx,
                                                                 ly, lz);
            if (j == sz.ny - 1) nv[in.c[1].off(i, sz.ny, k)] = 0.0;  // the j = ny wall row
        }
        if (i < sz.nx && j < sz.ny) {
            nw[in.c[2].off(i, j, k)] = (k == 0 || k == sz.nz)
                                           ? 0.0
                                           : advect_staged<POW2>(src, pm, p0, p1, ob, 2, i, j, k, h, inv_h, dt, lx,
                                                                 ly, lz);
        }
        // plane k-1 (load q) is no longer needed
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[q & (kAdvS - 1)]);
    }
}
