// cf_cg_lpass.cuh -- lean form of the single-reduction CG pass (included by
// cf_cg.cu inside namespace cf, after cf_cg_pass.cuh and cf_cg_lean.cuh).
//
// Same algorithm and per-element arithmetic as cg_pass_kernel (the
// Chronopoulos-Gear pass, cf_cg_pass.cuh: p_k, r_{k+1}, x_{k+1} and the three
// dot products gamma, delta, r.r in ONE sweep, 48 N of HBM traffic), laid out
// for fewer instructions:
//   * cell pairs everywhere (16-byte LDS/STS/LDG/STG), 32-bit cell indices;
//   * a CTA owns a 64 x 8 tile of a z-chunk; the p box (12 rows x 34 pairs)
//     and the r' box (10 x 34) are flat pair arrays in shared memory, every
//     thread owns one tile pair (stencil reads at fixed offsets) and 84
//     threads one halo pair of the r' box;
//   * the raw r_k / p_{k-1} of the next plane are loaded into registers one
//     plane ahead (a cp.async ring form measured slower: 224 vs 199 us at
//     256^3, three CTAs per SM for its 68 KB of rings);
//   * out-of-domain cells read the vectors' zeroed pads (p = +0), so the
//     stencils need no masks; r' is zeroed there explicitly.
// Per plane t: A: P(t) = z_k + beta p_{k-1} on the p box; barrier; B: q = A p,
// r' = r_k - alpha q on the r' box at plane t-1 (outputs p_k, r_{k+1},
// x_{k+1} and r.r, gamma on the tile); barrier; C: w = A z' on the tile at
// plane t-2, delta += z'.w.

constexpr int kLpPX = 34;  // pairs per box row: x0-2 .. x0+65
// R = tile rows (one warp each): p box rows y0-2 .. y0+R+1, r' box rows y0-1 .. y0+R
template <int R> struct Lp {
    static constexpr int PBox = (R + 4) * kLpPX;
    static constexpr int QBox = (R + 2) * kLpPX;
    static constexpr int Threads = 32 * R;
    static constexpr int Halo = 2 * kLpPX + 2 * R;  // r' box pairs outside the tile
    static constexpr size_t Smem = (size_t)(3 * PBox + 2 * QBox + 3 * QBox) * sizeof(double2) + 128;
};
// shared rings (pairs): P = p_k on the p box (3 planes), RAW = raw r_k on the
// r' box (2), Q = z' on the r' box (3): 47 KB at R = 8 (four CTAs per SM),
// 82 KB at R = 16 (two)

template <int ORDER, int PK, bool FIRST, int R>
__device__ __forceinline__ void lpass_body(const PairGeom &g, double off, double diag, double zc,
                                           const double *__restrict__ r_in, double *__restrict__ r_out,
                                           const double *__restrict__ p_old, double *__restrict__ p_new,
                                           double *__restrict__ x, double alpha, double beta, double2 *P,
                                           double2 *RAW, double2 *Q, double &rr, double &gam, double &dlt)
{
    const int tid = threadIdx.x, lane = tid & 31;
    const int ntiles = g.ntx * g.nty;
    const int tile = blockIdx.x % ntiles, chunk = blockIdx.x / ntiles;
    const int x0 = (tile % g.ntx) * kPairX, y0 = (tile / g.ntx) * R;
    const int z0 = (int)((long long)g.nz * chunk / g.nchunk);
    const int z1 = (int)((long long)g.nz * (chunk + 1) / g.nchunk);
    const unsigned nx = (unsigned)g.nx, pl = nx * (unsigned)g.ny;
    const unsigned zero = pl * (unsigned)g.nz + 2u * (unsigned)lane;
    const double malpha = -alpha;

    // stage-A items: p-box pairs tid and tid + 256
    const int na = tid + Lp<R>::Threads < Lp<R>::PBox ? 2 : 1;
    unsigned a_g[2];
    bool a_ok[2];
    int a_raw[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int e = tid + q * Lp<R>::Threads;
        const int br = e / kLpPX, px = e % kLpPX;
        const int i = x0 - 2 + 2 * px, j = y0 - 2 + br;
        a_ok[q] = e < Lp<R>::PBox && i >= 0 && i < g.nx && j >= 0 && j < g.ny;
        a_g[q] = a_ok[q] ? (unsigned)i + nx * (unsigned)j : 0u;
        a_raw[q] = (e < Lp<R>::PBox && br >= 1 && br <= R + 2) ? (br - 1) * kLpPX + px : -1;
    }
    // the tile pair: r' box offset, global index
    const int orow = tid >> 5, opx = 1 + lane;
    const int oq = (orow + 1) * kLpPX + opx;
    const int oi = x0 + 2 * lane, oj = y0 + orow;
    const bool own_ok = oi < g.nx && oj < g.ny;
    const unsigned og = own_ok ? (unsigned)oi + nx * (unsigned)oj : 0u;
    // the halo pair (tid < Lp<R>::Halo): r'-box rows 0 / R+1, or columns 0 / 33
    int hq = 0;
    bool h_ok = false;
    if (tid < Lp<R>::Halo) {
        int qr, qp;
        if (tid < 2 * kLpPX) {
            qr = tid < kLpPX ? 0 : R + 1;
            qp = tid % kLpPX;
        } else {
            const int k = tid - 2 * kLpPX;
            qr = 1 + (k >> 1);
            qp = (k & 1) ? kLpPX - 1 : 0;
        }
        hq = qr * kLpPX + qp;
        const int i = x0 - 2 + 2 * qp, j = y0 - 1 + qr;
        h_ok = i >= 0 && i < g.nx && j >= 0 && j < g.ny;
    }

    struct Raw {
        double2 r, q;
    };
    Raw cur[2], nxt[2];
    auto load_plane = [&](int z, Raw *out) {
        const bool zin = z >= 0 && z < g.nz;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            if (q < na) {
                const unsigned k = (a_ok[q] && zin) ? a_g[q] + pl * (unsigned)z : zero;
                out[q].r = ldg2_pinned(r_in + k);
                if (!FIRST) out[q].q = ldg2_pinned(p_old + k);
            }
        }
    };
    // r' box pair -> z' = M^-1 r' (0 outside the domain)
    auto rprime = [&](const double2 *Pm, const double2 *Pc, const double2 *Pp, const double2 *Rw, int qo, bool ok,
                      double &r0, double &r1) {
        const int po = qo + kLpPX;  // p-box offset of the same cell pair
        const double2 c = Pc[po];
        const double xl = (qo % kLpPX) == 0 ? 0.0 : Pc[po - 1].y;           // x0-3: a don't-care cell's term
        const double xr = (qo % kLpPX) == kLpPX - 1 ? 0.0 : Pc[po + 1].x;   // x0+66: likewise
        double a0, a1;
        stencil_pair<ORDER, true>(c, xl, xr, Pc[po - kLpPX], Pc[po + kLpPX], Pm[po], Pp[po], true, true, true, true,
                                  true, true, off, diag, a0, a1);
        const double2 rk = Rw[qo];
        r0 = ok ? rk.x + malpha * a0 : 0.0;  // src/solver.py:157
        r1 = ok ? rk.y + malpha * a1 : 0.0;
    };
    auto s3 = [](int t) { return (t + 6) % 3; };

    auto s2 = [](int t) { return (t + 6) & 1; };
    load_plane(z0 - 2, cur);
    double2 xk = make_double2(0.0, 0.0), xk_nxt = xk;  // x_k of the tile pair, one plane ahead
    for (int t = z0 - 2; t <= z1 + 1; ++t) {
        const int zb = t - 1;  // stage-B plane
        const bool own_b = own_ok && zb >= z0 && zb < z1;
        // ---- A: p_k = z_k + beta p_{k-1} at plane t (src/solver.py:142, :169)
        {
            double2 *const Pt = P + s3(t) * Lp<R>::PBox;
            double2 *const Rt = RAW + s2(t) * Lp<R>::QBox;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (q < na) {
                    const double2 rv = cur[q].r;
                    double a = zscale<PK>(rv.x, zc), b = zscale<PK>(rv.y, zc);
                    if (!FIRST) {
                        a = a + beta * cur[q].q.x;
                        b = b + beta * cur[q].q.y;
                    }
                    Pt[tid + q * Lp<R>::Threads] = make_double2(a, b);
                    if (a_raw[q] >= 0) Rt[a_raw[q]] = rv;
                }
            }
        }
        if (t + 1 <= z1 + 1) load_plane(t + 1, nxt);
        __syncthreads();
        // ---- B: r' = r_k - alpha A p_k at plane t-1 on the r' box
        if (zb >= z0 - 1 && zb <= z1) {
            const bool zin = zb >= 0 && zb < g.nz;
            const double2 *Pm = P + s3(zb - 1) * Lp<R>::PBox, *Pc = P + s3(zb) * Lp<R>::PBox, *Pp = P + s3(zb + 1) * Lp<R>::PBox;
            const double2 *Rw = RAW + s2(zb) * Lp<R>::QBox;
            double2 *const Qo = Q + s3(zb) * Lp<R>::QBox;
            double r0, r1;
            rprime(Pm, Pc, Pp, Rw, oq, own_ok && zin, r0, r1);
            Qo[oq] = make_double2(zscale<PK>(r0, zc), zscale<PK>(r1, zc));  // the ring holds z_{k+1}
            if (own_b) {
                // the tile's outputs: p_k, r_{k+1}, x_{k+1} = x_k + alpha p_k (:155); r.r, r.z (:158, :163)
                const unsigned o = og + pl * (unsigned)zb;
                const double2 pc = Pc[oq + kLpPX];
                *reinterpret_cast<double2 *>(p_new + o) = pc;
                *reinterpret_cast<double2 *>(r_out + o) = make_double2(r0, r1);
                *reinterpret_cast<double2 *>(x + o) = make_double2(xk.x + alpha * pc.x, xk.y + alpha * pc.y);
                rr = rr + r0 * r0;
                rr = rr + r1 * r1;
                gam = gam + r0 * zscale<PK>(r0, zc);
                gam = gam + r1 * zscale<PK>(r1, zc);
            }
            if (tid < Lp<R>::Halo) {
                double h0, h1;
                rprime(Pm, Pc, Pp, Rw, hq, h_ok && zin, h0, h1);
                Qo[hq] = make_double2(zscale<PK>(h0, zc), zscale<PK>(h1, zc));
            }
        }
        if (own_ok && t >= z0 && t < z1) xk_nxt = ld2_pinned(x + og + pl * (unsigned)t);
        __syncthreads();
        // ---- C: w = A z' on the tile at plane t-2, delta += z'.w
        const int zw = t - 2;
        if (own_ok && zw >= z0 && zw < z1) {
            const double2 *Qm = Q + s3(zw - 1) * Lp<R>::QBox, *Qc = Q + s3(zw) * Lp<R>::QBox, *Qp = Q + s3(zw + 1) * Lp<R>::QBox;
            const double2 c = Qc[oq];
            double w0, w1;
            stencil_pair<ORDER, true>(c, Qc[oq - 1].y, Qc[oq + 1].x, Qc[oq - kLpPX], Qc[oq + kLpPX], Qm[oq], Qp[oq],
                                      true, true, true, true, true, true, off, diag, w0, w1);
            dlt = dlt + c.x * w0;
            dlt = dlt + c.y * w1;
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) cur[q] = nxt[q];
        xk = xk_nxt;
    }
}

template <int ORDER, int PK, int R = 8>
__global__ void __launch_bounds__(32 * R, 32 / R) cg_lpass_kernel(PairGeom g, double off, double diag, double zc,
                                                                const double *__restrict__ r_in,
                                                                double *__restrict__ r_out,
                                                                const double *__restrict__ p_old,
                                                                double *__restrict__ p_new, double *__restrict__ x,
                                                                CgScalars *sc, double *partials, CgTickets *tk,
                                                                int use_cond, cudaGraphConditionalHandle cond)
{
    extern __shared__ unsigned char smem_raw[];
    __shared__ double red[32];
    __shared__ int is_last;
    if (sc->done) {
        if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    double2 *const P = reinterpret_cast<double2 *>(aligned_smem(smem_raw));
    double2 *const RAW = P + 3 * Lp<R>::PBox;
    double2 *const Q = RAW + 2 * Lp<R>::QBox;
    double rr = 0.0, gam = 0.0, dlt = 0.0;
    if (sc->it == 0)
        lpass_body<ORDER, PK, true, R>(g, off, diag, zc, r_in, r_out, p_old, p_new, x, sc->alpha, 0.0, P, RAW, Q, rr,
                                    gam, dlt);
    else
        lpass_body<ORDER, PK, false, R>(g, off, diag, zc, r_in, r_out, p_old, p_new, x, sc->alpha, sc->beta, P, RAW, Q,
                                     rr, gam, dlt);
    rr = block_sum<Lp<R>::Threads>(rr, red);
    gam = block_sum<Lp<R>::Threads>(gam, red);
    dlt = block_sum<Lp<R>::Threads>(dlt, red);
    if (threadIdx.x == 0) {
        partials[3 * blockIdx.x] = rr;
        partials[3 * blockIdx.x + 1] = gam;
        partials[3 * blockIdx.x + 2] = dlt;
    }
    if (last_block(&tk->upd, &is_last)) {
        rr = reduce_partials<Lp<R>::Threads>(partials, gridDim.x, 3, red);
        gam = reduce_partials<Lp<R>::Threads>(partials + 1, gridDim.x, 3, red);
        dlt = reduce_partials<Lp<R>::Threads>(partials + 2, gridDim.x, 3, red);
        if (threadIdx.x == 0) {
            scalar_after_pass(sc, rr, gam, dlt);
            if (sc->done && use_cond) cudaGraphSetConditional(cond, 0);
        }
    }
}
