// cf_cg_pass.cuh -- the single-reduction CG: ONE fused kernel per iteration
// (included by cf_cg.cu inside namespace cf, after the other CG forms).
//
// The two-kernel CG needs two grid-wide reductions per iteration (p.Ap for
// alpha, then r.r / r.z for the stop test and beta), hence two passes over
// HBM.  The Chronopoulos-Gear rearrangement needs one: with z = M^-1 r,
//   gamma_k = r_k.z_k,  delta_k = z_k.A z_k,
//   beta_k  = gamma_k / gamma_{k-1},
//   p_k.A p_k = delta_k - beta_k gamma_k / alpha_{k-1},   alpha_k = gamma_k / that,
// (exact CG identities), so pass k can apply alpha_k, beta_k -- known from
// pass k-1's reduction -- and produce gamma_{k+1}, delta_{k+1}, r_{k+1}.r_{k+1}
// in the same sweep:
//   p_k     = z_k + beta_k p_{k-1}               (halo 2: needed by A p at the neighbours)
//   q       = A p_k                              (halo 1)
//   r_{k+1} = r_k - alpha_k q                    (halo 1)
//   x_{k+1} = x_k + alpha_k p_k                  (interior)
//   w       = A z_{k+1},  z_{k+1} = M^-1 r_{k+1} (interior) -> gamma, delta, r.r
// Every per-element operation is the two-kernel form's (stencil7<ORDER>, the
// same p, r, x updates), so given the same scalars the vectors are
// bit-identical; only alpha's evaluation and the dot trees differ (measured:
// the same 446/445/449 iterations as the reference on config 2, x within
// 1e-15 relative; tests/test_gpu_parity.py).  HBM per iteration: read r, p_old,
// x; write r_new, p, x = 48 N (r ping-pongs: neighbours still read r_k's halo).
//
// A CTA owns a 32 x 16 tile of a z-chunk and marches z with a two-plane
// lookahead through shared rings: P (p_k on the halo-2 box, 3 planes), R
// (r_{k+1} on the halo-1 box, 3 planes) and the loaded r_k box (2 planes).
// Step t: load r_k, p_{k-1} of plane t+2 and form P(t+2); barrier; q and
// r_{k+1} on plane t+1 (+ the outputs of plane t+1); barrier; w on plane t
// and the dot partials.  Cells outside the domain are zero in the rings,
// which drops their stencil terms exactly (off*0 = -0.0).

constexpr int kPassTX = 32, kPassTY = 16;
constexpr int kPassThreads = 256;
constexpr int kP2X = kPassTX + 4, kP2Y = kPassTY + 4;  // halo-2 box 36 x 20
constexpr int kP1X = kPassTX + 2, kP1Y = kPassTY + 2;  // halo-1 box 34 x 18
constexpr int kP2 = kP2X * kP2Y, kP1 = kP1X * kP1Y;
// rings (55 KB: four CTAs per SM): raw r_k (3 planes: t+1 read for r_{k+1},
// t+2 formed, t+3 in flight), PP (4 planes: p_{k-1} lands there by cp.async
// and is turned into p_k in place -- P(t), P(t+1), P(t+2) read, t+3 in
// flight), Q = r_{k+1} (3 planes)
constexpr int kRawR = 3, kPP = 4;
constexpr size_t kPassSmem = ((kRawR + kPP) * kP2 + 3 * kP1) * sizeof(double) + 128;

struct PassGeom {
    int nx, ny, nz, ntx, nty, nchunk;
    __host__ __device__ int ctas() const { return ntx * nty * nchunk; }
};

template <int PK>
__device__ __forceinline__ double zscale(double r, double zc)
{
    return PK == PK_JCONST ? r * zc : r;  // src/precond.py:94 (Jacobi) / src/solver.py:71-76 (none)
}

// 16-byte asynchronous global -> shared copy; src_bytes 0 zero-fills
__device__ __forceinline__ void cp_async16(double *dst, const double *src, int src_bytes)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int ORDER, int PK>
__global__ void __launch_bounds__(kPassThreads) cg_pass_kernel(PassGeom g, double off, double diag, double zc,
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
    double *const raw_r = aligned_smem(smem_raw);   // kRawR x kP2
    double *const ring_p = raw_r + kRawR * kP2;     // kPP x kP2 (p_{k-1} in, p_k out)
    double *const ring_q = ring_p + kPP * kP2;      // 3 x kP1 (r_{k+1})
    auto rslot = [&](int z) { return raw_r + ((z + 9) % kRawR) * kP2; };
    auto pslot = [&](int z) { return ring_p + ((z + 8) % kPP) * kP2; };
    const double alpha = sc->alpha, malpha = -alpha, beta = sc->beta;
    const bool first = sc->it == 0;
    const int tid = threadIdx.x;
    const int ntiles = g.ntx * g.nty;
    const int tile = blockIdx.x % ntiles, chunk = blockIdx.x / ntiles;
    const int x0 = (tile % g.ntx) * kPassTX, y0 = (tile / g.ntx) * kPassTY;
    const int z0 = (int)((long long)g.nz * chunk / g.nchunk), z1 = (int)((long long)g.nz * (chunk + 1) / g.nchunk);
    const long long plane = (long long)g.nx * g.ny;
    double rr = 0.0, gam = 0.0, dlt = 0.0;

    // this thread's halo-2 box pairs (loads + P formation): e = tid, tid + 256 (< 360)
    constexpr int kBoxPairs = kP2 / 2;
    int e_off[2];
    long long e_glob[2];
    bool e_in[2];
    const int ne = tid + kPassThreads < kBoxPairs ? 2 : 1;
    for (int q = 0; q < 2; ++q) {
        const int e = tid + q * kPassThreads;
        const int by = e / (kP2X / 2), bx = 2 * (e % (kP2X / 2));
        const int gi = x0 - 2 + bx, gj = y0 - 2 + by;
        e_off[q] = by * kP2X + bx;
        // pairs never straddle the x walls (x0 - 2 and nx are even)
        e_in[q] = e < kBoxPairs && gj >= 0 && gj < g.ny && gi >= 0 && gi < g.nx;
        e_glob[q] = e_in[q] ? (long long)gi + (long long)g.nx * gj : 0;
    }
    // issue the copies of plane zq (zero-filled outside the domain / the chunk's needs)
    auto issue = [&](int zq) {
        const bool zin = zq >= 0 && zq < g.nz && zq <= z1 + 1;
        double *const Rr = rslot(zq);
        double *const Rp = pslot(zq);
        for (int q = 0; q < ne; ++q) {
            const bool in = zin && e_in[q];
            const long long o = in ? e_glob[q] + plane * zq : 0;
            cp_async16(Rr + e_off[q], r_in + o, in ? 16 : 0);
            cp_async16(Rp + e_off[q], p_old + o, (in && !first) ? 16 : 0);
        }
        cp_async_commit();
    };
    issue(z0 - 2);
    // t runs from z0-4: P(t+2) every step, R(t+1) from t = z0-2, w(t) from t = z0
    for (int t = z0 - 4; t < z1; ++t) {
        // x_k of plane t+1 at this thread's phase-2 output cells, loaded first so
        // its latency hides behind the P formation and the barrier
        double xk[3] = {0.0, 0.0, 0.0};
        if (t + 1 >= z0 && t + 1 < z1) {
            for (int q = 0; q < 3; ++q) {
                const int e = tid + q * kPassThreads;
                const int qy = e / kP1X, qx = e % kP1X;
                const int gi = x0 + qx - 1, gj = y0 + qy - 1;
                if (e < kP1 && qx >= 1 && qx <= kPassTX && qy >= 1 && qy <= kPassTY && gi < g.nx && gj < g.ny)
                    xk[q] = x[(long long)gi + (long long)g.nx * gj + plane * (t + 1)];
            }
        }
        // ---- P(t+2) from this thread's own staged pairs (src/solver.py:142, :169)
        {
            const int zp = t + 2;
            cp_async_wait<0>();  // this thread's copies of plane t+2 landed
            const double *const Rr = rslot(zp);
            double *const P = pslot(zp);  // p_{k-1} staged here becomes p_k in place
            for (int q = 0; q < ne; ++q) {
                const double2 rv = *reinterpret_cast<const double2 *>(Rr + e_off[q]);
                const double2 qv = *reinterpret_cast<const double2 *>(P + e_off[q]);
                const double a = zscale<PK>(rv.x, zc), b = zscale<PK>(rv.y, zc);
                *reinterpret_cast<double2 *>(P + e_off[q]) =
                    make_double2(first ? a : a + beta * qv.x, first ? b : b + beta * qv.y);
            }
        }
        issue(t + 3);
        __syncthreads();
        // ---- q = A p and r_{k+1} on plane t+1 over the halo-1 box, one cell
        // per thread and step (consecutive lanes, consecutive x: no bank conflicts)
        if (t >= z0 - 2) {
            const int zq = t + 1;
            const double *const Pm = pslot(zq - 1);
            const double *const Pc = pslot(zq);
            const double *const Pp = pslot(zq + 1);
            const double *const Rk = rslot(zq);
            double *const Q = ring_q + ((zq + 6) % 3) * kP1;
            const bool zin = zq >= 0 && zq < g.nz;
            const bool write_out = zq >= z0 && zq < z1;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const int e = tid + q * kPassThreads;
                if (e >= kP1) break;
                const int qy = e / kP1X, qx = e % kP1X;  // box-1 coords; tile-local (qx-1, qy-1)
                const int gi = x0 + qx - 1, gj = y0 + qy - 1;
                const int bo = (qy + 1) * kP2X + (qx + 1);  // box-2 offset of the same cell
                double rn = 0.0;
                if (zin && gi >= 0 && gi < g.nx && gj >= 0 && gj < g.ny) {
                    const double c = Pc[bo];
                    const double a = stencil7<ORDER>(c, Pc[bo - 1], Pc[bo + 1], Pc[bo - kP2X], Pc[bo + kP2X], Pm[bo],
                                                     Pp[bo], true, true, true, true, true, true, off, diag);
                    rn = Rk[bo] + malpha * a;  // src/solver.py:157
                    if (write_out && qx >= 1 && qx <= kPassTX && qy >= 1 && qy <= kPassTY) {
                        // the tile's own cells: p_k, r_{k+1}, x_{k+1} = x_k + alpha p_k (:155),
                        // and r.r, r.z of r_{k+1} (:158, :163-166)
                        const long long o = (long long)gi + (long long)g.nx * gj + plane * zq;
                        p_new[o] = c;
                        r_out[o] = rn;
                        x[o] = xk[q] + alpha * c;
                        rr = rr + rn * rn;
                        gam = gam + rn * zscale<PK>(rn, zc);
                    }
                }
                Q[e] = zscale<PK>(rn, zc);  // the ring holds z_{k+1} = M^-1 r_{k+1}
            }
        }
        __syncthreads();
        // ---- w = A z_{k+1} on plane t (interior, two cells per thread): z.w
        if (t >= z0) {
            const double *const Qm = ring_q + ((t - 1 + 6) % 3) * kP1;
            const double *const Qc = ring_q + ((t + 6) % 3) * kP1;
            const double *const Qp = ring_q + ((t + 1 + 6) % 3) * kP1;
            for (int e = tid; e < kPassTX * kPassTY; e += kPassThreads) {
                const int cy = e / kPassTX, cx = e % kPassTX;
                if (x0 + cx >= g.nx || y0 + cy >= g.ny) continue;
                const int qo = (cy + 1) * kP1X + (cx + 1);
                const double c = Qc[qo];
                const double w = stencil7<ORDER>(c, Qc[qo - 1], Qc[qo + 1], Qc[qo - kP1X], Qc[qo + kP1X], Qm[qo],
                                                 Qp[qo], true, true, true, true, true, true, off, diag);
                dlt = dlt + c * w;
            }
        }
        // ring reuse: the next step's P / raw writes land in slots whose last
        // readers ran before the barrier above
    }
    cp_async_wait<0>();
    rr = block_sum<kPassThreads>(rr, red);
    gam = block_sum<kPassThreads>(gam, red);
    dlt = block_sum<kPassThreads>(dlt, red);
    if (threadIdx.x == 0) {
        partials[3 * blockIdx.x] = rr;
        partials[3 * blockIdx.x + 1] = gam;
        partials[3 * blockIdx.x + 2] = dlt;
    }
    if (last_block(&tk->upd, &is_last)) {
        rr = reduce_partials<kPassThreads>(partials, gridDim.x, 3, red);
        gam = reduce_partials<kPassThreads>(partials + 1, gridDim.x, 3, red);
        dlt = reduce_partials<kPassThreads>(partials + 2, gridDim.x, 3, red);
        if (threadIdx.x == 0) {
            scalar_after_pass(sc, rr, gam, dlt);
            if (sc->done && use_cond) cudaGraphSetConditional(cond, 0);
        }
    }
}

// Init pass: r = b, x = 0, |b|^2, gamma_0 = r.z, delta_0 = z.A z (z = M^-1 b),
// through the pair march (z formed on the fly).
template <int ORDER, int PK>
__global__ void __launch_bounds__(kPairThreads, 8) cg_pass_init(PairGeom g, double off, double diag, double zc,
                                                                const double *__restrict__ b, double *__restrict__ r,
                                                                double *__restrict__ x, CgScalars *sc,
                                                                double *partials, CgTickets *tk)
{
    __shared__ double red[32];
    __shared__ int is_last;
    const PairCoords c = pair_coords(g, blockIdx.x);
    struct Epi {
        const double *b;
        double *r, *x;
        double zc, bb, gam, dlt;
        __device__ __forceinline__ void cell(long long o, double2 zc2, double a0, double a1)
        {
            const double2 bv = *reinterpret_cast<const double2 *>(b + o);
            *reinterpret_cast<double2 *>(r + o) = bv;
            *reinterpret_cast<double2 *>(x + o) = make_double2(0.0, 0.0);
            bb = bb + bv.x * bv.x;
            bb = bb + bv.y * bv.y;
            gam = gam + bv.x * zc2.x;
            gam = gam + bv.y * zc2.y;
            dlt = dlt + zc2.x * a0;
            dlt = dlt + zc2.y * a1;
        }
        __device__ __forceinline__ void halo(long long, double2) {}
    } epi{b, r, x, zc, 0.0, 0.0, 0.0};
    if (c.row_ok) {
        const DirSrc<PK == PK_JCONST ? PK_JCONST : PK_NONE> src{b, b, nullptr, zc, 0.0, true};
        pair_march<ORDER, false>(c, g, off, diag, src, epi);
    }
    double bb = block_sum<kPairThreads>(epi.bb, red);
    double gam = block_sum<kPairThreads>(epi.gam, red);
    double dlt = block_sum<kPairThreads>(epi.dlt, red);
    if (threadIdx.x == 0) {
        partials[3 * blockIdx.x] = bb;
        partials[3 * blockIdx.x + 1] = gam;
        partials[3 * blockIdx.x + 2] = dlt;
    }
    if (last_block(&tk->init, &is_last)) {
        bb = reduce_partials<kPairThreads>(partials, gridDim.x, 3, red);
        gam = reduce_partials<kPairThreads>(partials + 1, gridDim.x, 3, red);
        dlt = reduce_partials<kPairThreads>(partials + 2, gridDim.x, 3, red);
        if (threadIdx.x == 0) scalar_after_pass_init(sc, bb, gam, dlt);
    }
}
