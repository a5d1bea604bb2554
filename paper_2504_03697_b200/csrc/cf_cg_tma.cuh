// cf_cg_tma.cuh -- TMA-staged, warp-specialised forms of the two fused CG
// kernels (included by cf_cg.cu / cf_dist.cu inside namespace cf, after
// CgScalars / CgTickets / zval).  Same per-element arithmetic as
// cg_dir_kernel / cg_update_kernel.  Warps 0..7 consume cell pairs, warp 8
// drives the TMA ring through full/empty mbarriers (cf_tma_march.cuh), so no
// block-wide barrier sits inside the plane loop.

// ---------------------------------------------------------------- direction
// p = z + beta*p_old is formed in registers from the staged r (or z) and
// p_old boxes wherever the stencil needs it (centre pair, x-outer, y pairs,
// next plane): a little more fp64 work, no shared ring, no barrier.
template <int PK>
struct DirPolicy {
    const double *sz, *sp;
    double zc, beta;
    bool first;
    double *out;  // p_new at (i, j) of plane 0
    long long plane;
    int nz;
    double pap = 0.0;

    __device__ __forceinline__ double2 value2(int s, int o) const
    {
        double2 r = ld2(sz + s * kBoxStride + o);
        if (PK == PK_JCONST) {  // z = r * (1/diag) (src/precond.py:94)
            r.x = r.x * zc;
            r.y = r.y * zc;
        }
        if (!first) {  // p = z + beta * p_old (src/solver.py:169); p = z first (:142)
            const double2 p = ld2(sp + s * kBoxStride + o);
            r.x = r.x + beta * p.x;
            r.y = r.y + beta * p.y;
        }
        return r;
    }
    __device__ __forceinline__ double value(int s, int o) const
    {
        double r = sz[s * kBoxStride + o];
        if (PK == PK_JCONST) r = r * zc;
        if (!first) r = r + beta * sp[s * kBoxStride + o];
        return r;
    }
    __device__ __forceinline__ void epi(int, const MarchCoords &, int z, double2 c, double a0, double a1)
    {
        st2(out + plane * z, c.x, c.y);
        pap = pap + c.x * a0;
        pap = pap + c.y * a1;
    }
    // z-slab halo planes (-1, nz): p there is recomputed from the exchanged r
    // halo (bit-identical to the neighbour's owned p) and stored so the update
    // kernel's stencil can read it
    __device__ __forceinline__ void halo(const MarchCoords &m, int zq, double2 v)
    {
        if (m.valid && (zq == -1 || zq == nz)) st2(out + plane * zq, v.x, v.y);
    }
};

template <int ORDER, int PK>
__global__ void __launch_bounds__(kWSThreads, 4) cg_dir_tma(const __grid_constant__ CUtensorMap mz,
                                                         const __grid_constant__ CUtensorMap mp, TmaGeom g,
                                                         double off, double diag, double *__restrict__ p_new,
                                                         double zc, CgScalars *sc, double *partials, CgTickets *tk,
                                                         double *red_out)
{
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    __shared__ double red[32];
    __shared__ int is_last;
    if (sc->done) return;
    double *const sz = aligned_smem(smem_raw);      // kStages boxes of z (or r)
    double *const sp = sz + kStages * kBoxStride;  // kStages boxes of p_old
    const bool first = sc->it == 0;
    const MarchCoords m = march_coords(g);
    const long long plane = (long long)g.nx * g.ny;
    DirPolicy<PK> pol{sz, sp, zc, sc->beta, first, p_new + m.i + (long long)g.nx * m.j, plane, g.nz};
    init_ws_bars(full, empty);
    if (threadIdx.x >= kPThreads) {  // producer warp
        if (threadIdx.x == kPThreads) {
            prefetch_map(&mz);
            prefetch_map(&mp);
            const uint32_t bytes = first ? kBoxBytes : 2 * kBoxBytes;
            ws_produce(m.nplanes, full, empty, [&](int q, int s, uint64_t *bar) {
                const int z = m.zs + q + g.lo_halo;
                mbar_expect_tx(bar, bytes);
                tma_load_3d(sz + s * kBoxStride, &mz, m.bx0, m.by0, z, bar);
                if (!first) tma_load_3d(sp + s * kBoxStride, &mp, m.bx0, m.by0, z, bar);
            });
        }
    } else {
        ws_consume<ORDER>(g, m, off, diag, pol, full, empty);
    }
    double pap = block_sum<kWSThreads>(pol.pap, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = pap;
    if (last_block(&tk->dir, &is_last)) {
        pap = reduce_partials<kWSThreads>(partials, gridDim.x, 1, red);
        if (threadIdx.x == 0) {
            if (red_out) red_out[0] = pap;  // z-slab: summed across slabs/ranks first
            else scalar_after_dir(sc, pap);
        }
    }
}

// ---------------------------------------------------------------- update
template <int PK, int XM>
struct UpdPolicy {
    const double *sp, *sr, *sx, *sq;
    double alpha, malpha, zc, alpha_prev;
    double *r, *x;
    long long nx, plane;
    // z-slab peer form (cf_p2p.cu): the bottom / top owned r plane is also
    // stored into the neighbours' halo planes (null: no neighbour / not used)
    double *lo_r, *hi_r;
    int ztop;
    double rr = 0.0, rz = 0.0;

    __device__ __forceinline__ double2 value2(int s, int o) const { return ld2(sp + s * kBoxStride + o); }
    __device__ __forceinline__ double value(int s, int o) const { return sp[s * kBoxStride + o]; }
    __device__ __forceinline__ void epi(int s, const MarchCoords &m, int z, double2 c, double a0, double a1)
    {
        const int k = m.ty * kTTX + 2 * m.tx2;
        const long long gi = m.i + nx * m.j + plane * z;
        const double2 ro = ld2(sr + s * kInt + k);
        if (XM == XM_EACH) {
            const double2 xo = ld2(sx + s * kInt + k);
            st2(x + gi, xo.x + alpha * c.x, xo.y + alpha * c.y);  // src/solver.py:155
        } else if (XM == XM_DOUBLE) {  // the skipped step first, then this one
            const double2 xo = ld2(sx + s * kInt + k), q = ld2(sq + s * kInt + k);
            const double x0 = xo.x + alpha_prev * q.x, x1 = xo.y + alpha_prev * q.y;
            st2(x + gi, x0 + alpha * c.x, x1 + alpha * c.y);
        }
        const double r0 = ro.x + malpha * a0, r1 = ro.y + malpha * a1;  // :157
        st2(r + gi, r0, r1);
        if (lo_r && z == 0) st2(lo_r + (gi - plane * z), r0, r1);
        if (hi_r && z == ztop) st2(hi_r + (gi - plane * z), r0, r1);
        rr = rr + r0 * r0;
        rr = rr + r1 * r1;
        if (PK != PK_ZVEC) {
            rz = rz + r0 * zval<PK>(r0, nullptr, 0, zc);
            rz = rz + r1 * zval<PK>(r1, nullptr, 0, zc);
        }
    }
    __device__ __forceinline__ void halo(const MarchCoords &, int, double2) {}
};

// interior boxes staged per plane: r, plus x (XM_EACH / XM_DOUBLE), plus p_prev (XM_DOUBLE)
template <int XM>
__host__ __device__ constexpr int upd_interiors() { return XM == XM_SKIP ? 1 : (XM == XM_EACH ? 2 : 3); }

// The update march of one block (block `bid` of the geometry): producer warp
// streams the p halo box and the interior boxes through the mbarrier ring,
// consumers run the stencil + epilogue.  Returns the block sums (rr, rz) on
// thread 0.  Maps may live in the parameter block or in global memory.
template <int ORDER, int PK, int XM, int S = kStages>
__device__ __forceinline__ void update_tma_body(const CUtensorMap *mp, const CUtensorMap *mr, const CUtensorMap *mx,
                                             const CUtensorMap *mq, const TmaGeom g, int bid, double off, double diag,
                                             double *__restrict__ r, double *__restrict__ x, double zc, double alpha,
                                             double alpha_prev, double *__restrict__ lo_r, double *__restrict__ hi_r,
                                             double *red, double &rr_out, double &rz_out)
{
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[S], empty[S];
    double *const sp = aligned_smem(smem_raw);
    double *const sr = sp + S * kBoxStride;
    double *const sx = sr + S * kInt;
    double *const sq = sx + S * kInt;
    const MarchCoords m = march_coords(g, bid);
    UpdPolicy<PK, XM> pol{sp,  sr,   sx,   sq,   alpha,   -alpha, zc, alpha_prev, r, x, g.nx, (long long)g.nx * g.ny,
                          lo_r, hi_r, g.nz - 1};
    init_ws_bars<S>(full, empty);
    if (threadIdx.x >= kPThreads) {  // producer warp
        if (threadIdx.x == kPThreads) {
            prefetch_map(mp);
            prefetch_map(mr);
            if (XM != XM_SKIP) prefetch_map(mx);
            if (XM == XM_DOUBLE) prefetch_map(mq);
            auto issue = [&](int q, int s, uint64_t *bar) {
                const int z = m.zs + q;
                const bool own = z >= m.z0 && z < m.z1;  // r, x, p_prev only for owned planes
                mbar_expect_tx(bar, kBoxBytes + (own ? upd_interiors<XM>() * kIntBytes : 0));
                tma_load_3d(sp + s * kBoxStride, mp, m.bx0, m.by0, z + g.lo_halo, bar);
                if (own) {
                    tma_load_3d(sr + s * kInt, mr, m.x0, m.y0, z + g.lo_halo, bar);
                    if (XM != XM_SKIP) tma_load_3d(sx + s * kInt, mx, m.x0, m.y0, z + g.lo_halo, bar);
                    if (XM == XM_DOUBLE) tma_load_3d(sq + s * kInt, mq, m.x0, m.y0, z + g.lo_halo, bar);
                }
            };
            ws_produce<decltype(issue), S>(m.nplanes, full, empty, issue);
        }
    } else {
        ws_consume<ORDER, UpdPolicy<PK, XM>, S>(g, m, off, diag, pol, full, empty);
    }
    rr_out = block_sum<kWSThreads>(pol.rr, red);
    rz_out = PK != PK_ZVEC ? block_sum<kWSThreads>(pol.rz, red) : 0.0;
}

template <int ORDER, int PK, int XM = XM_EACH, int S = kStages>
__global__ void __launch_bounds__(kWSThreads) cg_update_tma(
    const __grid_constant__ CUtensorMap mp, const __grid_constant__ CUtensorMap mr,
    const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap mq, TmaGeom g, double off,
    double diag, double *__restrict__ r, double *__restrict__ x, double zc, CgScalars *sc, double *partials,
    CgTickets *tk, int use_cond, cudaGraphConditionalHandle cond, double *red_out)
{
    __shared__ double red[32];
    __shared__ int is_last;
    griddep_enter();
    if (sc->done) {
        if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    double rr, rz;
    update_tma_body<ORDER, PK, XM, S>(&mp, &mr, &mx, &mq, g, blockIdx.x, off, diag, r, x, zc, sc->alpha,
                                      sc->alpha_prev, nullptr, nullptr, red, rr, rz);
    griddep_trigger();
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = rr;
        partials[2 * blockIdx.x + 1] = rz;
    }
    if (last_block(&tk->upd, &is_last)) {
        rr = reduce_partials<kWSThreads>(partials, gridDim.x, 2, red);
        if (PK != PK_ZVEC) rz = reduce_partials<kWSThreads>(partials + 1, gridDim.x, 2, red);
        if (threadIdx.x == 0) {
            if (red_out) {  // z-slab: summed across slabs/ranks first
                red_out[0] = rr;
                red_out[1] = rz;
            } else if (scalar_after_update<PK != PK_ZVEC>(sc, rr, rz) && use_cond) {
                cudaGraphSetConditional(cond, 0);
            }
        }
    }
}

constexpr size_t kDirSmem = 2 * kStages * kBoxStride * sizeof(double) + 128;
constexpr size_t kUpdSmem = kStages * (kBoxStride + 3 * kInt) * sizeof(double) + 128;
// the skip-x update stages only the p halo box and the r box: deeper rings fit
template <int S>
constexpr size_t upd_skip_smem() { return (size_t)S * (kBoxStride + kInt) * sizeof(double) + 128; }
template <int S>
constexpr size_t upd_full_smem() { return (size_t)S * (kBoxStride + 3 * kInt) * sizeof(double) + 128; }
