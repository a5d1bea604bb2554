// cf_cg_tma.cuh -- TMA-staged forms of the two fused CG kernels (included by
// cf_cg.cu inside namespace cf, after CgScalars / CgTickets / zval).  Same
// per-element arithmetic as cg_dir_kernel / cg_update_kernel; operands
// arrive by TMA into a 4-stage mbarrier ring (cf_tma_march.cuh), each
// thread owning an x-adjacent cell pair.

constexpr int kPnSlots = 4;

// ---------------------------------------------------------------- direction
// Lagged form: plane q of the chunk is staged (r or z, and p_old), its
// p = z + beta*p_old is formed ONCE per box position into a 4-slot ring, and
// the stencil runs one plane behind (plane q-1 reads ring slots q-2, q-1,
// q), so one barrier per plane covers both the ring and TMA slot recycling.
template <int ORDER, int PK>
__global__ void __launch_bounds__(kPThreads) cg_dir_tma(const __grid_constant__ CUtensorMap mz,
                                                        const __grid_constant__ CUtensorMap mp, TmaGeom g,
                                                        double off, double diag, double *__restrict__ p_new,
                                                        double zc, CgScalars *sc, double *partials, CgTickets *tk,
                                                        double *red_out)
{
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[kStages];
    __shared__ double red[32];
    __shared__ int is_last;
    if (sc->done) return;
    double *const sz = aligned_smem(smem_raw);  // kStages boxes of z (or r)
    double *const sp = sz + kStages * kBoxStride;  // kStages boxes of p_old
    double *const ring = sp + kStages * kBoxStride;  // kPnSlots boxes of p
    const bool first = sc->it == 0;  // p = z on the first iteration (src/solver.py:142)
    const double beta = sc->beta;
    const MarchCoords m = march_coords(g);
    init_bars(bars);
    const uint32_t bytes = first ? kBoxBytes : 2 * kBoxBytes;
    auto issue = [&](int q) {
        const int s = q % kStages;
        const int z = m.zs + q + g.lo_halo;
        mbar_expect_tx(&bars[s], bytes);
        tma_load_3d(sz + s * kBoxStride, &mz, m.bx0, m.by0, z, &bars[s]);
        if (!first) tma_load_3d(sp + s * kBoxStride, &mp, m.bx0, m.by0, z, &bars[s]);
    };
    if (threadIdx.x == 0) {
        prefetch_map(&mz);
        prefetch_map(&mp);
        for (int q = 0; q < min(kStages, m.nplanes); ++q) issue(q);
    }
    const bool hxl = m.i > 0, hxr = m.i + 2 < g.nx, hym = m.j > 0, hyp = m.j < g.ny - 1;
    const bool inplane_fast = hxl && hxr && hym && hyp;
    const long long plane = (long long)g.nx * g.ny;
    double *out = p_new + m.i + (long long)g.nx * m.j;
    double pap = 0.0;
    for (int q = 0; q <= m.nplanes; ++q) {
        if (q < m.nplanes) {
            const int s = q % kStages;
            mbar_wait(&bars[s], (uint32_t)((q / kStages) & 1));
            const double *zb = sz + s * kBoxStride, *pb = sp + s * kBoxStride;
            double *slot = ring + (q % kPnSlots) * kBoxStride;
            for (int pos = 2 * threadIdx.x; pos < kBox; pos += 2 * kPThreads) {
                double2 r2 = ld2(zb + pos);
                if (PK == PK_JCONST) {  // z = r * (1/diag) (src/precond.py:94)
                    r2.x = r2.x * zc;
                    r2.y = r2.y * zc;
                }
                if (!first) {  // p = z + beta * p_old (src/solver.py:169)
                    const double2 p2 = ld2(pb + pos);
                    r2.x = r2.x + beta * p2.x;
                    r2.y = r2.y + beta * p2.y;
                }
                st2(slot + pos, r2.x, r2.y);
            }
        }
        fence_proxy_async_smem();  // my reads of TMA slot q before its refill
        __syncthreads();           // ring slot q complete; TMA slot q fully consumed
        if (threadIdx.x == 0 && q + kStages < m.nplanes) issue(q + kStages);
        if (q < m.nplanes && m.valid) {
            // z-slab halo planes: p there is recomputed from the exchanged r
            // halo (bit-identical to the neighbour's owned p) and stored, so
            // the update kernel's stencil can read it
            const int zq = m.zs + q;
            if (zq == -1 || zq == g.nz) {
                const double2 v = ld2(ring + (q % kPnSlots) * kBoxStride + m.o);
                st2(out + plane * zq, v.x, v.y);
            }
        }
        const int z = m.zs + q - 1;
        if (z >= m.z0 && z < m.z1 && m.valid) {
            const bool hzm = z - 1 >= m.zlo, hzp = z + 1 <= m.zhi;
            const double *cur = ring + ((q + kPnSlots - 1) % kPnSlots) * kBoxStride + m.o;
            const double2 c = ld2(cur);
            const double2 zero = make_double2(0.0, 0.0);
            const double2 zm = hzm ? ld2(ring + ((q + kPnSlots - 2) % kPnSlots) * kBoxStride + m.o) : zero;
            const double2 zp = hzp ? ld2(ring + (q % kPnSlots) * kBoxStride + m.o) : zero;
            double a0, a1;
            if (inplane_fast && hzm && hzp) {
                stencil_pair<ORDER, true>(c, cur[-1], cur[2], ld2(cur - kHX), ld2(cur + kHX), zm, zp, true, true,
                                          true, true, true, true, off, diag, a0, a1);
            } else {
                stencil_pair<ORDER, false>(c, hxl ? cur[-1] : 0.0, hxr ? cur[2] : 0.0, hym ? ld2(cur - kHX) : zero,
                                           hyp ? ld2(cur + kHX) : zero, zm, zp, hxl, hxr, hym, hyp, hzm, hzp, off,
                                           diag, a0, a1);
            }
            st2(out + plane * z, c.x, c.y);
            pap = pap + c.x * a0;
            pap = pap + c.y * a1;
        }
    }
    pap = block_sum<kPThreads>(pap, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = pap;
    if (last_block(&tk->dir, &is_last)) {
        pap = reduce_partials<kPThreads>(partials, gridDim.x, 1, red);
        if (threadIdx.x == 0) {
            if (red_out) red_out[0] = pap;  // z-slab: summed across slabs/ranks first
            else scalar_after_dir(sc, pap);
        }
    }
}

// ---------------------------------------------------------------- update
template <int PK>
struct UpdPolicy {
    const CUtensorMap *mp, *mr, *mx;
    double *sp, *sr, *sx;
    int lo;
    double alpha, malpha, zc;
    double *r, *x;
    long long nx, plane;
    double rr = 0.0, rz = 0.0;

    __device__ void prefetch() const
    {
        prefetch_map(mp);
        prefetch_map(mr);
        prefetch_map(mx);
    }
    __device__ __forceinline__ const double *box(int s) const { return sp + s * kBoxStride; }
    __device__ void issue(int s, const MarchCoords &m, int z, uint64_t *bar) const
    {
        const bool own = z >= m.z0 && z < m.z1;  // r and x only for owned planes
        mbar_expect_tx(bar, kBoxBytes + (own ? 2 * kIntBytes : 0));
        tma_load_3d(sp + s * kBoxStride, mp, m.bx0, m.by0, z + lo, bar);
        if (own) {
            tma_load_3d(sr + s * kInt, mr, m.x0, m.y0, z + lo, bar);
            tma_load_3d(sx + s * kInt, mx, m.x0, m.y0, z + lo, bar);
        }
    }
    __device__ __forceinline__ void epi(int s, const MarchCoords &m, int z, double2 c, double a0, double a1)
    {
        const int k = m.ty * kTTX + 2 * m.tx2;
        const long long gi = m.i + nx * m.j + plane * z;
        const double2 xo = ld2(sx + s * kInt + k), ro = ld2(sr + s * kInt + k);
        st2(x + gi, xo.x + alpha * c.x, xo.y + alpha * c.y);  // src/solver.py:155
        const double r0 = ro.x + malpha * a0, r1 = ro.y + malpha * a1;  // :157
        st2(r + gi, r0, r1);
        rr = rr + r0 * r0;
        rr = rr + r1 * r1;
        if (PK != PK_ZVEC) {
            rz = rz + r0 * zval<PK>(r0, nullptr, 0, zc);
            rz = rz + r1 * zval<PK>(r1, nullptr, 0, zc);
        }
    }
};

template <int ORDER, int PK>
__global__ void __launch_bounds__(kPThreads) cg_update_tma(
    const __grid_constant__ CUtensorMap mp, const __grid_constant__ CUtensorMap mr,
    const __grid_constant__ CUtensorMap mx, TmaGeom g, double off, double diag, double *__restrict__ r,
    double *__restrict__ x, double zc, CgScalars *sc, double *partials, CgTickets *tk, int use_cond,
    cudaGraphConditionalHandle cond, double *red_out)
{
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[kStages];
    __shared__ double red[32];
    __shared__ int is_last;
    if (sc->done) {
        if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    double *base = aligned_smem(smem_raw);
    const double alpha = sc->alpha;
    UpdPolicy<PK> pol{&mp, &mr, &mx, base, base + kStages * kBoxStride, base + kStages * (kBoxStride + kInt),
                      g.lo_halo, alpha, -alpha, zc, r, x, g.nx, (long long)g.nx * g.ny};
    staged_pair_march<ORDER>(g, off, diag, pol, bars);
    double rr = block_sum<kPThreads>(pol.rr, red);
    double rz = PK != PK_ZVEC ? block_sum<kPThreads>(pol.rz, red) : 0.0;
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = rr;
        partials[2 * blockIdx.x + 1] = rz;
    }
    if (last_block(&tk->upd, &is_last)) {
        rr = reduce_partials<kPThreads>(partials, gridDim.x, 2, red);
        if (PK != PK_ZVEC) rz = reduce_partials<kPThreads>(partials + 1, gridDim.x, 2, red);
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

constexpr size_t kDirSmem = (2 * kStages + kPnSlots) * kBoxStride * sizeof(double) + 128;
constexpr size_t kUpdSmem = kStages * (kBoxStride + 2 * kInt) * sizeof(double) + 128;
