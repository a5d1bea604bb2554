// cf_cg_lean.cuh -- low-instruction form of the pair-march direction kernel
// (included by cf_cg.cu inside namespace cf, after cf_cg_pair.cuh).
//
// Why: the pair march (cf_cg_pair.cuh) spends ~200 instructions per warp and
// plane (r01b SASS / ncu: 62 % issue slots busy, IPC 2.5, ~4.1 TB/s DRAM):
// 64-bit offset arithmetic for each of its 8 loads, wall masks (FSEL) on
// every loaded value, the first-iteration select on every p.  Here
//   * indices are 32-bit unsigned (N + pad < 2^32), so an address is one
//     IMAD.WIDE.U32 off the array base;
//   * every CG vector carries kLeanPad zeroed doubles after its N cells, and
//     a neighbour outside the domain is read from there: p = z*zc + beta*0 =
//     +0 and off*(+0) = -0 leaves the stencil sum unchanged bit for bit (the
//     same identity the masked forms rely on), so no per-value mask remains;
//   * the first iteration (p = z) is a separate instantiation of the march,
//     chosen once per block;
//   * only lanes 0 / 31 load the tile-edge cell.
// Same per-element arithmetic as cg_dir_pair / cg_dir_tma: p, A p and the
// block partials of p.Ap are bit-identical.

constexpr int kLeanPad = 64;  // >= 2 * 32 lanes: one zero pair per lane

// 16-byte loads the compiler may not move (volatile asm).  The next plane's
// loads are issued right AFTER this plane's values are consumed: issued before
// the first use (as plain __ldg code placed them), they shared a scoreboard
// with the values in use, and that first use waited for the new loads too
// (ncu: 29 % of all stall samples on that one DMUL).
__device__ __forceinline__ double2 ldg2_pinned(const double *p)
{
    double2 v;
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ double ldg1_pinned(const double *p)
{
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld2_pinned(const double *p)
{
    double2 v;
    asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}


template <int PK, bool FIRST>
__device__ __forceinline__ double lean_form(double z, double q, double zc, double beta)
{
    if (PK == PK_JCONST) z = z * zc;  // src/precond.py:94
    return FIRST ? z : z + beta * q;  // src/solver.py:142, :169
}

// COH: coherent (.cg, L2) loads instead of the read-only path -- for the
// persistent CG kernel, whose vectors are rewritten within one launch
template <bool COH>
__device__ __forceinline__ double2 lean_ld2(const double *p)
{
    return COH ? __ldcg(reinterpret_cast<const double2 *>(p)) : __ldg(reinterpret_cast<const double2 *>(p));
}
template <bool COH>
__device__ __forceinline__ double lean_ld1(const double *p)
{
    return COH ? __ldcg(p) : __ldg(p);
}

template <int PK, bool FIRST, bool COH = false>
struct LeanSrc {
    const double *__restrict__ zs;
    const double *__restrict__ po;
    double zc, beta;
    struct Raw {
        double2 z, q;
    };
    __device__ __forceinline__ Raw raw(unsigned k) const
    {
        Raw r;
        r.z = lean_ld2<COH>(zs + k);
        if (!FIRST) r.q = lean_ld2<COH>(po + k);
        return r;
    }
    __device__ __forceinline__ double2 form(const Raw &r) const
    {
        return make_double2(lean_form<PK, FIRST>(r.z.x, FIRST ? 0.0 : r.q.x, zc, beta),
                            lean_form<PK, FIRST>(r.z.y, FIRST ? 0.0 : r.q.y, zc, beta));
    }
    struct Raw1 {
        double z, q;
    };
    __device__ __forceinline__ Raw1 one(unsigned k) const
    {
        Raw1 r;
        r.z = lean_ld1<COH>(zs + k);
        r.q = FIRST ? 0.0 : lean_ld1<COH>(po + k);
        return r;
    }
    __device__ __forceinline__ double form1(const Raw1 &r) const { return lean_form<PK, FIRST>(r.z, r.q, zc, beta); }
    // the same loads, pinned in place (volatile): software pipelining (PF 2)
    __device__ __forceinline__ Raw raw_pinned(unsigned k) const
    {
        Raw r;
        r.z = ldg2_pinned(zs + k);
        if (!FIRST) r.q = ldg2_pinned(po + k);
        return r;
    }
    __device__ __forceinline__ Raw1 one_pinned(unsigned k) const
    {
        Raw1 r;
        r.z = ldg1_pinned(zs + k);
        r.q = FIRST ? 0.0 : ldg1_pinned(po + k);
        return r;
    }
};

// One block's top-down march (the update kernel marches bottom-up, so this
// one starts on the planes it wrote last, still in L2).  Returns the thread's
// partial p.Ap.  PF (software pipelining): 1 = the next plane's far operand
// is loaded one iteration early, 2 = every load of the next plane is, issued
// (volatile) only after this plane's loaded values are consumed.
template <int ORDER, int PK, bool FIRST, int PF, int ROWS, bool HALO = false, bool COH = false>
__device__ __forceinline__ double dir_lean_march(const PairGeom &g, int bid, double off, double diag,
                                                 const double *__restrict__ zs, const double *__restrict__ po,
                                                 double *__restrict__ pn, double zc, double beta)
{
    // z-slab halos (multi-GPU, cf_p2p.cu): planes -1 / nz exist in memory when
    // lo_halo / hi_halo; indices count from the lowest plane present, and the
    // zero pad follows the highest
    // HALO: the caller passes zs / po / pn at the LOWEST plane in memory (plane
    // -1 when lo_halo).  (Shifting them in here made the compiler rebuild every
    // address in 64-bit arithmetic; HALO = false is the single-domain kernel.)
    const int lo = HALO && g.lo_halo ? 1 : 0, hi = HALO && g.hi_halo ? 1 : 0;
    using Raw = typename LeanSrc<PK, FIRST, COH>::Raw;
    using Raw1 = typename LeanSrc<PK, FIRST, COH>::Raw1;
    const int lane = threadIdx.x & 31;
    const int ntiles = g.ntx * g.nty;
    const int tile = bid % ntiles, chunk = g.chunk_of(bid);
    const int i = (tile % g.ntx) * kPairX + 2 * lane;
    const int j = (tile / g.ntx) * ROWS + (threadIdx.x >> 5);
    if (j >= g.ny) return 0.0;  // the whole warp
    const int z0 = (int)((long long)g.nz * chunk / g.nchunk);
    const int z1 = (int)((long long)g.nz * (chunk + 1) / g.nchunk);
    const unsigned nx = (unsigned)g.nx, pl = nx * (unsigned)g.ny;
    const unsigned zero = pl * (unsigned)(g.nz + lo + hi) + 2u * (unsigned)lane;  // this lane's zero pair
    const bool valid = i < g.nx;
    const bool hym = valid && j > 0, hyp = valid && j + 1 < g.ny;
    const bool eload = lane == 0 || lane == 31;  // lanes that need the tile-edge cell
    const bool he = valid && (lane == 0 ? i > 0 : i + 2 < g.nx);
    const unsigned de = lane == 0 ? 0xffffffffu : 2u;  // -1 / +2 (mod 2^32)
    const LeanSrc<PK, FIRST, COH> src{zs, po, zc, beta};
    // the in-plane loads of plane index k (c = its centre index)
    auto in_plane = [&](unsigned k, Raw &ym, Raw &yp, Raw1 &e) {
        if (PF >= 2) {
            ym = src.raw_pinned(hym ? k - nx : zero);
            yp = src.raw_pinned(hyp ? k + nx : zero);
            if (eload) e = src.one_pinned(he ? k + de : zero);
        } else {
            ym = src.raw(hym ? k - nx : zero);
            yp = src.raw(hyp ? k + nx : zero);
            if (eload) e = src.one(he ? k + de : zero);
        }
    };

    unsigned c = (unsigned)i + nx * (unsigned)j + pl * (unsigned)(z1 - 1 + lo);
    const bool hzp1 = valid && z1 < g.nz + hi;
    double2 cp = src.form(src.raw(hzp1 ? c + pl : zero));
    double2 cc = src.form(src.raw(valid ? c : zero));
    // the slab's top halo plane of p, recomputed from the exchanged r halo
    // (bit-identical to the neighbour's own p) for the update kernel's stencil
    if (hi && hzp1 && z1 == g.nz) *reinterpret_cast<double2 *>(pn + c + pl) = cp;
    Raw rnx, nym, nyp;
    Raw1 ne{0.0, 0.0};
    if (PF == 1) rnx = src.raw(valid && z1 - 1 + lo >= 1 ? c - pl : zero);
    if (PF >= 2) {
        rnx = src.raw_pinned(valid && z1 - 1 + lo >= 1 ? c - pl : zero);
        in_plane(c, nym, nyp, ne);
    }
    double pap = 0.0;
    for (int z = z1 - 1; z >= z0; --z, c -= pl) {
        Raw rm, rym, ryp;
        Raw1 re{0.0, 0.0};
        if (PF >= 2) {
            rm = rnx;
        } else if (PF == 1) {
            rm = rnx;
            rnx = src.raw(valid && z + lo >= 2 && z > z0 ? c - 2 * pl : zero);  // plane z-2, if the next iteration runs
        } else {
            rm = src.raw(valid && z + lo >= 1 ? c - pl : zero);
        }
        if (PF >= 2) {
            rym = nym;
            ryp = nyp;
            re = ne;
        } else {
            in_plane(c, rym, ryp, re);
        }
        const double2 cm = src.form(rm);
        const double2 ym = src.form(rym), yp = src.form(ryp);
        const double e = eload ? src.form1(re) : 0.0;
        if (PF >= 2 && z > z0) {  // every load of the next plane, now that this one is consumed
            rnx = src.raw_pinned(valid && z + lo >= 2 ? c - 2 * pl : zero);
            in_plane(c - pl, nym, nyp, ne);
        }
        double xl = __shfl_up_sync(0xffffffffu, cc.y, 1);
        double xr = __shfl_down_sync(0xffffffffu, cc.x, 1);
        xl = lane == 0 ? e : xl;
        xr = lane == 31 ? e : xr;
        double a0, a1;
        stencil_pair<ORDER, true>(cc, xl, xr, ym, yp, cm, cp, true, true, true, true, true, true, off, diag, a0, a1);
        if (valid) {
            *reinterpret_cast<double2 *>(pn + c) = cc;
            pap = pap + cc.x * a0;
            pap = pap + cc.y * a1;
            if (lo && z == 0) *reinterpret_cast<double2 *>(pn + c - pl) = cm;  // bottom halo plane of p
        }
        cp = cc;
        cc = cm;
    }
    return pap;
}

template <int ORDER, int PK, int PF, int ROWS = kPairRows>
__global__ void __launch_bounds__(32 * ROWS, 8 * kPairRows / ROWS) cg_dir_lean(PairGeom g, double off, double diag,
                                                            const double *__restrict__ zs,
                                                            const double *__restrict__ p_old,
                                                            double *__restrict__ p_new, double zc, CgScalars *sc,
                                                            double *partials, CgTickets *tk)
{
    __shared__ double red[32];
    __shared__ int is_last;
    griddep_enter();
    if (sc->done) return;
    double pap = sc->it == 0
                     ? dir_lean_march<ORDER, PK, true, PF, ROWS>(g, blockIdx.x, off, diag, zs, p_old, p_new, zc, 0.0)
                     : dir_lean_march<ORDER, PK, false, PF, ROWS>(g, blockIdx.x, off, diag, zs, p_old, p_new, zc, sc->beta);
    griddep_trigger();  // this CTA's sweep is done: the next kernel may start launching
    pap = block_sum<32 * ROWS>(pap, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = pap;
    if (last_block(&tk->dir, &is_last)) {
        pap = reduce_partials<32 * ROWS>(partials, gridDim.x, 1, red);
        if (threadIdx.x == 0) scalar_after_dir(sc, pap);
    }
}

// ---------------------------------------------------------------- update
// Ap recomputed from p (as stored), r += (-alpha) Ap, x per XM (cf_cg_common.cuh),
// partial r.r and r.z; last block -> convergence test and beta.  Marched
// bottom-up (the direction kernel marched top-down and left its last planes,
// the bottom ones, in L2).  Per-element arithmetic of cg_update_tma /
// cg_update_pair.
template <int ORDER, int PK, int XM, int ROWS, bool COH = false>
__device__ __forceinline__ void upd_lean_march(const PairGeom &g, int bid, double off, double diag,
                                               const double *__restrict__ p, const double *__restrict__ q,
                                               double *__restrict__ r, double *__restrict__ x, double zc,
                                               double alpha, double alpha_prev, double &rr, double &rz)
{
    const int lane = threadIdx.x & 31;
    const int ntiles = g.ntx * g.nty;
    const int tile = bid % ntiles, chunk = g.chunk_of(bid);
    const int i = (tile % g.ntx) * kPairX + 2 * lane;
    const int j = (tile / g.ntx) * ROWS + (threadIdx.x >> 5);
    if (j >= g.ny) return;  // the whole warp
    const int z0 = (int)((long long)g.nz * chunk / g.nchunk);
    const int z1 = (int)((long long)g.nz * (chunk + 1) / g.nchunk);
    const unsigned nx = (unsigned)g.nx, pl = nx * (unsigned)g.ny;
    const unsigned zero = pl * (unsigned)g.nz + 2u * (unsigned)lane;
    const bool valid = i < g.nx;
    const bool hym = valid && j > 0, hyp = valid && j + 1 < g.ny;
    const bool eload = lane == 0 || lane == 31;
    const bool he = valid && (lane == 0 ? i > 0 : i + 2 < g.nx);
    const unsigned de = lane == 0 ? 0xffffffffu : 2u;
    const double malpha = -alpha;
    auto ld2 = [](const double *a, unsigned k) { return lean_ld2<COH>(a + k); };

    unsigned c = (unsigned)i + nx * (unsigned)j + pl * (unsigned)z0;
    double2 cm = ld2(p, valid && z0 >= 1 ? c - pl : zero);
    double2 cc = ld2(p, valid ? c : zero);
    for (int z = z0; z < z1; ++z, c += pl) {
        const unsigned cv = valid ? c : zero;
        const double2 cp = ld2(p, valid && z + 1 < g.nz ? c + pl : zero);
        const double2 ym = ld2(p, hym ? c - nx : zero);
        const double2 yp = ld2(p, hyp ? c + nx : zero);
        double e = 0.0;
        if (eload) e = lean_ld1<COH>(p + (he ? c + de : zero));
        // r, x, p_prev of this plane: plain loads (r and x are written here)
        const double2 ro = *reinterpret_cast<const double2 *>(r + cv);
        double2 xo, qo;
        if (XM != XM_SKIP) xo = *reinterpret_cast<const double2 *>(x + cv);
        if (XM == XM_DOUBLE) qo = ld2(q, cv);
        double xl = __shfl_up_sync(0xffffffffu, cc.y, 1);
        double xr = __shfl_down_sync(0xffffffffu, cc.x, 1);
        xl = lane == 0 ? e : xl;
        xr = lane == 31 ? e : xr;
        double a0, a1;
        stencil_pair<ORDER, true>(cc, xl, xr, ym, yp, cm, cp, true, true, true, true, true, true, off, diag, a0, a1);
        if (valid) {
            if (XM == XM_EACH) {  // src/solver.py:155
                *reinterpret_cast<double2 *>(x + c) = make_double2(xo.x + alpha * cc.x, xo.y + alpha * cc.y);
            } else if (XM == XM_DOUBLE) {  // the skipped step first, then this one
                const double x0 = xo.x + alpha_prev * qo.x, x1 = xo.y + alpha_prev * qo.y;
                *reinterpret_cast<double2 *>(x + c) = make_double2(x0 + alpha * cc.x, x1 + alpha * cc.y);
            }
            const double r0 = ro.x + malpha * a0, r1 = ro.y + malpha * a1;  // :157
            *reinterpret_cast<double2 *>(r + c) = make_double2(r0, r1);
            rr = rr + r0 * r0;
            rr = rr + r1 * r1;
            if (PK != PK_ZVEC) {
                rz = rz + r0 * zval<PK>(r0, nullptr, 0, zc);
                rz = rz + r1 * zval<PK>(r1, nullptr, 0, zc);
            }
        }
        cm = cc;
        cc = cp;
    }
}

template <int ORDER, int PK, int XM, int ROWS = kPairRows>
__global__ void __launch_bounds__(32 * ROWS, 8 * kPairRows / ROWS) cg_update_lean(PairGeom g, double off, double diag,
                                                               const double *__restrict__ p,
                                                               const double *__restrict__ p_prev,
                                                               double *__restrict__ r, double *__restrict__ x,
                                                               double zc, CgScalars *sc, double *partials,
                                                               CgTickets *tk, int use_cond,
                                                               cudaGraphConditionalHandle cond)
{
    __shared__ double red[32];
    __shared__ int is_last;
    griddep_enter();
    if (sc->done) {
        if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    double rr = 0.0, rz = 0.0;
    upd_lean_march<ORDER, PK, XM, ROWS>(g, blockIdx.x, off, diag, p, p_prev, r, x, zc, sc->alpha, sc->alpha_prev, rr, rz);
    griddep_trigger();
    rr = block_sum<32 * ROWS>(rr, red);
    rz = PK != PK_ZVEC ? block_sum<32 * ROWS>(rz, red) : 0.0;
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = rr;
        partials[2 * blockIdx.x + 1] = rz;
    }
    if (last_block(&tk->upd, &is_last)) {
        rr = reduce_partials<32 * ROWS>(partials, gridDim.x, 2, red);
        if (PK != PK_ZVEC) rz = reduce_partials<32 * ROWS>(partials + 1, gridDim.x, 2, red);
        if (threadIdx.x == 0 && scalar_after_update<PK != PK_ZVEC>(sc, rr, rz) && use_cond)
            cudaGraphSetConditional(cond, 0);
    }
}

// ---------------------------------------------------------------- two rows per warp
// The direction march with each warp owning TWO tile rows (j, j+1): the rows'
// shared y-neighbours come from registers (row j's yp is row j+1's centre and
// vice versa), so per plane a warp issues two DRAM row loads (the next plane
// of both rows) but only two L1/L2 halo rows, and more DRAM bytes are in
// flight per register (the one-row march is long-scoreboard bound at 64
// registers).  A CTA of RW warps covers 2*RW rows.  Single domain (no slab
// halos), same per-element arithmetic; the per-thread p.Ap order is row j
// then row j+1 per plane.
template <int ORDER, int PK, bool FIRST, int RW, bool HALO = false>
__device__ __forceinline__ double dir_lean2_march(const PairGeom &g, int bid, double off, double diag,
                                                  const double *__restrict__ zs, const double *__restrict__ po,
                                                  double *__restrict__ pn, double zc, double beta)
{
    // HALO (z-slab, cf_p2p.cu): as in dir_lean_march, pointers at the lowest
    // plane in memory, halo planes of p recomputed and stored
    const int lo = HALO && g.lo_halo ? 1 : 0, hi = HALO && g.hi_halo ? 1 : 0;
    using Src = LeanSrc<PK, FIRST>;
    using Raw = typename Src::Raw;
    using Raw1 = typename Src::Raw1;
    const int lane = threadIdx.x & 31;
    const int ntiles = g.ntx * g.nty;
    const int tile = bid % ntiles, chunk = g.chunk_of(bid);
    const int i = (tile % g.ntx) * kPairX + 2 * lane;
    const int j = (tile / g.ntx) * (2 * RW) + 2 * (threadIdx.x >> 5);  // rows j, j+1
    if (j >= g.ny) return 0.0;
    const int z0 = (int)((long long)g.nz * chunk / g.nchunk);
    const int z1 = (int)((long long)g.nz * (chunk + 1) / g.nchunk);
    const unsigned nx = (unsigned)g.nx, pl = nx * (unsigned)g.ny;
    const unsigned zero = pl * (unsigned)(g.nz + lo + hi) + 2u * (unsigned)lane;
    const bool xv = i < g.nx;
    const bool v0 = xv, v1 = xv && j + 1 < g.ny;          // the two rows' pairs exist
    const bool hym = v0 && j > 0, hyp = v1 && j + 2 < g.ny;  // outer y-neighbour rows
    const bool eload = lane == 0 || lane == 31;
    const bool he = xv && (lane == 0 ? i > 0 : i + 2 < g.nx);
    const unsigned de = lane == 0 ? 0xffffffffu : 2u;
    const Src src{zs, po, zc, beta};

    unsigned c = (unsigned)i + nx * (unsigned)j + pl * (unsigned)(z1 - 1 + lo);  // row j; row j+1 is c + nx
    const bool top = z1 < g.nz + hi;
    double2 cp0 = src.form(src.raw(v0 && top ? c + pl : zero));
    double2 cp1 = src.form(src.raw(v1 && top ? c + nx + pl : zero));
    double2 cc0 = src.form(src.raw(v0 ? c : zero));
    double2 cc1 = src.form(src.raw(v1 ? c + nx : zero));
    if (hi && z1 == g.nz) {  // the slab's top halo plane of p
        if (v0) *reinterpret_cast<double2 *>(pn + c + pl) = cp0;
        if (v1) *reinterpret_cast<double2 *>(pn + c + nx + pl) = cp1;
    }
    double pap = 0.0;
    for (int z = z1 - 1; z >= z0; --z, c -= pl) {
        const bool hzm = z + lo >= 1;
        const Raw rm0 = src.raw(v0 && hzm ? c - pl : zero);
        const Raw rm1 = src.raw(v1 && hzm ? c + nx - pl : zero);
        const Raw rym = src.raw(hym ? c - nx : zero);
        const Raw ryp = src.raw(hyp ? c + 2 * nx : zero);
        Raw1 re0{0.0, 0.0}, re1{0.0, 0.0};
        if (eload) {
            re0 = src.one(he ? c + de : zero);
            re1 = src.one(he && v1 ? c + nx + de : zero);
        }
        const double2 cm0 = src.form(rm0), cm1 = src.form(rm1);
        const double2 ym = src.form(rym), yp = src.form(ryp);
        const double e0 = eload ? src.form1(re0) : 0.0, e1 = eload ? src.form1(re1) : 0.0;
        double xl0 = __shfl_up_sync(0xffffffffu, cc0.y, 1), xr0 = __shfl_down_sync(0xffffffffu, cc0.x, 1);
        double xl1 = __shfl_up_sync(0xffffffffu, cc1.y, 1), xr1 = __shfl_down_sync(0xffffffffu, cc1.x, 1);
        xl0 = lane == 0 ? e0 : xl0;
        xr0 = lane == 31 ? e0 : xr0;
        xl1 = lane == 0 ? e1 : xl1;
        xr1 = lane == 31 ? e1 : xr1;
        double a0, a1, b0, b1;
        stencil_pair<ORDER, true>(cc0, xl0, xr0, ym, cc1, cm0, cp0, true, true, true, true, true, true, off, diag, a0,
                                  a1);
        stencil_pair<ORDER, true>(cc1, xl1, xr1, cc0, yp, cm1, cp1, true, true, true, true, true, true, off, diag, b0,
                                  b1);
        if (v0) {
            *reinterpret_cast<double2 *>(pn + c) = cc0;
            pap = pap + cc0.x * a0;
            pap = pap + cc0.y * a1;
        }
        if (v1) {
            *reinterpret_cast<double2 *>(pn + c + nx) = cc1;
            pap = pap + cc1.x * b0;
            pap = pap + cc1.y * b1;
        }
        if (lo && z == 0) {  // bottom halo plane of p
            if (v0) *reinterpret_cast<double2 *>(pn + c - pl) = cm0;
            if (v1) *reinterpret_cast<double2 *>(pn + c + nx - pl) = cm1;
        }
        cp0 = cc0;
        cc0 = cm0;
        cp1 = cc1;
        cc1 = cm1;
    }
    return pap;
}

// 3 CTAs per SM at RW = 8 (80 registers, 24 bytes of L1-resident spill in the
// plane loop); the spill-free 2-CTA/SM build (90 registers) measured slower:
// 188.8 vs ~183 us per 256^3 two-kernel iteration, 1390 vs ~1380 at 512^3.
template <int ORDER, int PK, int RW>
__global__ void __launch_bounds__(32 * RW, 24 / RW) cg_dir_lean2(PairGeom g, double off, double diag,
                                                             const double *__restrict__ zs,
                                                             const double *__restrict__ p_old,
                                                             double *__restrict__ p_new, double zc, CgScalars *sc,
                                                             double *partials, CgTickets *tk)
{
    __shared__ double red[32];
    __shared__ int is_last;
    griddep_enter();
    if (sc->done) return;
    double pap = sc->it == 0
                     ? dir_lean2_march<ORDER, PK, true, RW>(g, blockIdx.x, off, diag, zs, p_old, p_new, zc, 0.0)
                     : dir_lean2_march<ORDER, PK, false, RW>(g, blockIdx.x, off, diag, zs, p_old, p_new, zc, sc->beta);
    griddep_trigger();
    pap = block_sum<32 * RW>(pap, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = pap;
    if (last_block(&tk->dir, &is_last)) {
        pap = reduce_partials<32 * RW>(partials, gridDim.x, 1, red);
        if (threadIdx.x == 0) scalar_after_dir(sc, pap);
    }
}
