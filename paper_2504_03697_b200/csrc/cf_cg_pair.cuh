// cf_cg_pair.cuh -- full-occupancy register-march forms of the two fused CG
// kernels (included by cf_cg.cu / cf_dist.cu inside namespace cf, after
// CgScalars / CgTickets / zval and the stencil helpers).
//
// Why a second form beside the TMA pipeline (cf_cg_tma.cuh): the TMA kernels
// hold 56 registers x 288 threads and a 3-stage smem ring, so at most 4 CTAs
// (36 warps) sit on an SM and the HBM queue is fed by ~512 CTAs.  Measured on
// this B200 (tools/bw_probe2.cu, tools/cg_probe.cu), a z-march with too few
// CTAs in flight stays near 4.5 TB/s even for a plain copy, while the same
// march at full occupancy reaches 5.7-6.2 TB/s.  Here a CTA is kPairRows warps
// (128 threads, no shared ring), so 8+ CTAs fit per SM:
//   * a warp owns one 64-cell tile row: lane k holds the x-adjacent pair
//     (x0 + 2k, x0 + 2k + 1), loads/stores it as one 16-byte access;
//   * x-neighbours come from the adjacent lanes by shuffle (only lanes 0 / 31
//     read the tile-edge cell); y-neighbours (rows j +- 1) are 16-byte loads
//     that hit L1/L2 (the rows are the neighbouring warps' centre rows);
//   * z-neighbours are the register window (z-1, z, z+1) of the march.
// Per-element arithmetic is the TMA kernels' (stencil_pair<ORDER>, p = z +
// beta*p_old, x += alpha*p, r += (-alpha)*Ap), so results are bit-identical
// per element; only the block partition of the dot products differs.

constexpr int kPairX = 64;                  // cells per tile row (= one warp of pairs)
constexpr int kPairRows = 4;                // tile rows = warps per CTA
constexpr int kPairThreads = 32 * kPairRows;

struct PairGeom {
    int nx, ny, nz;
    int lo_halo, hi_halo;  // plane -1 / plane nz exist in memory (z-slab halos)
    int ntx, nty, nchunk;
    // 1: CTAs take the z chunks from the top down (the lean marches), so a
    // kernel's last wave ends where the next kernel's first wave starts
    int chunk_rev = 0;
    __host__ __device__ int ctas() const { return ntx * nty * nchunk; }
    __host__ __device__ int chunk_of(int bid) const
    {
        const int c = bid / (ntx * nty);
        return chunk_rev ? nchunk - 1 - c : c;
    }
};

// Host: geometry for an nx*ny*nz block (z-slab halos lo/hi), z cut into
// chunks of ~32 planes (env_name: override of the chunk count).  cf_cg.cu.
PairGeom pair_geom(int nx, int ny, int nz, int lo_halo, int hi_halo, const char *env_name);
// Host: lean-march geometry -- 64 x rows tiles, wave-aware z chunks (cf_cg.cu).
PairGeom lean_geom(int nx, int ny, int nz, int rows, int ctas4);

struct PairCoords {
    int lane, i, j, z0, z1, zlo, zhi;
    bool row_ok, valid;        // row j exists; the pair (i, i+1) exists
    bool hxl, hxr, hym, hyp;   // in-plane neighbours exist
    long long base;            // flat offset of (i, j, 0)
};

__device__ __forceinline__ PairCoords pair_coords(const PairGeom &g, int bid)
{
    PairCoords c;
    const int ntiles = g.ntx * g.nty;
    const int tile = bid % ntiles, chunk = bid / ntiles;
    c.lane = threadIdx.x & 31;
    c.i = (tile % g.ntx) * kPairX + 2 * c.lane;
    c.j = (tile / g.ntx) * kPairRows + (threadIdx.x >> 5);
    c.z0 = (int)((long long)g.nz * chunk / g.nchunk);
    c.z1 = (int)((long long)g.nz * (chunk + 1) / g.nchunk);
    c.zlo = g.lo_halo ? -1 : 0;
    c.zhi = g.hi_halo ? g.nz : g.nz - 1;
    c.row_ok = c.j < g.ny;
    c.valid = c.row_ok && c.i < g.nx;
    c.hxl = c.i > 0;
    c.hxr = c.i + 2 < g.nx;
    c.hym = c.j > 0;
    c.hyp = c.j + 1 < g.ny;
    // lanes past the x wall (nx % 64 != 0) read a valid pair and store nothing
    c.base = (long long)min(c.i, g.nx - 2) + (long long)g.nx * c.j;
    return c;
}

__device__ __forceinline__ double2 ldg2(const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); }

// The pair march over this CTA's planes.  Src supplies raw loads and the
// operand formed from them (raw2/form2 for a pair, raw1/form1 for one cell);
// Epi receives (plane offset, centre pair, A pair) for every valid pair and
// (offset, pair) for the slab halo planes.  Per plane, EVERY load (z+1 centre,
// rows j-1 / j+1, tile-edge cell) is issued unconditionally -- at the walls
// the address is clamped onto the pair itself and the value masked to 0
// afterwards -- before any is consumed, so the plane costs one memory round
// trip, not four dependent ones.  x-neighbours come from adjacent lanes by
// shuffle; every lane reads one "edge" cell (left half of the warp i-1, right
// half i+2: L1 hits) and lanes 0 / 31 keep theirs.  The stencil is the full
// 7-term sum with absent neighbours as 0: off*0 = -0.0 (off < 0) and
// s + (-0.0) == s exactly, so each partial sum is bit-identical to the
// reference's sum over the existing entries (src/sparse.py:194-213).
template <int ORDER, class Src, class Epi>
__device__ __forceinline__ void pair_plane_step(const PairCoords &c, const PairGeom &g, long long o, double2 cm,
                                                double2 cc, double2 cp, double off, double diag, const Src &src,
                                                Epi &epi)
{
    const double2 zero = make_double2(0.0, 0.0);
    const int de = c.lane < 16 ? (c.hxl ? -1 : 0) : (c.hxr ? 2 : 0);
    const int dym = c.hym ? -g.nx : 0, dyp = c.hyp ? g.nx : 0;
    auto rym = src.raw2(o + dym);
    auto ryp = src.raw2(o + dyp);
    auto re = src.raw1(o + de);
    const double2 ym = c.hym ? src.form2(rym, o + dym) : zero;
    const double2 yp = c.hyp ? src.form2(ryp, o + dyp) : zero;
    const double e = src.form1(re, o + de);
    double xl = __shfl_up_sync(0xffffffffu, cc.y, 1);
    double xr = __shfl_down_sync(0xffffffffu, cc.x, 1);
    xl = c.lane == 0 ? e : xl;
    xr = c.lane == 31 ? e : xr;
    xl = c.hxl ? xl : 0.0;
    xr = c.hxr ? xr : 0.0;
    double a0, a1;
    stencil_pair<ORDER, true>(cc, xl, xr, ym, yp, cm, cp, true, true, true, true, true, true, off, diag, a0, a1);
    if (c.valid) epi.cell(o, cc, a0, a1);
}

// REV: march the chunk from its top plane down.  The CG alternates march
// directions between consecutive kernels (direction kernel down, update
// kernel up), so each kernel starts on the planes its predecessor wrote
// last -- the ones still resident in the 126 MB L2.
//
// PF: software-pipelined loads -- the raw operand of the next plane's far
// neighbour (z-2 when marching down, z+2 up) is issued one iteration early, so
// two planes' HBM reads are in flight per warp instead of one (the march is
// long-scoreboard bound at ~45 % occupancy; r01b ncu).  Same values, same
// arithmetic: results are bit-identical with or without PF.
template <int ORDER, bool REV, class Src, class Epi, bool PF = false>
__device__ __forceinline__ void pair_march(const PairCoords &c, const PairGeom &g, double off, double diag,
                                           const Src &src, Epi &epi)
{
    const long long pl = (long long)g.nx * g.ny;
    const double2 zero = make_double2(0.0, 0.0);
    if (REV) {
        const bool hzp1 = c.z1 <= c.zhi;
        const long long o1 = c.base + pl * (c.z1 - 1);
        const int zstop = max(c.z0 - 1, c.zlo);  // lowest plane this chunk reads
        auto rp1 = src.raw2(hzp1 ? o1 + pl : o1);
        auto rc1 = src.raw2(o1);
        auto rnx = src.raw2(PF && c.z1 - 2 >= zstop ? o1 - pl : o1);
        double2 cp = hzp1 ? src.form2(rp1, o1 + pl) : zero;
        double2 cc = src.form2(rc1, o1);
        if (hzp1 && c.z1 == g.nz) epi.halo(o1 + pl, cp);
        for (int z = c.z1 - 1; z >= c.z0; --z) {
            const long long o = c.base + pl * z;
            const bool hzm = z - 1 >= c.zlo;
            const long long om = hzm ? o - pl : o;
            decltype(rnx) rm;
            if (PF) {
                rm = rnx;
                rnx = src.raw2(z - 2 >= zstop ? o - 2 * pl : o);
            } else {
                rm = src.raw2(om);
            }
            const double2 cm = hzm ? src.form2(rm, om) : zero;
            pair_plane_step<ORDER>(c, g, o, cm, cc, cp, off, diag, src, epi);
            if (hzm && z == 0) epi.halo(om, cm);
            cp = cc;
            cc = cm;
        }
        return;
    }
    const bool hzm0 = c.z0 - 1 >= c.zlo;
    const long long o0 = c.base + pl * c.z0;
    const int ztop = min(c.z1, c.zhi);  // highest plane this chunk reads
    auto rm0 = src.raw2(hzm0 ? o0 - pl : o0);
    auto rc0 = src.raw2(o0);
    auto rnx = src.raw2(PF && c.z0 + 1 <= ztop ? o0 + pl : o0);
    double2 cm = hzm0 ? src.form2(rm0, o0 - pl) : zero;
    double2 cc = src.form2(rc0, o0);
    if (hzm0 && c.z0 - 1 == -1) epi.halo(o0 - pl, cm);
    for (int z = c.z0; z < c.z1; ++z) {
        const long long o = c.base + pl * z;
        const bool hzp = z + 1 <= c.zhi;
        const long long on = hzp ? o + pl : o;
        decltype(rnx) rn;
        if (PF) {
            rn = rnx;
            rnx = src.raw2(z + 2 <= ztop ? o + 2 * pl : o);
        } else {
            rn = src.raw2(on);
        }
        const double2 cp = hzp ? src.form2(rn, on) : zero;
        pair_plane_step<ORDER>(c, g, o, cm, cc, cp, off, diag, src, epi);
        if (hzp && z + 1 == g.nz) epi.halo(on, cp);
        cm = cc;
        cc = cp;
    }
}

struct Raw2 {
    double2 z, q, j;
};
struct Raw1 {
    double z, q, j;
};

// direction operand: p = z + beta*p_old with z = r, r*zc, r*jd or the DIC z
template <int PK>
struct DirSrc {
    const double *zsrc, *p_old, *jd;
    double zc, beta;
    bool first;
    __device__ __forceinline__ Raw2 raw2(long long o) const
    {
        Raw2 r;
        r.z = ldg2(zsrc + o);
        r.q = ldg2(p_old + o);  // read even on the first iteration (value discarded)
        if (PK == PK_JVEC) r.j = ldg2(jd + o);
        return r;
    }
    __device__ __forceinline__ Raw1 raw1(long long o) const
    {
        Raw1 r;
        r.z = __ldg(zsrc + o);
        r.q = __ldg(p_old + o);
        if (PK == PK_JVEC) r.j = __ldg(jd + o);
        return r;
    }
    __device__ __forceinline__ double form(double z, double q, double j) const
    {
        if (PK == PK_JCONST) z = z * zc;  // src/precond.py:94
        if (PK == PK_JVEC) z = z * j;
        return first ? z : z + beta * q;  // src/solver.py:142, :169
    }
    __device__ __forceinline__ double2 form2(const Raw2 &r, long long) const
    {
        return make_double2(form(r.z.x, r.q.x, r.j.x), form(r.z.y, r.q.y, r.j.y));
    }
    __device__ __forceinline__ double form1(const Raw1 &r, long long) const { return form(r.z, r.q, r.j); }
};

// update operand: p as stored
struct UpdSrc {
    const double *p;
    __device__ __forceinline__ double2 raw2(long long o) const { return ldg2(p + o); }
    __device__ __forceinline__ double raw1(long long o) const { return __ldg(p + o); }
    __device__ __forceinline__ double2 form2(double2 v, long long) const { return v; }
    __device__ __forceinline__ double form1(double v, long long) const { return v; }
};

// ---------------------------------------------------------------- direction
// p = z + beta*p_old, A p, partial p.Ap; last block -> alpha (or the slab
// partial to red_out).  In slab mode the halo planes of p (-1, nz) are
// recomputed from the exchanged r halo and stored so the update kernel's
// stencil can read them (bit-identical to the neighbour's owned p).
// The direction march of one block; returns the thread's partial p.Ap.
template <int ORDER, int PK, bool PF = false>
__device__ __forceinline__ double dir_pair_body(const PairGeom &g, int bid, double off, double diag,
                                                const double *__restrict__ zsrc, const double *__restrict__ jd,
                                                const double *__restrict__ p_old, double *__restrict__ p_new,
                                                double zc, double beta, bool first)
{
    const PairCoords c = pair_coords(g, bid);
    struct Epi {
        double *p_new;
        bool valid;
        double pap;
        __device__ __forceinline__ void cell(long long o, double2 cc, double a0, double a1)
        {
            *reinterpret_cast<double2 *>(p_new + o) = cc;
            pap = pap + cc.x * a0;
            pap = pap + cc.y * a1;
        }
        __device__ __forceinline__ void halo(long long o, double2 v)
        {
            if (valid) *reinterpret_cast<double2 *>(p_new + o) = v;
        }
    } epi{p_new, c.valid, 0.0};
    if (c.row_ok) {
        const DirSrc<PK> src{zsrc, p_old, jd, zc, beta, first};
        pair_march<ORDER, true, DirSrc<PK>, decltype(epi), PF>(c, g, off, diag, src, epi);
    }
    return epi.pap;
}

template <int ORDER, int PK, bool PF = false>
__global__ void __launch_bounds__(kPairThreads, 8) cg_dir_pair(PairGeom g, double off, double diag,
                                                            const double *__restrict__ zsrc,
                                                            const double *__restrict__ jd,
                                                            const double *__restrict__ p_old,
                                                            double *__restrict__ p_new, double zc, CgScalars *sc,
                                                            double *partials, CgTickets *tk, double *red_out)
{
    __shared__ double red[32];
    __shared__ int is_last;
    if (sc->done) return;
    double pap = dir_pair_body<ORDER, PK, PF>(g, blockIdx.x, off, diag, zsrc, jd, p_old, p_new, zc, sc->beta,
                                          sc->it == 0);
    pap = block_sum<kPairThreads>(pap, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = pap;
    if (last_block(&tk->dir, &is_last)) {
        pap = reduce_partials<kPairThreads>(partials, gridDim.x, 1, red);
        if (threadIdx.x == 0) {
            if (red_out) red_out[0] = pap;
            else scalar_after_dir(sc, pap);
        }
    }
}

// ---------------------------------------------------------------- update
// Ap recomputed from p, x += alpha p, r += (-alpha) Ap, partial r.r (and r.z
// for Jacobi/none); last block -> convergence test and beta.
template <int ORDER, int PK, int XM = XM_EACH>
__global__ void __launch_bounds__(kPairThreads, 8) cg_update_pair(PairGeom g, double off, double diag,
                                                               const double *__restrict__ p,
                                                               const double *__restrict__ p_prev,
                                                               double *__restrict__ r,
                                                               double *__restrict__ x,
                                                               const double *__restrict__ jd, double zc,
                                                               CgScalars *sc, double *partials, CgTickets *tk,
                                                               int use_cond, cudaGraphConditionalHandle cond,
                                                               double *red_out)
{
    __shared__ double red[32];
    __shared__ int is_last;
    if (sc->done) {
        if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    const PairCoords c = pair_coords(g, blockIdx.x);
    struct Epi {
        double *r, *x;
        const double *jd, *q;
        double alpha, malpha, zc, alpha_prev;
        double rr, rz;
        __device__ __forceinline__ void cell(long long o, double2 cc, double a0, double a1)
        {
            const double2 ro = *reinterpret_cast<const double2 *>(r + o);
            if (XM == XM_EACH) {
                const double2 xo = *reinterpret_cast<const double2 *>(x + o);
                *reinterpret_cast<double2 *>(x + o) = make_double2(xo.x + alpha * cc.x, xo.y + alpha * cc.y);
            } else if (XM == XM_DOUBLE) {  // the skipped step first, then this one
                const double2 xo = *reinterpret_cast<const double2 *>(x + o);
                const double2 qo = *reinterpret_cast<const double2 *>(q + o);
                const double x0 = xo.x + alpha_prev * qo.x, x1 = xo.y + alpha_prev * qo.y;
                *reinterpret_cast<double2 *>(x + o) = make_double2(x0 + alpha * cc.x, x1 + alpha * cc.y);
            }
            const double r0 = ro.x + malpha * a0, r1 = ro.y + malpha * a1;  // src/solver.py:155-157
            *reinterpret_cast<double2 *>(r + o) = make_double2(r0, r1);
            rr = rr + r0 * r0;
            rr = rr + r1 * r1;
            if (PK != PK_ZVEC) {
                rz = rz + r0 * zval<PK>(r0, jd, o, zc);
                rz = rz + r1 * zval<PK>(r1, jd, o + 1, zc);
            }
        }
        __device__ __forceinline__ void halo(long long, double2) {}
    } epi{r, x, jd, p_prev, sc->alpha, -sc->alpha, zc, sc->alpha_prev, 0.0, 0.0};
    if (c.row_ok) pair_march<ORDER, false>(c, g, off, diag, UpdSrc{p}, epi);
    double rr = block_sum<kPairThreads>(epi.rr, red);
    double rz = PK != PK_ZVEC ? block_sum<kPairThreads>(epi.rz, red) : 0.0;
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = rr;
        partials[2 * blockIdx.x + 1] = rz;
    }
    if (last_block(&tk->upd, &is_last)) {
        rr = reduce_partials<kPairThreads>(partials, gridDim.x, 2, red);
        if (PK != PK_ZVEC) rz = reduce_partials<kPairThreads>(partials + 1, gridDim.x, 2, red);
        if (threadIdx.x == 0) {
            if (red_out) {
                red_out[0] = rr;
                red_out[1] = rz;
            } else if (scalar_after_update<PK != PK_ZVEC>(sc, rr, rz) && use_cond) {
                cudaGraphSetConditional(cond, 0);
            }
        }
    }
}
