// cf_cg_spass.cuh -- the single-reduction CG iteration as ONE streaming pass
// fed by TMA (included by cf_cg.cu inside namespace cf, after cf_cg_pass.cuh
// for scalar_after_pass / cg_pass_init and cf_tma.cuh for the TMA helpers).
//
// Same recurrence as cg_pass_kernel (Chronopoulos-Gear, src/solver.py:128-171
// rearranged so one grid reduction per iteration suffices):
//   p_k     = z_k + beta_k p_{k-1}          (halo 2)
//   q       = A p_k                          (halo 1)
//   r_{k+1} = r_k - alpha_k q,  z' = M^-1 r_{k+1}   (halo 1)
//   w       = A z'                           (tile)  -> r.r, gamma = r.z', delta = z'.w
// with x updated every second pass, x_{k+1} = x_{k-1} + alpha_{k-1} p_{k-1} +
// alpha_k p_k (p_{k-1} is read anyway).  HBM per iteration: read r_k,
// p_{k-1}; write r_{k+1}, p_k; + x read/write every second pass = 40 N
// (the two-kernel form moves 60 N, the reference's op sequence 88 N).
//
// Layout for few instructions and one block barrier per plane:
//   * a CTA owns a 64 x TY tile and marches z; every plane of r_k and p_{k-1}
//     arrives as ONE 68 x (TY+4) box per vector (x0-2 .. x0+65, y0-2 ..
//     y0+TY+1) by TMA into an S-deep ring (a producer warp, full/empty
//     mbarriers); ghosts outside the domain are zero-filled by the TMA unit
//     (negative box origins work when the x origin is a 16-byte multiple:
//     tools/tma_selftest.cu variants 6-10), so p = 0 there with no mask;
//   * the stage is handed back to the producer as soon as the raw values are
//     in registers; p_k and z' go to two double-buffered plane buffers (the
//     ring sees TMA writes and generic reads only: no proxy fence per step);
//   * warp w owns box row w (TY+4 row warps), lane l the cell pair
//     x0+2l, x0+2l+1; the 2(TY+4) halo pairs at x0-2 and x0+64 belong to
//     edge warps, which form p there and carry q / z' for the halo cell;
//   * the stencils are split along z: A p at plane t collects its z-1 and
//     in-plane terms when plane t is formed and its z+1 term one step later,
//     so each thread keeps 5 pair registers (accumulators for q and w, the
//     previous p and z', the raw r) instead of 3-plane windows;
//   * step t: take stage t+2 (raw r, p_old, x) and release it; form p(t+2);
//     finish q(t+1) -> r', z'(t+1); finish w(t) -> dots; barrier; in-plane
//     terms of q(t+2) and of w(t+1).  A tile row's steady state (every plane
//     condition true) is a separate instantiation of the step.
//   * one CTA per SM walks (tile, z-chunk) items in lockstep with its
//     neighbours (SpGeom); each item's march has 4 planes of fill.
// The stencil sums follow the reference CSR column order (k-1, j-1, i-1, i,
// i+1, j+1, k+1; src/sparse.py:194-201) with fused multiply-adds: the
// single-reduction recurrence rounds differently from the reference anyway
// (parity: iterations within +-2, solution within 1e-8; tests/test_gpu_parity.py).

constexpr int kSpTX = 64;            // tile width (32 pairs)
constexpr int kSpBX = kSpTX + 4;     // box width: x0-2 .. x0+65

// FORM 1: one box row per warp, AoS plane buffers (the first form, kept for
// A/B); FORM 2: two box rows per warp (their shared y-neighbours stay in
// registers) and even / odd (SoA) plane buffers, so every x- and y-neighbour
// read is a conflict-free 8-byte LDS: 32 % fewer shared-memory wavefronts.
template <int TY, int S, int FORM = 2>
struct Sp {
    static_assert(TY % 4 == 0, "box bytes must stay 128-byte multiples");
    static constexpr int Rows = TY + 4;                       // box rows y0-2 .. y0+TY+1
    static constexpr int RowWarps = FORM == 2 ? Rows / 2 : Rows;
    static constexpr int EdgeWarps = FORM == 2 ? (Rows + 31) / 32 : (2 * Rows + 31) / 32;  // halo pairs
    static constexpr int CWarps = RowWarps + EdgeWarps;       // consumer warps
    static constexpr int Threads = 32 * (CWarps + 1);         // + the producer warp
    static constexpr int BoxD = Rows * kSpBX;                 // doubles per box
    static constexpr int XD = TY * kSpTX;                     // doubles per x box
    static constexpr uint32_t BoxBytes = BoxD * 8, XBytes = XD * 8;
    static constexpr int StageD = 2 * BoxD + XD;              // R | P | X (TMA writes only)
    // + two p planes and two z' planes (double-buffered, generic writes only)
    static constexpr size_t Smem = ((size_t)S * StageD + 4 * BoxD) * sizeof(double) + 128;
    // small tiles run two CTAs per SM (two independent lockstep groups)
    static constexpr int MinBlocks = (Threads <= 512 && FORM == 1) || Threads <= 256 ? 2 : 1;
};

// Work items (tile, z-chunk), chunk-major: item j = chunk j / T, tile j % T
// (T = ntx * nty).  CTA b takes items b, b + G, b + 2G, ... so the items in
// flight at any time are neighbouring tiles on the same chunk, marching in
// lockstep: the halo rows / columns a tile reads were fetched by its
// neighbours moments earlier and come from L2 (measured at 256^3: 128
// lockstep CTAs 157 us per iteration against 169 for 148 CTAs on equal
// contiguous (tile, plane) ranges, whose neighbours ran tens of planes apart).
// perm != null selects the phase-aligned contiguous schedule instead: the
// (tile position, plane) units are split into gridDim.x equal contiguous
// ranges (every SM busy, ranges may cross a tile boundary), and perm maps a
// position to a tile so that tiles adjacent in x share their phase and tiles
// adjacent in y are L / (tiles / distinct phases) planes apart -- a few
// planes, inside what L2 holds between neighbours (host: sp_phase_perm).
struct SpGeom {
    int nx, ny, nz, ntx, nty, nchunk;
    const int *perm;
    __host__ __device__ int items() const { return ntx * nty * nchunk; }
};

// This CTA's (tile, z0, z1) segments under either schedule.
struct SpSegs {
    const SpGeom &g;
    const int nblk;
    int j;              // item schedule: next item
    long long u, u1;    // contiguous schedule: next unit, end
    __device__ __forceinline__ SpSegs(const SpGeom &g_, int bid, int nblk_) : g(g_), nblk(nblk_), j(bid)
    {
        const long long units = (long long)g.ntx * g.nty * g.nz;
        u = units * bid / nblk;
        u1 = units * (bid + 1) / nblk;
    }
    __device__ __forceinline__ bool next(int &tile, int &za, int &zb)
    {
        if (!g.perm) {
            if (j >= g.items()) return false;
            const int t = g.ntx * g.nty;
            tile = j % t;
            const int chunk = j / t;
            za = g.nz * chunk / g.nchunk;
            zb = g.nz * (chunk + 1) / g.nchunk;
            j += nblk;
            return true;
        }
        if (u >= u1) return false;
        const long long pos = u / g.nz;
        za = (int)(u - pos * g.nz);
        zb = (int)min((long long)g.nz, za + (u1 - u));
        u += zb - za;
        tile = g.perm[pos];
        return true;
    }
};

// z-slab form (cf_p2p.cu): the slab's arrays hold 2 halo planes below and
// above its nz owned planes; a missing neighbour's halo stays zero (the
// Dirichlet ghost).  Boundary planes 0, 1 and nz-2, nz-1 of r_{k+1} and p_k
// are also stored straight into the neighbours' halo planes (peer memory).
struct SpSlabIO {
    int zoff;                // TMA plane coordinate of local plane 0 (2 in a slab array)
    int lo_ghost, hi_ghost;  // planes < 0 / >= nz are ghosts (no neighbour there)
    double *lo_r, *lo_p;     // the lower neighbour's planes matching our planes 0, 1 (null: none)
    double *hi_r, *hi_p;     // the upper neighbour's planes matching our planes nz-2, nz-1
};

__device__ __forceinline__ double2 sp_lds2(const double *p) { return *reinterpret_cast<const double2 *>(p); }
__device__ __forceinline__ void sp_sts2(double *p, double2 v) { *reinterpret_cast<double2 *>(p) = v; }
__device__ __forceinline__ void sp_stg2(double *p, double2 v) { *reinterpret_cast<double2 *>(p) = v; }
__device__ __forceinline__ void sp_bar(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }

template <int PK>
__device__ __forceinline__ double sp_z(double r, double zc) { return PK == PK_JCONST ? r * zc : r; }

// p = M^-1 r + beta p_old (src/precond.py:94, src/solver.py:169; p = z first, :142)
template <int PK, bool FIRST>
__device__ __forceinline__ double sp_form(double r, double po, double zc, double beta)
{
    const double z = sp_z<PK>(r, zc);
    return FIRST ? z : __fma_rn(beta, po, z);
}

// The producer: one lane streams the boxes of every step of this CTA's items
// through the ring (the consumers release a stage as soon as they have read it).
template <class G, int TY, int S, bool FIRST, bool XDBL>
__device__ __forceinline__ void sp_produce(const CUtensorMap *mr, const CUtensorMap *mp, const CUtensorMap *mx,
                                           const SpGeom &g, double *ring, uint64_t *full, uint64_t *empty,
                                           int bid, int nblk, int zoff)
{
    prefetch_map(mr);
    if (!FIRST) prefetch_map(mp);
    if (XDBL) prefetch_map(mx);
    int slot = 0;
    uint32_t phase = 0;
    bool wrapped = false;  // the ring has been filled once: wait for releases
    SpSegs segs(g, bid, nblk);
    int tile, za, zb;
    while (segs.next(tile, za, zb)) {
        const int x0 = (tile % g.ntx) * kSpTX, y0 = (tile / g.ntx) * TY;
        for (int s = 0; s < zb - za + 4; ++s) {
            if (wrapped) mbar_wait(&empty[slot], phase ^ 1u);
            const int zp = za - 2 + s + zoff;
            const bool xo = XDBL && zp - zoff >= za && zp - zoff < zb;
            double *st = ring + slot * G::StageD;
            mbar_expect_tx(&full[slot], (FIRST ? 1 : 2) * G::BoxBytes + (xo ? G::XBytes : 0));
            tma_load_3d(st, mr, x0 - 2, y0 - 2, zp, &full[slot]);
            if (!FIRST) tma_load_3d(st + G::BoxD, mp, x0 - 2, y0 - 2, zp, &full[slot]);
            if (xo) tma_load_3d(st + 2 * G::BoxD, mx, x0, y0, zp, &full[slot]);
            if (++slot == S) {
                slot = 0;
                phase ^= 1u;
                wrapped = true;
            }
        }
    }
}

// The march of one CTA (FORM 1).  Consumers return their partial rr / gamma / delta.
template <int PK, int TY, int S, bool FIRST, bool XDBL>
__device__ __forceinline__ void spass_body(const CUtensorMap *mr, const CUtensorMap *mp, const CUtensorMap *mx,
                                           const SpGeom &g, double off, double diag, double zc,
                                           double *__restrict__ r_out, double *__restrict__ p_new,
                                           double *__restrict__ x, double alpha, double alpha_prev, double beta,
                                           double *ring, uint64_t *full, uint64_t *empty, double &rr, double &gam,
                                           double &dlt)
{
    using G = Sp<TY, S, 1>;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long plane = (long long)g.nx * g.ny;
    const double malpha = -alpha;

    if (warp == G::CWarps) {  // ---------------- producer: one lane drives the ring
        if (lane == 0) sp_produce<G, TY, S, FIRST, XDBL>(mr, mp, mx, g, ring, full, empty, blockIdx.x, gridDim.x, 0);
        return;
    }

    // ---------------- consumers
    double *const PB = ring + S * G::StageD;  // p planes [2], then z' planes [2]
    double *const ZB = PB + 2 * G::BoxD;
    const bool edge = warp >= G::Rows;
    const int e = (warp - G::Rows) * 32 + lane;          // edge item
    const bool eact = edge && e < 2 * G::Rows;
    const int row = edge ? (eact ? e >> 1 : 0) : warp;
    const int side = e & 1;                               // edge: 0 = x0-2 pair, 1 = x0+64 pair
    const int col = edge ? (side ? kSpBX - 2 : 0) : 2 + 2 * lane;  // pair start column in the box
    const int o = row * kSpBX + col;
    const int oi = row * kSpBX + (side ? kSpBX - 2 : 1);  // edge: the halo cell next to the tile
    const int ox = 2 * G::BoxD + (row - 2) * kSpTX + 2 * lane;  // row warps: the pair in the x box
    const bool qrow = row >= 1 && row <= TY + 2;          // q / r' / z' rows (halo 1)
    const int nthr = 32 * G::CWarps;
    const unsigned pl = (unsigned)plane;
    // ring position, carried across segments (no 64-bit division in the loop)
    int slot = 0;
    uint32_t phase = 0;
    // take the staged raw values of this step, then hand the stage back to the
    // producer at once: p and z' live in their own plane buffers, so the ring
    // sees generic-proxy READS only (no proxy fence needed before the refill)
    auto take = [&](double2 &r2, double2 &po, double2 &xo, bool want_x) {
        mbar_wait(&full[slot], phase);
        const double *st = ring + slot * G::StageD;
        r2 = sp_lds2(st + o);
        po = make_double2(0.0, 0.0);
        if (!FIRST) po = sp_lds2(st + G::BoxD + o);
        xo = make_double2(0.0, 0.0);
        if (XDBL && want_x) xo = sp_lds2(st + ox);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == S) {
            slot = 0;
            phase ^= 1u;
        }
    };
    for (int j = blockIdx.x; j < g.items(); j += gridDim.x) {
        const int tile = j % (g.ntx * g.nty), chunk = j / (g.ntx * g.nty);
        const int za = g.nz * chunk / g.nchunk, zb = g.nz * (chunk + 1) / g.nchunk;
        const int x0 = (tile % g.ntx) * kSpTX, y0 = (tile / g.ntx) * TY;
        const int gy = y0 - 2 + row;
        const int gx = edge ? (side ? x0 + kSpTX : x0 - 1) : x0 + 2 * lane;  // edge: the halo cell
        const bool xyin = gy >= 0 && gy < g.ny && gx >= 0 && gx < g.nx;    // z' may be nonzero
        const bool irow = !edge && row >= 2 && row < TY + 2 && gy < g.ny;  // tile rows
        const bool own = irow && gx < g.nx;                                 // tile pairs
        const int L = zb - za, last = L + 3;
        // 32-bit flat offset of this pair on plane zp = za - 2 + s (wraps for
        // ghost rows / planes; used only when the cell is owned)
        unsigned gz = (unsigned)gx + (unsigned)g.nx * (unsigned)gy + pl * (unsigned)(za - 2);
        // per-pair state (edge warps use .x only): accumulators of q (plane
        // zp) and w (plane zq), previous p and z', raw r of the newest plane
        double2 aq = make_double2(0.0, 0.0), aw = aq, pc = aq, zl = aq, rw = aq;
        if (!edge) {
            // step s: p(zp), zp = za-2+s; q, r', z' of zq = zp-1; w of zq-1.
            // ST: the steady state of a tile row (every plane condition true)
            auto step = [&](auto steady, int s) {
                constexpr bool ST = decltype(steady)::value;
                const int zq = za - 3 + s;
                double2 r2, po, xo;
                take(r2, po, xo, own && s >= 2 && s <= L + 1);
                const double2 p2 = make_double2(sp_form<PK, FIRST>(r2.x, po.x, zc, beta),
                                                sp_form<PK, FIRST>(r2.y, po.y, zc, beta));
                double *const Pb = PB + (s & 1) * G::BoxD + o;
                double *const Zb = ZB + (s & 1) * G::BoxD + o;
                sp_sts2(Pb, p2);
                if (ST ? own : (own && s >= 2 && s <= L + 1)) {
                    sp_stg2(p_new + gz, p2);
                    if (XDBL)  // x = (x + alpha_prev p_{k-1}) + alpha p_k (src/solver.py:155, twice)
                        sp_stg2(x + gz, make_double2(__fma_rn(alpha, p2.x, __fma_rn(alpha_prev, po.x, xo.x)),
                                                     __fma_rn(alpha, p2.y, __fma_rn(alpha_prev, po.y, xo.y))));
                }
                // ---- q(zq) complete (its z+1 term), r_{k+1} and z' of plane zq
                if (ST || (qrow && s >= 1)) {
                    const double q0 = __fma_rn(off, p2.x, aq.x), q1 = __fma_rn(off, p2.y, aq.y);
                    const double r0 = __fma_rn(malpha, q0, rw.x), r1 = __fma_rn(malpha, q1, rw.y);  // :157
                    const bool zin = ST || (unsigned)zq < (unsigned)g.nz;
                    const double2 zn = xyin && zin ? make_double2(sp_z<PK>(r0, zc), sp_z<PK>(r1, zc))
                                                   : make_double2(0.0, 0.0);
                    sp_sts2(Zb, zn);
                    if (ST ? own : (own && s >= 3 && s <= L + 2)) {
                        sp_stg2(r_out + (gz - pl), make_double2(r0, r1));
                        rr = __fma_rn(r0, r0, rr);  // :158
                        rr = __fma_rn(r1, r1, rr);
                        gam = __fma_rn(r0, zn.x, gam);  // :163-164
                        gam = __fma_rn(r1, zn.y, gam);
                    }
                    // ---- w(zq-1) complete (its z+1 term): delta += z'.w
                    if (ST ? own : (own && s >= 4)) {
                        dlt = __fma_rn(zl.x, __fma_rn(off, zn.x, aw.x), dlt);
                        dlt = __fma_rn(zl.y, __fma_rn(off, zn.y, aw.y), dlt);
                    }
                    aw = zn;  // parked: z'(zq) for w's in-plane terms after the barrier
                }
                rw = r2;
                gz += pl;
                sp_bar(nthr);
                if (ST || qrow) {  // in-plane terms of q(zp) = A p(zp): k-1, j-1, i-1, i, i+1, j+1
                    const double2 ym = sp_lds2(Pb - kSpBX), yp = sp_lds2(Pb + kSpBX);
                    const double xl = Pb[-1], xr = Pb[2];
                    double a0 = off * pc.x, a1 = off * pc.y;
                    a0 = __fma_rn(off, ym.x, a0);
                    a1 = __fma_rn(off, ym.y, a1);
                    a0 = __fma_rn(off, xl, a0);
                    a1 = __fma_rn(off, p2.x, a1);
                    a0 = __fma_rn(diag, p2.x, a0);
                    a1 = __fma_rn(diag, p2.y, a1);
                    a0 = __fma_rn(off, p2.y, a0);
                    a1 = __fma_rn(off, xr, a1);
                    a0 = __fma_rn(off, yp.x, a0);
                    a1 = __fma_rn(off, yp.y, a1);
                    aq = make_double2(a0, a1);
                    pc = p2;
                }
                if (ST || (irow && s >= 1)) {  // in-plane terms of w(zq) = A z'(zq)
                    const double2 zc2 = aw;
                    const double2 ym = sp_lds2(Zb - kSpBX), yp = sp_lds2(Zb + kSpBX);
                    const double xl = Zb[-1], xr = Zb[2];
                    double a0 = off * zl.x, a1 = off * zl.y;
                    a0 = __fma_rn(off, ym.x, a0);
                    a1 = __fma_rn(off, ym.y, a1);
                    a0 = __fma_rn(off, xl, a0);
                    a1 = __fma_rn(off, zc2.x, a1);
                    a0 = __fma_rn(diag, zc2.x, a0);
                    a1 = __fma_rn(diag, zc2.y, a1);
                    a0 = __fma_rn(off, zc2.y, a0);
                    a1 = __fma_rn(off, xr, a1);
                    a0 = __fma_rn(off, yp.x, a0);
                    a1 = __fma_rn(off, yp.y, a1);
                    zl = zc2;
                    aw = make_double2(a0, a1);
                }
            };
            int s = 0;
            if (irow) {
                for (; s < 4 && s <= last; ++s) step(std::false_type{}, s);
                for (; s <= L + 1; ++s) step(std::true_type{}, s);
            }
            for (; s <= last; ++s) step(std::false_type{}, s);
        } else {
            // ---- edge warps: the halo pairs' p, and q / z' of the halo cell
            for (int s = 0; s <= last; ++s) {
                const int zq = za - 3 + s;
                double2 r2, po, xo;
                take(r2, po, xo, false);
                double *const Pb = PB + (s & 1) * G::BoxD;
                double *const Zb = ZB + (s & 1) * G::BoxD;
                double pin = 0.0;
                if (eact) {
                    const double2 p2 = make_double2(sp_form<PK, FIRST>(r2.x, po.x, zc, beta),
                                                    sp_form<PK, FIRST>(r2.y, po.y, zc, beta));
                    sp_sts2(Pb + o, p2);
                    pin = side ? p2.x : p2.y;
                    if (qrow && s >= 1) {
                        const double q0 = __fma_rn(off, pin, aq.x);
                        const double r0 = __fma_rn(malpha, q0, rw.x);
                        Zb[oi] = xyin && (unsigned)zq < (unsigned)g.nz ? sp_z<PK>(r0, zc) : 0.0;
                    }
                    rw.x = side ? r2.x : r2.y;
                }
                sp_bar(nthr);
                if (eact && qrow) {
                    double a0 = off * pc.x;
                    a0 = __fma_rn(off, Pb[oi - kSpBX], a0);
                    a0 = __fma_rn(off, Pb[oi - 1], a0);
                    a0 = __fma_rn(diag, pin, a0);
                    a0 = __fma_rn(off, Pb[oi + 1], a0);
                    a0 = __fma_rn(off, Pb[oi + kSpBX], a0);
                    aq.x = a0;
                    pc.x = pin;
                }
            }
        }
    }
}

// ---------------------------------------------------------------- FORM 2
constexpr int kSpPX = kSpBX / 2;  // 34 pairs per box row
__device__ __forceinline__ double sp_lds(const double *p) { return *p; }

// The march of one CTA (FORM 2: two box rows per row warp, SoA plane buffers).
// SLAB: the z-slab form (bid / nblk: this slab's block range, io: halo
// offsets, ghosts and the neighbours' planes); the single domain passes
// blockIdx.x / gridDim.x and {0, 1, 1, null...}.
template <int PK, int TY, int S, bool FIRST, bool XDBL, bool SLAB = false>
__device__ __forceinline__ void spass2_body(const CUtensorMap *mr, const CUtensorMap *mp, const CUtensorMap *mx,
                                            const SpGeom &g, double off, double diag, double zc,
                                            double *__restrict__ r_out, double *__restrict__ p_new,
                                            double *__restrict__ x, double alpha, double alpha_prev, double beta,
                                            double *ring, uint64_t *full, uint64_t *empty, double &rr, double &gam,
                                            double &dlt, int bid, int nblk, const SpSlabIO &io)
{
    using G = Sp<TY, S, 2>;
    constexpr int R = G::Rows, PL = R * kSpPX;  // one SoA plane: R rows x 34 pairs
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned pl = (unsigned)g.nx * (unsigned)g.ny;
    const double malpha = -alpha;
    if (warp == G::CWarps) {  // ---------------- producer
        if (lane == 0) sp_produce<G, TY, S, FIRST, XDBL>(mr, mp, mx, g, ring, full, empty, bid, nblk, io.zoff);
        return;
    }
    // z' vanishes on ghost planes only (a neighbour's halo plane is real data)
    auto zreal = [&](int zq) { return (zq >= 0 || !io.lo_ghost) && (zq < g.nz || !io.hi_ghost); };
    // boundary planes also into the neighbours' halo planes (SLAB)
    const unsigned top = (unsigned)g.nx * (unsigned)g.ny * (unsigned)(g.nz - 2);
    auto peer2 = [&](double *lo, double *hi, int z, unsigned o, double2 v) {
        if (!SLAB) return;
        if (lo && z < 2) sp_stg2(lo + o, v);
        if (hi && z >= g.nz - 2) sp_stg2(hi + (o - top), v);
    };

    // plane buffers [2 steps]: p even / odd cells, z' even / odd cells
    double *const pe = ring + S * G::StageD, *const po = pe + 2 * PL;
    double *const ze = po + 2 * PL, *const zo = ze + 2 * PL;
    const int nthr = 32 * G::CWarps;
    int slot = 0;
    uint32_t phase = 0;
    auto wait_stage = [&]() -> const double * {
        mbar_wait(&full[slot], phase);
        return ring + slot * G::StageD;
    };
    auto release_stage = [&]() {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == S) {
            slot = 0;
            phase ^= 1u;
        }
    };
    const bool edge = warp >= G::RowWarps;
    SpSegs segs(g, bid, nblk);
    int tile, za, zb;
    while (segs.next(tile, za, zb)) {
        const int x0 = (tile % g.ntx) * kSpTX, y0 = (tile / g.ntx) * TY;
        const int L = zb - za, last = L + 3;
        if (!edge) {
            // ---- row warp: box rows a = 2w, b = 2w + 1; lane l owns the pair x0+2l
            const int a = 2 * warp, b = a + 1;
            const int jp = lane + 1;                       // pair index in the box row
            const int ga = y0 - 2 + a, gx = x0 + 2 * lane;  // row b is ga + 1
            const bool xin = gx < g.nx;
            const bool qa = a >= 1 && a <= TY + 2, qb = b <= TY + 2;  // q / z' rows (b >= 1 always)
            const bool ia = a >= 2 && a < TY + 2 && ga < g.ny, ib = b >= 2 && b < TY + 2 && ga + 1 < g.ny;
            const bool inner = a >= 2 && b < TY + 2;      // both rows are tile rows (warp-uniform)
            const bool oa = ia && xin, ob = ib && xin;     // owned pairs
            const bool za_ok = ga >= 0 && ga < g.ny && xin, zb_ok = ga + 1 >= 0 && ga + 1 < g.ny && xin;
            const int sa = a * kSpBX + 2 + 2 * lane;      // stage offset of row a's pair (row b: + kSpBX)
            const int xa = 2 * G::BoxD + (a - 2) * kSpTX + 2 * lane;  // x box offset (row b: + kSpTX)
            const int ea = a * kSpPX + jp, eb = ea + kSpPX;  // SoA plane index of the pair
            unsigned gz = (unsigned)gx + (unsigned)g.nx * (unsigned)ga + pl * (unsigned)(za - 2);
            double2 aqa = make_double2(0.0, 0.0), aqb = aqa, awa = aqa, awb = aqa, pca = aqa, pcb = aqa;
            double2 zla = aqa, zlb = aqa, rwa = aqa, rwb = aqa;
            // raw r_k / p_{k-1} (/ x) of the NEXT plane: taken right after the barrier,
            // so the stage wait and its loads overlap the in-plane arithmetic
            double2 nra, nrb, npoa = aqa, npob = aqa, nxoa = aqa, nxob = aqa;
            auto take2 = [&](int s) {
                const double *st = wait_stage();
                nra = sp_lds2(st + sa);
                nrb = sp_lds2(st + sa + kSpBX);
                if (!FIRST) {
                    npoa = sp_lds2(st + G::BoxD + sa);
                    npob = sp_lds2(st + G::BoxD + sa + kSpBX);
                }
                if (XDBL && inner && s >= 2 && s <= L + 1) {
                    nxoa = sp_lds2(st + xa);
                    nxob = sp_lds2(st + xa + kSpTX);
                }
                release_stage();
            };
            auto step = [&](auto steady, int s) {
                constexpr bool ST = decltype(steady)::value;
                const int zq = za - 3 + s;
                // this plane's raw values were taken at the end of the previous step
                const double2 ra = nra, rb = nrb, poa = npoa, pob = npob, xoa = nxoa, xob = nxob;
                const bool stp = ST || (s >= 2 && s <= L + 1);  // p / x of this plane are stored
                const double2 pa = make_double2(sp_form<PK, FIRST>(ra.x, poa.x, zc, beta),
                                                sp_form<PK, FIRST>(ra.y, poa.y, zc, beta));
                const double2 pb = make_double2(sp_form<PK, FIRST>(rb.x, pob.x, zc, beta),
                                                sp_form<PK, FIRST>(rb.y, pob.y, zc, beta));
                const int bo = (s & 1) * PL;
                pe[bo + ea] = pa.x;
                po[bo + ea] = pa.y;
                pe[bo + eb] = pb.x;
                po[bo + eb] = pb.y;
                if (stp) {
                    const int zp = za - 2 + s;
                    if (oa) {
                        sp_stg2(p_new + gz, pa);
                        peer2(io.lo_p, io.hi_p, zp, gz, pa);
                    }
                    if (ob) {
                        sp_stg2(p_new + gz + g.nx, pb);
                        peer2(io.lo_p, io.hi_p, zp, gz + g.nx, pb);
                    }
                    if (XDBL) {  // x = (x + alpha_prev p_{k-1}) + alpha p_k (src/solver.py:155, twice)
                        if (oa)
                            sp_stg2(x + gz, make_double2(__fma_rn(alpha, pa.x, __fma_rn(alpha_prev, poa.x, xoa.x)),
                                                         __fma_rn(alpha, pa.y, __fma_rn(alpha_prev, poa.y, xoa.y))));
                        if (ob)
                            sp_stg2(x + gz + g.nx,
                                    make_double2(__fma_rn(alpha, pb.x, __fma_rn(alpha_prev, pob.x, xob.x)),
                                                 __fma_rn(alpha, pb.y, __fma_rn(alpha_prev, pob.y, xob.y))));
                    }
                }
                // ---- q(zq) complete, r_{k+1}, z' (+ r.r, gamma); w(zq-1) complete (+ delta)
                const bool zin = ST || zreal(zq);
                const bool str = ST || (s >= 3 && s <= L + 2), std_ = ST || s >= 4;
                auto finish = [&](const double2 &p2, const double2 &aq, const double2 &rw, const double2 &aw,
                                  const double2 &zl, bool zok, bool own, unsigned o, int e, double2 &zpark) {
                    const double q0 = __fma_rn(off, p2.x, aq.x), q1 = __fma_rn(off, p2.y, aq.y);
                    const double r0 = __fma_rn(malpha, q0, rw.x), r1 = __fma_rn(malpha, q1, rw.y);  // :157
                    const double2 zn = zok && zin ? make_double2(sp_z<PK>(r0, zc), sp_z<PK>(r1, zc))
                                                  : make_double2(0.0, 0.0);
                    ze[bo + e] = zn.x;
                    zo[bo + e] = zn.y;
                    if (own && str) {
                        sp_stg2(r_out + o, make_double2(r0, r1));
                        peer2(io.lo_r, io.hi_r, zq, o, make_double2(r0, r1));
                        rr = __fma_rn(r0, r0, rr);  // :158
                        rr = __fma_rn(r1, r1, rr);
                        gam = __fma_rn(r0, zn.x, gam);  // :163-164
                        gam = __fma_rn(r1, zn.y, gam);
                    }
                    if (own && std_) {
                        dlt = __fma_rn(zl.x, __fma_rn(off, zn.x, aw.x), dlt);
                        dlt = __fma_rn(zl.y, __fma_rn(off, zn.y, aw.y), dlt);
                    }
                    zpark = zn;
                };
                double2 zna = make_double2(0.0, 0.0), znb = zna;
                if (ST || s >= 1) {
                    if (ST || qa) finish(pa, aqa, rwa, awa, zla, za_ok, oa, gz - pl, ea, zna);
                    if (ST || qb) finish(pb, aqb, rwb, awb, zlb, zb_ok, ob, gz - pl + g.nx, eb, znb);
                }
                rwa = ra;
                rwb = rb;
                gz += pl;
                sp_bar(nthr);
                if (s < last) take2(s + 1);
                // ---- in-plane terms (k-1, j-1, i-1, i, i+1, j+1) of q(zp) and w(zq)
                const double *Pe = pe + bo, *Po = po + bo, *Ze = ze + bo, *Zo = zo + bo;
                auto inplane = [&](const double2 &c, const double2 &zm, const double2 &ym, const double2 &yp,
                                   double xl, double xr) {
                    double a0 = off * zm.x, a1 = off * zm.y;
                    a0 = __fma_rn(off, ym.x, a0);
                    a1 = __fma_rn(off, ym.y, a1);
                    a0 = __fma_rn(off, xl, a0);
                    a1 = __fma_rn(off, c.x, a1);
                    a0 = __fma_rn(diag, c.x, a0);
                    a1 = __fma_rn(diag, c.y, a1);
                    a0 = __fma_rn(off, c.y, a0);
                    a1 = __fma_rn(off, xr, a1);
                    a0 = __fma_rn(off, yp.x, a0);
                    a1 = __fma_rn(off, yp.y, a1);
                    return make_double2(a0, a1);
                };
                if (ST || qa) {
                    const double2 ym = make_double2(sp_lds(Pe + ea - kSpPX), sp_lds(Po + ea - kSpPX));
                    aqa = inplane(pa, pca, ym, pb, sp_lds(Po + ea - 1), sp_lds(Pe + ea + 1));
                }
                if (ST || qb) {
                    const double2 yp = make_double2(sp_lds(Pe + eb + kSpPX), sp_lds(Po + eb + kSpPX));
                    aqb = inplane(pb, pcb, pa, yp, sp_lds(Po + eb - 1), sp_lds(Pe + eb + 1));
                }
                pca = pa;
                pcb = pb;
                if (ST || (inner && s >= 1)) {
                    const double2 ym = make_double2(sp_lds(Ze + ea - kSpPX), sp_lds(Zo + ea - kSpPX));
                    const double2 yp = make_double2(sp_lds(Ze + eb + kSpPX), sp_lds(Zo + eb + kSpPX));
                    awa = inplane(zna, zla, ym, znb, sp_lds(Zo + ea - 1), sp_lds(Ze + ea + 1));
                    awb = inplane(znb, zlb, zna, yp, sp_lds(Zo + eb - 1), sp_lds(Ze + eb + 1));
                    zla = zna;
                    zlb = znb;
                }
            };
            take2(0);
            int s = 0;
            if (inner) {
                for (; s < 4 && s <= last; ++s) step(std::false_type{}, s);
                for (; s <= L + 1; ++s) step(std::true_type{}, s);
            }
            for (; s <= last; ++s) step(std::false_type{}, s);
        } else {
            // ---- edge warp: lane = box row; the halo pairs x0-2 (left) and x0+64
            // (right), q / z' of their inner cells x0-1 and x0+64
            const int e = (warp - G::RowWarps) * 32 + lane;
            const bool act = e < R;
            const int row = act ? e : 0;
            const int gy = y0 - 2 + row;
            const bool yin = gy >= 0 && gy < g.ny;
            const bool zl_ok = yin && x0 - 1 >= 0, zr_ok = yin && x0 + kSpTX < g.nx;
            const bool q = act && row >= 1 && row <= TY + 2;
            const int so = row * kSpBX, ei = row * kSpPX;  // stage / SoA offsets of the row
            double aqL = 0.0, aqR = 0.0, pcL = 0.0, pcR = 0.0, rwL = 0.0, rwR = 0.0;
            double2 nrL = make_double2(0.0, 0.0), nrR = nrL, noL = nrL, noR = nrL;
            auto take_e = [&]() {  // the next plane's raw halo pairs (see take2)
                const double *st = wait_stage();
                if (act) {
                    nrL = sp_lds2(st + so);
                    nrR = sp_lds2(st + so + kSpBX - 2);
                    if (!FIRST) {
                        noL = sp_lds2(st + G::BoxD + so);
                        noR = sp_lds2(st + G::BoxD + so + kSpBX - 2);
                    }
                }
                release_stage();
            };
            take_e();
            for (int s = 0; s <= last; ++s) {
                const int zq = za - 3 + s;
                const double2 rL = nrL, rR = nrR, oL = noL, oR = noR;
                const int bo = (s & 1) * PL;
                const double2 pL = make_double2(sp_form<PK, FIRST>(rL.x, oL.x, zc, beta),
                                                sp_form<PK, FIRST>(rL.y, oL.y, zc, beta));
                const double2 pR = make_double2(sp_form<PK, FIRST>(rR.x, oR.x, zc, beta),
                                                sp_form<PK, FIRST>(rR.y, oR.y, zc, beta));
                if (act) {
                    pe[bo + ei] = pL.x;
                    po[bo + ei] = pL.y;
                    pe[bo + ei + kSpPX - 1] = pR.x;
                    po[bo + ei + kSpPX - 1] = pR.y;
                }
                if (q && s >= 1) {
                    const bool zin = zreal(zq);
                    const double rl = __fma_rn(malpha, __fma_rn(off, pL.y, aqL), rwL);
                    const double rr_ = __fma_rn(malpha, __fma_rn(off, pR.x, aqR), rwR);
                    zo[bo + ei] = zl_ok && zin ? sp_z<PK>(rl, zc) : 0.0;
                    ze[bo + ei + kSpPX - 1] = zr_ok && zin ? sp_z<PK>(rr_, zc) : 0.0;
                }
                rwL = rL.y;
                rwR = rR.x;
                sp_bar(nthr);
                if (s < last) take_e();
                if (q) {
                    const double *Pe = pe + bo, *Po = po + bo;
                    double a0 = off * pcL;  // x0-1: k-1, j-1, i-1 (own), i, i+1 (row warp), j+1
                    a0 = __fma_rn(off, sp_lds(Po + ei - kSpPX), a0);
                    a0 = __fma_rn(off, pL.x, a0);
                    a0 = __fma_rn(diag, pL.y, a0);
                    a0 = __fma_rn(off, sp_lds(Pe + ei + 1), a0);
                    a0 = __fma_rn(off, sp_lds(Po + ei + kSpPX), a0);
                    aqL = a0;
                    const int er = ei + kSpPX - 1;
                    double a1 = off * pcR;  // x0+64: i-1 (row warp), i, i+1 (own)
                    a1 = __fma_rn(off, sp_lds(Pe + er - kSpPX), a1);
                    a1 = __fma_rn(off, sp_lds(Po + er - 1), a1);
                    a1 = __fma_rn(diag, pR.x, a1);
                    a1 = __fma_rn(off, pR.y, a1);
                    a1 = __fma_rn(off, sp_lds(Pe + er + kSpPX), a1);
                    aqR = a1;
                }
                pcL = pL.y;
                pcR = pR.x;
            }
        }
    }
}

template <int PK, int TY, int S, bool XDBL, int FORM = 2>
__global__ void __launch_bounds__(Sp<TY, S, FORM>::Threads, Sp<TY, S, FORM>::MinBlocks)
    cg_spass_kernel(const __grid_constant__ CUtensorMap mr, const __grid_constant__ CUtensorMap mp,
                    const __grid_constant__ CUtensorMap mx, SpGeom g, double off, double diag, double zc,
                    double *__restrict__ r_out, double *__restrict__ p_new, double *__restrict__ x, CgScalars *sc,
                    double *partials, CgTickets *tk, int use_cond, cudaGraphConditionalHandle cond)
{
    using G = Sp<TY, S, FORM>;
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[S], empty[S];
    __shared__ double red[96];
    __shared__ int is_last;
    if (sc->done) {
        if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    double *const ring = aligned_smem(smem_raw);
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], G::CWarps);
        }
        fence_barrier_init();
    }
    __syncthreads();
    double rr = 0.0, gam = 0.0, dlt = 0.0;
    const double alpha = sc->alpha, alpha_prev = sc->alpha_prev, beta = sc->beta;
    if (FORM == 1) {
        if (!XDBL && sc->it == 0)
            spass_body<PK, TY, S, true, false>(&mr, &mp, &mx, g, off, diag, zc, r_out, p_new, x, alpha, alpha_prev,
                                               0.0, ring, full, empty, rr, gam, dlt);
        else
            spass_body<PK, TY, S, false, XDBL>(&mr, &mp, &mx, g, off, diag, zc, r_out, p_new, x, alpha, alpha_prev,
                                               beta, ring, full, empty, rr, gam, dlt);
    } else {
        const SpSlabIO io{0, 1, 1, nullptr, nullptr, nullptr, nullptr};
        if (!XDBL && sc->it == 0)
            spass2_body<PK, TY, S, true, false>(&mr, &mp, &mx, g, off, diag, zc, r_out, p_new, x, alpha, alpha_prev,
                                                0.0, ring, full, empty, rr, gam, dlt, blockIdx.x, gridDim.x, io);
        else
            spass2_body<PK, TY, S, false, XDBL>(&mr, &mp, &mx, g, off, diag, zc, r_out, p_new, x, alpha, alpha_prev,
                                                beta, ring, full, empty, rr, gam, dlt, blockIdx.x, gridDim.x, io);
    }
    block_sum3<G::Threads>(rr, gam, dlt, red);
    if (threadIdx.x == 0) {
        partials[3 * blockIdx.x] = rr;
        partials[3 * blockIdx.x + 1] = gam;
        partials[3 * blockIdx.x + 2] = dlt;
    }
    if (last_block(&tk->upd, &is_last) && threadIdx.x < 32) {
        warp_reduce_partials3(partials, gridDim.x, rr, gam, dlt);
        if (threadIdx.x == 0) {
            scalar_after_pass(sc, rr, gam, dlt);
            if (sc->done && use_cond) cudaGraphSetConditional(cond, 0);
        }
    }
}
