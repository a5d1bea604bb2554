// cf_cg_persist.cuh -- the whole CG solve in ONE persistent launch for grids
// whose vectors stay in L2 (included by cf_cg.cu inside namespace cf, after
// cf_cg_lean.cuh).
//
// At L2-resident sizes (BASELINE config 2, 128^3: 4 x 16.8 MB) the two-kernel
// loop is launch- and tail-bound: ~33 us per iteration for ~8 us of L2
// traffic.  Here every CTA stays resident for the whole solve and walks a
// fixed set of lean-march tiles (the direction march, then the update march
// with x updated every iteration), separated by grid-wide barriers:
//   direction -> partial p.Ap -> barrier -> every CTA sums all partials in
//   block order (the same value everywhere) -> alpha -> update -> partial
//   r.r, r.z -> barrier -> sums -> stop test, beta -> next iteration.
// The vectors are rewritten inside the launch, so the marches read through L2
// (.cg, COH) instead of the read-only path.  Same per-element arithmetic as
// the two-kernel form; only the dot products' partition differs.

constexpr int kPersistRows = 8;
constexpr int kPersistThreads = 32 * kPersistRows;

struct GridBar {
    unsigned int count, gen;
};

// All CTAs of the launch are co-resident (grid <= resident slots, checked on
// the host), so a counter + generation barrier cannot deadlock.
__device__ __forceinline__ void grid_barrier(GridBar *gb, unsigned int nblk)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int *vgen = &gb->gen;
        const unsigned int g = *vgen;
        __threadfence();  // this CTA's stores before its arrival
        if (atomicAdd(&gb->count, 1u) == nblk - 1) {
            gb->count = 0u;
            __threadfence();
            atomicExch(&gb->gen, g + 1u);
        } else {
            while (*vgen == g) __nanosleep(32);
        }
        __threadfence();  // everyone's stores before this CTA's later loads
    }
    __syncthreads();
}

// Fixed-order sum of `count` partials (stride `stride`), broadcast to every
// thread of the block.
__device__ __forceinline__ double persist_sum(const double *p, int count, int stride, double *red, double *bcast)
{
    double v = 0.0;
    for (int i = threadIdx.x; i < count; i += kPersistThreads) v += __ldcg(p + (size_t)i * stride);
    v = block_sum<kPersistThreads>(v, red);
    if (threadIdx.x == 0) *bcast = v;
    __syncthreads();
    v = *bcast;
    __syncthreads();
    return v;
}

template <int ORDER, int PK>
__global__ void __launch_bounds__(kPersistThreads, 4) cg_persist_kernel(PairGeom g, double off, double diag,
                                                                       double zc, double *__restrict__ r,
                                                                       double *__restrict__ x, double *p0, double *p1,
                                                                       CgScalars *sc, double *part_dir,
                                                                       double *part_upd, GridBar *gb)
{
    __shared__ double red[32];
    __shared__ double bcast;
    const unsigned int nblk = gridDim.x;
    const int nunits = g.ctas();
    CgScalars s = *sc;  // norm_b, rz, tol, max_iter from the init kernel / host
    int half = 0;
    while (!s.done) {
        const double *p_old = half ? p1 : p0;
        double *p_new = half ? p0 : p1;
        // ---- direction: p = z + beta p_old, partial p.Ap (src/solver.py:142-153)
        double pap = 0.0;
        for (int u = blockIdx.x; u < nunits; u += nblk)
            pap += s.it == 0
                       ? dir_lean_march<ORDER, PK, true, 0, kPersistRows, false, true>(g, u, off, diag, r, p_old,
                                                                                      p_new, zc, 0.0)
                       : dir_lean_march<ORDER, PK, false, 0, kPersistRows, false, true>(g, u, off, diag, r, p_old,
                                                                                       p_new, zc, s.beta);
        pap = block_sum<kPersistThreads>(pap, red);
        if (threadIdx.x == 0) part_dir[blockIdx.x] = pap;
        grid_barrier(gb, nblk);
        pap = persist_sum(part_dir, nblk, 1, red, &bcast);
        scalar_after_dir(&s, pap);
        if (s.done) break;  // breakdown (every CTA saw the same sum)
        // ---- update: r -= alpha A p, x += alpha p, partial r.r and r.z (:155-166)
        double rr = 0.0, rz = 0.0;
        for (int u = blockIdx.x; u < nunits; u += nblk)
            upd_lean_march<ORDER, PK, XM_EACH, kPersistRows, true>(g, u, off, diag, p_new, nullptr, r, x, zc, s.alpha,
                                                                   0.0, rr, rz);
        rr = block_sum<kPersistThreads>(rr, red);
        rz = block_sum<kPersistThreads>(rz, red);
        if (threadIdx.x == 0) {
            part_upd[2 * blockIdx.x] = rr;
            part_upd[2 * blockIdx.x + 1] = rz;
        }
        grid_barrier(gb, nblk);
        rr = persist_sum(part_upd, nblk, 2, red, &bcast);
        rz = persist_sum(part_upd + 1, nblk, 2, red, &bcast);
        scalar_after_update<true>(&s, rr, rz);
        half ^= 1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *sc = s;
}
