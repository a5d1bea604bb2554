// cf_dic.cuh -- level-scheduled simplified-DIC preconditioner
// (src/precond.py:24-54).  The reference's recurrence and sweeps are
// sequential by row; a row only depends on rows of its strictly lower
// (forward) or upper (backward) pattern, so rows are grouped into levels of
// equal dependency depth (for the 7-point operator: hyperplanes i+j+k =
// const, 3n-2 levels) and each level is one data-parallel launch.  Every row
// performs the reference's operations in the reference's operand order, so
// the factor and the applied preconditioner are bit-identical.
#pragma once

#include <vector>

#include "cf_common.cuh"

namespace cf {

// Tiled-wavefront form of the sweeps (cf_dic_wave.cu): structured 7-point
// pattern with one lower and one upper value, verified at attach time.
struct DicWave {
    int nx = 0, ny = 0, nz = 0, ntx = 0, nty = 0;
    double lval = 0.0, uval = 0.0;
    int slack = 1;                             // extra steps kept between neighbouring tiles
    int pub = 8;                               // steps per published progress value
    int shape = 0;                             // tile shape (cf_dic_wave.cu kShapes)
    int depth = 0;                             // cp.async pipeline depth of the 16x8 sweeps (0: one-step prefetch)
    int *prog_f = nullptr, *prog_b = nullptr;  // per-tile progress of the two sweeps
    int *ticket = nullptr;                     // [2] CTA tickets of the two sweeps (tile order)
    long long prog_cap = 0, ex_cap = 0, ey_cap = 0;  // allocated ints / doubles (re-sized per setup)
    // edge mailboxes of the pipelined 16x8 sweeps: a tile's boundary values
    // for its neighbour, [tile][k][lane], armed with kEdgeEmpty; the reader
    // spins on the value itself and re-arms it (cf_dic_wave.cu)
    double *ex_f = nullptr, *ey_f = nullptr, *ex_b = nullptr, *ey_b = nullptr;
    bool ok = false;
};

// Skewed-warp form of the sweeps (cf_dic_skew.cu): a warp owns a 32 x J tile
// column, lane l the cells x0 + l, and walks it with a skew of one step per
// lane, so every in-tile dependency is a register (y, z) or a shuffle (x).
struct DicSkew {
    int J = 0, logJ = 0;                 // tile rows (power of two)
    int ntx = 0, nty = 0, nz = 0;        // tiles in x / y, planes
    int nrows = 0;                       // steps per tile (padded to whole blocks)
    int trows = 0;                       // rows per tile of the skewed arrays (nrows + padding on both sides)
    int grid = 0;                        // CTAs launched (tickets -> tiles)
    double *buf = nullptr;               // the allocation behind dy and wsk
    double *dy = nullptr;                // (d~, its refined reciprocal) pairs: [tile][row][lane]
    double *wsk = nullptr;               // w: [tile][row][lane]
    // face mailboxes of the two sweeps: x [tile][q], y [tile][k][lane]
    double *mx_f = nullptr, *my_f = nullptr, *mx_b = nullptr, *my_b = nullptr;
    long long sk_cap = 0, mx_cap = 0, my_cap = 0;  // allocated doubles (re-sized per setup)
    double gf = 0.0, gb = 0.0;           // ghost values: L * gf = +0, U * gb = -0 (exact no-ops in the sums)
    bool ok = false;
};

struct DicData {
    long long n = 0;
    const int32_t *lp = nullptr, *lc = nullptr;  // strict lower triangle (CSR)
    const double *lv = nullptr;
    const int32_t *up = nullptr, *uc = nullptr;  // strict upper triangle (CSR)
    const double *uv = nullptr;
    const double *d = nullptr;                   // modified diagonal
    const int32_t *rows = nullptr;               // rows sorted by level
    std::vector<long long> level_ptr;            // host: level l = rows[level_ptr[l]:level_ptr[l+1]]
    DicWave wave;                                // used instead of the levels when wave.ok
    DicSkew skew;                                // used instead of the tiled wavefront when skew.ok
};

// z = M^-1 r through w; if `done` is non-null every launch exits when *done
// is set (used inside the CG graph once the solve has stopped).
int dic_apply_launch(const DicData &dd, const double *r, double *w, double *z, const int *done,
                     cudaStream_t s);

// Enable the wavefront sweeps for an nx*ny*nz grid if the triangles match
// (dd.wave.ok tells); and apply them.  cf_dic_wave.cu.
int dic_wave_setup(DicData &dd, int nx, int ny, int nz, cudaStream_t s);
int dic_wave_apply(const DicData &dd, const double *r, double *w, double *z, const int *done, cudaStream_t s);

// Skewed-warp sweeps (cf_dic_skew.cu): set up after dic_wave_setup verified
// the pattern (uses wave.lval / uval / ticket); apply = both sweeps.
int dic_skew_setup(DicData &dd, cudaStream_t s);
int dic_skew_apply(const DicData &dd, const double *r, double *z, const int *done, cudaStream_t s);
void dic_skew_free(DicSkew &sk);

}  // namespace cf
