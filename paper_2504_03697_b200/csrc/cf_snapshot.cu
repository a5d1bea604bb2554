// cf_snapshot.cu -- the snapshot path.
//
// Reference: src/snapshots.py:46-62 (cell-centred view), :65-70 (shortest
// round-trip decimal with the integral ".0" dropped), :82-108 (CSV writer,
// serial and buffered_parallel modes produce the same bytes).
//
// Device side: one pass over the staggered fields writes the cell-centred
// face averages and p as four contiguous i-fastest columns, so a snapshot
// costs one 4N-double D2H instead of three strided face copies and a host
// numpy averaging pass.  Host side: a native, multi-threaded CSV writer whose
// per-value formatting is Python's repr(float) (the reference's formatter),
// built on std::to_chars' shortest round-trip digits; row blocks are
// formatted in parallel and written in row order, so the bytes do not depend
// on the thread count.
#include <algorithm>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "cf_common.cuh"

namespace cf {

// ---------------------------------------------------------------- device

// out = [uc | vc | wc | p], each nx*ny*nz, cell index i + nx*(j + ny*k).
// Face component c is physical [k][j][i] with row pitch ld_c (elements);
// the average is 0.5 * (lo + hi) in that order (src/snapshots.py:53-55).
__global__ void snapshot_cells_kernel(const double *__restrict__ u, const double *__restrict__ v,
                                      const double *__restrict__ w, const double *__restrict__ p, int nx, int ny,
                                      int nz, int ldu, int ldv, int ldw, double *__restrict__ out)
{
    const long long ncell = (long long)nx * ny * nz;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += stride) {
        const int i = (int)(c % nx);
        const long long jk = c / nx;
        const int j = (int)(jk % ny);
        const int k = (int)(jk / ny);
        const long long ru = ((long long)k * ny + j) * ldu + i;
        const long long rv = ((long long)k * (ny + 1) + j) * ldv + i;
        const long long rw = ((long long)k * ny + j) * ldw + i;
        out[c] = 0.5 * (u[ru] + u[ru + 1]);
        out[ncell + c] = 0.5 * (v[rv] + v[rv + ldv]);
        out[2 * ncell + c] = 0.5 * (w[rw] + w[rw + (long long)ldw * ny]);
        out[3 * ncell + c] = p[c];
    }
}

// ---------------------------------------------------------------- host

namespace csv {

// repr(float(v)) with a trailing ".0" removed (src/snapshots.py:65-70).
// CPython's 'r' formatting: shortest round-trip digits d1..dk with the
// decimal point after position `decpt`; exponent notation when
// decpt <= -4 or decpt > 16, exponent signed and at least two digits.
// `o` needs 32 bytes; returns the length.
int format_double(double v, char *o)
{
    char *p = o;
    if (std::isnan(v)) {
        std::memcpy(p, "nan", 3);
        return 3;
    }
    if (std::signbit(v)) {
        *p++ = '-';
        v = -v;
    }
    if (std::isinf(v)) {
        std::memcpy(p, "inf", 3);
        return (int)(p - o) + 3;
    }
    if (v == 0.0) {
        *p++ = '0';
        return (int)(p - o);
    }
    char sci[40];
    char *end = std::to_chars(sci, sci + sizeof sci, v, std::chars_format::scientific).ptr;
    char dig[24];
    int nd = 0;
    const char *q = sci;
    for (; q < end && *q != 'e'; ++q)
        if (*q != '.') dig[nd++] = *q;
    int e10 = 0;
    std::from_chars(q + 1 + (q[1] == '+'), end, e10);
    const int decpt = e10 + 1;
    if (decpt <= -4 || decpt > 16) {
        *p++ = dig[0];
        if (nd > 1) {
            *p++ = '.';
            std::memcpy(p, dig + 1, nd - 1);
            p += nd - 1;
        }
        *p++ = 'e';
        int x = decpt - 1;
        *p++ = x < 0 ? '-' : '+';
        x = x < 0 ? -x : x;
        if (x >= 100) *p++ = char('0' + x / 100);
        *p++ = char('0' + (x / 10) % 10);
        *p++ = char('0' + x % 10);
    } else if (decpt <= 0) {
        *p++ = '0';
        *p++ = '.';
        for (int z = 0; z < -decpt; ++z) *p++ = '0';
        std::memcpy(p, dig, nd);
        p += nd;
    } else if (decpt >= nd) {  // integral: digits, zeros, and no ".0"
        std::memcpy(p, dig, nd);
        p += nd;
        for (int z = nd; z < decpt; ++z) *p++ = '0';
    } else {
        std::memcpy(p, dig, decpt);
        p += decpt;
        *p++ = '.';
        std::memcpy(p, dig + decpt, nd - decpt);
        p += nd - decpt;
    }
    return (int)(p - o);
}

constexpr long long kBlockRows = 1 << 15;
constexpr const char *kHeader = "x,y,z,u,v,w,p\n";

// Rows [r0, r1) of `row(r, vals[7])` appended to `out`.
template <class Row>
void format_rows(const Row &row, long long r0, long long r1, std::string &out)
{
    out.clear();
    out.reserve((size_t)(r1 - r0) * 7 * 24);
    char buf[32];
    double vals[7];
    for (long long r = r0; r < r1; ++r) {
        row(r, vals);
        for (int c = 0; c < 7; ++c) {
            out.append(buf, format_double(vals[c], buf));
            out.push_back(c == 6 ? '\n' : ',');
        }
    }
}

// Header + rows, formatted by `threads` workers in waves of row blocks and
// written in row order.
template <class Row>
int write_csv(const char *path, const Row &row, long long nrows, int threads)
{
    FILE *f = std::fopen(path, "wb");
    if (!f) {
        set_error(std::string("cannot open ") + path + ": " + std::strerror(errno));
        return CF_EIO;
    }
    int t = std::max(1, threads);
    std::vector<std::string> bufs(t);
    bool ok = std::fwrite(kHeader, 1, std::strlen(kHeader), f) == std::strlen(kHeader);
    const long long nblocks = (nrows + kBlockRows - 1) / kBlockRows;
    for (long long b0 = 0; ok && b0 < nblocks; b0 += t) {
        const int nb = (int)std::min<long long>(t, nblocks - b0);
        auto job = [&](int s) {
            long long r0 = (b0 + s) * kBlockRows;
            format_rows(row, r0, std::min(nrows, r0 + kBlockRows), bufs[s]);
        };
        if (nb == 1) {
            job(0);
        } else {
            std::vector<std::thread> pool;
            for (int s = 1; s < nb; ++s) pool.emplace_back(job, s);
            job(0);
            for (auto &th : pool) th.join();
        }
        for (int s = 0; ok && s < nb; ++s) ok = std::fwrite(bufs[s].data(), 1, bufs[s].size(), f) == bufs[s].size();
    }
    if (std::fclose(f) != 0) ok = false;
    if (!ok) {
        set_error(std::string("write failed: ") + path + ": " + std::strerror(errno));
        return CF_EIO;
    }
    return CF_OK;
}

}  // namespace csv
}  // namespace cf

extern "C" {

int cf_snapshot_cells(const double *u, const double *v, const double *w, const double *p, int nx, int ny, int nz,
                      int ldu, int ldv, int ldw, double *out, void *stream)
{
    CF_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1 && ldu >= nx + 1 && ldv >= nx && ldw >= nx && u && v && w && p && out,
               "cf_snapshot_cells: bad arguments");
    long long ncell = (long long)nx * ny * nz;
    int threads = 256;
    long long want = (ncell + threads - 1) / threads;
    long long cap = (long long)cf::num_sms() * 8;
    int grid = (int)std::max<long long>(1, std::min(want, cap));
    cf::snapshot_cells_kernel<<<grid, threads, 0, cf::as_stream(stream)>>>(u, v, w, p, nx, ny, nz, ldu, ldv, ldw,
                                                                          out);
    CF_CHECK_LAUNCH("snapshot_cells_kernel");
    return CF_OK;
}

int cf_format_double(double v, char *out, int cap)
{
    CF_REQUIRE(out && cap >= 32, "cf_format_double: need a 32-byte buffer");
    int len = cf::csv::format_double(v, out);
    out[len] = '\0';
    return len;
}

int cf_snapshot_write(const char *path, const double *cells_host, int nx, int ny, int nz, double h, int threads)
{
    CF_REQUIRE(path && cells_host && nx >= 1 && ny >= 1 && nz >= 1, "cf_snapshot_write: bad arguments");
    const long long ncell = (long long)nx * ny * nz;
    // x, y, z: (arange(n) + 0.5) * h per axis, meshgrid 'ij', F-order flatten
    auto row = [=](long long r, double *vals) {
        const long long i = r % nx, jk = r / nx;
        const long long j = jk % ny, k = jk / ny;
        vals[0] = ((double)i + 0.5) * h;
        vals[1] = ((double)j + 0.5) * h;
        vals[2] = ((double)k + 0.5) * h;
        for (int c = 0; c < 4; ++c) vals[3 + c] = cells_host[c * ncell + r];
    };
    return cf::csv::write_csv(path, row, ncell, threads);
}

int cf_csv_write_columns(const char *path, const double *x, const double *y, const double *z, const double *u,
                         const double *v, const double *w, const double *p, int64_t nrows, int threads)
{
    CF_REQUIRE(path && x && y && z && u && v && w && p && nrows >= 0, "cf_csv_write_columns: bad arguments");
    const double *cols[7] = {x, y, z, u, v, w, p};
    auto row = [&](long long r, double *vals) {
        for (int c = 0; c < 7; ++c) vals[c] = cols[c][r];
    };
    return cf::csv::write_csv(path, row, nrows, threads);
}

}  // extern "C"
