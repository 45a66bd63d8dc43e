/*
 * chr_oracle.c -- CPU restatement of the reference (isochr) hot loops.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path
 * (paper_2408_05462_b200/) may link, import or call this file; only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg use it, and there only as the checker or as the
 * timed CPU baseline.
 *
 * Every function below restates one reference loop; the file:line it
 * follows is cited (paths relative to /root/reference/pkg/src/isochr/).
 * Arithmetic is IEEE f64 with no contraction (built with
 * -ffp-contract=off, no -ffast-math) so results are bit-identical to the
 * numba/numpy reference, which was pinned against golden vectors
 * generated from the reference itself (tests/golden/, see
 * tests/test_oracle_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "mc_tables.h"

/* 1.5 * 2**52 and 2**27: kernels.py:18, 22 */
#define OR_ROUND_SHIFT 6755399441055744.0
#define OR_ESCAPE_UMAX 134217728.0

/* ------------------------------------------------------------------ */
/* quantised 3D Lorenzo encode: kernels.py:47-93                        */
/* Returns the number of escaped samples.                              */
int64_t or_lorenzo_encode(const double *flat, int64_t nx, int64_t ny, int64_t nz,
                          double e, int64_t *q, uint8_t *escaped, int64_t *u)
{
    const double twoe = 2.0 * e;
    const double inv = 1.0 / twoe;
    const int64_t sy = nx, sz = nx * ny;
    int64_t nesc = 0, i = 0;
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x, ++i) {
                const double v = flat[i];
                const double qf = v * inv;
                const double t = qf + OR_ROUND_SHIFT; /* no reassociation: -ffp-contract=off, no fast-math */
                double uf = t - OR_ROUND_SHIFT;
                const double d = qf - uf;
                if (d == 0.5)
                    uf += 1.0;
                else if (d == -0.5)
                    uf -= 1.0;
                int64_t ui;
                if (fabs(uf) > OR_ESCAPE_UMAX || fabs(uf * twoe - v) > e) {
                    escaped[i] = 1;
                    ui = 0;
                    ++nesc;
                } else {
                    escaped[i] = 0;
                    ui = (int64_t)uf;
                }
                u[i] = ui;
                int64_t p = 0;
                if (x > 0) p += u[i - 1];
                if (y > 0) p += u[i - sy];
                if (z > 0) p += u[i - sz];
                if (x > 0 && y > 0) p -= u[i - 1 - sy];
                if (x > 0 && z > 0) p -= u[i - 1 - sz];
                if (y > 0 && z > 0) p -= u[i - sy - sz];
                if (x > 0 && y > 0 && z > 0) p += u[i - 1 - sy - sz];
                q[i] = ui - p;
            }
    return nesc;
}

/* inverse Lorenzo + scale + escape overwrite: kernels.py:131-166 */
void or_lorenzo_decode(const int64_t *q, const uint8_t *escaped, const double *escape_values,
                       double e, int64_t nx, int64_t ny, int64_t nz, int64_t *u, double *recon)
{
    const double twoe = 2.0 * e;
    const int64_t sy = nx, sz = nx * ny;
    int64_t i = 0, iesc = 0;
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x, ++i) {
                /* int64 wraparound like numba: do it in uint64 */
                uint64_t p = (uint64_t)q[i];
                if (x > 0) p += (uint64_t)u[i - 1];
                if (y > 0) p += (uint64_t)u[i - sy];
                if (z > 0) p += (uint64_t)u[i - sz];
                if (x > 0 && y > 0) p -= (uint64_t)u[i - 1 - sy];
                if (x > 0 && z > 0) p -= (uint64_t)u[i - 1 - sz];
                if (y > 0 && z > 0) p -= (uint64_t)u[i - sy - sz];
                if (x > 0 && y > 0 && z > 0) p += (uint64_t)u[i - 1 - sy - sz];
                u[i] = (int64_t)p;
                if (escaped && escaped[i])
                    recon[i] = escape_values[iesc++];
                else
                    recon[i] = (double)(int64_t)p * twoe;
            }
}

/* ------------------------------------------------------------------ */
/* zigzag / LEB128 / zero-run token encode: kernels.py:198-234          */
static int64_t put_varint(uint8_t *out, int64_t pos, uint64_t u)
{
    while (u >= 0x80) {
        out[pos++] = (uint8_t)((u & 0x7F) | 0x80);
        u >>= 7;
    }
    out[pos++] = (uint8_t)u;
    return pos;
}

/* out must hold 6*n+16 bytes; returns the number of bytes written */
int64_t or_rle_encode(const int64_t *vals, int64_t n, uint8_t *out)
{
    int64_t pos = 0, i = 0;
    while (i < n) {
        const int64_t v = vals[i];
        if (v == 0) {
            int64_t j = i + 1;
            while (j < n && vals[j] == 0) ++j;
            const int64_t run = j - i;
            if (run == 1) {
                out[pos++] = 1;
            } else {
                out[pos++] = 0;
                pos = put_varint(out, pos, (uint64_t)run);
            }
            i = j;
        } else {
            const uint64_t zz = ((uint64_t)v << 1) ^ (uint64_t)(v >> 63);
            pos = put_varint(out, pos, zz + 1);
            ++i;
        }
    }
    return pos;
}

/* token decode: kernels.py:299-345.  0 = ok, else an error code:
 * 1 truncated, 2 varint too long, 3 zero run missing length,
 * 4 zero run out of range, 5 trailing bytes. */
int or_rle_decode(const uint8_t *buf, int64_t nb, int64_t n, int64_t *vals)
{
    memset(vals, 0, (size_t)n * sizeof(int64_t));
    int64_t pos = 0, i = 0;
    while (i < n) {
        if (pos >= nb) return 1;
        int64_t u = 0;
        int shift = 0;
        for (;;) {
            const int64_t b = buf[pos++];
            u |= (b & 0x7F) << shift;
            if (b < 0x80) break;
            shift += 7;
            if (shift > 28) return 2;
            if (pos >= nb) return 1;
        }
        if (u == 0) {
            if (pos >= nb) return 3;
            int64_t run = 0;
            shift = 0;
            for (;;) {
                const int64_t b = buf[pos++];
                run |= (b & 0x7F) << shift;
                if (b < 0x80) break;
                shift += 7;
                if (shift > 28) return 2;
                if (pos >= nb) return 1;
            }
            if (run < 1 || i + run > n) return 4;
            i += run;
        } else {
            const int64_t zz = u - 1;
            vals[i++] = (zz >> 1) ^ -(zz & 1);
        }
    }
    if (pos != nb) return 5;
    return 0;
}

/* ------------------------------------------------------------------ */
/* min |s - k|: kernels.py:417-425 */
double or_min_abs_distance(const double *flat, int64_t n, double k)
{
    double best = fabs(flat[0] - k);
    for (int64_t i = 1; i < n; ++i) {
        const double d = fabs(flat[i] - k);
        if (d < best) best = d;
    }
    return best;
}

/* min |s - k| over a strided 3D window of a volume (x fastest), i.e.
 * kernels.min_abs_distance applied to grid[ox:ox+ex, oy:oy+ey, oz:oz+ez]
 * as region_bound does (bound.py:150-219, chr_archive.py:172-185). */
double or_window_min_abs_distance(const double *vol, int64_t nx, int64_t ny,
                                  int64_t ox, int64_t oy, int64_t oz,
                                  int64_t ex, int64_t ey, int64_t ez, double k)
{
    double best = INFINITY;
    int first = 1;
    for (int64_t z = 0; z < ez; ++z)
        for (int64_t y = 0; y < ey; ++y) {
            const double *row = vol + ((oz + z) * ny + (oy + y)) * nx + ox;
            for (int64_t x = 0; x < ex; ++x) {
                const double d = fabs(row[x] - k);
                if (first || d < best) {
                    best = d;
                    first = 0;
                }
            }
        }
    return best;
}

/* gather a window into a contiguous x-fastest buffer (chr_archive.py:174) */
void or_gather_window(const double *vol, int64_t nx, int64_t ny,
                      int64_t ox, int64_t oy, int64_t oz,
                      int64_t ex, int64_t ey, int64_t ez, double *out)
{
    for (int64_t z = 0; z < ez; ++z)
        for (int64_t y = 0; y < ey; ++y)
            memcpy(out + (z * ey + y) * ex, vol + ((oz + z) * ny + (oy + y)) * nx + ox,
                   (size_t)ex * sizeof(double));
}

/* ------------------------------------------------------------------ */
/* per-block window extrema: blocking.py:64-111 (block_grid_shape,
 * _window, decompose.make).  Blocks are in block_id order
 * bx + nbx*(by + nby*bz). */
static void or_axis_window(int64_t bc, int64_t bs, int64_t n, int64_t *lo, int64_t *ext)
{
    int64_t a = bc * bs;
    int64_t b = (bc + 1) * bs;
    if (b > n - 1) b = n - 1;
    *lo = a;
    *ext = b - a + 1;
}

void or_decompose(const double *vol, int64_t nx, int64_t ny, int64_t nz, int64_t bs,
                  double *vmin, double *vmax)
{
    const int64_t nbx = nx - 1 > 0 ? (nx - 1 + bs - 1) / bs : 1;
    const int64_t nby = ny - 1 > 0 ? (ny - 1 + bs - 1) / bs : 1;
    const int64_t nbz = nz - 1 > 0 ? (nz - 1 + bs - 1) / bs : 1;
    for (int64_t bz = 0; bz < nbz; ++bz)
        for (int64_t by = 0; by < nby; ++by)
            for (int64_t bx = 0; bx < nbx; ++bx) {
                int64_t ox, ex, oy, ey, oz, ez;
                or_axis_window(bx, bs, nx, &ox, &ex);
                or_axis_window(by, bs, ny, &oy, &ey);
                or_axis_window(bz, bs, nz, &oz, &ez);
                double lo = INFINITY, hi = -INFINITY;
                for (int64_t z = 0; z < ez; ++z)
                    for (int64_t y = 0; y < ey; ++y) {
                        const double *row = vol + ((oz + z) * ny + (oy + y)) * nx + ox;
                        for (int64_t x = 0; x < ex; ++x) {
                            if (row[x] < lo) lo = row[x];
                            if (row[x] > hi) hi = row[x];
                        }
                    }
                const int64_t id = bx + nbx * (by + nby * bz);
                vmin[id] = lo;
                vmax[id] = hi;
            }
}

/* greedy region merge: blocking.py:130-193.  keys[block_id] is the
 * relevance bitmask.  out_regions receives 6 int32 per region:
 * (bx, by, bz, hx, hy, hz) in creation order; returns the count. */
int64_t or_merge_regions(const uint64_t *keys, int64_t nbx, int64_t nby, int64_t nbz,
                         int32_t *out_regions)
{
    const int64_t nb = nbx * nby * nbz;
    uint8_t *claimed = (uint8_t *)calloc((size_t)nb, 1);
#define OR_ID(x, y, z) ((x) + nbx * ((y) + nby * (z)))
    int64_t nreg = 0;
    for (int64_t bz = 0; bz < nbz; ++bz)
        for (int64_t by = 0; by < nby; ++by)
            for (int64_t bx = 0; bx < nbx; ++bx) {
                if (claimed[OR_ID(bx, by, bz)]) continue;
                const uint64_t key = keys[OR_ID(bx, by, bz)];
                int64_t hx = bx, hy = by, hz = bz;
                /* grow +x one block at a time */
                while (hx + 1 < nbx && !claimed[OR_ID(hx + 1, by, bz)] &&
                       keys[OR_ID(hx + 1, by, bz)] == key)
                    ++hx;
                /* grow +y by whole rows [bx..hx] */
                for (;;) {
                    if (hy + 1 >= nby) break;
                    int ok = 1;
                    for (int64_t x = bx; x <= hx && ok; ++x)
                        if (claimed[OR_ID(x, hy + 1, bz)] || keys[OR_ID(x, hy + 1, bz)] != key) ok = 0;
                    if (!ok) break;
                    ++hy;
                }
                /* grow +z by whole slabs */
                for (;;) {
                    if (hz + 1 >= nbz) break;
                    int ok = 1;
                    for (int64_t y = by; y <= hy && ok; ++y)
                        for (int64_t x = bx; x <= hx && ok; ++x)
                            if (claimed[OR_ID(x, y, hz + 1)] || keys[OR_ID(x, y, hz + 1)] != key) ok = 0;
                    if (!ok) break;
                    ++hz;
                }
                for (int64_t z = bz; z <= hz; ++z)
                    for (int64_t y = by; y <= hy; ++y)
                        for (int64_t x = bx; x <= hx; ++x) claimed[OR_ID(x, y, z)] = 1;
                int32_t *r = out_regions + 6 * nreg++;
                r[0] = (int32_t)bx; r[1] = (int32_t)by; r[2] = (int32_t)bz;
                r[3] = (int32_t)hx; r[4] = (int32_t)hy; r[5] = (int32_t)hz;
            }
#undef OR_ID
    free(claimed);
    return nreg;
}

/* ------------------------------------------------------------------ */
/* CRC-32/IEEE, reflected 0xEDB88320 -- the algorithm of zlib.crc32
 * (codec.py:132, 222; chr_archive.py:338, 352). */
static uint32_t or_crc_table[256];
static int or_crc_ready = 0;

uint32_t or_crc32(uint32_t crc, const uint8_t *buf, int64_t n)
{
    if (!or_crc_ready) {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ 0xEDB88320u : c >> 1;
            or_crc_table[i] = c;
        }
        or_crc_ready = 1;
    }
    crc = ~crc;
    for (int64_t i = 0; i < n; ++i) crc = or_crc_table[(crc ^ buf[i]) & 0xFF] ^ (crc >> 8);
    return ~crc;
}

/* ------------------------------------------------------------------ */
/* marching cubes: kernels.py:428-524.  grid is x-fastest (nx,ny,nz).
 * Pass 1 (or_mc_count) returns the triangle total; pass 2 fills
 * verts (capacity 3*total rows of 3 doubles) and tris (total rows of 3
 * int32) and returns the vertex count.  vert_ids scratch: 3*nx*ny*nz. */
static inline int or_code(const double *g, int64_t nx, int64_t ny, int64_t cx, int64_t cy,
                          int64_t cz, double k)
{
#define G(x, y, z) g[((z) * ny + (y)) * nx + (x)]
    int c = 0;
    if (G(cx, cy, cz) >= k) c |= 1;
    if (G(cx + 1, cy, cz) >= k) c |= 2;
    if (G(cx + 1, cy + 1, cz) >= k) c |= 4;
    if (G(cx, cy + 1, cz) >= k) c |= 8;
    if (G(cx, cy, cz + 1) >= k) c |= 16;
    if (G(cx + 1, cy, cz + 1) >= k) c |= 32;
    if (G(cx + 1, cy + 1, cz + 1) >= k) c |= 64;
    if (G(cx, cy + 1, cz + 1) >= k) c |= 128;
#undef G
    return c;
}

int64_t or_mc_count(const double *g, int64_t nx, int64_t ny, int64_t nz, double k,
                    uint8_t *codes /* optional, (nx-1)(ny-1)(nz-1) */)
{
    int64_t total = 0, ic = 0;
    for (int64_t cz = 0; cz < nz - 1; ++cz)
        for (int64_t cy = 0; cy < ny - 1; ++cy)
            for (int64_t cx = 0; cx < nx - 1; ++cx, ++ic) {
                const int c = or_code(g, nx, ny, cx, cy, cz, k);
                if (codes) codes[ic] = (uint8_t)c;
                total += CHR_NTRI_TABLE[c];
            }
    return total;
}

int64_t or_mc_emit(const double *g, int64_t nx, int64_t ny, int64_t nz, double k,
                   double *verts, int32_t *tris, int32_t *vert_ids)
{
    for (int64_t i = 0; i < 3 * nx * ny * nz; ++i) vert_ids[i] = -1;
    int64_t nv = 0, itri = 0;
    for (int64_t cz = 0; cz < nz - 1; ++cz)
        for (int64_t cy = 0; cy < ny - 1; ++cy)
            for (int64_t cx = 0; cx < nx - 1; ++cx) {
                const int c = or_code(g, nx, ny, cx, cy, cz, k);
                const int nt = CHR_NTRI_TABLE[c];
                for (int slot = 0; slot < 3 * nt; ++slot) {
                    const int e = CHR_TRI_TABLE[c][slot];
                    const int ax = CHR_EDGE_AXIS[e];
                    const int64_t px = cx + CHR_EDGE_LOW[e][0];
                    const int64_t py = cy + CHR_EDGE_LOW[e][1];
                    const int64_t pz = cz + CHR_EDGE_LOW[e][2];
                    const int64_t p = (pz * ny + py) * nx + px;
                    int32_t vid = vert_ids[3 * p + ax];
                    if (vid < 0) {
                        const double s0 = g[p];
                        const double s1 = g[p + (ax == 0 ? 1 : ax == 1 ? nx : nx * ny)];
                        const double denom = s1 - s0;
                        const double t = denom == 0.0 ? 0.0 : (k - s0) / denom;
                        double f[3] = {(double)px, (double)py, (double)pz};
                        f[ax] = f[ax] + t;
                        verts[3 * nv + 0] = f[0];
                        verts[3 * nv + 1] = f[1];
                        verts[3 * nv + 2] = f[2];
                        vid = (int32_t)nv;
                        vert_ids[3 * p + ax] = vid;
                        ++nv;
                    }
                    tris[3 * itri + slot % 3] = vid;
                    if (slot % 3 == 2) ++itri;
                }
            }
    return nv;
}

/* binary-order case codes, bit i = corner (i&1, i>>1&1, i>>2&1):
 * isosurf.py:77-88 */
void or_case_field(const double *g, int64_t nx, int64_t ny, int64_t nz, double k, uint8_t *codes)
{
    int64_t ic = 0;
    for (int64_t cz = 0; cz < nz - 1; ++cz)
        for (int64_t cy = 0; cy < ny - 1; ++cy)
            for (int64_t cx = 0; cx < nx - 1; ++cx, ++ic) {
                int c = 0;
                for (int i = 0; i < 8; ++i) {
                    const int64_t x = cx + (i & 1), y = cy + ((i >> 1) & 1), z = cz + ((i >> 2) & 1);
                    if (g[(z * ny + y) * nx + x] >= k) c |= 1 << i;
                }
                codes[ic] = (uint8_t)c;
            }
}
