// mc.cu -- step 5 of the hot path: marching cubes as count -> scan -> emit,
// reproducing the reference mesh exactly (kernels.py:428-524 mc_extract,
// isosurf.py:183-204 marching_cubes, isosurf.py:207-225 merge_meshes).
//
// Reference ordering: cells z-outer / y / x-inner, triangle slots in
// TRI_TABLE order, a vertex is created the first time its canonical edge
// (axis, low corner) is touched.  Because every TRI_TABLE row references
// exactly the crossing edges of its case, the first touch of an edge is by
// the minimum-index cell containing it, the OWNER:
//   owner of an axis-a edge at lattice point p = p with every other
//   coordinate q replaced by max(p_q - 1, 0).
// So a cell owns the crossing edges whose perpendicular low offsets are 1
// (or 0 at a grid boundary), the vertex id of an owned edge is
//   (owned crossing edges in earlier cells) + (its first-appearance rank in
//   the owner's triangle row), and both come from tables + one scan.
//
//   k_mc_count4  lane per 64-cell row piece (persistent warps on a batch
//                queue): live cells, triangles and owned vertices from the
//                inside masks; per live piece the owned-vertex prefix of each
//                live cell (u16) and 4-bit triangle counts
//   k_mc_reduce / k_mc_grid_scan / k_mc_grids / k_mc_down   chunked scans
//   k_mc_emit4   lane per LIVE CELL: its code and its owners' codes from nine
//                3-bit row windows, owner vertex ids from piece base + prefix
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "chr_internal.cuh"
#include "mc_tables.h"

namespace chr {

constexpr int MTX = 64, MTY = 8, MZC = 32;
constexpr int64_t MCH = 1024;

// Bourke corner index of unit offset (x, y, z) (mc_tables.py:8-12)
#define CHR_CORNER_OF(x, y, z) (4 * (z) + ((2 * (y)) | ((x) ^ (y))))

struct __align__(16) McTables {
    int8_t tri[256][16];
    uint8_t ntri[256];
    uint8_t owncnt[256][8];   // owned crossing edges per (code, boundary flags)
    int8_t rank[256][8][12];  // first-appearance rank among owned edges, -1 if not owned
    int8_t inv[256][8][12];   // owned edge of rank r
    uint16_t cross[256];      // crossing-edge mask
    uint8_t edge_axis[12];
    uint8_t edge_low[12][3];
    int8_t edge_id[3][2][2][2];  // [axis][lx][ly][lz] -> Bourke edge (l_axis == 0)
};

static McTables g_mct;
constexpr int kMaxDevices = 64;
static McTables *g_dmct[kMaxDevices] = {};  // per CUDA device (cudaGetDevice)
static std::once_flag g_mct_once;
static std::mutex g_mct_mu;

// flags bit a set <=> the cell's coordinate along axis a is 0
static bool owned_by(int e, int flags) {
    const int a = CHR_EDGE_AXIS[e];
    for (int q = 0; q < 3; ++q) {
        if (q == a) continue;
        if (!(CHR_EDGE_LOW[e][q] == 1 || ((flags >> q) & 1))) return false;
    }
    return true;
}

static void mc_tables_host() {
    McTables &T = g_mct;
    std::memset(&T, 0, sizeof(T));
    std::memcpy(T.tri, CHR_TRI_TABLE, sizeof(T.tri));
    std::memcpy(T.ntri, CHR_NTRI_TABLE, sizeof(T.ntri));
    std::memcpy(T.edge_axis, CHR_EDGE_AXIS, sizeof(T.edge_axis));
    std::memcpy(T.edge_low, CHR_EDGE_LOW, sizeof(T.edge_low));
    std::memset(T.edge_id, -1, sizeof(T.edge_id));
    for (int e = 0; e < 12; ++e)
        T.edge_id[CHR_EDGE_AXIS[e]][CHR_EDGE_LOW[e][0]][CHR_EDGE_LOW[e][1]][CHR_EDGE_LOW[e][2]] = (int8_t)e;
    for (int c = 0; c < 256; ++c) {
        uint16_t cm = 0;
        for (int e = 0; e < 12; ++e) {
            const int a = CHR_EDGE_CORNERS[e][0], b = CHR_EDGE_CORNERS[e][1];
            if (((c >> a) & 1) != ((c >> b) & 1)) cm |= (uint16_t)(1u << e);
        }
        T.cross[c] = cm;
        for (int f = 0; f < 8; ++f) {
            for (int e = 0; e < 12; ++e) T.rank[c][f][e] = -1;
            int cnt = 0;
            for (int s = 0; s < 3 * CHR_NTRI_TABLE[c]; ++s) {
                const int e = CHR_TRI_TABLE[c][s];
                if (T.rank[c][f][e] < 0 && owned_by(e, f)) T.rank[c][f][e] = (int8_t)cnt++;
            }
            T.owncnt[c][f] = (uint8_t)cnt;
            std::memset(T.inv[c][f], -1, 12);
            for (int e = 0; e < 12; ++e)
                if (T.rank[c][f][e] >= 0) T.inv[c][f][T.rank[c][f][e]] = (int8_t)e;
        }
    }
}

static const McTables *mc_tables_device() {
    std::call_once(g_mct_once, mc_tables_host);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
    std::lock_guard<std::mutex> lk(g_mct_mu);
    if (!g_dmct[dev]) {
        McTables *d = nullptr;
        if (cudaMalloc(&d, sizeof(McTables)) != cudaSuccess) return nullptr;
        if (cudaMemcpy(d, &g_mct, sizeof(McTables), cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaFree(d);
            return nullptr;
        }
        g_dmct[dev] = d;
    }
    return g_dmct[dev];
}

struct McGrid {
    uint64_t goff;
    int32_t nx, ny, nz, ncx, ncy, ncz, ntx;
    uint32_t ncy_magic;             // ceil(2^32 / ncy): rr / ncy by __umulhi (+ one correction)
    double origin[3], spacing[3];
    int64_t piece_base, npieces, chunk_base, nchunks, item_base;
    int64_t tri_base, vert_base;    // in the merged output (device scan)
    int64_t ntri, nvert;
    int64_t mask_off;               // inside mask (v >= k): word offset, plane-linear bits
    int64_t mask_item_base;         // k_mc_mask items: planes x ceil(pw / 64)
    int32_t pw;                     // mask words per plane
    int32_t zoff;                   // lattice z of grid plane 0 (sub-grid of a region window)
};

struct McPieceCnt {
    int32_t tri, vert;
};
struct McPieceBase {
    int64_t tri, vert;
};

__device__ __forceinline__ int64_t find_grid(const McGrid *__restrict__ g, int64_t n, int64_t key, int which) {
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        const int64_t b = which == 0 ? g[mid].piece_base : (which == 1 ? g[mid].chunk_base : g[mid].item_base);
        if (b <= key) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Bourke-order case code of cell (cx,cy,cz) (kernels.py:451-467), corner values out
__device__ __forceinline__ int cell_code(const double *__restrict__ g, int64_t nx, int64_t nxy, int cx, int cy,
                                         int cz, double k, double c[8]) {
    const double *p = g + (int64_t)cz * nxy + (int64_t)cy * nx + cx;
    c[0] = __ldg(p);
    c[1] = __ldg(p + 1);
    c[2] = __ldg(p + nx + 1);
    c[3] = __ldg(p + nx);
    c[4] = __ldg(p + nxy);
    c[5] = __ldg(p + nxy + 1);
    c[6] = __ldg(p + nxy + nx + 1);
    c[7] = __ldg(p + nxy + nx);
    int code = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) code |= (c[i] >= k) ? (1 << i) : 0;
    return code;
}

__device__ __forceinline__ int bflags(int cx, int cy, int cz) {
    return (cx == 0 ? 1 : 0) | (cy == 0 ? 2 : 0) | (cz == 0 ? 4 : 0);
}

__global__ void __launch_bounds__(256) k_mc_reduce(const McPieceCnt *__restrict__ cnt, McPieceBase *__restrict__ chunk) {
    const int64_t c = blockIdx.x;
    int64_t t = 0, v = 0;
    for (int i = threadIdx.x; i < MCH; i += blockDim.x) {
        const McPieceCnt x = cnt[c * MCH + i];
        t += x.tri;
        v += x.vert;
    }
    __shared__ int64_t st[8], sv[8];
    for (int off = 16; off; off >>= 1) {
        t += __shfl_xor_sync(0xFFFFFFFFu, t, off);
        v += __shfl_xor_sync(0xFFFFFFFFu, v, off);
    }
    if ((threadIdx.x & 31) == 0) {
        st[threadIdx.x >> 5] = t;
        sv[threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t a = 0, b = 0;
        for (int i = 0; i < 8; ++i) {
            a += st[i];
            b += sv[i];
        }
        chunk[c].tri = a;
        chunk[c].vert = b;
    }
}

// per grid: exclusive chunk prefixes + grid totals (thread per grid)
// warp per grid: exclusive scan of its chunk totals, 32 chunks per step
__global__ void k_mc_grid_scan(McGrid *__restrict__ G, int64_t ng, McPieceBase *__restrict__ chunk) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= ng) return;
    McGrid &g = G[i];
    int64_t t = 0, v = 0;  // running totals before this step
    for (int64_t c0 = g.chunk_base; c0 < g.chunk_base + g.nchunks; c0 += 32) {
        const int64_t c = c0 + lane;
        const bool ok = c < g.chunk_base + g.nchunks;
        McPieceBase x;
        x.tri = 0;
        x.vert = 0;
        if (ok) x = chunk[c];
        int64_t it = x.tri, iv = x.vert;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int64_t a = __shfl_up_sync(0xFFFFFFFFu, it, off), b = __shfl_up_sync(0xFFFFFFFFu, iv, off);
            if (lane >= off) {
                it += a;
                iv += b;
            }
        }
        if (ok) {
            chunk[c].tri = t + it - x.tri;
            chunk[c].vert = v + iv - x.vert;
        }
        t += __shfl_sync(0xFFFFFFFFu, it, 31);
        v += __shfl_sync(0xFFFFFFFFu, iv, 31);
    }
    if (lane == 0) {
        g.ntri = t;
        g.nvert = v;
    }
}

// one CTA: merged-mesh bases of every grid (exclusive scan over grids)
__global__ void __launch_bounds__(1024) k_mc_grids(McGrid *__restrict__ G, int64_t ng, int64_t *__restrict__ totals) {
    __shared__ int64_t st[32], sv[32];
    __shared__ int64_t ct, cv;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) ct = cv = 0;
    __syncthreads();
    for (int64_t b = 0; b < ng; b += 1024) {
        const int64_t i = b + threadIdx.x;
        const int64_t t = i < ng ? G[i].ntri : 0, v = i < ng ? G[i].nvert : 0;
        int64_t it = t, iv = v;
        for (int off = 1; off < 32; off <<= 1) {
            const int64_t a = __shfl_up_sync(0xFFFFFFFFu, it, off), c = __shfl_up_sync(0xFFFFFFFFu, iv, off);
            if (lane >= off) {
                it += a;
                iv += c;
            }
        }
        if (lane == 31) {
            st[warp] = it;
            sv[warp] = iv;
        }
        __syncthreads();
        int64_t pt = ct, pv = cv;
        for (int w = 0; w < warp; ++w) {
            pt += st[w];
            pv += sv[w];
        }
        if (i < ng) {
            G[i].tri_base = pt + it - t;
            G[i].vert_base = pv + iv - v;
        }
        __syncthreads();
        if (threadIdx.x == 1023) {
            ct = pt + it;
            cv = pv + iv;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        totals[0] = ct;
        totals[1] = cv;
    }
}

__global__ void __launch_bounds__(256) k_mc_down(const McPieceCnt *__restrict__ cnt,
                                                 const McPieceBase *__restrict__ chunk,
                                                 McPieceBase *__restrict__ base) {
    const int64_t c = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // 4 consecutive pieces per thread
    McPieceCnt x[4];
    int64_t t = 0, v = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        x[i] = cnt[c * MCH + threadIdx.x * 4 + i];
        t += x[i].tri;
        v += x[i].vert;
    }
    int64_t it = t, iv = v;
    for (int off = 1; off < 32; off <<= 1) {
        const int64_t a = __shfl_up_sync(0xFFFFFFFFu, it, off);
        const int64_t b = __shfl_up_sync(0xFFFFFFFFu, iv, off);
        if (lane >= off) {
            it += a;
            iv += b;
        }
    }
    __shared__ int64_t st[8], sv[8];
    if (lane == 31) {
        st[warp] = it;
        sv[warp] = iv;
    }
    __syncthreads();
    int64_t pt = chunk[c].tri, pv = chunk[c].vert;
    for (int i = 0; i < warp; ++i) {
        pt += st[i];
        pv += sv[i];
    }
    pt += it - t;
    pv += iv - v;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        McPieceBase b;
        b.tri = pt;
        b.vert = pv;
        base[c * MCH + threadIdx.x * 4 + i] = b;
        pt += x[i].tri;
        pv += x[i].vert;
    }
}

__device__ __forceinline__ double world(double origin, double lat, double spacing) {
    return __dadd_rn(origin, __dmul_rn(lat, spacing));
}

// ------------------------------------------------------------------ v2 tiles
// CTA = 64 cells x 8 cell rows, marching z over up to MZC cell planes.  Every
// f64 sample row is loaded once per plane by one warp (coalesced), turned
// into an inside mask with ballots, and the Bourke code of a cell is
// assembled from four 64-bit row masks (rows y, y+1 at planes z, z+1).
__global__ void k_mc_fill_map(const McGrid *__restrict__ G, int64_t ng, int32_t *__restrict__ item_grid,
                              int32_t *__restrict__ chunk_grid, int32_t *__restrict__ mask_grid) {
    const int64_t i = blockIdx.x;
    if (i >= ng) return;
    const McGrid &g = G[i];
    const int64_t nit = (int64_t)g.ntx * ((g.ncy + MTY - 1) / MTY) * ((g.ncz + MZC - 1) / MZC);
    for (int64_t t = threadIdx.x; t < nit; t += blockDim.x) item_grid[g.item_base + t] = (int32_t)i;
    for (int64_t t = threadIdx.x; t < g.nchunks; t += blockDim.x) chunk_grid[g.chunk_base + t] = (int32_t)i;
    const int64_t nm = (int64_t)g.nz * ((g.pw + 63) / 64);
    for (int64_t t = threadIdx.x; t < nm; t += blockDim.x) mask_grid[g.mask_item_base + t] = (int32_t)i;
}

// ------------------------------------------------------------------ inside masks
// One bit per sample (v >= k), plane-linear (bit y * nx + x of the plane's
// words): 1/64 of the f64 bytes, so the count and emit passes stream masks
// and touch f64 samples only to interpolate vertices.  Item = 64 words of
// one plane; warp = 8 words, all loads issued before the ballots.
__global__ void __launch_bounds__(256) k_mc_mask(const double *__restrict__ grids, const McGrid *__restrict__ G,
                                                 const int32_t *__restrict__ mask_grid, double k,
                                                 uint32_t *__restrict__ mask) {
    const int64_t item = blockIdx.x;
    const McGrid &g = G[__ldg(mask_grid + item)];
    const int64_t local = item - g.mask_item_base;
    const int wpb = (g.pw + 63) / 64;
    const int z = (int)(local / wpb), wc = (int)(local - (int64_t)z * wpb);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nxy = (int64_t)g.nx * g.ny;
    const double *gp = grids + g.goff + (int64_t)z * nxy;
    const int w0 = wc * 64 + warp * 8;
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t t = (int64_t)(w0 + i) * 32 + lane;
        v[i] = (w0 + i < g.pw && t < nxy) ? __ldg(gp + t) : 0.0;
    }
    uint32_t *mp = mask + g.mask_off + (int64_t)z * g.pw;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t t = (int64_t)(w0 + i) * 32 + lane;
        const uint32_t b = __ballot_sync(0xFFFFFFFFu, t < nxy && v[i] >= k);
        if (lane == 0 && w0 + i < g.pw) mp[w0 + i] = b;
    }
}

// 64 bits of a plane mask from bit `b` (m) and the 2 bits after (h)
__device__ __forceinline__ void mask_bits66(const uint32_t *__restrict__ mp, int64_t b, uint64_t &m, uint32_t &h) {
    const uint32_t *w = mp + (b >> 5);
    const int sh = (int)(b & 31);
    const uint32_t w0 = __ldg(w), w1 = __ldg(w + 1), w2 = __ldg(w + 2), w3 = __ldg(w + 3);
    m = (uint64_t)__funnelshift_r(w0, w1, sh) | ((uint64_t)__funnelshift_r(w1, w2, sh) << 32);
    h = __funnelshift_r(w2, w3, sh) & 3u;
}

// bits c and c+1 of a (lo | hi << 64) mask
__device__ __forceinline__ uint32_t bit_at(uint64_t lo, uint32_t hi, int c) {
    return c < 64 ? (uint32_t)(lo >> c) & 1u : (hi >> (c - 64)) & 1u;
}

// bits (c, c+1) of the 65/66-bit mask (lo | hi << 64) as a 2-bit pair
__device__ __forceinline__ uint32_t pair_at(uint64_t lo, uint32_t hi, int c) {
    const uint32_t a = (uint32_t)lo, b = (uint32_t)(lo >> 32);
    if (c < 32) return __funnelshift_r(a, b, c) & 3u;
    if (c < 64) return __funnelshift_r(b, hi, c - 32) & 3u;
    return (hi >> (c - 64)) & 3u;
}
__device__ __forceinline__ uint32_t pair_swap(uint32_t p) { return ((p * 5u) >> 1) & 3u; }

// Bourke code from the four row masks: bits (c,c+1) of rows y,z / y+1,z / y,z+1 / y+1,z+1
__device__ __forceinline__ int code_fast(uint64_t m00, uint32_t h00, uint64_t m10, uint32_t h10, uint64_t m01,
                                         uint32_t h01, uint64_t m11, uint32_t h11, int c) {
    return (int)(pair_at(m00, h00, c) | pair_swap(pair_at(m10, h10, c)) << 2 | pair_at(m01, h01, c) << 4 |
                 pair_swap(pair_at(m11, h11, c)) << 6);
}

__device__ __forceinline__ int code_from(uint64_t m00, uint32_t h00, uint64_t m10, uint32_t h10, uint64_t m01,
                                         uint32_t h01, uint64_t m11, uint32_t h11, int c) {
    // Bourke corners: 0(0,0,0) 1(1,0,0) 2(1,1,0) 3(0,1,0) 4(0,0,1) 5(1,0,1) 6(1,1,1) 7(0,1,1)
    return (int)(bit_at(m00, h00, c) | bit_at(m00, h00, c + 1) << 1 | bit_at(m10, h10, c + 1) << 2 |
                 bit_at(m10, h10, c) << 3 | bit_at(m01, h01, c) << 4 | bit_at(m01, h01, c + 1) << 5 |
                 bit_at(m11, h11, c + 1) << 6 | bit_at(m11, h11, c) << 7);
}

// count v4: a LANE per 64-cell row piece (a warp takes 32 consecutive pieces
// of a batch).  The lane loads its piece's four 66-bit row masks (rows y, y+1
// x planes z, z+1), finds the live cells -- some corner inside and some
// outside: (OR of the 8 corners) & ~(AND of the 8 corners), with the x+1
// corners by a one-bit shift -- and looks up triangles / owned vertices only
// for those (c3: 3 % of the cells), so a dead piece costs a few dozen
// instructions of one lane instead of a warp's step.
__global__ void __launch_bounds__(256) k_mc_count4(const McGrid *__restrict__ G,
                                                   const int32_t *__restrict__ chunk_grid,
                                                   const McTables *__restrict__ T,
                                                   const uint32_t *__restrict__ mask,
                                                   McPieceCnt *__restrict__ cnt, uint64_t *__restrict__ lmask,
                                                   uint32_t *__restrict__ cellw,
                                                   unsigned long long *__restrict__ queue, int64_t nbatch) {
    __shared__ __align__(16) uint8_t s_ntri[256];
    __shared__ __align__(16) uint8_t s_own[256][8];
    __shared__ McGrid sg[8];
    {
        const uint4 *so = reinterpret_cast<const uint4 *>(T->owncnt);
        uint4 *d_o = reinterpret_cast<uint4 *>(&s_own[0][0]);
        for (int i = threadIdx.x; i < 128; i += blockDim.x) d_o[i] = __ldg(so + i);
        if (threadIdx.x < 16)
            reinterpret_cast<uint4 *>(s_ntri)[threadIdx.x] = __ldg(reinterpret_cast<const uint4 *>(T->ntri) + threadIdx.x);
    }
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    McGrid &g = sg[w];
    int cur_grid = -1;
    constexpr int NB = (int)(MCH / 32);
    for (;;) {
        unsigned long long bq = 0;
        if (lane == 0) bq = atomicAdd(queue, 1ull);
        const int64_t bi = (int64_t)__shfl_sync(0xFFFFFFFFu, bq, 0);
        if (bi >= nbatch) break;
        const int64_t c = bi / NB;
        const int gi = __ldg(chunk_grid + c);
        if (gi != cur_grid) {
            __syncwarp();
            const uint32_t *src = reinterpret_cast<const uint32_t *>(G + gi);
            uint32_t *dst = reinterpret_cast<uint32_t *>(&g);
            for (int i = lane; i < (int)(sizeof(McGrid) / 4); i += 32) dst[i] = src[i];
            __syncwarp();
            cur_grid = gi;
        }
        const int64_t lp = (c - g.chunk_base) * MCH + (bi - c * NB) * 32 + lane;
        if (lp >= g.npieces) continue;
        const int xt = (int)(lp % g.ntx);
        const int64_t rr = lp / g.ntx;
        const int cy = (int)(rr % g.ncy), cz = (int)(rr / g.ncy);
        const int x0 = xt * MTX;
        const int ncell = min(MTX, g.ncx - x0);
        const uint32_t *mbase = mask + g.mask_off;
        uint64_t m[4];
        uint32_t h[4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
            mask_bits66(mbase + (int64_t)(cz + (r >> 1)) * g.pw, (int64_t)(cy + (r & 1)) * g.nx + x0, m[r], h[r]);
        const uint64_t a = m[0] & m[1] & m[2] & m[3], o = m[0] | m[1] | m[2] | m[3];
        const uint32_t ah = h[0] & h[1] & h[2] & h[3], oh = h[0] | h[1] | h[2] | h[3];
        const uint64_t o1 = (o >> 1) | ((uint64_t)(oh & 1u) << 63), a1 = (a >> 1) | ((uint64_t)(ah & 1u) << 63);
        const uint64_t cells = ncell >= 64 ? ~0ull : ((1ull << ncell) - 1);
        const uint64_t live0 = (o | o1) & ~(a & a1) & cells;
        uint64_t live = live0;
        int t = 0, v = 0;
        const int fyz = (cy == 0 ? 2 : 0) | (cz == 0 ? 4 : 0);
        const int64_t gp = g.piece_base + lp;
        uint32_t *cw = cellw + 64 * gp;
        while (live) {
            const int cc = __ffsll((long long)live) - 1;
            live &= live - 1;
            const int code = code_fast(m[0], h[0], m[1], h[1], m[2], h[2], m[3], h[3], cc);
            const uint32_t nt = s_ntri[code], no = s_own[code][fyz | (x0 + cc == 0 ? 1 : 0)];
            // the cell's word: owned vertices (<= 516) and triangles (<= 320) of
            // the piece's earlier cells, and its code
            cw[cc] = (uint32_t)v | ((uint32_t)t << 10) | ((uint32_t)code << 19);
            t += nt;
            v += no;
        }
        McPieceCnt out;
        out.tri = t;
        out.vert = v;
        cnt[gp] = out;
        lmask[gp] = live0;
    }
}

// emit v4: a LANE per LIVE CELL.  A warp takes 32 consecutive pieces of a
// batch, scans their live-cell counts (k_mc_count4's live masks) and deals
// the batch's live cells to its lanes 32 at a time, so every lane does one
// cell's work whatever the pieces' densities.  k_mc_count4 left one word per
// live cell (code, owned vertices and triangles of the piece's earlier
// cells), so a cell's triangle offset and vertex base are its piece's bases
// + its word, and a triangle corner owned by another cell costs that cell's
// word and its piece's vertex base (two loads) + one rank lookup.
#ifndef CHR_E4W
#define CHR_E4W 8
#endif
constexpr int E4W = CHR_E4W;  // warps per CTA
__global__ void __launch_bounds__(E4W * 32) k_mc_emit4(const double *__restrict__ grids, const McGrid *__restrict__ G,
                                                       const int32_t *__restrict__ chunk_grid, double k,
                                                       const McTables *__restrict__ T,
                                                       const McPieceBase *__restrict__ base,
                                                       const uint64_t *__restrict__ lmask,
                                                       const uint32_t *__restrict__ cellw,
                                                       unsigned long long *__restrict__ queue, int64_t nbatch,
                                                       double *__restrict__ verts, int32_t *__restrict__ tris,
                                                       int64_t *__restrict__ vedge) {
    __shared__ __align__(16) int8_t s_tri[256][16];
    __shared__ __align__(16) int8_t s_rank[256][8][12];
    __shared__ uint8_t s_cinfo[12][8], s_vinfo[12];
    __shared__ McGrid sg[E4W];
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(T->tri);
        uint4 *dst = reinterpret_cast<uint4 *>(&s_tri[0][0]);
        for (int i = threadIdx.x; i < 256; i += blockDim.x) dst[i] = __ldg(src + i);
        const uint4 *sr = reinterpret_cast<const uint4 *>(T->rank);
        uint4 *dr = reinterpret_cast<uint4 *>(&s_rank[0][0][0]);
        for (int i = threadIdx.x; i < (int)(sizeof(s_rank) / 16); i += blockDim.x) dr[i] = __ldg(sr + i);
    }
    if (threadIdx.x < 96) {
        const int e = threadIdx.x >> 3, f = threadIdx.x & 7;
        const int a = T->edge_axis[e];
        int l[3] = {T->edge_low[e][0], T->edge_low[e][1], T->edge_low[e][2]};
        int d = 0;
        for (int q = 0; q < 3; ++q)
            if (q != a && l[q] == 0 && !((f >> q) & 1)) {
                d |= 1 << q;
                l[q] = 1;
            }
        s_cinfo[e][f] = (uint8_t)(d | (T->edge_id[a][l[0]][l[1]][l[2]] << 3));
        if (f == 0) s_vinfo[e] = (uint8_t)(a | (T->edge_low[e][0] << 2) | (T->edge_low[e][1] << 3) | (T->edge_low[e][2] << 4));
    }
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    McGrid &g = sg[w];
    int cur_grid = -1;
    constexpr int NB = (int)(MCH / 32);
    for (;;) {
        unsigned long long bq = 0;
        if (lane == 0) bq = atomicAdd(queue, 1ull);
        const int64_t bi = (int64_t)__shfl_sync(0xFFFFFFFFu, bq, 0);
        if (bi >= nbatch) break;
        const int64_t c = bi / NB;
        const int gi = __ldg(chunk_grid + c);
        if (gi != cur_grid) {
            __syncwarp();
            const uint32_t *src = reinterpret_cast<const uint32_t *>(G + gi);
            uint32_t *dst = reinterpret_cast<uint32_t *>(&g);
            for (int i = lane; i < (int)(sizeof(McGrid) / 4); i += 32) dst[i] = src[i];
            __syncwarp();
            cur_grid = gi;
        }
        const int64_t lp0 = (c - g.chunk_base) * MCH + (bi - c * NB) * 32;  // batch's first piece (grid-local)
        const uint64_t live = lp0 + lane < g.npieces ? __ldg(lmask + g.piece_base + lp0 + lane) : 0ull;
        const int n = __popcll(live);
        int incl = n;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
            if (lane >= off) incl += t;
        }
        const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        if (total == 0) continue;
        const int excl = incl - n;
        const uint32_t llo = (uint32_t)live, lhi = (uint32_t)(live >> 32);
        const double *gp = grids + g.goff;
        const int64_t nxy = (int64_t)g.nx * g.ny;
        for (int i0 = 0; i0 < total; i0 += 32) {
            const int i = i0 + lane;
            int q = 0;  // the lane (piece) holding live cell i: last q with excl_q <= i
#pragma unroll
            for (int step = 16; step; step >>= 1) {
                const int e = __shfl_sync(0xFFFFFFFFu, excl, q + step);
                if (e <= i) q += step;
            }
            const int r = i - __shfl_sync(0xFFFFFFFFu, excl, q);
            const uint32_t lo = __shfl_sync(0xFFFFFFFFu, llo, q), hi = __shfl_sync(0xFFFFFFFFu, lhi, q);
            if (i >= total) continue;
            const int clo = __popc(lo);
            const int b = r < clo ? (int)__fns(lo, 0, r + 1) : 32 + (int)__fns(hi, 0, r - clo + 1);
            const int lp = (int)(lp0 + q);
            const int rr = g.ntx == 1 ? lp : lp / g.ntx;
            const int xt = lp - rr * g.ntx;
            int cz = g.ncy == 1 ? rr : (int)__umulhi((uint32_t)rr, g.ncy_magic);
            if (cz * g.ncy > rr) --cz;
            const int cy = rr - cz * g.ncy;
            const int cx = xt * MTX + b;
            const int f = bflags(cx, cy, cz);
            const int64_t pg = g.piece_base + lp;
            const McPieceBase pb = base[pg];
            const uint32_t cwd = __ldg(cellw + 64 * pg + b);
            const int code = (int)(cwd >> 19);
            const int64_t vbase = pb.vert + (cwd & 1023u);
            const int64_t tofs = pb.tri + ((cwd >> 10) & 511u);
            const int nt = (int)T->ntri[code];
            int32_t *to = tris + 3 * (g.tri_base + tofs);
            const int pstep = g.ncy * g.ntx;  // pieces per cell plane (< 2^31)
            for (int t = 0; t < nt; ++t) {
                int32_t out3[3];
#pragma unroll
                for (int qq = 0; qq < 3; ++qq) {
                    // owner cell (the cell itself when info & 7 == 0): its piece's
                    // vertex base + its prefix inside the piece + the edge's rank
                    const int info = s_cinfo[s_tri[code][3 * t + qq]][f];
                    const int dx = info & 1, rs = (info >> 1) & 3, e2 = info >> 3;
                    const int ox = cx - dx, oy = cy - (rs & 1), oz = cz - (rs >> 1);
                    const int64_t op = pg - (rs & 1) * g.ntx - (rs >> 1) * pstep - ((dx & (b == 0)) ? 1 : 0);
                    const uint32_t ow = __ldg(cellw + 64 * op + (ox & 63));
                    const int64_t vid = __ldg(&base[op].vert) + (ow & 1023u) + s_rank[ow >> 19][bflags(ox, oy, oz)][e2];
                    out3[qq] = (int32_t)(g.vert_base + vid);
                }
                to[3 * t] = out3[0];
                to[3 * t + 1] = out3[1];
                to[3 * t + 2] = out3[2];
            }
            const int nown = (int)T->owncnt[code][f];
            for (int rk = 0; rk < nown; ++rk) {
                const int vi = s_vinfo[__ldg(&T->inv[code][f][rk])];
                const int a = vi & 3, lx = (vi >> 2) & 1, ly = (vi >> 3) & 1, lz = (vi >> 4) & 1;
                const double *sp = gp + (int64_t)(cz + lz) * nxy + (int64_t)(cy + ly) * g.nx + (cx + lx);
                const double s0 = __ldg(sp);
                const double s1 = __ldg(sp + (a == 0 ? 1 : (a == 1 ? (int64_t)g.nx : nxy)));
                const double den = __dadd_rn(s1, -s0);
                const double tt = den == 0.0 ? 0.0 : __ddiv_rn(__dadd_rn(k, -s0), den);
                double lx_ = (double)(cx + lx), ly_ = (double)(cy + ly), lz_ = (double)(cz + lz + g.zoff);
                if (a == 0) lx_ = __dadd_rn(lx_, tt);
                else if (a == 1) ly_ = __dadd_rn(ly_, tt);
                else lz_ = __dadd_rn(lz_, tt);
                const int64_t vid = g.vert_base + vbase + rk;
                double *o = verts + 3 * vid;
                if (vedge)
                    vedge[vid] = (((int64_t)(cz + lz) * g.ny + (cy + ly)) * g.nx + (cx + lx)) * 3 + a;
                o[0] = world(g.origin[0], lx_, g.spacing[0]);
                o[1] = world(g.origin[1], ly_, g.spacing[1]);
                o[2] = world(g.origin[2], lz_, g.spacing[2]);
            }
        }
    }
}

__global__ void k_case_codes(const double *__restrict__ g, int64_t nx, int64_t ny, int64_t nz, double k,
                             int binary, uint8_t *__restrict__ codes) {
    const int64_t ncx = nx - 1, ncy = ny - 1, ncz = nz - 1;
    const int64_t n = ncx * ncy * ncz;
    const int64_t nxy = nx * ny;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int cx = (int)(i % ncx), cy = (int)((i / ncx) % ncy), cz = (int)(i / (ncx * ncy));
        double c[8];
        int code = cell_code(g, nx, nxy, cx, cy, cz, k, c);
        if (binary) {  // Bourke -> binary: swap bits 2<->3 and 6<->7
            const int b2 = (code >> 2) & 1, b3 = (code >> 3) & 1, b6 = (code >> 6) & 1, b7 = (code >> 7) & 1;
            code = (code & 0x33) | (b3 << 2) | (b2 << 3) | (b7 << 6) | (b6 << 7);
        }
        codes[i] = (uint8_t)code;
    }
}

// ------------------------------------------------------------------ host
struct McPlan {
    std::vector<McGrid> grids;
    int64_t npieces = 0, nchunks = 0, nitems = 0, nmask_items = 0, nmask_words = 0;
    size_t ws = 0;
    McGrid *d_grids;
    McPieceCnt *cnt;
    McPieceBase *chunk, *base;
    uint64_t *lmask;  // live cells of every piece (k_mc_count4)
    uint32_t *cellw;  // per live cell of a live piece: vertex / triangle prefix in the piece + code
    int64_t *totals;
    int32_t *item_grid, *chunk_grid, *mask_grid;
    uint32_t *mask;
};

static bool mc_build(const chr_mc_grid_t *h, int64_t n, McPlan &pl) {
    pl.grids.resize(n);
    int64_t piece = 0, chunk = 0, item = 0;
    for (int64_t i = 0; i < n; ++i) {
        McGrid &g = pl.grids[i];
        std::memset(&g, 0, sizeof(g));
        g.goff = h[i].grid_offset;
        g.nx = h[i].dims[0];
        g.ny = h[i].dims[1];
        g.nz = h[i].dims[2];
        if (g.nx < 2 || g.ny < 2 || g.nz < 2) return false;
        g.ncx = g.nx - 1;
        g.ncy = g.ny - 1;
        g.ncz = g.nz - 1;
        g.ntx = (int32_t)ceil_div(g.ncx, MTX);
        g.ncy_magic = g.ncy > 1 ? (uint32_t)(((uint64_t(1) << 32) + (uint64_t)g.ncy - 1) / (uint64_t)g.ncy) : 0u;
        for (int a = 0; a < 3; ++a) {
            g.origin[a] = h[i].origin[a];
            g.spacing[a] = h[i].spacing[a];
        }
        g.zoff = h[i].zoff;
        g.piece_base = piece;
        g.npieces = (int64_t)g.ntx * g.ncy * g.ncz;
        if (g.npieces >= (int64_t(1) << 31)) return false;  // piece indices are int32 in the kernels
        g.chunk_base = chunk;
        g.nchunks = ceil_div(g.npieces, MCH);
        piece += g.nchunks * MCH;
        chunk += g.nchunks;
        g.item_base = item;
        item += (int64_t)g.ntx * ceil_div(g.ncy, MTY) * ceil_div(g.ncz, MZC);
        g.pw = (int32_t)ceil_div((int64_t)g.nx * g.ny, 32);
        g.mask_off = pl.nmask_words;
        pl.nmask_words += (int64_t)g.pw * g.nz;
        g.mask_item_base = pl.nmask_items;
        pl.nmask_items += (int64_t)g.nz * ceil_div(g.pw, 64);
    }
    pl.npieces = piece;
    pl.nchunks = chunk;
    pl.nitems = item;
    return true;
}

static int mc_num_sms() {
    static int n_sm[kMaxDevices] = {};  // per CUDA device
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 148;
    if (!n_sm[dev]) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
            n_sm[dev] = n;
        else
            return 148;
    }
    return n_sm[dev];
}

// two zeroed counters after the piece counts: [0] k_mc_emit4's batch queue, [1] k_mc_count4's
static unsigned long long *mc_queue(const McPlan &pl) {
    return reinterpret_cast<unsigned long long *>(pl.cnt + pl.npieces);
}

static void mc_carve(McPlan &pl, void *base, size_t cap) {
    WsCarver c{reinterpret_cast<char *>(base), 0, cap};
    pl.d_grids = c.take<McGrid>(pl.grids.size());
    pl.cnt = c.take<McPieceCnt>(pl.npieces + 2);  // + the two batch queues (mc_queue)
    pl.chunk = c.take<McPieceBase>(pl.nchunks);
    pl.base = c.take<McPieceBase>(pl.npieces);
    pl.lmask = c.take<uint64_t>(pl.npieces);
    pl.cellw = c.take<uint32_t>(64 * pl.npieces);
    pl.totals = c.take<int64_t>(2);
    pl.item_grid = c.take<int32_t>(pl.nitems + 1);
    pl.chunk_grid = c.take<int32_t>(pl.nchunks + 1);
    pl.mask_grid = c.take<int32_t>(pl.nmask_items + 1);
    pl.mask = c.take<uint32_t>(pl.nmask_words + 8);  // + slack: 4-word reads past a plane
    pl.ws = ((c.off + 255) & ~size_t(255)) + 256;
}

}  // namespace chr

using namespace chr;

extern "C" size_t chr_mc_workspace_size(const chr_mc_grid_t *h, int64_t n) {
    CHR_XFER_SCOPE;
    McPlan pl;
    if (!h || n < 1 || !mc_build(h, n, pl)) return 256;
    mc_carve(pl, nullptr, ~size_t(0));
    return pl.ws;
}

static int mc_count_impl(const double *d_grids, const chr_mc_grid_t *h, int64_t n, double k, const uint32_t *d_masks,
                         void *d_ws, size_t ws_bytes, int64_t *h_ntri, int64_t *h_nvert, int64_t *h_total_tri,
                         int64_t *h_total_vert, void *stream);
static int mc_emit_impl(const double *d_grids, const chr_mc_grid_t *h, int64_t n, double k, const uint32_t *d_masks,
                        void *d_ws, size_t ws_bytes, double *d_verts, int32_t *d_tris, int64_t *d_vedge,
                        void *stream);

extern "C" int chr_mc_count(const double *d_grids, const chr_mc_grid_t *h, int64_t n, double k, void *d_ws,
                            size_t ws_bytes, int64_t *h_ntri, int64_t *h_nvert, int64_t *h_total_tri,
                            int64_t *h_total_vert, void *stream) {
    CHR_XFER_SCOPE;
    return mc_count_impl(d_grids, h, n, k, nullptr, d_ws, ws_bytes, h_ntri, h_nvert, h_total_tri, h_total_vert,
                         stream);
}
extern "C" int chr_mc_count_masked(const double *d_grids, const chr_mc_grid_t *h, int64_t n, double k,
                                   const uint32_t *d_masks, void *d_ws, size_t ws_bytes, int64_t *h_ntri,
                                   int64_t *h_nvert, int64_t *h_total_tri, int64_t *h_total_vert, void *stream) {
    CHR_XFER_SCOPE;
    if (!d_masks) return CHR_E_PARAMETER;
    return mc_count_impl(d_grids, h, n, k, d_masks, d_ws, ws_bytes, h_ntri, h_nvert, h_total_tri, h_total_vert,
                         stream);
}
extern "C" int chr_mc_emit_masked(const double *d_grids, const chr_mc_grid_t *h, int64_t n, double k,
                                  const uint32_t *d_masks, void *d_ws, size_t ws_bytes, double *d_verts,
                                  int32_t *d_tris, void *stream) {
    CHR_XFER_SCOPE;
    if (!d_masks) return CHR_E_PARAMETER;
    return mc_emit_impl(d_grids, h, n, k, d_masks, d_ws, ws_bytes, d_verts, d_tris, nullptr, stream);
}

static int mc_count_impl(const double *d_grids, const chr_mc_grid_t *h, int64_t n, double k, const uint32_t *d_masks,
                         void *d_ws, size_t ws_bytes, int64_t *h_ntri, int64_t *h_nvert, int64_t *h_total_tri,
                         int64_t *h_total_vert, void *stream) {
    if (n == 0) {
        if (h_total_tri) *h_total_tri = 0;
        if (h_total_vert) *h_total_vert = 0;
        return CHR_OK;
    }
    if (!d_grids || !h || n < 0) return CHR_E_PARAMETER;
    cudaStream_t st = (cudaStream_t)stream;
    McPlan pl;
    if (!mc_build(h, n, pl)) return CHR_E_PARAMETER;
    mc_carve(pl, d_ws, ws_bytes);
    if (!d_ws || pl.ws > ws_bytes) return CHR_E_WORKSPACE;
    const McTables *T = mc_tables_device();
    if (!T) return CHR_E_CUDA;
    CHR_CUDA_TRY(h2d(pl.d_grids, pl.grids.data(), sizeof(McGrid) * n, st));
    CHR_CUDA_TRY(fill_async(pl.cnt, 0, sizeof(McPieceCnt) * (pl.npieces + 2), st));  // + the batch queues
    {
        CHR_PROF("k_mc_fill_map", st);
        k_mc_fill_map<<<(unsigned)n, 256, 0, st>>>(pl.d_grids, n, pl.item_grid, pl.chunk_grid, pl.mask_grid);
    }
    const uint32_t *masks = d_masks ? d_masks : pl.mask;  // caller's masks (decoder output) or our own
    if (!d_masks) {
        CHR_CUDA_TRY(fill_async(pl.mask + pl.nmask_words, 0, 8 * sizeof(uint32_t), st));
        if (pl.nmask_items > 0) {
            CHR_PROF("k_mc_mask", st);
            k_mc_mask<<<(unsigned)pl.nmask_items, 256, 0, st>>>(d_grids, pl.d_grids, pl.mask_grid, k, pl.mask);
        }
    }
    if (pl.nchunks > 0) {
        CHR_PROF("k_mc_count4", st);
        const int64_t nbatch = pl.nchunks * (MCH / 32);
        k_mc_count4<<<(unsigned)std::min<int64_t>(ceil_div(nbatch, 8), (int64_t)mc_num_sms() * 8), 256, 0, st>>>(
            pl.d_grids, pl.chunk_grid, T, masks, pl.cnt, pl.lmask, pl.cellw, mc_queue(pl) + 1, nbatch);
    }
    {
        CHR_PROF("k_mc_reduce", st);
        k_mc_reduce<<<(unsigned)pl.nchunks, 256, 0, st>>>(pl.cnt, pl.chunk);
    }
    {
        CHR_PROF("k_mc_grid_scan", st);
        k_mc_grid_scan<<<(unsigned)ceil_div(n, 4), 128, 0, st>>>(pl.d_grids, n, pl.chunk);
    }
    {
        CHR_PROF("k_mc_grids", st);
        k_mc_grids<<<1, 1024, 0, st>>>(pl.d_grids, n, pl.totals);
    }
    {
        CHR_PROF("k_mc_down", st);
        k_mc_down<<<(unsigned)pl.nchunks, 256, 0, st>>>(pl.cnt, pl.chunk, pl.base);
    }
    CHR_CUDA_TRY(cudaGetLastError());
    CHR_CUDA_TRY(d2h(pl.grids.data(), pl.d_grids, sizeof(McGrid) * n, st));
    CHR_CUDA_TRY(stream_sync(st));
    int64_t tt = 0, tv = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (h_ntri) h_ntri[i] = pl.grids[i].ntri;
        if (h_nvert) h_nvert[i] = pl.grids[i].nvert;
        tt += pl.grids[i].ntri;
        tv += pl.grids[i].nvert;
    }
    if (h_total_tri) *h_total_tri = tt;
    if (h_total_vert) *h_total_vert = tv;
    return CHR_OK;
}

extern "C" int chr_mc_emit(const double *d_grids, const chr_mc_grid_t *h, int64_t n, double k, void *d_ws,
                           size_t ws_bytes, double *d_verts, int32_t *d_tris, void *stream) {
    CHR_XFER_SCOPE;
    return mc_emit_impl(d_grids, h, n, k, nullptr, d_ws, ws_bytes, d_verts, d_tris, nullptr, stream);
}

// chr_mc_emit that also writes every vertex's canonical edge (grid-local
// ((z * ny + y) * nx + x) * 3 + axis, int64) -- the z-slab request matches
// vertices on the planes two ranks share by it
extern "C" int chr_mc_emit_edges(const double *d_grids, const chr_mc_grid_t *h, int64_t n, double k, void *d_ws,
                                 size_t ws_bytes, double *d_verts, int32_t *d_tris, int64_t *d_vedge, void *stream) {
    CHR_XFER_SCOPE;
    return mc_emit_impl(d_grids, h, n, k, nullptr, d_ws, ws_bytes, d_verts, d_tris, d_vedge, stream);
}

static int mc_emit_impl(const double *d_grids, const chr_mc_grid_t *h, int64_t n, double k, const uint32_t *d_masks,
                        void *d_ws, size_t ws_bytes, double *d_verts, int32_t *d_tris, int64_t *d_vedge,
                        void *stream) {
    if (n == 0) return CHR_OK;
    if (!d_grids || !h || n < 0) return CHR_E_PARAMETER;
    cudaStream_t st = (cudaStream_t)stream;
    McPlan pl;
    if (!mc_build(h, n, pl)) return CHR_E_PARAMETER;
    mc_carve(pl, d_ws, ws_bytes);
    if (!d_ws || pl.ws > ws_bytes) return CHR_E_WORKSPACE;
    const McTables *T = mc_tables_device();
    if (!T) return CHR_E_CUDA;
    if (pl.nchunks > 0) {
        const int64_t nbatch = pl.nchunks * (MCH / 32);
        const int64_t ctas = std::min<int64_t>(ceil_div(nbatch, E4W), (int64_t)mc_num_sms() * 6);
        CHR_PROF("k_mc_emit4", st);
        k_mc_emit4<<<(unsigned)ctas, E4W * 32, 0, st>>>(d_grids, pl.d_grids, pl.chunk_grid, k, T, pl.base, pl.lmask,
                                                        pl.cellw, mc_queue(pl), nbatch,
                                                        d_verts, d_tris, d_vedge);
    }
    CHR_CUDA_TRY(cudaGetLastError());
    CHR_CUDA_TRY(stream_sync(st));
    return CHR_OK;
}

extern "C" int chr_case_codes(const double *d_grid, int64_t nx, int64_t ny, int64_t nz, double k, int binary,
                              uint8_t *d_codes, void *stream) {
    CHR_XFER_SCOPE;
    if (!d_grid || !d_codes || nx < 2 || ny < 2 || nz < 2) return CHR_E_PARAMETER;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = (nx - 1) * (ny - 1) * (nz - 1);
    const int64_t blocks = std::min<int64_t>(ceil_div(n, 256), 148 * 32);
    {
        CHR_PROF("k_case_codes", st);
        k_case_codes<<<(unsigned)blocks, 256, 0, st>>>(d_grid, nx, ny, nz, k, binary, d_codes);
    }
    return cudaGetLastError() == cudaSuccess ? CHR_OK : CHR_E_CUDA;
}
