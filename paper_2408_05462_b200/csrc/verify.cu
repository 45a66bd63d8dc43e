// verify.cu -- SURVEY 8(f3): owner-wins stitch of request windows
// (chr_archive.stitch, chr_archive.py:277-294) and the case-code
// comparison behind verify_topology (isosurf.py:91-114), on the device.
//
// stitch: the reference writes the windows in descending (z, y, x) origin
// order so the LOWEST origin lands last.  Here every sample is written
// exactly once, by its owner: the selected region with the lowest origin
// whose window covers it.  A sample at g lies in the windows of the blocks
// b with b*bs <= g <= min((b+1)*bs, d-1) -- at most two per axis -- so the
// owner is a min over <= 8 entries of a per-block priority map (the rank of
// the block's region by origin, INT32_MAX for unselected blocks).  One pass,
// no atomics: read the window (8 B), write the owned samples (8 B).
//
// compare: a sample "flips" when (a >= k) != (b >= k); a cell's binary
// case code differs iff any of its 8 corners flips.  32x8-cell tiles march
// z with the flip plane in shared memory (double-buffered, one barrier per
// plane); per-CTA counts + the smallest differing cell index.
#include <algorithm>
#include <climits>
#include <cstring>
#include <vector>

#include "chr_internal.cuh"

namespace chr {

struct StitchDev {
    uint64_t win_off;    // window start in the windows buffer (samples)
    int32_t ox, oy, oz;  // origin
    int32_t ex, ey, ez;  // extent
    int32_t prio;        // rank by (z, y, x) origin, ascending
    int32_t pad;
    int64_t row_base;    // first row (of ey*ez) in the launch
};

__device__ __forceinline__ void cover(int g, int bs, int nb, int &lo, int &hi) {
    hi = min(g / bs, nb - 1);
    lo = (g % bs == 0 && g > 0) ? g / bs - 1 : hi;
    lo = min(lo, hi);
}

// warp per window row
__global__ void __launch_bounds__(256) k_stitch(const double *__restrict__ wins, const StitchDev *__restrict__ tab,
                                                int64_t n, int64_t total_rows, const int32_t *__restrict__ bprio,
                                                int64_t NX, int64_t NY, int bs, int nbx, int nby, int nbz,
                                                double *__restrict__ out) {
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= total_rows) return;
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (__ldg(&tab[mid].row_base) <= row) lo = mid; else hi = mid - 1;
    }
    const StitchDev &W = tab[lo];
    const int64_t r = row - W.row_base;
    const int y = (int)(r % W.ey), z = (int)(r / W.ey);
    const int gy = W.oy + y, gz = W.oz + z;
    int ylo, yhi, zlo, zhi;
    cover(gy, bs, nby, ylo, yhi);
    cover(gz, bs, nbz, zlo, zhi);
    const double *src = wins + W.win_off + ((int64_t)z * W.ey + y) * W.ex;
    double *dst = out + ((int64_t)gz * NY + gy) * NX + W.ox;
    for (int x = lane; x < W.ex; x += 32) {
        const int gx = W.ox + x;
        int xlo, xhi;
        cover(gx, bs, nbx, xlo, xhi);
        int best = INT_MAX;
        for (int bz = zlo; bz <= zhi; ++bz)
            for (int by = ylo; by <= yhi; ++by)
                for (int bx = xlo; bx <= xhi; ++bx)
                    best = min(best, __ldg(bprio + ((int64_t)bz * nby + by) * nbx + bx));
        if (best == W.prio) dst[x] = __ldg(src + x);
    }
}

constexpr int TX = 32, TY = 8, TZ = 16;

template <typename TA, typename TB>
__global__ void __launch_bounds__(TX *TY) k_topo_compare(const TA *__restrict__ a, const TB *__restrict__ b,
                                                         int64_t NX, int64_t NY, int64_t NZ, double k,
                                                         unsigned long long *__restrict__ ndiff,
                                                         unsigned long long *__restrict__ first) {
    __shared__ uint8_t F[2][TY + 1][TX + 1];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t x = (int64_t)blockIdx.x * TX + tx, y = (int64_t)blockIdx.y * TY + ty;
    const int64_t z0 = (int64_t)blockIdx.z * TZ, z1 = min(z0 + TZ, NZ - 1);  // cells [z0, z1)
    const int64_t plane = NX * NY;
    auto flip = [&](int64_t xx, int64_t yy, int64_t zz) -> uint8_t {
        if (xx >= NX || yy >= NY) return 0;
        const int64_t i = zz * plane + yy * NX + xx;
        return (uint8_t)(((double)__ldg(a + i) >= k) != ((double)__ldg(b + i) >= k));
    };
    const bool cell_ok = x < NX - 1 && y < NY - 1;
    unsigned long long cnt = 0, fst = ~0ull;
    uint8_t cprev = 0;
    for (int64_t z = z0; z <= z1; ++z) {
        uint8_t(*P)[TX + 1] = F[z & 1];
        P[ty][tx] = flip(x, y, z);
        if (tx == TX - 1) P[ty][TX] = flip(x + 1, y, z);
        if (ty == TY - 1) P[TY][tx] = flip(x, y + 1, z);
        if (tx == TX - 1 && ty == TY - 1) P[TY][TX] = flip(x + 1, y + 1, z);
        __syncthreads();
        const uint8_t c = P[ty][tx] | P[ty][tx + 1] | P[ty + 1][tx] | P[ty + 1][tx + 1];
        if (z > z0 && cell_ok && (c | cprev)) {
            ++cnt;
            const unsigned long long id = (unsigned long long)(((z - 1) * (NY - 1) + y) * (NX - 1) + x);
            fst = min(fst, id);
        }
        cprev = c;
    }
    for (int off = 16; off; off >>= 1) {
        cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, off);
        fst = min(fst, __shfl_xor_sync(0xFFFFFFFFu, fst, off));
    }
    if (tx == 0 && cnt) {
        atomicAdd(ndiff, cnt);
        atomicMin(first, fst);
    }
}

}  // namespace chr

using namespace chr;

extern "C" size_t chr_stitch_workspace_size(int64_t n_windows, int64_t nx, int64_t ny, int64_t nz, int64_t bs) {
    CHR_XFER_SCOPE;
    if (bs < 1) return 0;
    auto nb = [&](int64_t d) { return std::max<int64_t>(1, (d - 1 + bs - 1) / bs); };
    return (size_t)n_windows * sizeof(StitchDev) + (size_t)nb(nx) * nb(ny) * nb(nz) * 4 + 1024;
}

extern "C" int chr_stitch(const double *d_windows, const chr_stitch_t *h_windows, int64_t n, int64_t nx, int64_t ny,
                          int64_t nz, int64_t bs, void *d_ws, size_t ws_bytes, double *d_out, void *stream) {
    CHR_XFER_SCOPE;
    if (n == 0) return CHR_OK;
    if (!d_windows || !h_windows || !d_out || bs < 1 || nx < 1 || ny < 1 || nz < 1) return CHR_E_PARAMETER;
    if (!d_ws || ws_bytes < chr_stitch_workspace_size(n, nx, ny, nz, bs)) return CHR_E_WORKSPACE;
    const int64_t d3[3] = {nx, ny, nz};
    int64_t nb[3];
    for (int a = 0; a < 3; ++a) nb[a] = std::max<int64_t>(1, (d3[a] - 1 + bs - 1) / bs);
    std::vector<int64_t> order(n);
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    auto key = [&](int64_t i) {
        const chr_stitch_t &w = h_windows[i];
        return std::make_tuple(w.origin[2], w.origin[1], w.origin[0]);
    };
    std::stable_sort(order.begin(), order.end(), [&](int64_t p, int64_t q) { return key(p) < key(q); });
    std::vector<StitchDev> tab(n);
    std::vector<int32_t> prio((size_t)(nb[0] * nb[1] * nb[2]), INT32_MAX);
    int64_t rows = 0;
    for (int64_t rk = 0; rk < n; ++rk) {
        const int64_t i = order[rk];
        const chr_stitch_t &w = h_windows[i];
        for (int a = 0; a < 3; ++a) {
            if (w.origin[a] < 0 || w.extent[a] < 1 || w.origin[a] + (int64_t)w.extent[a] > d3[a]) return CHR_E_PARAMETER;
            if (w.block_lo[a] < 0 || w.block_hi[a] < w.block_lo[a] || w.block_hi[a] >= nb[a]) return CHR_E_PARAMETER;
        }
        StitchDev &S = tab[i];
        std::memset(&S, 0, sizeof(S));
        S.win_off = w.window_offset;
        S.ox = w.origin[0];
        S.oy = w.origin[1];
        S.oz = w.origin[2];
        S.ex = w.extent[0];
        S.ey = w.extent[1];
        S.ez = w.extent[2];
        S.prio = (int32_t)rk;
        for (int bz = w.block_lo[2]; bz <= w.block_hi[2]; ++bz)
            for (int by = w.block_lo[1]; by <= w.block_hi[1]; ++by)
                for (int bx = w.block_lo[0]; bx <= w.block_hi[0]; ++bx) {
                    int32_t &p = prio[(size_t)((bz * nb[1] + by) * nb[0] + bx)];
                    p = std::min(p, (int32_t)rk);
                }
    }
    for (int64_t i = 0; i < n; ++i) {  // row prefix in table order
        tab[i].row_base = rows;
        rows += (int64_t)tab[i].ey * tab[i].ez;
    }
    cudaStream_t st = (cudaStream_t)stream;
    StitchDev *d_tab = reinterpret_cast<StitchDev *>(d_ws);
    int32_t *d_prio = reinterpret_cast<int32_t *>(reinterpret_cast<char *>(d_ws) + n * sizeof(StitchDev));
    CHR_CUDA_TRY(h2d(d_tab, tab.data(), n * sizeof(StitchDev), st));
    CHR_CUDA_TRY(h2d(d_prio, prio.data(), prio.size() * 4, st));
    {
        CHR_PROF("k_stitch", st);
        k_stitch<<<(unsigned)ceil_div(rows, 8), 256, 0, st>>>(d_windows, d_tab, n, rows, d_prio, nx, ny, (int)bs,
                                                              (int)nb[0], (int)nb[1], (int)nb[2], d_out);
    }
    CHR_CUDA_TRY(cudaGetLastError());
    return CHR_OK;
}

extern "C" int chr_topology_compare(const void *d_a, int dtype_a, const void *d_b, int dtype_b, int64_t nx,
                                    int64_t ny, int64_t nz, double k, void *d_ws, size_t ws_bytes,
                                    uint64_t *h_ndiff, int64_t *h_first, void *stream) {
    CHR_XFER_SCOPE;
    if (!d_a || !d_b || !h_ndiff || !h_first || nx < 2 || ny < 2 || nz < 2) return CHR_E_PARAMETER;
    if ((dtype_a != CHR_F32 && dtype_a != CHR_F64) || (dtype_b != CHR_F32 && dtype_b != CHR_F64))
        return CHR_E_PARAMETER;
    if (!d_ws || ws_bytes < 16) return CHR_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long *d_res = reinterpret_cast<unsigned long long *>(d_ws);
    const unsigned long long init[2] = {0ull, ~0ull};
    CHR_CUDA_TRY(h2d(d_res, init, 16, st));
    const dim3 grid((unsigned)ceil_div(nx - 1, TX), (unsigned)ceil_div(ny - 1, TY), (unsigned)ceil_div(nz - 1, TZ));
    {
        CHR_PROF("k_topo_compare", st);
#define CHR_TOPO(TA, TB) \
    k_topo_compare<TA, TB><<<grid, TX * TY, 0, st>>>((const TA *)d_a, (const TB *)d_b, nx, ny, nz, k, d_res, d_res + 1)
        if (dtype_a == CHR_F32 && dtype_b == CHR_F32) CHR_TOPO(float, float);
        else if (dtype_a == CHR_F32) CHR_TOPO(float, double);
        else if (dtype_b == CHR_F32) CHR_TOPO(double, float);
        else CHR_TOPO(double, double);
#undef CHR_TOPO
    }
    CHR_CUDA_TRY(cudaGetLastError());
    unsigned long long res[2];
    CHR_CUDA_TRY(d2h(res, d_res, 16, st));
    CHR_CUDA_TRY(stream_sync(st));
    *h_ndiff = res[0];
    *h_first = res[0] ? (int64_t)res[1] : -1;
    return CHR_OK;
}
