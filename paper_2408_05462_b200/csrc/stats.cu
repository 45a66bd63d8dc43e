// stats.cu -- step 1 of the hot path: block decomposition + min/max index
// + the strict accuracy-1 distance reduction, in one streaming read.
//
// Reference: blocking.py:64-111 (block_grid_shape, _window, decompose),
// blocking.py:114-127 (span test, done on the host from these extrema),
// bound.py:150-219 + kernels.py:417-425 (min |s-k| per region; here per
// block, the region value is the min over its blocks because block
// windows tile the region window), volume.py:71-74 (first non-finite
// flat index).
//
// Closed form used for the bound (verified against the
// oracle in tests): per sample, min_k |s - k| is attained at one of the two
// candidates bracketing s, because fl(s - k) is monotone in k.
#include "chr_internal.cuh"

namespace chr {

struct CandParams {
    double k[64];
    int m;
};

__device__ __forceinline__ double min_cand_dist(const double *k, int m, double s) {
    if (m == 1) return fabs(__dadd_rn(s, -k[0]));
    // first candidate > s
    int lo = 0, hi = m;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (k[mid] > s) hi = mid; else lo = mid + 1;
    }
    double d = INFINITY;
    if (lo > 0) d = fabs(__dadd_rn(s, -k[lo - 1]));
    if (lo < m) d = fmin(d, fabs(__dadd_rn(s, -k[lo])));
    return d;
}

template <typename T>
__device__ __forceinline__ bool is_finite_val(T v) {
    return isfinite(v);
}

// one CTA per block; warps stride over window rows, lanes over x
template <typename T>
__global__ void __launch_bounds__(256) k_stats(const T *__restrict__ vol, int64_t nx, int64_t ny,
                                               int64_t nz, int bs, int nbx, int nby,
                                               CandParams cp, double *__restrict__ stats,
                                               unsigned long long *__restrict__ first_bad) {
    __shared__ double ks[64];
    __shared__ double red[3][8];
    __shared__ unsigned long long bad_s;
    if (threadIdx.x < cp.m) ks[threadIdx.x] = cp.k[threadIdx.x];
    if (threadIdx.x == 0) bad_s = ~0ull;
    __syncthreads();
    const int m = cp.m;
    const int64_t id = blockIdx.x;
    const int bx = (int)(id % nbx);
    const int by = (int)((id / nbx) % nby);
    const int bz = (int)(id / ((int64_t)nbx * nby));
    const int64_t ox = (int64_t)bx * bs, oy = (int64_t)by * bs, oz = (int64_t)bz * bs;
    const int64_t ex = min((int64_t)(bx + 1) * bs, nx - 1) - ox + 1;
    const int64_t ey = min((int64_t)(by + 1) * bs, ny - 1) - oy + 1;
    const int64_t ez = min((int64_t)(bz + 1) * bs, nz - 1) - oz + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T lo = vol[(oz * ny + oy) * nx + ox], hi = lo;
    double dmin = INFINITY;
    bool bad = false;
    unsigned long long badidx = ~0ull;
    const int64_t rows = ey * ez;
    for (int64_t r = warp; r < rows; r += 8) {
        const int64_t y = r % ey, z = r / ey;
        const int64_t rowbase = ((oz + z) * ny + (oy + y)) * nx + ox;
        for (int64_t x = lane; x < ex; x += 32) {
            const T v = __ldg(vol + rowbase + x);
            if (!is_finite_val(v)) {
                bad = true;
                badidx = min(badidx, (unsigned long long)(rowbase + x));
                continue;
            }
            lo = v < lo ? v : lo;
            hi = v > hi ? v : hi;
            dmin = fmin(dmin, min_cand_dist(ks, m, (double)v));
        }
    }
    if (__any_sync(0xFFFFFFFFu, bad)) {
        for (int off = 16; off; off >>= 1) badidx = min(badidx, __shfl_xor_sync(0xFFFFFFFFu, badidx, off));
        if (lane == 0) atomicMin(&bad_s, badidx);
    }
    double dlo = (double)lo, dhi = (double)hi;
    for (int off = 16; off; off >>= 1) {
        dlo = fmin(dlo, __shfl_xor_sync(0xFFFFFFFFu, dlo, off));
        dhi = fmax(dhi, __shfl_xor_sync(0xFFFFFFFFu, dhi, off));
        dmin = fmin(dmin, __shfl_xor_sync(0xFFFFFFFFu, dmin, off));
    }
    if (lane == 0) {
        red[0][warp] = dlo;
        red[1][warp] = dhi;
        red[2][warp] = dmin;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) {
            dlo = fmin(dlo, red[0][w]);
            dhi = fmax(dhi, red[1][w]);
            dmin = fmin(dmin, red[2][w]);
        }
        stats[3 * id + 0] = dlo;
        stats[3 * id + 1] = dhi;
        stats[3 * id + 2] = dmin;
        if (bad_s != ~0ull) atomicMin(first_bad, bad_s);
    }
}

}  // namespace chr

using namespace chr;

extern "C" int64_t chr_num_blocks(int64_t nx, int64_t ny, int64_t nz, int64_t bs) {
    if (bs < 1) return 0;
    auto nb = [bs](int64_t d) { return d - 1 > 0 ? (d - 1 + bs - 1) / bs : (int64_t)1; };
    return nb(nx) * nb(ny) * nb(nz);
}

extern "C" int chr_stats(const void *d_vol, int dtype, int64_t nx, int64_t ny, int64_t nz,
                         int64_t bs, const double *h_cands, int m, double *d_block_stats,
                         int64_t *d_first_nonfinite, void *stream) {
    if (!d_vol || !d_block_stats || !d_first_nonfinite || !h_cands) return CHR_E_PARAMETER;
    if (bs < 2 || nx < 2 || ny < 2 || nz < 2 || m < 1 || m > 64) return CHR_E_PARAMETER;
    if (dtype != CHR_F32 && dtype != CHR_F64) return CHR_E_PARAMETER;
    cudaStream_t st = (cudaStream_t)stream;
    CandParams cp;
    cp.m = m;
    for (int i = 0; i < m; ++i) cp.k[i] = h_cands[i];
    const int nbx = (int)((nx - 1 + bs - 1) / bs), nby = (int)((ny - 1 + bs - 1) / bs);
    const int64_t nblocks = chr_num_blocks(nx, ny, nz, bs);
    CHR_CUDA_TRY(cudaMemsetAsync(d_first_nonfinite, 0xFF, sizeof(int64_t), st));
    auto *bad = reinterpret_cast<unsigned long long *>(d_first_nonfinite);
    if (dtype == CHR_F32)
        {
            CHR_PROF("k_stats<float>", st);
            k_stats<float><<<(unsigned)nblocks, 256, 0, st>>>((const float *)d_vol, nx, ny, nz, (int)bs,
                                                              nbx, nby, cp, d_block_stats, bad);
        }
    else
        {
            CHR_PROF("k_stats<double>", st);
            k_stats<double><<<(unsigned)nblocks, 256, 0, st>>>((const double *)d_vol, nx, ny, nz,
                                                               (int)bs, nbx, nby, cp, d_block_stats, bad);
        }
    return cudaGetLastError() == cudaSuccess ? CHR_OK : CHR_E_CUDA;
}
