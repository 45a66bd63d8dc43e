// bounds.cu -- SURVEY 8(f2): error bounds at accuracy < 1 and in
// paper_edges mode (bound.py:117-219).  For every served (region,
// candidate) pair the n-th smallest distance of the pair's multiset D:
//   strict_vertices: |s - k| over the region window (n_R values);
//   paper_edges:     k - s0 and s1 - k for every axis-aligned window edge
//                    with s0 < k < s1 (bound.py:68-83).
// n = max(1, 1 + floor((1 - accuracy) * |D|)) (bound.py:117-120).
// Device algorithm: segmented radix select over the f64 bit patterns
// (non-negative doubles order like their uint64 patterns), 8 passes of
// 8-bit digits, most significant first; each pass histograms the values
// that still match the selected prefix (CTA = (pair, 64K-sample chunk),
// shared-memory histogram, one atomic per bin) and a warp per pair picks
// the digit holding the n-th value.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "chr_internal.cuh"

namespace chr {

constexpr int64_t SEL_CHUNK = 65536;

struct SelPair {
    int32_t ox, oy, oz, ex, ey, ez;  // window (volume coords)
    double k;
    int64_t item_base, nitems;
    int64_t count;                    // |D|
    int64_t n;                        // rank still to find (1-based)
    uint64_t prefix;                  // selected high bits
};

template <typename T>
__device__ __forceinline__ double vat(const T *vol, int64_t NX, int64_t NY, const SelPair &P, int x, int y, int z) {
    return (double)__ldg(vol + ((int64_t)(P.oz + z) * NY + (P.oy + y)) * NX + P.ox + x);
}

// visit the distances of one window sample (strict: 1, paper: <= 6)
template <typename T, typename F>
__device__ __forceinline__ void sample_distances(const T *vol, int64_t NX, int64_t NY, const SelPair &P, int64_t s,
                                                 int paper, F &&f) {
    const int64_t plane = (int64_t)P.ex * P.ey;
    const int z = (int)(s / plane);
    const int64_t r = s - (int64_t)z * plane;
    const int y = (int)(r / P.ex), x = (int)(r - (int64_t)y * P.ex);
    const double a = vat(vol, NX, NY, P, x, y, z);
    if (!paper) {
        f(fabs(__dadd_rn(a, -P.k)));
        return;
    }
    auto edge = [&](double b) {
        const double s0 = fmin(a, b), s1 = fmax(a, b);
        if (s0 < P.k && P.k < s1) {
            f(__dadd_rn(P.k, -s0));
            f(__dadd_rn(s1, -P.k));
        }
    };
    if (x + 1 < P.ex) edge(vat(vol, NX, NY, P, x + 1, y, z));
    if (y + 1 < P.ey) edge(vat(vol, NX, NY, P, x, y + 1, z));
    if (z + 1 < P.ez) edge(vat(vol, NX, NY, P, x, y, z + 1));
}

__device__ __forceinline__ int64_t find_pair(const SelPair *__restrict__ pairs, int64_t np, int64_t item) {
    int64_t lo = 0, hi = np - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (pairs[mid].item_base <= item) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// |D| of paper_edges pairs
template <typename T>
__global__ void __launch_bounds__(256) k_sel_count(const T *__restrict__ vol, int64_t NX, int64_t NY,
                                                   SelPair *__restrict__ pairs, int64_t np) {
    __shared__ int64_t sp;
    if (threadIdx.x == 0) sp = find_pair(pairs, np, blockIdx.x);
    __syncthreads();
    SelPair &P = pairs[sp];
    const int64_t n = (int64_t)P.ex * P.ey * P.ez;
    const int64_t s0 = (blockIdx.x - P.item_base) * SEL_CHUNK, s1 = min(n, s0 + SEL_CHUNK);
    unsigned long long c = 0;
    for (int64_t s = s0 + threadIdx.x; s < s1; s += blockDim.x)
        sample_distances(vol, NX, NY, P, s, 1, [&](double) { ++c; });
    for (int off = 16; off; off >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, off);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(reinterpret_cast<unsigned long long *>(&P.count), c);
}

template <typename T>
__global__ void __launch_bounds__(256) k_sel_hist(const T *__restrict__ vol, int64_t NX, int64_t NY,
                                                  const SelPair *__restrict__ pairs, int64_t np, int paper, int shift,
                                                  unsigned long long *__restrict__ hist) {
    __shared__ unsigned int h[256];
    __shared__ int64_t sp;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    if (threadIdx.x == 0) sp = find_pair(pairs, np, blockIdx.x);
    __syncthreads();
    const SelPair &P = pairs[sp];
    if (P.count > 0) {
        const int64_t n = (int64_t)P.ex * P.ey * P.ez;
        const int64_t s0 = (blockIdx.x - P.item_base) * SEL_CHUNK, s1 = min(n, s0 + SEL_CHUNK);
        const uint64_t hi_mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
        const uint64_t want = P.prefix & hi_mask;
        for (int64_t s = s0 + threadIdx.x; s < s1; s += blockDim.x)
            sample_distances(vol, NX, NY, P, s, paper, [&](double d) {
                const uint64_t b = (uint64_t)__double_as_longlong(d);
                if ((b & hi_mask) == want) atomicAdd(&h[(b >> shift) & 255u], 1u);
            });
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (h[i]) atomicAdd(hist + sp * 256 + i, (unsigned long long)h[i]);
}

// warp per pair: the digit holding the n-th value; clear the histogram
__global__ void k_sel_pick(SelPair *__restrict__ pairs, int64_t np, int shift, unsigned long long *__restrict__ hist) {
    const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (p >= np) return;
    SelPair &P = pairs[p];
    unsigned long long c[8], tot = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        c[i] = hist[p * 256 + lane * 8 + i];
        hist[p * 256 + lane * 8 + i] = 0;
        tot += c[i];
    }
    unsigned long long inc = tot;
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned long long o = __shfl_up_sync(0xFFFFFFFFu, inc, off);
        if (lane >= off) inc += o;
    }
    if (P.count <= 0) return;
    unsigned long long before = inc - tot;  // values in digits < lane * 8
    const unsigned long long n = (unsigned long long)P.n;
    if (before < n && n <= inc) {  // the n-th value's digit is in this lane's 8
        for (int i = 0; i < 8; ++i) {
            if (n <= before + c[i]) {
                P.prefix |= (uint64_t)(lane * 8 + i) << shift;
                P.n = (int64_t)(n - before);
                break;
            }
            before += c[i];
        }
    }
}

__global__ void k_sel_init_n(SelPair *__restrict__ pairs, int64_t np, double accuracy) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= np) return;
    SelPair &P = pairs[p];
    // select_index (bound.py:117-120): max(1, 1 + floor((1 - accuracy) * |D|))
    const double f = floor(__dmul_rn(__dadd_rn(1.0, -accuracy), (double)P.count));
    P.n = max((int64_t)1, (int64_t)1 + (int64_t)f);
    P.prefix = 0;
}

}  // namespace chr

using namespace chr;

static bool sel_build(const int32_t *h_windows, const double *h_k, int64_t np, std::vector<SelPair> &v,
                      int64_t &items) {
    v.resize(np);
    items = 0;
    for (int64_t i = 0; i < np; ++i) {
        SelPair &P = v[i];
        std::memset(&P, 0, sizeof(P));
        P.ox = h_windows[6 * i];
        P.oy = h_windows[6 * i + 1];
        P.oz = h_windows[6 * i + 2];
        P.ex = h_windows[6 * i + 3];
        P.ey = h_windows[6 * i + 4];
        P.ez = h_windows[6 * i + 5];
        if (P.ex < 1 || P.ey < 1 || P.ez < 1) return false;
        P.k = h_k[i];
        P.item_base = items;
        P.nitems = ceil_div((int64_t)P.ex * P.ey * P.ez, SEL_CHUNK);
        items += P.nitems;
    }
    return true;
}

extern "C" size_t chr_select_workspace_size(int64_t n_pairs) {
    CHR_XFER_SCOPE;
    return (size_t)n_pairs * (sizeof(SelPair) + 256 * 8) + 1024;
}

// h_windows: [n_pairs][ox, oy, oz, ex, ey, ez]; h_k: candidate per pair;
// mode 0 strict_vertices, 1 paper_edges.  Outputs: h_value = n-th smallest
// distance (or -1 when |D| == 0), h_count = |D|, h_n = n.
extern "C" int chr_select_distances(const void *d_vol, int dtype, int64_t nx, int64_t ny, int64_t nz,
                                    const int32_t *h_windows, const double *h_k, int64_t n_pairs, double accuracy,
                                    int mode, void *d_ws, size_t ws_bytes, double *h_value, int64_t *h_count,
                                    int64_t *h_n, void *stream) {
    CHR_XFER_SCOPE;
    if (n_pairs == 0) return CHR_OK;
    if (!d_vol || !h_windows || !h_k || !h_value || !(accuracy > 0.0 && accuracy <= 1.0) || mode < 0 || mode > 1)
        return CHR_E_PARAMETER;
    if (dtype != CHR_F32 && dtype != CHR_F64) return CHR_E_PARAMETER;
    if (!d_ws || ws_bytes < chr_select_workspace_size(n_pairs)) return CHR_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    std::vector<SelPair> v;
    int64_t items = 0;
    if (!sel_build(h_windows, h_k, n_pairs, v, items)) return CHR_E_PARAMETER;
    for (const SelPair &P : v)
        if (P.ox < 0 || P.oy < 0 || P.oz < 0 || P.ox + P.ex > nx || P.oy + P.ey > ny || P.oz + P.ez > nz)
            return CHR_E_PARAMETER;
    if (mode == 0)
        for (SelPair &P : v) P.count = (int64_t)P.ex * P.ey * P.ez;
    SelPair *d_pairs = reinterpret_cast<SelPair *>(d_ws);
    unsigned long long *d_hist =
        reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(d_ws) + (size_t)n_pairs * sizeof(SelPair));
    CHR_CUDA_TRY(h2d(d_pairs, v.data(), sizeof(SelPair) * n_pairs, st));
    CHR_CUDA_TRY(fill_async(d_hist, 0, sizeof(unsigned long long) * 256 * n_pairs, st));
    const unsigned nit = (unsigned)items, pick = (unsigned)ceil_div(n_pairs, 4);
    if (mode == 1) {
        CHR_PROF("k_sel_count", st);
        if (dtype == CHR_F32) k_sel_count<float><<<nit, 256, 0, st>>>((const float *)d_vol, nx, ny, d_pairs, n_pairs);
        else k_sel_count<double><<<nit, 256, 0, st>>>((const double *)d_vol, nx, ny, d_pairs, n_pairs);
    }
    k_sel_init_n<<<(unsigned)ceil_div(n_pairs, 128), 128, 0, st>>>(d_pairs, n_pairs, accuracy);
    for (int shift = 56; shift >= 0; shift -= 8) {
        {
            CHR_PROF("k_sel_hist", st);
            if (dtype == CHR_F32)
                k_sel_hist<float><<<nit, 256, 0, st>>>((const float *)d_vol, nx, ny, d_pairs, n_pairs, mode, shift,
                                                       d_hist);
            else
                k_sel_hist<double><<<nit, 256, 0, st>>>((const double *)d_vol, nx, ny, d_pairs, n_pairs, mode, shift,
                                                        d_hist);
        }
        k_sel_pick<<<pick, 128, 0, st>>>(d_pairs, n_pairs, shift, d_hist);
    }
    CHR_CUDA_TRY(cudaGetLastError());
    CHR_CUDA_TRY(d2h(v.data(), d_pairs, sizeof(SelPair) * n_pairs, st));
    CHR_CUDA_TRY(stream_sync(st));
    for (int64_t i = 0; i < n_pairs; ++i) {
        double d;
        std::memcpy(&d, &v[i].prefix, 8);
        h_value[i] = v[i].count > 0 ? d : -1.0;
        if (h_count) h_count[i] = v[i].count;
        if (h_n) h_n[i] = v[i].count > 0 ? std::max<int64_t>(1, 1 + (int64_t)std::floor((1.0 - accuracy) * (double)v[i].count)) : 0;
    }
    return CHR_OK;
}
