// slab.cu -- the z-slab request: finishing a rank's portion
// of a region window.  A portion's tokens are decoded with e = 1/2, so the
// decoder writes u_local (the 3D inclusive prefix of the portion's quanta,
// an exact integer in f64); the true u adds the z-carry plane C (u at the
// plane before the portion: the sum of the earlier portions' last-plane
// u_local, all-gathered), and recon = u * 2e exactly as the single-GPU
// decoder computes it (kernels.py:131-166: recon = u * 2e after the prefix).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "chr_internal.cuh"

namespace chr {

struct PortionDev {
    uint64_t out_offset;   // first sample of the portion in the windows buffer
    int64_t plane;         // samples per plane (ex * ey)
    int64_t nplanes;
    int64_t carry_offset;  // int64 carry plane in d_carry, -1: none (first portion)
    double twoe;
};

__global__ void __launch_bounds__(256) k_portion_finish(double *__restrict__ w, const PortionDev *__restrict__ tab,
                                                        int64_t n, const int64_t *__restrict__ carry) {
    for (int64_t p = blockIdx.y; p < n; p += gridDim.y) {
        const PortionDev P = tab[p];
        const int64_t cnt = P.plane * P.nplanes;
        double *o = w + P.out_offset;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
            int64_t u = __double2ll_rn(o[i]);
            if (P.carry_offset >= 0) u += __ldg(carry + P.carry_offset + i % P.plane);
            o[i] = __dmul_rn((double)u, P.twoe);
        }
    }
}

}  // namespace chr

using namespace chr;

extern "C" int chr_portion_finish(double *d_windows, const uint64_t *h_out_offset, const int64_t *h_plane,
                                  const int64_t *h_nplanes, const int64_t *h_carry_offset, const double *h_error_bound,
                                  int64_t n, const int64_t *d_carry, void *d_ws, size_t ws_bytes, void *stream) {
    CHR_XFER_SCOPE;
    if (n == 0) return CHR_OK;
    if (!d_windows || n < 0 || !h_out_offset || !h_plane || !h_nplanes || !h_carry_offset || !h_error_bound)
        return CHR_E_PARAMETER;
    if (!d_ws || ws_bytes < sizeof(PortionDev) * (size_t)n) return CHR_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    std::vector<PortionDev> t((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        if (h_plane[i] < 1 || h_nplanes[i] < 0 || (h_carry_offset[i] >= 0 && !d_carry)) return CHR_E_PARAMETER;
        t[i].out_offset = h_out_offset[i];
        t[i].plane = h_plane[i];
        t[i].nplanes = h_nplanes[i];
        t[i].carry_offset = h_carry_offset[i];
        t[i].twoe = 2.0 * h_error_bound[i];
    }
    PortionDev *d_tab = reinterpret_cast<PortionDev *>(d_ws);
    CHR_CUDA_TRY(h2d(d_tab, t.data(), sizeof(PortionDev) * (size_t)n, st));
    {
        CHR_PROF("k_portion_finish", st);
        k_portion_finish<<<dim3(64, (unsigned)std::min<int64_t>(n, 65535)), 256, 0, st>>>(d_windows, d_tab, n, d_carry);
    }
    return cudaGetLastError() == cudaSuccess ? CHR_OK : CHR_E_CUDA;
}

namespace chr {

// segment table entry: dst[dst_off, +len) <- src_k[src_off, +len) (k = src)
struct CopySeg {
    uint64_t dst_off, src_off, len;
    uint64_t src;
};

// bytes; one CTA per segment (grid-stride over long ones)
__global__ void __launch_bounds__(256) k_copy_segments(uint8_t *__restrict__ dst, const uint8_t *__restrict__ s0,
                                                       const uint8_t *__restrict__ s1, const CopySeg *__restrict__ t,
                                                       int64_t n) {
    for (int64_t i = blockIdx.y; i < n; i += gridDim.y) {
        const CopySeg S = t[i];
        const uint8_t *src = (S.src ? s1 : s0) + S.src_off;
        uint8_t *d = dst + S.dst_off;
        if ((((uintptr_t)src | (uintptr_t)d | S.len) & 7) == 0) {  // f64 planes: 8-byte moves
            const uint64_t *s8 = reinterpret_cast<const uint64_t *>(src);
            uint64_t *d8 = reinterpret_cast<uint64_t *>(d);
            for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < S.len / 8;
                 j += (uint64_t)gridDim.x * blockDim.x)
                d8[j] = __ldg(s8 + j);
            continue;
        }
        for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < S.len; j += (uint64_t)gridDim.x * blockDim.x)
            d[j] = __ldg(src + j);
    }
}

// bytes, word-granular: thread per aligned 4-byte word of the destination
// range covered by the (sorted, adjacent) segments; each byte is looked up
// in its segment (binary search over the segment starts) -- one aligned store
// per word, no two threads touch the same word
__global__ void __launch_bounds__(256) k_gather_words(uint8_t *__restrict__ dst, const uint8_t *__restrict__ s0,
                                                      const uint8_t *__restrict__ s1, const CopySeg *__restrict__ t,
                                                      int64_t n, uint64_t lo, uint64_t hi) {
    const uint64_t w0 = lo >> 2, w1 = (hi + 3) >> 2;
    for (uint64_t w = w0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < w1;
         w += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t word = 0, keep = 0;
        int64_t a = 0, b = n - 1;
        const uint64_t first = w << 2;
        while (a < b) {  // last segment starting at or before the word's first byte
            const int64_t m = (a + b + 1) >> 1;
            if (t[m].dst_off <= first) a = m; else b = m - 1;
        }
        int64_t si = a;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint64_t d = first + k;
            while (si + 1 < n && t[si + 1].dst_off <= d) ++si;
            const CopySeg S = t[si];
            if (d >= S.dst_off && d < S.dst_off + S.len) {
                const uint8_t v = __ldg((S.src ? s1 : s0) + S.src_off + (d - S.dst_off));
                word |= (uint32_t)v << (8 * k);
                keep |= 0xFFu << (8 * k);
            }
        }
        uint32_t *p = reinterpret_cast<uint32_t *>(dst) + w;
        if (keep == 0xFFFFFFFFu) *p = word;
        else if (keep) *p = (*p & ~keep) | word;  // the range's edge words: bytes outside it keep their value
    }
}

// int64 elements: dst[dst_off + j] += src[src_off + j] (segments may share a
// destination: 64-bit atomic adds, two's complement wraps like int64 sums)
__global__ void __launch_bounds__(256) k_add_segments(long long *__restrict__ dst, const long long *__restrict__ src,
                                                      const CopySeg *__restrict__ t, int64_t n) {
    for (int64_t i = blockIdx.y; i < n; i += gridDim.y) {
        const CopySeg S = t[i];
        for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < S.len; j += (uint64_t)gridDim.x * blockDim.x)
            atomicAdd(reinterpret_cast<unsigned long long *>(dst + S.dst_off + j),
                      (unsigned long long)__ldg(src + S.src_off + j));
    }
}

}  // namespace chr

// n segments (h_table: 4 u64 each = dst offset, src offset, length, source
// 0/1) copied from d_src0 / d_src1 into d_dst, one launch (z-slab request:
// re-framed token streams, packed planes).  elem = 1: bytes; elem = 8: the
// offsets and lengths count int64 elements and the segments ADD into d_dst.
extern "C" int chr_copy_segments(void *d_dst, const void *d_src0, const void *d_src1, const uint64_t *h_table,
                                 int64_t n, int elem, void *d_ws, size_t ws_bytes, void *stream) {
    CHR_XFER_SCOPE;
    if (n == 0) return CHR_OK;
    if (!d_dst || !h_table || n < 0 || (elem != 1 && elem != 8)) return CHR_E_PARAMETER;
    if (!d_ws || ws_bytes < sizeof(CopySeg) * (size_t)n) return CHR_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    CopySeg *d_t = reinterpret_cast<CopySeg *>(d_ws);
    CHR_CUDA_TRY(h2d(d_t, h_table, sizeof(CopySeg) * (size_t)n, st));
    const dim3 grid(16, (unsigned)std::min<int64_t>(n, 65535));
    bool gather = elem == 1 && ((uintptr_t)d_dst & 3) == 0;
    uint64_t lo = ~0ull, hi = 0, tot = 0;
    for (int64_t i = 0; gather && i < n; ++i) {  // sorted, non-overlapping destinations: word gather
        const uint64_t a = h_table[4 * i], b = a + h_table[4 * i + 2];
        if (i && a < h_table[4 * (i - 1)] + h_table[4 * (i - 1) + 2]) gather = false;
        lo = std::min(lo, a);
        hi = std::max(hi, b);
        tot += b - a;
    }
    if (gather && hi > lo && 2 * tot >= hi - lo) {  // dense (re-framed streams): word gather
        CHR_PROF("k_gather_words", st);
        const uint64_t words = ((hi + 3) >> 2) - (lo >> 2);
        k_gather_words<<<(unsigned)std::min<uint64_t>((words + 255) / 256, 148 * 16), 256, 0, st>>>(
            (uint8_t *)d_dst, (const uint8_t *)d_src0, (const uint8_t *)d_src1, d_t, n, lo, hi);
    } else if (elem == 1) {
        CHR_PROF("k_copy_segments", st);
        k_copy_segments<<<grid, 256, 0, st>>>((uint8_t *)d_dst, (const uint8_t *)d_src0, (const uint8_t *)d_src1, d_t,
                                              n);
    } else {
        CHR_PROF("k_add_segments", st);
        k_add_segments<<<grid, 256, 0, st>>>((long long *)d_dst, (const long long *)d_src0, d_t, n);
    }
    return cudaGetLastError() == cudaSuccess ? CHR_OK : CHR_E_CUDA;
}

namespace chr {

// one marching-cubes grid of the z-slab request (request_extract_portions)
struct SlabGrid {
    int64_t vbase, vend;     // its vertices in the merged local arrays
    int64_t halo_lim;        // drop x/y vertices with edge id < halo_lim (3 * plane on a halo grid, else 0)
    int64_t top_lo;          // export x/y vertices with edge id >= top_lo (top plane; INT64_MAX if none)
    int64_t key_base;        // selection index * key multiplier
    int64_t gid_base;        // global id of the grid's first kept vertex - its kept-prefix start
};

__device__ __forceinline__ int slab_grid_of(const SlabGrid *__restrict__ g, int ng, int64_t v) {
    int a = 0, b = ng - 1;
    while (a < b) {
        const int m = (a + b + 1) >> 1;
        if (g[m].vbase <= v) a = m; else b = m - 1;
    }
    return a;
}

// flags: bit 0 = dropped (a halo-plane x/y vertex the previous rank created),
// bit 1 = exported (a top-plane x/y vertex the next rank refers to); key =
// (selection, in-plane edge) of either kind; per-grid drop / export counts
__global__ void __launch_bounds__(256) k_slab_classify(const int64_t *__restrict__ vedge, int64_t nv,
                                                       const SlabGrid *__restrict__ g, int ng,
                                                       int8_t *__restrict__ flags, int64_t *__restrict__ key,
                                                       unsigned long long *__restrict__ counts) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
        const int gi = slab_grid_of(g, ng, v);
        const SlabGrid G = g[gi];
        const int64_t e = vedge[v];
        const bool xy = e % 3 != 2;
        const bool drop = xy && e < G.halo_lim;
        const bool top = xy && !drop && e >= G.top_lo;
        flags[v] = (int8_t)((drop ? 1 : 0) | (top ? 2 : 0));
        key[v] = drop ? G.key_base + e : (top ? G.key_base + e - G.top_lo : -1);
        if (drop) atomicAdd(counts + 2 * gi, 1ull);
        if (top) atomicAdd(counts + 2 * gi + 1, 1ull);
    }
}

// global ids of the kept vertices: gid = grid base + (kept vertices before v)
__global__ void __launch_bounds__(256) k_slab_gid(const int64_t *__restrict__ kept_incl, int64_t nv,
                                                  const SlabGrid *__restrict__ g, int ng, int64_t *__restrict__ gid) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x)
        gid[v] = g[slab_grid_of(g, ng, v)].gid_base + kept_incl[v] - 1;
}

}  // namespace chr

extern "C" int chr_slab_classify(const int64_t *d_vedge, int64_t nv, const int64_t *h_grids, int ng,
                                 int8_t *d_flags, int64_t *d_key, uint64_t *h_counts, void *d_ws, size_t ws_bytes,
                                 void *stream) {
    CHR_XFER_SCOPE;
    if (ng < 1 || nv < 0 || !h_grids || !h_counts) return CHR_E_PARAMETER;
    const size_t tb = sizeof(SlabGrid) * (size_t)ng, cb = 16 * (size_t)ng;
    if (!d_ws || ws_bytes < tb + cb + 256) return CHR_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    SlabGrid *d_g = reinterpret_cast<SlabGrid *>(d_ws);
    unsigned long long *d_c = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(d_ws) + ((tb + 255) & ~size_t(255)));
    CHR_CUDA_TRY(h2d(d_g, h_grids, tb, st));
    CHR_CUDA_TRY(zero_async({{d_c, cb}}, st));
    if (nv > 0) {
        CHR_PROF("k_slab_classify", st);
        k_slab_classify<<<(unsigned)std::min<int64_t>((nv + 255) / 256, 148 * 16), 256, 0, st>>>(d_vedge, nv, d_g, ng,
                                                                                                d_flags, d_key, d_c);
    }
    CHR_CUDA_TRY(cudaGetLastError());
    CHR_CUDA_TRY(d2h(h_counts, d_c, cb, st));
    CHR_CUDA_TRY(stream_sync(st));
    return CHR_OK;
}

extern "C" int chr_slab_gid(const int64_t *d_kept_incl, int64_t nv, const int64_t *h_grids, int ng, int64_t *d_gid,
                            void *d_ws, size_t ws_bytes, void *stream) {
    CHR_XFER_SCOPE;
    if (ng < 1 || nv < 0 || !h_grids) return CHR_E_PARAMETER;
    const size_t tb = sizeof(SlabGrid) * (size_t)ng;
    if (!d_ws || ws_bytes < tb) return CHR_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    SlabGrid *d_g = reinterpret_cast<SlabGrid *>(d_ws);
    CHR_CUDA_TRY(h2d(d_g, h_grids, tb, st));
    if (nv > 0) {
        CHR_PROF("k_slab_gid", st);
        k_slab_gid<<<(unsigned)std::min<int64_t>((nv + 255) / 256, 148 * 16), 256, 0, st>>>(d_kept_incl, nv, d_g, ng,
                                                                                           d_gid);
    }
    return cudaGetLastError() == cudaSuccess ? CHR_OK : CHR_E_CUDA;
}
