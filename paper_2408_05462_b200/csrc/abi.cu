// abi.cu -- library info + kernel-seam entry points on single windows
// (isochr/kernels.py: min_abs_distance kernels.py:417-425,
// lorenzo_encode kernels.py:47-128).
#include <cstring>

#include "chr_internal.cuh"

namespace chr {

__global__ void __launch_bounds__(256) k_min_abs(const double *__restrict__ x, int64_t n, double k,
                                                 unsigned long long *__restrict__ out) {
    double best = INFINITY;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        best = fmin(best, fabs(__dadd_rn(x[i], -k)));
    for (int off = 16; off; off >>= 1) best = fmin(best, __shfl_xor_sync(0xFFFFFFFFu, best, off));
    // non-negative doubles order like their bit patterns
    if ((threadIdx.x & 31) == 0) atomicMin(out, (unsigned long long)__double_as_longlong(best));
}

// thread per sample; the 8 lattice values are requantised (exactly as the
// encoder does), so q matches kernels.lorenzo_encode bit for bit
__global__ void __launch_bounds__(256) k_lorenzo_seam(const double *__restrict__ x, int64_t nx, int64_t ny,
                                                      int64_t nz, Quant Q, int64_t *__restrict__ q,
                                                      uint8_t *__restrict__ esc) {
    const int64_t n = nx * ny * nz;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t xx = i % nx, yy = (i / nx) % ny, zz = i / (nx * ny);
        int64_t acc = 0;
        bool e0 = false;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int dx = c & 1, dy = (c >> 1) & 1, dz = (c >> 2) & 1;
            if (xx - dx < 0 || yy - dy < 0 || zz - dz < 0) continue;
            bool e;
            const int32_t u = quantize(Q, x[i - dx - dy * nx - dz * nx * ny], e);
            if (c == 0) e0 = e;
            acc += ((dx + dy + dz) & 1) ? -(int64_t)u : (int64_t)u;
        }
        q[i] = acc;
        esc[i] = e0 ? 1 : 0;
    }
}

// value_range + finite check of a whole volume (volume.py:54-78): min/max
// over the samples as ordered-integer atomics, the first non-finite flat
// index as an atomicMin (a NaN/Inf never enters min/max, like the
// reference which raises before computing the range)
__device__ __forceinline__ unsigned long long ord_key(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | (1ull << 63));
}
template <typename T>
__global__ void __launch_bounds__(256) k_value_range(const T *__restrict__ x, int64_t n,
                                                     unsigned long long *__restrict__ out) {
    double lo = INFINITY, hi = -INFINITY;
    unsigned long long bad = ~0ull;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = (double)__ldg(x + i);
        if (!isfinite(v)) {
            bad = min(bad, (unsigned long long)i);
            continue;
        }
        lo = fmin(lo, v);
        hi = fmax(hi, v);
    }
    for (int off = 16; off; off >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, off));
        hi = fmax(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, off));
        bad = min(bad, __shfl_xor_sync(0xFFFFFFFFu, bad, off));
    }
    if ((threadIdx.x & 31) == 0) {
        if (lo <= hi) {
            atomicMin(out + 0, ord_key(lo));
            atomicMax(out + 1, ord_key(hi));
        }
        if (bad != ~0ull) atomicMin(out + 2, bad);
    }
}

}  // namespace chr

using namespace chr;

extern "C" int chr_value_range(const void *d_vol, int dtype, int64_t n, void *d_ws, size_t ws_bytes,
                               double *h_range, int64_t *h_first_nonfinite, void *stream) {
    CHR_XFER_SCOPE;
    if (!d_vol || n < 1 || !h_range || !h_first_nonfinite) return CHR_E_PARAMETER;
    if (dtype != CHR_F32 && dtype != CHR_F64) return CHR_E_PARAMETER;
    if (!d_ws || ws_bytes < 24) return CHR_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    auto *slot = reinterpret_cast<unsigned long long *>(d_ws);
    CHR_CUDA_TRY(zero_async({{slot + 1, 8}}, st));
    CHR_CUDA_TRY(fill_async(slot, 0xFF, 8, st));
    CHR_CUDA_TRY(fill_async(slot + 2, 0xFF, 8, st));
    const int64_t blocks = std::min<int64_t>(ceil_div(n, 256), 148 * 8);
    {
        CHR_PROF("k_value_range", st);
        if (dtype == CHR_F32)
            k_value_range<float><<<(unsigned)blocks, 256, 0, st>>>((const float *)d_vol, n, slot);
        else
            k_value_range<double><<<(unsigned)blocks, 256, 0, st>>>((const double *)d_vol, n, slot);
    }
    CHR_CUDA_TRY(cudaGetLastError());
    unsigned long long r[3];
    CHR_CUDA_TRY(d2h(r, slot, 24, st));
    CHR_CUDA_TRY(stream_sync(st));
    for (int i = 0; i < 2; ++i) {
        const unsigned long long b = (r[i] >> 63) ? (r[i] & ~(1ull << 63)) : ~r[i];
        memcpy(&h_range[i], &b, 8);
    }
    *h_first_nonfinite = r[2] == ~0ull ? -1 : (int64_t)r[2];
    return CHR_OK;
}

extern "C" int chr_abi_version(void) {
    CHR_XFER_SCOPE; return 1; }

extern "C" const char *chr_status_string(int s) {
    CHR_XFER_SCOPE;
    switch (s) {
        case CHR_OK: return "ok";
        case CHR_E_PARAMETER: return "invalid parameter";
        case CHR_E_NONFINITE: return "non-finite sample";
        case CHR_E_CORRUPT: return "corrupt payload";
        case CHR_E_UNSUPPORTED_CODEC: return "unsupported codec";
        case CHR_E_CUDA: return "CUDA error";
        case CHR_E_WORKSPACE: return "workspace too small";
        default: return "unknown status";
    }
}

extern "C" int chr_min_abs_distance(const double *d_flat, int64_t n, double k, double *h_out, void *d_ws,
                                    size_t ws_bytes, void *stream) {
    CHR_XFER_SCOPE;
    if (!d_flat || n < 1 || !h_out) return CHR_E_PARAMETER;
    if (!d_ws || ws_bytes < 8) return CHR_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    auto *slot = reinterpret_cast<unsigned long long *>(d_ws);
    CHR_CUDA_TRY(fill_async(slot, 0x7F, 8, st));  // a huge positive double
    const int64_t blocks = std::min<int64_t>(ceil_div(n, 256), 148 * 16);
    {
        CHR_PROF("k_min_abs", st);
        k_min_abs<<<(unsigned)blocks, 256, 0, st>>>(d_flat, n, k, slot);
    }
    CHR_CUDA_TRY(cudaGetLastError());
    unsigned long long bits = 0;
    CHR_CUDA_TRY(d2h(&bits, slot, 8, st));
    CHR_CUDA_TRY(stream_sync(st));
    double v;
    memcpy(&v, &bits, 8);
    *h_out = v;
    return CHR_OK;
}

extern "C" int chr_lorenzo_encode(const double *d_flat, int64_t nx, int64_t ny, int64_t nz, double e,
                                  int64_t *d_q, uint8_t *d_escaped, void *stream) {
    CHR_XFER_SCOPE;
    if (!d_flat || !d_q || !d_escaped || nx < 1 || ny < 1 || nz < 1 || !(e > 0.0)) return CHR_E_PARAMETER;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = nx * ny * nz;
    const int64_t blocks = std::min<int64_t>(ceil_div(n, 256), 148 * 32);
    {
        CHR_PROF("k_lorenzo_seam", st);
        k_lorenzo_seam<<<(unsigned)blocks, 256, 0, st>>>(d_flat, nx, ny, nz, make_quant(e), d_q, d_escaped);
    }
    return cudaGetLastError() == cudaSuccess ? CHR_OK : CHR_E_CUDA;
}

// ------------------------------------------------------------------ SM copy
// Bulk host<->device copy through UVA-mapped pinned memory by a small grid
// (no copy engine): lets a pipelined caller stream inputs/outputs over PCIe
// while the library's own small DMA copies proceed unqueued.
namespace chr {
__global__ void __launch_bounds__(256) k_sm_copy(const uint8_t *__restrict__ src, uint8_t *__restrict__ dst,
                                                 uint64_t n) {
    const uint64_t n16 = n >> 4;
    const uint4 *s = reinterpret_cast<const uint4 *>(src);
    uint4 *d = reinterpret_cast<uint4 *>(dst);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {  // 4 loads in flight per thread
        const uint4 a = s[i], b = s[i + stride], c = s[i + 2 * stride], e = s[i + 3 * stride];
        d[i] = a;
        d[i + stride] = b;
        d[i + 2 * stride] = c;
        d[i + 3 * stride] = e;
    }
    for (; i < n16; i += stride) d[i] = s[i];
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < (n & 15)) dst[(n16 << 4) + t] = src[(n16 << 4) + t];
}
}  // namespace chr

extern "C" int chr_sm_copy(void *dst, const void *src, uint64_t nbytes, int ctas, void *stream) {
    CHR_XFER_SCOPE;
    if (nbytes == 0) return CHR_OK;
    if (!dst || !src || (((uintptr_t)dst | (uintptr_t)src) & 15)) return CHR_E_PARAMETER;
    cudaStream_t st = (cudaStream_t)stream;
    {
        CHR_PROF("k_sm_copy", st);
        k_sm_copy<<<(unsigned)std::max(1, ctas), 256, 0, st>>>((const uint8_t *)src, (uint8_t *)dst, nbytes);
    }
    return cudaGetLastError() == cudaSuccess ? CHR_OK : CHR_E_CUDA;
}

// request(k) tables from an archive's region table (chr_archive.py:249-259
// selection; host only): the regions whose relevance mask has bit
// k_index (all regions when k_index < 0), as chr_dec_region_t (payload
// after the 34-byte block header, windows back to back) and chr_mc_grid_t
// (world origin = sample origin * spacing).  Returns the selected count;
// h_sel receives their region indices, *h_total_samples the window sum.
extern "C" int64_t chr_request_tables(const chr_region_t *h_regions, int64_t n, int k_index, const double *spacing,
                                      chr_dec_region_t *h_dec, chr_mc_grid_t *h_mc, int64_t *h_sel,
                                      uint64_t *h_total_samples) {
    if (!h_regions || n < 0 || k_index > 63) return -1;
    int64_t m = 0;
    uint64_t off = 0;
    for (int64_t i = 0; i < n; ++i) {
        const chr_region_t &r = h_regions[i];
        if (k_index >= 0 && !((r.mask >> k_index) & 1ull)) continue;
        const uint64_t ns = (uint64_t)r.extent[0] * r.extent[1] * r.extent[2];
        if (h_dec) {
            chr_dec_region_t &d = h_dec[m];
            std::memset(&d, 0, sizeof(d));
            d.payload_offset = r.block_offset + 34;
            d.payload_nbytes = r.block_nbytes - 34;
            d.codec_id = r.codec_id;
            for (int a = 0; a < 3; ++a) d.dims[a] = r.extent[a];
            d.error_bound = r.error_bound;
            d.crc = r.payload_crc;
            d.out_offset = off;
        }
        if (h_mc) {
            chr_mc_grid_t &g = h_mc[m];
            std::memset(&g, 0, sizeof(g));
            g.grid_offset = off;
            for (int a = 0; a < 3; ++a) {
                g.dims[a] = r.extent[a];
                const double sp = spacing ? spacing[a] : 1.0;
                g.origin[a] = (double)r.origin[a] * sp;
                g.spacing[a] = sp;
            }
        }
        if (h_sel) h_sel[m] = i;
        off += ns;
        ++m;
    }
    if (h_total_samples) *h_total_samples = off;
    return m;
}
