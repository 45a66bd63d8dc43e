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
#include <cmath>
#include <cstdlib>
#include <algorithm>

#include "chr_internal.cuh"

#ifndef CHR_STATS_RU
#define CHR_STATS_RU 4
#endif

namespace chr {

struct CandParams {
    double k[64];
    float thr[64];  // smallest float >= k[j]: for a float s, k[j] <= s  <=>  s >= thr[j]
    int m;
};

// min_k |s - k| for a float sample: the bracketing index by single-precision
// compares against thr (exact, see CandParams), the two distances in f64
__device__ __forceinline__ double min_cand_dist_f32(const double *k, const float *thr, int m, float s) {
    if (m == 1) return fabs(__dadd_rn((double)s, -k[0]));
    // #{j : k[j] <= s} = first candidate > s: branch-free binary search over
    // the thresholds padded with +inf to 128 (a finite s is never >= +inf)
    int lo = 0;
#pragma unroll
    for (int step = 64; step; step >>= 1)
        if (step < 2 * m && s >= thr[lo + step - 1]) lo += step;
    double d = INFINITY;
    if (lo > 0) d = fabs(__dadd_rn((double)s, -k[lo - 1]));
    if (lo < m) d = fmin(d, fabs(__dadd_rn((double)s, -k[lo])));
    return d;
}

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

// Fast path (f32, block size % 4 == 0, nx % 4 == 0, 16-byte aligned rows):
// one CTA per (by, bz) block row streams its (bs+1)^2 full-width sample rows
// with 16-byte loads; thread t owns x-quads t, t + 512, ...  Per-quad
// partials go through shared memory and one thread per block combines its
// bs/4 quads plus the x-ghost sample (first sample of the next block).
constexpr int SQ = 512;  // threads; nx/4 <= SQ quads per row
constexpr int SB = 4096;  // candidate buckets (k_stats_rows, m > 1)
constexpr int NSTG = 4;   // bulk-copy stages in flight per CTA (TMA variant)
constexpr int STG_BYTES = 16384;  // bytes per stage

// mbarrier / bulk-copy primitives (PTX; sm_90+)
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void async_proxy_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

template <bool TMA>
__global__ void __launch_bounds__(SQ) k_stats_rows(const float *__restrict__ vol, int64_t nx, int64_t ny,
                                                   int64_t nz, int bs, int nbx, int nby, CandParams cp,
                                                   double *__restrict__ stats,
                                                   unsigned long long *__restrict__ first_bad, int srows) {
    __shared__ double ks[128];
    __shared__ float kt[128];  // thresholds, +inf padded (the search may probe up to 2m - 2)
    // per (row group, quad) partials: index g * nq + q  (rg * nq <= SQ)
    __shared__ float plo[SQ], phi[SQ], pgl[SQ], pgh[SQ];
    __shared__ double pdm[SQ], pgd[SQ];
    if (threadIdx.x < 128) ks[threadIdx.x] = threadIdx.x < cp.m ? cp.k[threadIdx.x] : INFINITY;
    if (threadIdx.x < 128) kt[threadIdx.x] = threadIdx.x < cp.m ? cp.thr[threadIdx.x] : INFINITY;
    __syncthreads();
    // bucket table: a sample f in [thr[0], thr[m-1]) maps to bucket
    // b(f) = min(SB-1, int((f - lo_e) * invw)), monotone in f.  A bucket no
    // threshold maps to has one answer, #{j : b(thr[j]) < b}; a bucket some
    // threshold maps to is flagged (0x80) and resolved by exact compares.
    __shared__ uint8_t kb[SB];
    const float lo_e = kt[0], hi_e = cp.m > 1 ? kt[cp.m - 1] : kt[0];
    const float invw = hi_e > lo_e ? (float)SB / (hi_e - lo_e) : 0.f;
    auto bucket = [&](float f) { return min(SB - 1, (int)((f - lo_e) * invw)); };
    if (cp.m > 1) {
        for (int b = threadIdx.x; b < SB; b += blockDim.x) {
            int c = 0, hit = 0;
            for (int j = 0; j < cp.m; ++j) {
                const float t = kt[j];
                if (!(t >= lo_e) || !(t < hi_e)) {  // outside the bucketed range
                    c += t < lo_e ? 1 : 0;
                    continue;
                }
                const int bt = bucket(t);
                c += bt < b ? 1 : 0;
                hit |= bt == b ? 1 : 0;
            }
            kb[b] = (uint8_t)(c | (hit << 7));
        }
    }
    __syncthreads();
    const int nq = (int)(nx >> 2);
    const int m = cp.m;
    const int by = blockIdx.x % nby, bz = blockIdx.x / nby;
    const int64_t y0 = (int64_t)by * bs, y1 = min((int64_t)(by + 1) * bs, ny - 1);
    const int64_t z0 = (int64_t)bz * bs, z1 = min((int64_t)(bz + 1) * bs, nz - 1);
    const int G = bs >> 2;
    const int rg = SQ / nq;  // row groups
    const int q = threadIdx.x % nq, g = threadIdx.x / nq;
    const int nrow_y = (int)(y1 - y0 + 1);
    const int nrows = nrow_y * (int)(z1 - z0 + 1);
    float lo = INFINITY, hi = -INFINITY, gl = INFINITY, gh = -INFINITY;
    double dm = INFINITY, gd = INFINITY;
    // m == 1: fl(s - k) is monotone in s, so min |fl(s - k)| over a block
    // is attained at the smallest sample >= k or the largest sample < k:
    // track those two in f32 (exact compares against thr = the smallest
    // float >= k) and form the f64 distances once at the end
    float ab = INFINITY, bl = -INFINITY, gab = INFINITY, gbl = -INFINITY;
    const float thr0 = kt[0];
    unsigned long long bad = ~0ull;
    const bool ghost = ((4 * q) % bs) == 0 && q > 0;
    auto row_off = [&](int r) {  // flat index of row r's first sample
        const int zr = r / nrow_y, yr = r - zr * nrow_y;
        return ((z0 + zr) * ny + (y0 + yr)) * nx;
    };
    auto proc = [&](const float4 v4, int r) {  // this thread's quad of row r
        const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float f = v[i];
            if (!isfinite(f)) {
                bad = min(bad, (unsigned long long)(row_off(r) + 4 * q + i));
                continue;
            }
            lo = fminf(lo, f);
            hi = fmaxf(hi, f);
            if (m == 1) {
                const bool up = f >= thr0;
                ab = fminf(ab, up ? f : INFINITY);
                bl = fmaxf(bl, up ? -INFINITY : f);
                if (i == 0 && ghost) {
                    gl = fminf(gl, f);
                    gh = fmaxf(gh, f);
                    gab = fminf(gab, up ? f : INFINITY);
                    gbl = fmaxf(gbl, up ? -INFINITY : f);
                }
                continue;
            }
            // min |s - k| over the two candidates bracketing s
            const double sd = (double)f;
            double d;
            {
                int c;  // #{j : k[j] <= s}
                if (!(f >= lo_e)) {
                    c = 0;
                } else if (f >= hi_e) {
                    c = m;
                } else {
                    const int vv = kb[min(SB - 1, (int)((f - lo_e) * invw))];
                    c = vv & 0x7F;
                    if (vv & 0x80) {  // a threshold falls in this bucket: exact compares
                        while (c < m && f >= kt[c]) ++c;
                        while (c > 0 && f < kt[c - 1]) --c;
                    }
                }
                const double kl = c > 0 ? ks[c - 1] : -INFINITY;
                d = fmin(fabs(__dadd_rn(sd, -kl)), fabs(__dadd_rn(sd, -ks[c])));  // ks[m] = +inf
            }
            dm = fmin(dm, d);
            if (i == 0 && ghost) {
                gl = fminf(gl, f);
                gh = fmaxf(gh, f);
                gd = fmin(gd, d);
            }
        }
    };
    if constexpr (!TMA) {
        if (g < rg) {
            // RU rows per step: their 16-byte loads are all in flight before any is
            // used (one outstanding load per thread left HBM at ~35 % of peak)
            constexpr int RU = CHR_STATS_RU;
            for (int r0 = g; r0 < nrows; r0 += RU * rg) {
                float4 v4[RU];
#pragma unroll
                for (int u = 0; u < RU; ++u) {
                    const int r = r0 + u * rg;
                    v4[u] = r < nrows ? __ldg(reinterpret_cast<const float4 *>(vol + row_off(r)) + q)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < RU; ++u) {
                    if (r0 + u * rg >= nrows) break;
                    proc(v4[u], r0 + u * rg);
                }
            }
        }
    } else {
        // Bulk-copy (TMA) row streaming: thread 0 keeps NSTG stages of `srows`
        // rows in flight (cp.async.bulk into shared memory, completion counted
        // on one mbarrier per stage; rows of one plane are contiguous in HBM,
        // so a stage is one or two copies); every thread reduces its quad of
        // the stage's rows from shared memory.
        extern __shared__ __align__(128) unsigned char st_raw[];
        __shared__ __align__(8) uint64_t full[NSTG];
        const int64_t rowb = nx * 4;
        const int nst = (nrows + srows - 1) / srows;
        auto issue = [&](int s) {  // thread 0: stage s into buffer s % NSTG
            const int r0 = s * srows, r1 = min(nrows, r0 + srows);
            uint64_t *bar = &full[s % NSTG];
            unsigned char *dst = st_raw + (size_t)(s % NSTG) * srows * rowb;
            mbar_expect_tx(bar, (uint32_t)((r1 - r0) * rowb));
            for (int r = r0; r < r1;) {
                const int zr = r / nrow_y, yr = r - zr * nrow_y;
                const int cnt = min(r1 - r, nrow_y - yr);  // rows left in this plane
                bulk_g2s(dst + (size_t)(r - r0) * rowb, vol + row_off(r), (uint32_t)(cnt * rowb), bar);
                r += cnt;
            }
        };
        if (threadIdx.x == 0) {
            for (int i = 0; i < NSTG; ++i) mbar_init(&full[i], 1);
            mbar_fence_init();
            for (int s = 0; s < NSTG && s < nst; ++s) issue(s);
        }
        __syncthreads();
        for (int s = 0; s < nst; ++s) {
            const int buf = s % NSTG;
            mbar_wait(&full[buf], (uint32_t)((s / NSTG) & 1));
            if (g < rg) {
                const int r0 = s * srows, rn = min(nrows - r0, srows);
                const float4 *sb = reinterpret_cast<const float4 *>(st_raw + (size_t)buf * srows * rowb);
                for (int rr = g; rr < rn; rr += rg) proc(sb[(size_t)rr * nq + q], r0 + rr);
            }
            __syncthreads();  // every thread is done with the buffer
            if (threadIdx.x == 0 && s + NSTG < nst) {
                async_proxy_fence();
                issue(s + NSTG);
            }
        }
    }
    if (g < rg) {
        if (m == 1 && !isnan(ks[0])) {  // (a NaN candidate leaves the distances at +inf, like fmin)
            const double k0 = ks[0];
            dm = fmin(__dadd_rn((double)ab, -k0), __dadd_rn(k0, -(double)bl));
            gd = fmin(__dadd_rn((double)gab, -k0), __dadd_rn(k0, -(double)gbl));
        }
        if (bad != ~0ull) atomicMin(first_bad, bad);
        const int k = g * nq + q;
        plo[k] = lo;
        phi[k] = hi;
        pdm[k] = dm;
        pgl[k] = gl;
        pgh[k] = gh;
        pgd[k] = gd;
    }
    __syncthreads();
    for (int bx = threadIdx.x; bx < nbx; bx += SQ) {
        float l = INFINITY, h = -INFINITY;
        double d = INFINITY;
        const int q0 = bx * G, q1 = min(q0 + G, nq);
        for (int gg = 0; gg < rg; ++gg) {
            for (int qq = q0; qq < q1; ++qq) {
                const int k = gg * nq + qq;
                l = fminf(l, plo[k]);
                h = fmaxf(h, phi[k]);
                d = fmin(d, pdm[k]);
            }
            if (q1 < nq) {  // x-ghost: first sample of the next block
                const int k = gg * nq + q1;
                l = fminf(l, pgl[k]);
                h = fmaxf(h, pgh[k]);
                d = fmin(d, pgd[k]);
            }
        }
        const int64_t id = bx + (int64_t)nbx * (by + (int64_t)nby * bz);
        stats[3 * id + 0] = (double)l;
        stats[3 * id + 1] = (double)h;
        stats[3 * id + 2] = d;
    }
}

}  // namespace chr

using namespace chr;

extern "C" int64_t chr_num_blocks(int64_t nx, int64_t ny, int64_t nz, int64_t bs) {
    CHR_XFER_SCOPE;
    if (bs < 1) return 0;
    auto nb = [bs](int64_t d) { return d - 1 > 0 ? (d - 1 + bs - 1) / bs : (int64_t)1; };
    return nb(nx) * nb(ny) * nb(nz);
}

extern "C" int chr_stats(const void *d_vol, int dtype, int64_t nx, int64_t ny, int64_t nz,
                         int64_t bs, const double *h_cands, int m, double *d_block_stats,
                         int64_t *d_first_nonfinite, void *stream) {
    CHR_XFER_SCOPE;
    if (!d_vol || !d_block_stats || !d_first_nonfinite || !h_cands) return CHR_E_PARAMETER;
    if (bs < 2 || nx < 2 || ny < 2 || nz < 2 || m < 1 || m > 64) return CHR_E_PARAMETER;
    if (dtype != CHR_F32 && dtype != CHR_F64) return CHR_E_PARAMETER;
    cudaStream_t st = (cudaStream_t)stream;
    CandParams cp;
    cp.m = m;
    for (int i = 0; i < m; ++i) {
        cp.k[i] = h_cands[i];
        float f = (float)h_cands[i];  // round to nearest, then up to the smallest float >= k
        if (std::isnan(h_cands[i])) f = INFINITY;
        else if ((double)f < h_cands[i]) f = std::nextafter(f, INFINITY);
        cp.thr[i] = f;
    }
    const int nbx = (int)((nx - 1 + bs - 1) / bs), nby = (int)((ny - 1 + bs - 1) / bs);
    const int64_t nblocks = chr_num_blocks(nx, ny, nz, bs);
    CHR_CUDA_TRY(fill_async(d_first_nonfinite, 0xFF, sizeof(int64_t), st));
    auto *bad = reinterpret_cast<unsigned long long *>(d_first_nonfinite);
    const int nbz = (int)((nz - 1 + bs - 1) / bs);
    const bool rows_ok = dtype == CHR_F32 && bs % 4 == 0 && nx % 4 == 0 && nx <= 4 * SQ &&
                         ((uintptr_t)d_vol & 15) == 0;
    if (rows_ok) {
        // bulk-copy (TMA) row staging unless CHR_STATS_TMA=0; rows per stage: 16 KB
        static const bool tma = [] {
            const char *e = std::getenv("CHR_STATS_TMA");
            return !(e && e[0] == '0');
        }();
        const int srows = (int)std::max<int64_t>(1, STG_BYTES / (4 * nx));
        const int smem = NSTG * srows * (int)(4 * nx);
        CHR_PROF("k_stats_rows", st);
        if (tma) {
            CHR_CUDA_TRY(cudaFuncSetAttribute(k_stats_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            k_stats_rows<true><<<(unsigned)(nby * nbz), SQ, smem, st>>>((const float *)d_vol, nx, ny, nz, (int)bs, nbx,
                                                                       nby, cp, d_block_stats, bad, srows);
        } else {
            k_stats_rows<false><<<(unsigned)(nby * nbz), SQ, 0, st>>>((const float *)d_vol, nx, ny, nz, (int)bs, nbx,
                                                                     nby, cp, d_block_stats, bad, srows);
        }
    } else if (dtype == CHR_F32)
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
