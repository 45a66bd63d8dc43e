// encode.cu -- steps 2+3 of the hot path on the device: topology-bounded
// quantisation + 3D Lorenzo residuals + the zigzag/LEB128/zero-run token
// stream + codec selection + CompressedBlock / .chr byte layout + CRCs.
//
// Reference: kernels.py:47-93 (quantise + Lorenzo), kernels.py:198-234
// (token stream), codec.py:91-143 (codec 1/2, escape bitmap + values,
// verbatim fallback 0/3, CRC), codec.py:61-70 (34-byte header),
// chr_archive.py:297-340 + FORMAT.md (file header, region table,
// payloads in region order, CRC trailer).
//
// Pipeline (all on one stream, no host round trip):
//   k_quant        quantise + Lorenzo q per sample -> token values (zigzag+1),
//                  escape bits, f32-exactness flag
//   k_summarize    per 64-sample piece of a window's stream: token-byte
//                  summary (TokSeg)
//   k_scan_reduce  chunk aggregates (chunks never straddle regions)
//   k_scan_regions per region: chunk prefixes, totals, codec decision
//   k_layout       region offsets in the file, CRC segment plan
//   k_scan_down    per piece: token offset, zero-run carry, escape offset
//   k_emit_q       write every token byte at its final offset
//   k_bitmap       escape bitmaps (codec 2 regions only)
//   k_write_table  file header + region table
//   k_crc_segments payload + header-table CRCs (crc.cu)
//   k_finalize_*   34-byte block headers, file CRC trailer
//
// Tiles: a CTA owns 64 columns x 8 rows x 16 planes of one region window
// and marches z; one warp per row (+1 halo warp for row y0-1), 2 samples
// per lane + the x0-1 halo sample.  With D = u(z) - u(z-1) shared through
// shared memory, q = D - D(x-1) - D(y-1) + D(x-1,y-1), so u is computed
// once per sample (plus the 1/8 + 1/64 + 1/16 halo).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "chr_internal.cuh"

namespace chr {

constexpr int TX = 64, TY = 8, ZC = 16, NW = TY + 1;
#ifndef CHR_QB_T
#define CHR_QB_T 320
#endif
#ifndef CHR_QB_ZMAX
#define CHR_QB_ZMAX 33
#endif
constexpr int QB_T = CHR_QB_T, QB_SPT = 4, QB_CAP = QB_T * QB_SPT;  // k_quant_band: threads, slots, samples
constexpr int QB_ZMAX = CHR_QB_ZMAX;  // k_quant_band: planes per item at most (balanced chunks)
constexpr int CSPLIT = 4;  // k_summarize2 CTAs per scan chunk
constexpr int64_t CH = 1024;  // pieces per scan chunk

struct RegDev {
    int32_t ox, oy, oz, ex, ey, ez;
    int32_t ntx, nty, nzc, mode;  // mode 1: e == 0 (verbatim)
    double e;
    int64_t n;
    int64_t piece_base, npieces, item_base, chunk_base, nchunks;
    int64_t q_base;               // first token value of the region in the q buffer
    int64_t ebase;                // first escape-bit word of the region
    int32_t has_esc, f32bad;      // set by k_quant
    // z-slab portions (multi-GPU): this record encodes window planes
    // [oz_w, oz_w + ez) of a window of n_win samples, starting at window
    // sample s_off; zhalo = plane -1 belongs to the window, last = the
    // portion ends the window, pre = stream summary of the portions before.
    int64_t s_off, n_win;
    int32_t zhalo, last;
    TokSeg pre;
    int32_t qband, rb;            // quantiser items are full-row bands of rb rows (k_quant_band)
    int32_t zl, qzch;             // planes per item: segment path (k_qseg / k_qemit) / k_quant_band
    // results
    int32_t codec, f32ok;
    int64_t tok_len, nesc, payload_len;
    uint64_t block_off, payload_off, tok_start;
    uint32_t crc;
    uint32_t pad;
    uint64_t mask;
    int32_t lo[3], hi[3];
};

struct EncParams {
    int64_t NX, NY, NZ;
    int64_t nreg, nitems, nchunks;
    int32_t dtype, src_dtype, write_file, m;
    int32_t dist, bound_mode;  // dist: codec/length decided on the host; bound_mode: table byte (0 strict, 1 paper)
    double accuracy;           // stored accuracy (region table)
    double spacing[3];
    double vmin, vmax;
    int64_t bs;
    uint64_t header_table;  // bytes before the first block (0 if !write_file)
    double cands[64];
};

struct EncScalars {
    uint64_t file_body;      // bytes before the trailer
    uint64_t out_nbytes;     // total bytes written
    uint32_t file_raw;       // raw CRC accumulator of the body
    uint32_t pad;
    int64_t n_codec2;
    int64_t total_sc;
};

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ int64_t find_region_by(const RegDev *__restrict__ regs, int64_t nreg,
                                                  int64_t key, int which) {
    int64_t lo = 0, hi = nreg - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        const int64_t b = which == 0 ? regs[mid].item_base : regs[mid].chunk_base;
        if (b <= key) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ uint8_t *put_varint(uint8_t *p, uint64_t u) {
    while (u >= 0x80) {
        *p++ = (uint8_t)((u & 0x7F) | 0x80);
        u >>= 7;
    }
    *p++ = (uint8_t)u;
    return p;
}

__device__ __forceinline__ uint8_t *put_run(uint8_t *p, int64_t run) {
    if (run == 1) {
        *p++ = 1;
    } else if (run >= 2) {
        *p++ = 0;
        p = put_varint(p, (uint64_t)run);
    }
    return p;
}

template <typename V>
__device__ __forceinline__ void put_le(uint8_t *p, V v) {
    uint8_t b[sizeof(V)];
    memcpy(b, &v, sizeof(V));
#pragma unroll
    for (int i = 0; i < (int)sizeof(V); ++i) p[i] = b[i];
}

__device__ __forceinline__ int hibit(uint64_t m) { return 63 - __clzll((long long)m); }

template <typename T>
__device__ __forceinline__ bool not_f32_exact(T v) {
    return (double)(float)v != (double)v;
}

// ------------------------------------------------------------------ tiles
// 32-bit token-size helpers (valid quanta: |q| <= 2^30, zigzag+1 <= 2^31+1)
__device__ __forceinline__ uint32_t zz1_32(int32_t q) { return (((uint32_t)q << 1) ^ (uint32_t)(q >> 31)) + 1u; }
__device__ __forceinline__ int vlen32(uint32_t u) {  // ceil(bits / 7) for u >= 1: ((38 - clz) * 37) >> 8
    return ((38 - __clz(u)) * 37) >> 8;
}
// token bytes of a zero run shorter than 128 (every run inside one 64-sample piece)
__device__ __forceinline__ int rb_small(int L) { return L <= 0 ? 0 : (L == 1 ? 1 : 2); }

__device__ __forceinline__ uint8_t *put_varint32(uint8_t *p, uint32_t u) {
    while (u >= 0x80u) {
        *p++ = (uint8_t)((u & 0x7Fu) | 0x80u);
        u >>= 7;
    }
    *p++ = (uint8_t)u;
    return p;
}

// quantiser fast path only; false -> the caller runs the exact sequence
__device__ __forceinline__ bool quant_fast(const Quant &Q, double v, int32_t &u) {
    const double qf = __dmul_rn(v, Q.inv);
    const double t = __dadd_rn(qf, kRoundShift);
    const double d = __dadd_rn(qf, -__dadd_rn(t, -kRoundShift));
    u = __double2loint(t);
    return Q.fast && fabs(qf) < kEscapeUmax && fabs(d) < kTieMargin;
}

// Quantiser pass: CTA = 64 columns x 8 rows x 16 planes of one region
// window (+ a halo row, column and plane), marching z; q = D - D(x-1) -
// D(y-1) + D(x-1,y-1) with D = u(z) - u(z-1) in shared memory.  Writes the
// token value zigzag(q) + 1 of every sample in the window's raster order,
// the escape bits (rare) and the region's f32-inexact flag.
template <typename T>
__global__ void __launch_bounds__(NW * 32, 4) k_quant(const T *__restrict__ vol, const EncParams *__restrict__ P,
                                                   RegDev *__restrict__ regs,
                                                   const int32_t *__restrict__ item_reg,
                                                   uint32_t *__restrict__ qz, uint32_t *__restrict__ escbits) {
    __shared__ int32_t sD[2][NW][TX + 2];
    __shared__ RegDev R;
    const int64_t item = blockIdx.x;
    const int ri = __ldg(item_reg + item);
    coop_copy(&R, regs + ri);
    __syncthreads();
    if (R.qband) return;  // k_quant_band's item
    const int64_t NX = P->NX, NY = P->NY, plane = NX * NY;
    const int64_t local = item - R.item_base;
    const int xt = (int)(local % R.ntx);
    const int64_t t2 = local / R.ntx;
    const int yt = (int)(t2 % R.nty);
    const int zc = (int)(t2 / R.nty);
    const int x0 = xt * TX, y0 = yt * TY, z0 = zc * ZC;
    const int z1 = min(z0 + ZC, R.ez);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int y = y0 - 1 + w;
    const bool rowok = y >= 0 && y < R.ey;
    const int xA = x0 + lane, xB = x0 + 32 + lane, xH = x0 - 1;
    const bool okA = rowok && xA < R.ex, okB = rowok && xB < R.ex;
    const bool okH = rowok && lane == 0 && xH >= 0;
    const bool quant = R.mode == 0;
    const Quant Q = make_quant(R.e);
    const bool chk32 = sizeof(T) == 8 && P->src_dtype == CHR_F32;
    const T *row = vol + ((int64_t)(R.oz + z0) * NY + (R.oy + y)) * NX + R.ox;  // plane z0

    // returns (warp-uniform) whether the exact sequence ran; escapes only come from it
    auto quant3 = [&](T a, T b, T h, int32_t &ua, int32_t &ub, int32_t &uh, bool &ea, bool &eb, bool &eh) {
        ua = ub = uh = 0;
        ea = eb = eh = false;
        bool fa = true, fb = true, fh = true;
        if (okA) fa = quant_fast(Q, (double)a, ua);
        if (okB) fb = quant_fast(Q, (double)b, ub);
        if (okH) fh = quant_fast(Q, (double)h, uh);
        if (__any_sync(0xFFFFFFFFu, !(fa && fb && fh))) {  // rare: ties, escapes, tiny e
            if (!fa) ua = quantize(Q, (double)a, ea);
            if (!fb) ub = quantize(Q, (double)b, eb);
            if (!fh) uh = quantize(Q, (double)h, eh);
            return true;
        }
        return false;
    };
    int32_t pA = 0, pB = 0, pH = 0;  // u at the previous plane
    if (quant && (z0 > 0 || R.zhalo)) {  // u at the plane before (inside the window)
        const T *prow = row - plane;
        bool e0, e1, e2;
        quant3(okA ? __ldg(prow + xA) : (T)0, okB ? __ldg(prow + xB) : (T)0, okH ? __ldg(prow + xH) : (T)0, pA, pB,
               pH, e0, e1, e2);
    }
    T nA = 0, nB = 0, nH = 0;
    if (z0 < z1) {
        if (okA) nA = __ldg(row + xA);
        if (okB) nB = __ldg(row + xB);
        if (okH) nH = __ldg(row + xH);
    }
    bool inexact = false;
    for (int z = z0; z < z1; ++z, row += plane) {
        const T vA = nA, vB = nB, vH = nH;
        if (z + 1 < z1) {  // prefetch the next plane
            const T *nrow = row + plane;
            if (okA) nA = __ldg(nrow + xA);
            if (okB) nB = __ldg(nrow + xB);
            if (okH) nH = __ldg(nrow + xH);
        }
        bool eA = false, eB = false, eH = false, slow = false;
        int32_t uA = 0, uB = 0, uH = 0;
        if (quant) slow = quant3(vA, vB, vH, uA, uB, uH, eA, eB, eH);
        int32_t(*D)[TX + 2] = sD[z & 1];
        D[w][lane + 1] = uA - pA;
        D[w][lane + 33] = uB - pB;
        if (lane == 0) D[w][0] = uH - pH;
        pA = uA;
        pB = uB;
        pH = uH;
        __syncthreads();
        if (w == 0 || !rowok) continue;
        const int32_t qA = D[w][lane + 1] - D[w][lane] - D[w - 1][lane + 1] + D[w - 1][lane];
        const int32_t qB = D[w][lane + 33] - D[w][lane + 32] - D[w - 1][lane + 33] + D[w - 1][lane + 32];
        const int64_t s0 = ((int64_t)z * R.ey + y) * R.ex + x0;  // window sample index of column x0
        uint32_t *qrow = qz + R.q_base + s0;
        if (okA) qrow[lane] = zz1_32(qA);
        if (okB) qrow[32 + lane] = zz1_32(qB);
        if (slow) {
            const uint32_t eAm = __ballot_sync(0xFFFFFFFFu, okA && eA), eBm = __ballot_sync(0xFFFFFFFFu, okB && eB);
            if (lane == 0 && (eAm | eBm)) {  // 64 bits at window bit s0
                const int64_t bit = (int64_t)R.ebase * 32 + s0;
                uint32_t *wp = escbits + (bit >> 5);
                const int sh = (int)(bit & 31);
                const uint64_t m = (uint64_t)eAm | ((uint64_t)eBm << 32);
                if (m << sh) {
                    atomicOr(wp, (uint32_t)(m << sh));
                    atomicOr(wp + 1, (uint32_t)((m << sh) >> 32));
                }
                if (sh && (m >> (64 - sh))) atomicOr(wp + 2, (uint32_t)(m >> (64 - sh)));
                atomicOr(&regs[ri].has_esc, 1);
            }
        }
        if (chk32) inexact |= (okA && not_f32_exact(vA)) || (okB && not_f32_exact(vB));
    }
    if (chk32 && __any_sync(0xFFFFFFFFu, inexact) && lane == 0) atomicOr(&regs[ri].f32bad, 1);
}

// Quantiser pass, full-row bands: CTA = rb whole rows (+ the halo row y0-1)
// x 16 planes of one window, the band-plane's samples flattened over the
// threads (QB_SPT slots each) so narrow windows (33 = 32k+1 columns) keep
// every lane busy; D(z) = u(z) - u(z-1) per slot, q from the band-plane's D
// in shared memory.  Slot i = row yy (0 = halo) * ex + x; its volume offset
// (yy * NX + x), its window offset (i, from row y0-1 of the plane) and its
// shared index (a zero column at x = -1: yy * (ex+1) + x + 1, so the x-1 /
// y-1 / (x-1, y-1) neighbours need no edge selects) are 32-bit and fixed;
// only the per-plane base pointers move.
constexpr int QB_SD = 2 * QB_CAP + 64;  // padded band-plane: (rows + 1) * (ex + 1) <= 2 * QB_CAP
template <typename T>
__global__ void __launch_bounds__(QB_T, 3) k_quant_band(const T *__restrict__ vol, const EncParams *__restrict__ P,
                                                    RegDev *__restrict__ regs, const int32_t *__restrict__ item_reg,
                                                    uint32_t *__restrict__ qz, uint32_t *__restrict__ escbits) {
    __shared__ int32_t sD[2][QB_SD];
    __shared__ RegDev R;
    const int64_t item = blockIdx.x;
    const int ri = __ldg(item_reg + item);
    coop_copy(&R, regs + ri);
    __syncthreads();
    if (!R.qband) return;
    const int64_t NX = P->NX, NY = P->NY, plane = NX * NY;
    const int64_t local = item - R.item_base;
    const int yt = (int)(local % R.nty), zc = (int)(local / R.nty);
    const int ex = R.ex, y0 = yt * R.rb, rows = min(R.rb, R.ey - y0);
    const int z0 = zc * R.qzch, z1 = min(z0 + R.qzch, R.ez);
    const int span = (rows + 1) * ex;  // halo row first
    const bool quant = R.mode == 0;
    const Quant Q = make_quant(R.e);
    const bool chk32 = sizeof(T) == 8 && P->src_dtype == CHR_F32;
    const int tid = threadIdx.x;
    int voff[QB_SPT], sj[QB_SPT];
    unsigned okm = 0, ownm = 0;  // slot bits: a sample of the window / an own (non-halo) sample
#pragma unroll
    for (int k = 0; k < QB_SPT; ++k) {
        const int i = tid + QB_T * k;
        const int yy = i / ex, x = i - yy * ex;
        voff[k] = yy * (int)NX + x;
        sj[k] = yy * (ex + 1) + x + 1;
        if (i < span && y0 - 1 + yy >= 0) okm |= 1u << k;
        if (i < span && yy >= 1) ownm |= 1u << k;
    }
    // zero columns (x = -1) of both buffers; slots never write them
    for (int t = tid; t <= rows; t += QB_T) {
        sD[0][t * (ex + 1)] = 0;
        sD[1][t * (ex + 1)] = 0;
    }
    // row y0-1 of plane z: slot offsets are added to these
    const T *vrow = vol + ((int64_t)(R.oz + z0) * NY + (R.oy + y0 - 1)) * NX + R.ox;
    const int64_t plane_w = (int64_t)ex * R.ey;
    uint32_t *qrow = qz + R.q_base + (int64_t)z0 * plane_w + (int64_t)(y0 - 1) * ex;
    int32_t up[QB_SPT];
#pragma unroll
    for (int k = 0; k < QB_SPT; ++k) up[k] = 0;
    // returns the slots' escape bits (only the exact sequence escapes)
    auto quant_slots = [&](const T (&v)[QB_SPT], int32_t (&u)[QB_SPT]) -> unsigned {
        bool fast = true;
#pragma unroll
        for (int k = 0; k < QB_SPT; ++k) {
            u[k] = 0;
            if (((okm >> k) & 1u) && quant) fast &= quant_fast(Q, (double)v[k], u[k]);
        }
        unsigned em = 0;
        if (__any_sync(0xFFFFFFFFu, !fast)) {  // rare: ties, escapes, tiny e
#pragma unroll
            for (int k = 0; k < QB_SPT; ++k)
                if (((okm >> k) & 1u) && quant) {
                    bool e = false;
                    u[k] = quantize(Q, (double)v[k], e);
                    em |= e ? 1u << k : 0u;
                }
        }
        return em;
    };
    if (quant && (z0 > 0 || R.zhalo)) {  // u at the plane before (inside the window)
        T v[QB_SPT];
#pragma unroll
        for (int k = 0; k < QB_SPT; ++k) v[k] = ((okm >> k) & 1u) ? __ldg(vrow - plane + voff[k]) : (T)0;
        quant_slots(v, up);
    }
    T nv[QB_SPT];
#pragma unroll
    for (int k = 0; k < QB_SPT; ++k) nv[k] = (((okm >> k) & 1u) && z0 < z1) ? __ldg(vrow + voff[k]) : (T)0;
    bool inexact = false;
    for (int z = z0; z < z1; ++z, vrow += plane, qrow += plane_w) {
        T v[QB_SPT];
        const bool more = z + 1 < z1;
#pragma unroll
        for (int k = 0; k < QB_SPT; ++k) {
            v[k] = nv[k];
            nv[k] = (((okm >> k) & 1u) && more) ? __ldg(vrow + plane + voff[k]) : (T)0;  // prefetch the next plane
        }
        int32_t u[QB_SPT];
        const unsigned em = quant_slots(v, u);
        int32_t *D = sD[z & 1];
#pragma unroll
        for (int k = 0; k < QB_SPT; ++k) {
            if (tid + QB_T * k < span) D[sj[k]] = u[k] - up[k];  // invalid slots: 0 - 0
            up[k] = u[k];
        }
        __syncthreads();
        const int rs = ex + 1;
#pragma unroll
        for (int k = 0; k < QB_SPT; ++k) {
            if (!((ownm >> k) & 1u)) continue;
            const int j = sj[k];
            const int32_t q = D[j] - D[j - 1] - D[j - rs] + D[j - rs - 1];
            const int i = tid + QB_T * k;
            qrow[i] = zz1_32(q);
            if ((em >> k) & 1u) {
                const int64_t s = (int64_t)z * plane_w + (int64_t)(y0 - 1) * ex + i;  // window raster index
                const int64_t bit = (int64_t)R.ebase * 32 + s;
                atomicOr(escbits + (bit >> 5), 1u << (bit & 31));
                atomicOr(&regs[ri].has_esc, 1);
            }
            if (chk32) inexact |= not_f32_exact(v[k]);
        }
    }
    if (chk32 && __any_sync(0xFFFFFFFFu, inexact) && (tid & 31) == 0) atomicOr(&regs[ri].f32bad, 1);
}

// Piece records, a THREAD per 64-sample piece (CSPLIT CTAs of 256 threads per
// scan chunk): the piece's 64 token values in 16 vector loads (regions start
// 16-byte aligned in the token-value buffer), then a sequential branch-free
// fold of the token-size summary (a warp-per-piece ballot version spent its
// issue slots on 32 lanes' worth of mask bookkeeping per piece: 0.33 ms vs
// 0.15 ms at c3).
__global__ void __launch_bounds__(256) k_summarize2(const RegDev *__restrict__ regs,
                                                    const int32_t *__restrict__ chunk_reg,
                                                    const uint32_t *__restrict__ qz,
                                                    const uint32_t *__restrict__ escbits,
                                                    PieceRec *__restrict__ recs) {
    __shared__ RegDev R;
    const int64_t c = blockIdx.x / CSPLIT;
    coop_copy(&R, regs + __ldg(chunk_reg + c));
    __syncthreads();
    const int64_t lp = (c - R.chunk_base) * CH + (int64_t)(blockIdx.x % CSPLIT) * (CH / CSPLIT) + threadIdx.x;
    if (lp >= R.npieces) return;
    const int64_t s0 = lp * TX;
    const int vcount = (int)min((int64_t)TX, R.n - s0);
    const uint32_t *q = qz + R.q_base + s0;
    int bytes = 0, lead = -1, run = 0;
    auto fold = [&](uint32_t z, int i) {
        const bool nz = z != 1u && i < vcount;
        const int add = (lead >= 0 ? rb_small(run) : 0) + vlen32(z);
        bytes += nz ? add : 0;
        lead = (nz && lead < 0) ? i : lead;
        run = nz ? 0 : run + (i < vcount ? 1 : 0);
    };
    if (vcount == TX) {
        const uint4 *q4 = reinterpret_cast<const uint4 *>(q);
#pragma unroll 4
        for (int k = 0; k < TX / 4; ++k) {
            const uint4 v = __ldg(q4 + k);
            fold(v.x, 4 * k);
            fold(v.y, 4 * k + 1);
            fold(v.z, 4 * k + 2);
            fold(v.w, 4 * k + 3);
        }
    } else {
        for (int i = 0; i < vcount; ++i) fold(__ldg(q + i), i);
    }
    int nesc = 0;
    if (R.has_esc) {
        const int64_t bit = (int64_t)R.ebase * 32 + s0;
        const uint32_t *wp = escbits + (bit >> 5);
        const int sh = (int)(bit & 31);
        const uint64_t lo = (uint64_t)__funnelshift_r(wp[0], wp[1], sh) |
                            ((uint64_t)__funnelshift_r(wp[1], wp[2], sh) << 32);
        const uint64_t keep = vcount == 64 ? ~0ull : ((1ull << vcount) - 1);
        nesc = __popcll(lo & keep);
    }
    PieceRec pr;
    pr.bytes = (uint16_t)bytes;
    pr.vcount = (uint8_t)vcount;
    pr.lead = (uint8_t)(lead >= 0 ? lead : vcount);
    pr.trail = (uint8_t)(lead >= 0 ? run : vcount);
    pr.nesc = (uint8_t)nesc;
    pr.flags = (uint8_t)(lead >= 0 ? 1 : 0);
    pr.pad = 0;
    recs[R.piece_base + lp] = pr;
}

// item -> region map (replaces a per-CTA binary search over the regions)
__global__ void k_tile_fill_map(const RegDev *__restrict__ regs, int64_t nreg, int32_t *__restrict__ item_reg,
                                int32_t *__restrict__ chunk_reg) {
    const int64_t r = blockIdx.x;
    if (r >= nreg) return;
    const RegDev &R = regs[r];
    const int64_t nit = (int64_t)R.ntx * R.nty * R.nzc;
    for (int64_t i = threadIdx.x; i < nit; i += blockDim.x) item_reg[R.item_base + i] = (int32_t)r;
    for (int64_t i = threadIdx.x; i < R.nchunks; i += blockDim.x) chunk_reg[R.chunk_base + i] = (int32_t)r;
}

// ------------------------------------------------------------------ emit
// Token bytes, a THREAD per 64-sample piece (4 warps per CTA, 128 pieces):
// the lane folds its piece's token values into bytes sequentially, into a
// per-warp shared staging buffer at the piece's offset relative to the
// warp's first piece (a warp's 32 pieces are consecutive in one region's
// stream, so its bytes are one contiguous range [tok_off(p0), tok_off(p32))),
// then the warp writes that range with aligned 4-byte stores (byte stores
// only for its two edge words; the warp-per-piece ballot/scan version it
// replaced took 0.62 ms at c3, this one 0.55 ms).  A range larger than the buffer is written
// byte by byte from the lanes (rare).  Verbatim regions: the CTA's threads
// copy the samples of its 128 pieces, coalesced.
#ifndef CHR_EMIT_PF
#define CHR_EMIT_PF 2
#endif
#ifndef CHR_E2_WARPS
#define CHR_E2_WARPS 2
#endif
constexpr int E2_WARPS = CHR_E2_WARPS;
constexpr int E2_STAGE = 8188;  // bytes per warp (+ up to 3 alignment bytes)
template <typename T>
__global__ void __launch_bounds__(E2_WARPS * 32) k_emit_q2(const T *__restrict__ vol, const EncParams *__restrict__ P,
                                                           const RegDev *__restrict__ regs,
                                                           const int32_t *__restrict__ chunk_reg,
                                                           const PieceRec *__restrict__ recs,
                                                           const PieceOff *__restrict__ poffs,
                                                           const uint32_t *__restrict__ qz,
                                                           const uint32_t *__restrict__ escbits,
                                                           uint8_t *__restrict__ out) {
    __shared__ RegDev R;
    __shared__ __align__(16) uint8_t stage[E2_WARPS][E2_STAGE + 4];
    constexpr int PER = E2_WARPS * 32;  // pieces per CTA
    constexpr int SPLIT = (int)(CH / PER);
    const int64_t c = blockIdx.x / SPLIT;
    coop_copy(&R, regs + __ldg(chunk_reg + c));
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t lpb = (c - R.chunk_base) * CH + (int64_t)(blockIdx.x % SPLIT) * PER;  // CTA's first piece
    if (lpb >= R.npieces) return;
    const int codec = R.codec;
    const int64_t NX = P->NX, NY = P->NY;
    const int64_t exy = (int64_t)R.ex * R.ey;
    auto vol_at = [&](int64_t s) {  // portion raster index -> sample
        const int64_t z = s / exy, r = s - z * exy;
        const int64_t y = r / R.ex, x = r - y * R.ex;
        return __ldg(vol + ((R.oz + z) * NY + (R.oy + y)) * NX + R.ox + x);
    };
    if (codec != 1 && codec != 2) {  // verbatim (codec 3: f32, codec 0: f64), raster order
        const int64_t s_lo = lpb * TX, s_hi = min(s_lo + (int64_t)PER * TX, R.n);
        for (int64_t s = s_lo + threadIdx.x; s < s_hi; s += PER) {
            const T v = vol_at(s);
            if (codec == 3) put_le(out + R.payload_off + 4 * (R.s_off + s), (float)v);
            else put_le(out + R.payload_off + 8 * (R.s_off + s), (double)v);
        }
        return;
    }
    const int64_t wp0 = lpb + 32 * w;  // warp's first piece
    if (wp0 >= R.npieces) return;
    const int64_t lp = wp0 + lane;
    const bool have = lp < R.npieces;
    const int64_t wlast = min(wp0 + 32, R.npieces);  // one past the warp's last piece
    const int64_t off0 = poffs[R.piece_base + wp0].tok_off;
    // upper bound of the warp's bytes (a z-slab portion that does not end its
    // window stops short of tok_len: its trailing run belongs to the next one)
    const int64_t off_end = wlast < R.npieces ? poffs[R.piece_base + wlast].tok_off : R.tok_len;
    const bool staged = off_end - off0 <= E2_STAGE;
    int64_t cur_end = 0;  // end of this lane's bytes (relative to off0)
    uint8_t *const gdst = out + R.tok_start + off0;
    uint8_t *const sbuf = stage[w];
    // staging index = byte address mod 4 + offset: word k of the stage is an
    // aligned word of the archive, for the lanes' packed stores and the copy-out
    const int base = (int)((uintptr_t)gdst & 3);
    if (staged) {  // the lanes OR their words into a zeroed stage (edge words are shared)
        const int nw = (base + (int)(off_end - off0) + 3) >> 2;
        uint32_t *sw = reinterpret_cast<uint32_t *>(sbuf);
        for (int j = lane; j < nw; j += 32) sw[j] = 0;
        __syncwarp();
    }
    if (have) {
        const PieceOff po = poffs[R.piece_base + lp];
        const int64_t s0 = lp * TX;
        const int vcount = (int)min((int64_t)TX, R.n - s0);
        const uint32_t *q = qz + R.q_base + s0;
        const int64_t p0 = base + po.tok_off - off0;
        int64_t run = po.carry;
        // run the piece's tokens through a byte packer (bytes collect in a
        // 64-bit register and leave as aligned 4-byte stores; the lane's first
        // and last partial words as byte stores: the neighbours own the rest)
        auto emit = [&](auto st8, auto st32) {
            uint64_t acc = 0;
            int n = 0, need = (int)((4 - (p0 & 3)) & 3);
            int64_t pos = p0;
            auto add = [&](uint64_t v, int len) {  // len <= 5, n <= 3 on entry
                acc |= v << (8 * n);
                n += len;
                while (need > 0 && n > 0) {  // head bytes up to the first word boundary
                    st8(pos++, (uint8_t)acc);
                    acc >>= 8;
                    --n;
                    --need;
                }
                if (n >= 4) {
                    st32(pos, (uint32_t)acc);
                    acc >>= 32;
                    n -= 4;
                    pos += 4;
                }
                if (n >= 4) {
                    st32(pos, (uint32_t)acc);
                    acc >>= 32;
                    n -= 4;
                    pos += 4;
                }
            };
            auto leb = [](uint64_t u, int &len) {  // u < 2^35: LEB128 bytes, low byte first
                len = 1 + (u >= (1ull << 7)) + (u >= (1ull << 14)) + (u >= (1ull << 21)) + (u >= (1ull << 28));
                const uint64_t v = (u & 0x7Full) | ((u & 0x3F80ull) << 1) | ((u & 0x1FC000ull) << 2) |
                                   ((u & 0xFE00000ull) << 3) | ((u & 0x7F0000000ull) << 4);
                return v | (0x80808080ull & ((1ull << (8 * (len - 1))) - 1));
            };
            auto runs = [&](int64_t L) {  // the zero-run token before a literal (or the stream end)
                if (L == 1) {
                    add(1, 1);
                } else if (L >= 2) {
                    int len;
                    const uint64_t v = leb((uint64_t)L, len);
                    add(0, 1);
                    add(v, len);
                }
            };
            auto step = [&](uint32_t z) {
                if (z != 1u) {
                    runs(run);
                    run = 0;
                    int len;
                    const uint64_t v = leb(z, len);
                    add(v, len);
                } else {
                    ++run;
                }
            };
            if (vcount == TX) {
                const uint4 *q4 = reinterpret_cast<const uint4 *>(q);
#pragma unroll 2
                for (int k = 0; k < TX / 4; ++k) {
                    const uint4 v = __ldg(q4 + k);
                    step(v.x);
                    step(v.y);
                    step(v.z);
                    step(v.w);
                }
            } else {
                for (int i = 0; i < vcount; ++i) step(__ldg(q + i));
            }
            if (R.last && lp == R.npieces - 1) runs(run);  // the window's final zero run
            while (n > 0) {  // the last partial word
                st8(pos++, (uint8_t)acc);
                acc >>= 8;
                --n;
            }
            return pos;
        };
        // staged: a lean packer -- every word leaves by a shared atomicOr, so
        // a lane needs no byte stores for the words it shares with its
        // neighbours (acc starts with p0 & 3 zero bytes)
        auto emit_smem = [&]() -> int64_t {
            uint32_t *sw = reinterpret_cast<uint32_t *>(sbuf);
            int pw = (int)(p0 >> 2);
            uint64_t acc = 0;
            int n = (int)(p0 & 3);
            auto add = [&](uint64_t v, int len) {  // n <= 3 on entry, len <= 5
                acc |= v << (8 * n);
                n += len;
                if (n >= 4) {
                    atomicOr(sw + pw, (uint32_t)acc);
                    acc >>= 32;
                    n -= 4;
                    ++pw;
                }
                if (n >= 4) {
                    atomicOr(sw + pw, (uint32_t)acc);
                    acc >>= 32;
                    n -= 4;
                    ++pw;
                }
            };
            auto leb = [](uint64_t u, int &len) {  // u < 2^35: LEB128 bytes, low byte first
                len = 1 + (u >= (1ull << 7)) + (u >= (1ull << 14)) + (u >= (1ull << 21)) + (u >= (1ull << 28));
                const uint64_t v = (u & 0x7Full) | ((u & 0x3F80ull) << 1) | ((u & 0x1FC000ull) << 2) |
                                   ((u & 0xFE00000ull) << 3) | ((u & 0x7F0000000ull) << 4);
                return v | (0x80808080ull & ((1ull << (8 * (len - 1))) - 1));
            };
            auto runs = [&](int64_t L) {  // the zero-run token before a literal (or the stream end)
                if (L == 1) {
                    add(1, 1);
                } else if (L >= 2) {
                    int len;
                    const uint64_t v = leb((uint64_t)L, len);
                    if (len <= 3) {
                        add(v << 8, len + 1);  // the 0x00 marker and the length in one add
                    } else {
                        add(0, 1);
                        add(v, len);
                    }
                }
            };
            auto step = [&](uint32_t z) {
                if (z != 1u) {
                    if (run) runs(run);
                    run = 0;
                    // LEB128 of a 32-bit token value in 32-bit ops: 7-bit groups
                    // spread to bytes, continuation bits on all but the last
                    const int len = vlen32(z);
                    const uint32_t lo = (z & 0x7Fu) | ((z << 1) & 0x7F00u) | ((z << 2) & 0x7F0000u) |
                                        ((z << 3) & 0x7F000000u);
                    const uint32_t cont = __funnelshift_rc(0x80808080u, 0u, 8 * (5 - len));
                    add(((uint64_t)(z >> 28) << 32) | (lo | cont), len);
                } else {
                    ++run;
                }
            };
            if (vcount == TX) {
                const uint4 *q4 = reinterpret_cast<const uint4 *>(q);
#if CHR_EMIT_PF
                constexpr int EP = CHR_EMIT_PF;  // token values EP uint4 ahead of their use
                uint4 a[EP];
#pragma unroll
                for (int j = 0; j < EP; ++j) a[j] = __ldg(q4 + j);
#pragma unroll 1
                for (int k = 0; k < TX / 4; k += EP) {
                    uint4 b[EP];
#pragma unroll
                    for (int j = 0; j < EP; ++j) b[j] = k + EP < TX / 4 ? __ldg(q4 + k + EP + j) : a[j];
#pragma unroll
                    for (int j = 0; j < EP; ++j) {
                        step(a[j].x);
                        step(a[j].y);
                        step(a[j].z);
                        step(a[j].w);
                    }
#pragma unroll
                    for (int j = 0; j < EP; ++j) a[j] = b[j];
                }
#else
#pragma unroll 2
                for (int k = 0; k < TX / 4; ++k) {
                    const uint4 v = __ldg(q4 + k);
                    step(v.x);
                    step(v.y);
                    step(v.z);
                    step(v.w);
                }
#endif
            } else {
                for (int i = 0; i < vcount; ++i) step(__ldg(q + i));
            }
            if (R.last && lp == R.npieces - 1) runs(run);  // the window's final zero run
            if (n > 0) atomicOr(sw + pw, (uint32_t)acc);
            return 4 * (int64_t)pw + n;
        };
        if (staged) {
            cur_end = emit_smem();
        } else {
            uint8_t *g = gdst - base;  // 4-aligned
            cur_end = emit([&](int64_t i, uint8_t v) { g[i] = v; },
                           [&](int64_t i, uint32_t v) { *reinterpret_cast<uint32_t *>(g + i) = v; });
        }
        // codec 2: escaped samples' f64 values at their escape rank
        if (codec == 2 && recs[R.piece_base + lp].nesc) {
            const int64_t bit = (int64_t)R.ebase * 32 + s0;
            const uint32_t *wq = escbits + (bit >> 5);
            const int sh = (int)(bit & 31);
            uint64_t em = (uint64_t)__funnelshift_r(wq[0], wq[1], sh) |
                          ((uint64_t)__funnelshift_r(wq[1], wq[2], sh) << 32);
            if (vcount < 64) em &= (1ull << vcount) - 1;
            const uint64_t vbase = R.payload_off + (uint64_t)((R.n_win + 7) >> 3);
            int64_t erank = po.esc_off;
            while (em) {
                const int i = __ffsll((long long)em) - 1;
                em &= em - 1;
                put_le(out + vbase + 8 * (erank++), (double)vol_at(s0 + i));
            }
        }
    }
    if (!staged) return;
    __syncwarp();
    // the warp's bytes: stage [base, end) -> gdst - base + [base, end)
    const int end = (int)__reduce_max_sync(0xFFFFFFFFu, (unsigned)(have ? cur_end : (int64_t)base));
    uint8_t *const g = gdst - base;
    const int w0 = (base + 3) >> 2, w1 = end >> 2;  // whole words [w0, w1)
    if (w0 > w1) {  // all inside one word
        if (lane >= base && lane < end) g[lane] = sbuf[lane];
        return;
    }
    if (lane >= base && lane < 4 * w0) g[lane] = sbuf[lane];
    const uint32_t *sw = reinterpret_cast<const uint32_t *>(sbuf);
    uint32_t *gw = reinterpret_cast<uint32_t *>(g);
    for (int j = w0 + lane; j < w1; j += 32) gw[j] = sw[j];
    if (4 * w1 + lane < end) g[4 * w1 + lane] = sbuf[4 * w1 + lane];
}

// ------------------------------------------------------------------ scans
struct WarpSeg {
    __device__ static TokSeg shfl_up(const TokSeg &s, int off) {
        TokSeg r;
        r.len = __shfl_up_sync(0xFFFFFFFFu, s.len, off);
        r.lead = __shfl_up_sync(0xFFFFFFFFu, s.lead, off);
        r.trail = __shfl_up_sync(0xFFFFFFFFu, s.trail, off);
        r.bytes = __shfl_up_sync(0xFFFFFFFFu, s.bytes, off);
        r.nesc = __shfl_up_sync(0xFFFFFFFFu, s.nesc, off);
        r.nz = __shfl_up_sync(0xFFFFFFFFu, s.nz, off);
        r.f32ok = __shfl_up_sync(0xFFFFFFFFu, s.f32ok, off);
        return r;
    }
};

// inclusive block scan of one TokSeg per thread (256 threads); returns the
// thread's EXCLUSIVE prefix and writes the block total to *total
__device__ TokSeg block_excl_scan(TokSeg x, TokSeg *total) {
    __shared__ TokSeg wsum[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    TokSeg inc = x;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const TokSeg o = WarpSeg::shfl_up(inc, off);
        if (lane >= off) inc = tokseg_combine(o, inc);
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    TokSeg wpre = tokseg_identity();
    for (int i = 0; i < warp; ++i) wpre = tokseg_combine(wpre, wsum[i]);
    TokSeg excl = WarpSeg::shfl_up(inc, 1);
    if (lane == 0) excl = tokseg_identity();
    if (total) {
        TokSeg t = tokseg_identity();
        for (int i = 0; i < 8; ++i) t = tokseg_combine(t, wsum[i]);
        *total = t;
    }
    __syncthreads();
    return tokseg_combine(wpre, excl);
}

template <typename Rec>
__global__ void __launch_bounds__(256) k_scan_reduce(const EncParams *__restrict__ P,
                                                     const RegDev *__restrict__ regs,
                                                     const Rec *__restrict__ recs,
                                                     TokSeg *__restrict__ chunk_agg) {
    const int64_t c = blockIdx.x;
    __shared__ int64_t rlo, rhi;
    if (threadIdx.x == 0) {
        const RegDev &R = regs[find_region_by(regs, P->nreg, c, 1)];
        rlo = R.piece_base;
        rhi = R.piece_base + R.npieces;
    }
    __syncthreads();
    TokSeg acc = tokseg_identity();
    const int64_t p0 = c * CH + threadIdx.x * 4;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t p = p0 + k;
        if (p >= rlo && p < rhi) acc = tokseg_combine(acc, piece_to_seg(recs[p]));
    }
    TokSeg total;
    block_excl_scan(acc, &total);
    if (threadIdx.x == 0) chunk_agg[c] = total;
}

__global__ void k_scan_regions(const EncParams *__restrict__ P, RegDev *__restrict__ regs,
                               TokSeg *__restrict__ chunk_agg, int32_t *__restrict__ codec2_list,
                               EncScalars *__restrict__ sc) {
    // warp per region: 32 chunk aggregates per step, warp scan, carry
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= P->nreg) return;
    RegDev &R = regs[r];
    TokSeg acc = P->dist ? R.pre : tokseg_identity();  // portions: the stream before this rank's part
    for (int64_t c0 = 0; c0 < R.nchunks; c0 += 32) {
        const int64_t c = R.chunk_base + c0 + lane;
        const bool ok = c0 + lane < R.nchunks;
        const TokSeg a = ok ? chunk_agg[c] : tokseg_identity();
        TokSeg inc = a;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const TokSeg o = WarpSeg::shfl_up(inc, off);
            if (lane >= off) inc = tokseg_combine(o, inc);
        }
        TokSeg ex = WarpSeg::shfl_up(inc, 1);
        if (lane == 0) ex = tokseg_identity();
        if (ok) chunk_agg[c] = tokseg_combine(acc, ex);
        TokSeg tot;
        tot.len = __shfl_sync(0xFFFFFFFFu, inc.len, 31);
        tot.lead = __shfl_sync(0xFFFFFFFFu, inc.lead, 31);
        tot.trail = __shfl_sync(0xFFFFFFFFu, inc.trail, 31);
        tot.bytes = __shfl_sync(0xFFFFFFFFu, inc.bytes, 31);
        tot.nesc = __shfl_sync(0xFFFFFFFFu, inc.nesc, 31);
        tot.nz = __shfl_sync(0xFFFFFFFFu, inc.nz, 31);
        tot.f32ok = __shfl_sync(0xFFFFFFFFu, inc.f32ok, 31);
        acc = tokseg_combine(acc, tot);
    }
    if (lane != 0 || P->dist) return;
    const bool f32ok = P->dtype == CHR_F32 ? true : R.f32bad == 0;
    const bool vf32 = P->src_dtype == CHR_F32 && f32ok;
    const int64_t vlen = R.n * (vf32 ? 4 : 8);
    const int vcodec = vf32 ? 3 : 0;
    int codec;
    int64_t plen, tok = 0, nesc = 0;
    if (R.mode == 1) {
        codec = vcodec;
        plen = vlen;
    } else {
        tok = tokseg_stream_bytes(acc);
        nesc = acc.nesc;
        if (nesc) {
            codec = 2;
            plen = ((R.n + 7) >> 3) + 8 * nesc + tok;
        } else {
            codec = 1;
            plen = tok;
        }
        if (plen >= vlen) {
            codec = vcodec;
            plen = vlen;
        }
    }
    R.codec = codec;
    R.f32ok = f32ok;
    R.tok_len = tok;
    R.nesc = nesc;
    R.payload_len = plen;
    if (codec == 2) {
        const unsigned long long i = atomicAdd((unsigned long long *)&sc->n_codec2, 1ull);
        codec2_list[i] = (int32_t)r;
    }
}

// single CTA: file offsets of every block (region-id order) + CRC plan
__global__ void __launch_bounds__(1024) k_layout(const EncParams *__restrict__ P,
                                                 RegDev *__restrict__ regs, CrcSeg *__restrict__ segs,
                                                 EncScalars *__restrict__ sc) {
    __shared__ int64_t wsum[2][32];
    __shared__ int64_t carry[2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t nreg = P->nreg;
    const uint64_t H = P->header_table;
    const int seg0 = P->write_file ? 1 : 0;  // segment 0 = header+table
    if (threadIdx.x == 0) {
        carry[0] = 0;
        carry[1] = 0;
    }
    __syncthreads();
    auto nsc_of = [](uint64_t a, uint64_t b) -> int64_t { return crc_num_superchunks(a, b); };
    int64_t sc_head = 0;
    if (P->write_file) sc_head = nsc_of(0, H);
    for (int64_t t0 = 0; t0 < nreg; t0 += 1024) {
        const int64_t r = t0 + threadIdx.x;
        int64_t sz = 0, nsc = 0;
        if (r < nreg) {
            sz = kBlockHeader + regs[r].payload_len;
        }
        // block scan of sz
        int64_t v = sz;
        for (int off = 1; off < 32; off <<= 1) {
            const int64_t o = __shfl_up_sync(0xFFFFFFFFu, v, off);
            if (lane >= off) v += o;
        }
        if (lane == 31) wsum[0][warp] = v;
        __syncthreads();
        if (warp == 0) {
            int64_t s = wsum[0][lane];
            for (int off = 1; off < 32; off <<= 1) {
                const int64_t o = __shfl_up_sync(0xFFFFFFFFu, s, off);
                if (lane >= off) s += o;
            }
            wsum[0][lane] = s;
        }
        __syncthreads();
        const int64_t excl = carry[0] + (warp ? wsum[0][warp - 1] : 0) + v - sz;
        if (r < nreg) {
            RegDev &R = regs[r];
            R.block_off = H + (uint64_t)excl;
            R.payload_off = R.block_off + kBlockHeader;
            R.tok_start = R.payload_off +
                          (R.codec == 2 ? (uint64_t)((R.n_win + 7) >> 3) + 8ull * (uint64_t)R.nesc : 0ull);
            nsc = nsc_of(R.payload_off, R.payload_off + R.payload_len);
        }
        // scan of superchunk counts
        int64_t u = nsc;
        for (int off = 1; off < 32; off <<= 1) {
            const int64_t o = __shfl_up_sync(0xFFFFFFFFu, u, off);
            if (lane >= off) u += o;
        }
        if (lane == 31) wsum[1][warp] = u;
        __syncthreads();
        if (warp == 0) {
            int64_t s = wsum[1][lane];
            for (int off = 1; off < 32; off <<= 1) {
                const int64_t o = __shfl_up_sync(0xFFFFFFFFu, s, off);
                if (lane >= off) s += o;
            }
            wsum[1][lane] = s;
        }
        __syncthreads();
        const int64_t uex = carry[1] + (warp ? wsum[1][warp - 1] : 0) + u - nsc;
        if (r < nreg) {
            CrcSeg &S = segs[seg0 + r];
            S.begin = regs[r].payload_off;
            S.end = regs[r].payload_off + regs[r].payload_len;
            S.sc_base = sc_head + uex;
            S.n_sc = nsc;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            carry[0] += wsum[0][31];
            carry[1] += wsum[1][31];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const uint64_t body = H + (uint64_t)carry[0];
        sc->file_body = body;
        sc->out_nbytes = body + (P->write_file ? 4 : 0);
        sc->total_sc = sc_head + carry[1];
        if (P->write_file) {
            segs[0].begin = 0;
            segs[0].end = H;
            segs[0].sc_base = 0;
            segs[0].n_sc = sc_head;
        }
    }
}

template <typename Rec>
__global__ void __launch_bounds__(256) k_scan_down(const EncParams *__restrict__ P,
                                                   const RegDev *__restrict__ regs,
                                                   const Rec *__restrict__ recs,
                                                   const TokSeg *__restrict__ chunk_pre,
                                                   PieceOff *__restrict__ poffs) {
    const int64_t c = blockIdx.x;
    __shared__ int64_t rlo, rhi;
    if (threadIdx.x == 0) {
        const RegDev &R = regs[find_region_by(regs, P->nreg, c, 1)];
        rlo = R.piece_base;
        rhi = R.piece_base + R.npieces;
    }
    __syncthreads();
    const int64_t p0 = c * CH + threadIdx.x * 4;
    TokSeg s[4];
    TokSeg acc = tokseg_identity();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t p = p0 + k;
        s[k] = (p >= rlo && p < rhi) ? piece_to_seg(recs[p]) : tokseg_identity();
        acc = tokseg_combine(acc, s[k]);
    }
    TokSeg pre = tokseg_combine(chunk_pre[c], block_excl_scan(acc, nullptr));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t p = p0 + k;
        if (p >= rlo && p < rhi) {
            PieceOff o;
            o.tok_off = pre.bytes + (pre.nz ? run_bytes(pre.lead) : 0);
            o.carry = pre.nz ? pre.trail : pre.len;
            o.esc_off = pre.nesc;
            poffs[p] = o;
        }
        pre = tokseg_combine(pre, s[k]);
    }
}

// escape bitmaps of codec-2 regions: one byte = 8 consecutive stream samples
// codec 2: the escape bitmap (np.packbits little-endian) from k_quant's bits;
// a portion writes the bytes overlapping window bits [s_off, s_off + n) with
// its own bits only (other portions' bits stay 0, so slices OR together)
__global__ void __launch_bounds__(256) k_bitmap(const RegDev *__restrict__ regs,
                                                const int32_t *__restrict__ list,
                                                const EncScalars *__restrict__ sc,
                                                const uint32_t *__restrict__ escbits,
                                                uint8_t *__restrict__ out) {
    const int64_t nl = sc->n_codec2;
    for (int64_t li = 0; li < nl; ++li) {
        const RegDev &R = regs[list[li]];
        const int64_t b0 = R.s_off >> 3, b1 = (R.s_off + R.n + 7) >> 3;  // window bitmap bytes touched
        for (int64_t B = b0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; B < b1;
             B += (int64_t)gridDim.x * blockDim.x) {
            uint32_t v = 0;
            for (int k = 0; k < 8; ++k) {
                const int64_t sb = 8 * B + k - R.s_off;  // portion-local bit
                if (sb < 0 || sb >= R.n) continue;
                v |= ((escbits[R.ebase + (sb >> 5)] >> (sb & 31)) & 1u) << k;
            }
            out[R.payload_off + B] = (uint8_t)v;
        }
    }
}

// file header (FORMAT.md, chr_archive.py:50) + region table (chr_archive.py:51)
__global__ void __launch_bounds__(256) k_write_table(const EncParams *__restrict__ P,
                                                     const RegDev *__restrict__ regs,
                                                     uint8_t *__restrict__ out) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int m = P->m;
    const int mb = (m + 7) / 8;
    const int64_t table0 = kFileHeader + 4 + 8 * m + 4;
    if (r == 0) {
        uint8_t *p = out;
        p[0] = 'C'; p[1] = 'H'; p[2] = 'R'; p[3] = '1';
        put_le(p + 4, (uint16_t)1);
        put_le(p + 6, (uint32_t)P->NX);
        put_le(p + 10, (uint32_t)P->NY);
        put_le(p + 14, (uint32_t)P->NZ);
        put_le(p + 18, P->spacing[0]);
        put_le(p + 26, P->spacing[1]);
        put_le(p + 34, P->spacing[2]);
        p[42] = (uint8_t)P->src_dtype;
        put_le(p + 43, (uint32_t)P->bs);
        put_le(p + 47, P->vmin);
        put_le(p + 55, P->vmax);
        put_le(p + 63, (uint32_t)m);
        for (int i = 0; i < m; ++i) put_le(p + 67 + 8 * i, P->cands[i]);
        put_le(p + 67 + 8 * m, (uint32_t)P->nreg);
    }
    if (r >= P->nreg) return;
    const RegDev &R = regs[r];
    uint8_t *p = out + table0 + r * (kRegionFixed + mb);
    put_le(p, (uint32_t)r);
    for (int a = 0; a < 3; ++a) {
        put_le(p + 4 + 4 * a, (uint32_t)R.lo[a]);
        put_le(p + 16 + 4 * a, (uint32_t)R.hi[a]);
    }
    put_le(p + 28, (uint32_t)R.ox);
    put_le(p + 32, (uint32_t)R.oy);
    put_le(p + 36, (uint32_t)R.oz);
    put_le(p + 40, (uint32_t)R.ex);
    put_le(p + 44, (uint32_t)R.ey);
    put_le(p + 48, (uint32_t)R.ez);
    p[52] = (uint8_t)P->bound_mode;  // 0 strict_vertices, 1 paper_edges
    put_le(p + 53, P->accuracy);     // stored accuracy
    put_le(p + 61, R.e);
    put_le(p + 69, (uint64_t)R.block_off);
    put_le(p + 77, (uint64_t)(kBlockHeader + R.payload_len));
    for (int i = 0; i < mb; ++i) p[85 + i] = (uint8_t)(R.mask >> (8 * i));
}

// 34-byte block headers + per-region CRC + file-CRC contributions
// warp per region: payload CRC, block header, and the region's share of
// the file CRC; the x^(8n) shifts are warp-parallel
__global__ void __launch_bounds__(128) k_finalize_regions(const EncParams *__restrict__ P,
                                                          RegDev *__restrict__ regs,
                                                          const uint32_t *__restrict__ seg_raw,
                                                          const CrcTables *__restrict__ tabs,
                                                          EncScalars *__restrict__ sc,
                                                          uint8_t *__restrict__ out) {
    __shared__ uint32_t t0[256], x2n[64];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) t0[i] = tabs->t[0][i];
    if (threadIdx.x < 64) x2n[threadIdx.x] = tabs->x2n[threadIdx.x];
    __syncthreads();
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int seg0 = P->write_file ? 1 : 0;
    const uint64_t body = sc->file_body;
    if (r == 0 && P->write_file) {
        const uint32_t c = gf2_mul(warp_x8n(x2n, body - P->header_table), seg_raw[0]);
        if (lane == 0 && c) atomicXor(&sc->file_raw, c);
    }
    if (r >= P->nreg) return;
    RegDev &R = regs[r];
    const uint32_t praw = seg_raw[seg0 + r];
    // zlib crc = raw ^ (0xFFFFFFFF * x^(8 len)) ^ 0xFFFFFFFF
    const uint32_t crc = gf2_mul(warp_x8n(x2n, (uint64_t)R.payload_len), 0xFFFFFFFFu) ^ praw ^ 0xFFFFFFFFu;
    uint8_t h[kBlockHeader];
    h[0] = (uint8_t)R.codec;
    put_le(h + 1, (uint32_t)R.ex);
    put_le(h + 5, (uint32_t)R.ey);
    put_le(h + 9, (uint32_t)R.ez);
    put_le(h + 13, R.e);
    h[21] = (uint8_t)P->src_dtype;
    put_le(h + 22, (uint64_t)R.payload_len);
    put_le(h + 30, crc);
    if (lane == 0) R.crc = crc;
    uint8_t *dst = out + R.block_off;
    if (lane < kBlockHeader) dst[lane] = h[lane];
    if (lane + 32 < kBlockHeader) dst[lane + 32] = h[lane + 32];
    if (P->write_file) {
        const uint32_t hraw = crc_raw_bytes(t0, 0, h, kBlockHeader);
        uint32_t c = gf2_mul(warp_x8n(x2n, body - (R.block_off + kBlockHeader)), hraw);
        c ^= gf2_mul(warp_x8n(x2n, body - (R.payload_off + R.payload_len)), praw);
        if (lane == 0 && c) atomicXor(&sc->file_raw, c);
    }
}

__global__ void k_finalize_file(const CrcTables *__restrict__ tabs, const EncScalars *__restrict__ sc,
                                uint8_t *__restrict__ out) {
    const uint32_t crc = crc_finalize(tabs->x2n, sc->file_raw, sc->file_body);
    put_le(out + sc->file_body, crc);
}

// ------------------------------------------------------------------ segment encoder
// Single-read encoder path (no quantum intermediate in HBM).  An item is a
// band of whole rows (rb rows + the halo row y0-1) x up to SG_ZMAX planes of
// one region window, marching z.  The band's rows of one plane are a
// contiguous piece of the window's raster stream (a segment); warp w owns
// the slots [w W, (w + 1) W) of it -- a PIECE of the stream:
//   k_qseg   quantise + Lorenzo q and reduce each piece's token stream to
//            its summary (the token-size monoid, PieceRec2); nothing per
//            sample leaves the SM but (rare) escape bits
//   k_scan_reduce / k_scan_regions / k_scan_down
//            exclusive prefix of every piece in its region's stream order
//            (plane, band, warp), codec decision, file layout
//   k_qemit  recomputes q from the input (the second and last read) and
//            writes every token byte at its final offset
// Per plane, phase 1 runs over the band-plane's slots with a block stride
// (coalesced loads): u, D = u - u(z-1) into shared memory (u(z-1) kept per
// slot in sU).  Phase 2 gives each lane SG_L consecutive slots: it reads D,
// forms q = D - D(x-1) - D(y-1) + D(x-1,y-1) and folds its samples into a
// 32-bit token summary sequentially (a few instructions per sample); lanes
// combine by one ordered warp reduction (k_qseg) or scan (k_qemit, which
// then writes its samples' tokens sequentially).  Shared arrays are padded
// (index i + i/8) so both access patterns are bank-conflict free; D and the
// escape flags are double-buffered by plane: one barrier per plane.
constexpr int SG_T = 256;                // threads per item
constexpr int SG_NW = SG_T / 32;
constexpr int SG_L = 8;                  // consecutive slots per lane in phase 2
constexpr int SG_SPAN = 4096;            // max band-plane slots incl. the halo row
constexpr int SG_TARGET = 2048;          // band height target: (rb + 1) * ex <= SG_TARGET
constexpr int SG_ZMAX = 16;              // planes per item
static_assert(SG_SPAN / SG_T <= 32, "phase-1 slot masks are 32-bit");

__device__ __forceinline__ int sp_idx(int i) { return i + (i >> 3); }  // padded shared index

// 32-bit token-size monoid inside one piece (<= SG_SPAN samples)
struct TS32 {
    int32_t len, lead, trail, bytes, nesc, nz;
};
__device__ __forceinline__ TS32 ts32_identity() { return TS32{0, 0, 0, 0, 0, 0}; }
__device__ __forceinline__ int rb32(int L) { return L <= 0 ? 0 : (L == 1 ? 1 : 1 + vlen32((uint32_t)L)); }
__device__ __forceinline__ TS32 ts32_combine(const TS32 &a, const TS32 &b) {
    TS32 r;
    r.len = a.len + b.len;
    r.nesc = a.nesc + b.nesc;
    r.nz = a.nz | b.nz;
    r.lead = a.nz ? a.lead : a.len + b.lead;
    r.trail = b.nz ? b.trail : (a.nz ? a.trail + b.len : r.len);
    r.bytes = a.bytes + b.bytes + ((a.nz && b.nz) ? rb32(a.trail + b.lead) : 0);
    return r;
}
__device__ __forceinline__ TS32 ts32_shfl(const TS32 &s, int off, bool up) {
    TS32 r;
    if (up) {
        r.len = __shfl_up_sync(0xFFFFFFFFu, s.len, off);
        r.lead = __shfl_up_sync(0xFFFFFFFFu, s.lead, off);
        r.trail = __shfl_up_sync(0xFFFFFFFFu, s.trail, off);
        r.bytes = __shfl_up_sync(0xFFFFFFFFu, s.bytes, off);
        r.nesc = __shfl_up_sync(0xFFFFFFFFu, s.nesc, off);
        r.nz = __shfl_up_sync(0xFFFFFFFFu, s.nz, off);
    } else {
        r.len = __shfl_down_sync(0xFFFFFFFFu, s.len, off);
        r.lead = __shfl_down_sync(0xFFFFFFFFu, s.lead, off);
        r.trail = __shfl_down_sync(0xFFFFFFFFu, s.trail, off);
        r.bytes = __shfl_down_sync(0xFFFFFFFFu, s.bytes, off);
        r.nesc = __shfl_down_sync(0xFFFFFFFFu, s.nesc, off);
        r.nz = __shfl_down_sync(0xFFFFFFFFu, s.nz, off);
    }
    return r;
}

__device__ __forceinline__ TS32 ts32_bcast(const TS32 &s, int src) {
    TS32 r;
    r.len = __shfl_sync(0xFFFFFFFFu, s.len, src);
    r.lead = __shfl_sync(0xFFFFFFFFu, s.lead, src);
    r.trail = __shfl_sync(0xFFFFFFFFu, s.trail, src);
    r.bytes = __shfl_sync(0xFFFFFFFFu, s.bytes, src);
    r.nesc = __shfl_sync(0xFFFFFFFFu, s.nesc, src);
    r.nz = __shfl_sync(0xFFFFFFFFu, s.nz, src);
    return r;
}

struct SegGeom {
    int band, y0, rows, z0, z1, ex, span, W;
    uint32_t M;  // row = umulhi(slot, M) for slot < SG_SPAN (M = ceil(2^32 / ex); ex == 1 special)
};

__device__ __forceinline__ SegGeom seg_geom(const RegDev &R, int64_t item) {
    SegGeom g;
    const int64_t local = item - R.item_base;
    g.band = (int)(local % R.nty);
    const int zc = (int)(local / R.nty);
    g.ex = R.ex;
    g.y0 = g.band * R.rb;
    g.rows = min(R.rb, R.ey - g.y0);
    g.z0 = zc * R.zl;
    g.z1 = min(g.z0 + R.zl, R.ez);
    g.span = (g.rows + 1) * g.ex;
    // slots per warp: whole 256-slot chunks (lanes full in phase 2; a small
    // band-plane leaves the last warps idle rather than every lane half-used)
    g.W = 32 * SG_L * ((g.span + SG_T * SG_L - 1) / (SG_T * SG_L));
    g.M = (uint32_t)((0x100000000ull + (uint64_t)g.ex - 1) / (uint64_t)g.ex);
    return g;
}

__device__ __forceinline__ int seg_row(const SegGeom &G, int i) {
    return G.ex == 1 ? i : (int)__umulhi((uint32_t)i, G.M);
}

// piece (warp range of one band-plane) index in the region's stream order
__device__ __forceinline__ int64_t seg_piece(const RegDev &R, int z, int band, int warp) {
    return R.piece_base + ((int64_t)z * R.nty + band) * SG_NW + warp;
}

// Shared memory of an item: one dynamic array (int32 words), addressed by
// integer offsets so every access compiles to LDS/STS: D x 2 (by plane
// parity) and U, each padded (sp_idx), then the escape flags x 2 (bytes).
extern __shared__ __align__(16) int32_t sg_w[];
struct SegSmem {
    int ps;                  // padded words per array
    int d0, d1, u;           // word offsets
};
__device__ __forceinline__ SegSmem seg_smem(int span_cap) {
    SegSmem s;
    s.ps = sp_idx(span_cap) + 16;  // + lookahead of a lane's SG_L slots
    s.d0 = 0;
    s.d1 = s.ps;
    s.u = 2 * s.ps;
    return s;
}
__device__ __forceinline__ uint8_t *seg_flags(const SegSmem &S, int par, int span_cap) {
    return reinterpret_cast<uint8_t *>(sg_w + 3 * S.ps) + par * (span_cap + 16);
}
// staged input of plane parity par (cp.async, one element per slot)
template <typename T>
__device__ __forceinline__ T *seg_stage(const SegSmem &S, int par, int span_cap) {
    unsigned char *b = reinterpret_cast<unsigned char *>(sg_w + 3 * S.ps) + 2 * (span_cap + 16);
    b = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(b) + 15) & ~uintptr_t(15));
    return reinterpret_cast<T *>(b) + par * span_cap;
}

// asynchronous copy of the thread's strided slots of one plane into the
// staging buffer (rows above the window are not copied: their u is 0)
template <typename T>
__device__ __forceinline__ void seg_issue(const SegGeom &G, const T *base, int64_t NX, T *stage) {
    for (int i = threadIdx.x; i < G.span; i += SG_T) {
        const int row = seg_row(G, i);
        if (G.y0 - 1 + row >= 0) {
            const T *src = base + (int64_t)row * NX + (i - row * G.ex);
            const unsigned dst = (unsigned)__cvta_generic_to_shared(stage + i);
            if (sizeof(T) == 4)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src) : "memory");
            else
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
        }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void seg_wait_prev() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// u at plane z0 - 1 of the thread's slots (0 outside the window); escape
// flags cleared
template <typename T>
__device__ __forceinline__ void seg_init(const RegDev &R, const SegGeom &G, const Quant &Q, bool quant,
                                         const T *base, int64_t NX, int64_t plane, const SegSmem &S,
                                         int span_cap) {
    uint8_t *e0 = seg_flags(S, 0, span_cap), *e1 = seg_flags(S, 1, span_cap);
    for (int i = threadIdx.x; i < S.ps; i += SG_T) {  // D zero past the span (lookahead reads)
        sg_w[S.d0 + i] = 0;
        sg_w[S.d1 + i] = 0;
    }
    for (int i = threadIdx.x; i < G.span; i += SG_T) {
        int32_t u = 0;
        const int row = seg_row(G, i);
        if (quant && (G.z0 > 0 || R.zhalo) && G.y0 - 1 + row >= 0) {
            bool e;
            u = quantize(Q, (double)__ldg(base - plane + (int64_t)row * NX + (i - row * G.ex)), e);
        }
        sg_w[S.u + sp_idx(i)] = u;
        e0[i] = 0;
        e1[i] = 0;
    }
}

// phase 1 of one plane: D = u - u(z-1) for the thread's strided slots; the
// (rare) lanes whose fast quantiser path failed run the exact sequence
// afterwards; returns the thread's escape mask (bit k = slot tid + SG_T k)
template <typename T, bool CHK32>
__device__ __forceinline__ uint32_t seg_phase1(const SegGeom &G, const Quant &Q, bool quant, const T *base,
                                               int64_t NX, const SegSmem &S, int par, int span_cap,
                                               uint32_t clear_escm, bool &inexact) {
    const int dofs = par ? S.d1 : S.d0, uofs = S.u;
    const T *stage = seg_stage<T>(S, par, span_cap);
    uint8_t *sE = seg_flags(S, par, span_cap);
    while (clear_escm) {  // flags this thread set two planes ago in this buffer
        const int k = __ffs(clear_escm) - 1;
        clear_escm &= clear_escm - 1;
        sE[threadIdx.x + SG_T * k] = 0;
    }
    uint32_t slowm = 0;
    int k = 0;
#pragma unroll 4
    for (int i = threadIdx.x; i < G.span; i += SG_T, ++k) {
        const int row = seg_row(G, i);
        int32_t u = 0;
        if (G.y0 - 1 + row >= 0) {
            const T tv = stage[i];
            if (CHK32 && row >= 1) inexact |= not_f32_exact(tv);
            if (quant && !quant_fast(Q, (double)tv, u)) slowm |= 1u << k;
        }
        const int p = sp_idx(i);
        sg_w[dofs + p] = u - sg_w[uofs + p];
        sg_w[uofs + p] = u;
    }
    uint32_t escm = 0;
    while (slowm) {  // exact sequence; prev = u_fast - D keeps D = u - prev exact
        const int kk = __ffs(slowm) - 1;
        slowm &= slowm - 1;
        const int i = threadIdx.x + SG_T * kk;
        const int row = seg_row(G, i);
        bool e;
        const int32_t u = quantize(Q, (double)stage[i], e);
        const int p = sp_idx(i);
        const int32_t prev = sg_w[uofs + p] - sg_w[dofs + p];
        sg_w[dofs + p] = u - prev;
        sg_w[uofs + p] = u;
        if (e && row >= 1) {
            escm |= 1u << kk;
            sE[i] = 1;
        }
    }
    return escm;
}

// phase 2 helper: the lane's SG_L consecutive slots [i0, i0 + SG_L) (i0 a
// multiple of SG_L) below lim: token values (zigzag + 1; 1 = zero or not own)
// and bit masks of own / nonzero / escaped slots (own slots are contiguous).
// Straight-line: own range and row starts as masks, reads clamped in-bounds.
struct LaneQ {
    uint32_t z1[SG_L];
    uint32_t own, nz, esc;  // bit j
};
__device__ __forceinline__ LaneQ seg_lane_q(const SegGeom &G, const SegSmem &S, int par, int span_cap, int i0,
                                            int lim, bool any_esc) {
    LaneQ L;
    if (i0 >= lim) {  // no slot of this lane (its reads would leave the arrays)
#pragma unroll
        for (int j = 0; j < SG_L; ++j) L.z1[j] = 1u;
        L.own = L.nz = L.esc = 0;
        return L;
    }
    const int dofs = par ? S.d1 : S.d0;
    const int lo = min(max(G.ex - i0, 0), SG_L), hi = min(lim - i0, SG_L);  // own slots [lo, hi)
    L.own = (hi > lo) ? (((1u << hi) - 1u) & ~((1u << lo) - 1u)) : 0u;
    const int x0 = i0 - seg_row(G, i0) * G.ex;
    uint32_t rs = 0;  // slots j with x == 0
    for (int t = x0 == 0 ? 0 : G.ex - x0; t < SG_L; t += G.ex) rs |= 1u << t;
    const int pb = dofs + sp_idx(i0);  // slot i0 + j sits at pb + j (i0 % 8 == 0)
    const int pu = i0 - G.ex;          // up-row slot of j = 0 (negative only when not own)
    int32_t dl = sg_w[dofs + sp_idx(max(i0 - 1, 0))];
    int32_t ul = sg_w[dofs + sp_idx(max(pu - 1, 0))];
    uint32_t nzm = 0;
#pragma unroll
    for (int j = 0; j < SG_L; ++j) {
        const int32_t d = sg_w[pb + j];
        const int32_t du = sg_w[dofs + sp_idx(max(pu + j, 0))];
        const int32_t q = d - du - (((rs >> j) & 1u) ? 0 : dl - ul);
        const uint32_t z1v = ((L.own >> j) & 1u) ? zz1_32(q) : 1u;
        L.z1[j] = z1v;
        nzm |= (z1v != 1u ? 1u : 0u) << j;
        dl = d;
        ul = du;
    }
    L.nz = nzm;
    uint32_t em = 0;
    if (any_esc) {
        const uint8_t *sE = seg_flags(S, par, span_cap);
#pragma unroll
        for (int j = 0; j < SG_L; ++j)
            if ((L.own >> j) & 1u) em |= (sE[i0 + j] ? 1u : 0u) << j;
    }
    L.esc = em;
    return L;
}

// the lane's summary from its masks: bytes = sum of literal varint sizes +
// run tokens between literals (gaps < SG_L: rb = [gap >= 1] + [gap >= 2])
__device__ __forceinline__ TS32 lane_summary(const LaneQ &L) {
    TS32 t;
    const uint32_t own = L.own, m = L.nz;
    t.len = __popc(own);
    t.nesc = __popc(L.esc);
    t.nz = m != 0;
    int vb = 0;
#pragma unroll
    for (int j = 0; j < SG_L; ++j) vb += ((m >> j) & 1u) ? vlen32(L.z1[j]) : 0;
    const uint32_t later = m & (m - 1);                 // nonzeros after the first
    const uint32_t g1 = later & ~(m << 1);              // ... whose previous slot is zero
    const uint32_t g2 = g1 & ~(m << 2);                 // ... and the one before it too
    t.bytes = vb + __popc(g1) + __popc(g2);
    const int a = own ? __ffs(own) - 1 : 0, b = own ? 32 - __clz(own) : 0;  // own slots [a, b)
    t.lead = m ? (__ffs(m) - 1) - a : t.len;
    t.trail = m ? (b - 1) - (31 - __clz(m)) : t.len;
    return t;
}

// pass 1: the summary of every piece (warp range of a band-plane)
template <typename T>
__global__ void __launch_bounds__(SG_T, 3) k_qseg(const T *__restrict__ vol, const EncParams *__restrict__ P,
                                                  RegDev *__restrict__ regs, const int32_t *__restrict__ item_reg,
                                                  PieceRec2 *__restrict__ recs, uint32_t *__restrict__ escbits,
                                                  int span_cap) {
    __shared__ RegDev R;
    const int64_t item = blockIdx.x;
    const int ri = __ldg(item_reg + item);
    coop_copy(&R, regs + ri);
    __syncthreads();
    const SegGeom G = seg_geom(R, item);
    const SegSmem S = seg_smem(span_cap);
    const int64_t NX = P->NX, NY = P->NY, plane = NX * NY;
    const bool quant = R.mode == 0;
    const Quant Q = make_quant(R.e);
    const bool chk32 = sizeof(T) == 8 && P->src_dtype == CHR_F32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const T *base = vol + ((int64_t)(R.oz + G.z0) * NY + R.oy + G.y0 - 1) * NX + R.ox;  // halo row, plane z0
    seg_init(R, G, Q, quant, base, NX, plane, S, span_cap);
    seg_issue(G, base, NX, seg_stage<T>(S, G.z0 & 1, span_cap));
    __syncthreads();
    bool inexact = false;
    uint32_t hist0 = 0u, hist1 = 0u;  // escape masks of the last two planes (by parity)
    const int wlo = warp * G.W, whi = min(wlo + G.W, G.span);
    for (int z = G.z0; z < G.z1; ++z, base += plane) {
        const int par = z & 1;
        if (z + 1 < G.z1) seg_issue(G, base + plane, NX, seg_stage<T>(S, par ^ 1, span_cap));
        else asm volatile("cp.async.commit_group;\n" ::: "memory");
        seg_wait_prev();
        const uint32_t clr = par ? hist1 : hist0;
        const uint32_t escm = chk32 ? seg_phase1<T, true>(G, Q, quant, base, NX, S, par, span_cap, clr, inexact)
                                    : seg_phase1<T, false>(G, Q, quant, base, NX, S, par, span_cap, clr, inexact);
        if (par) hist1 = escm; else hist0 = escm;
        const bool any_esc = __syncthreads_or(escm != 0);
        if (escm) {  // rare: escape bits at the window's raster index
            uint32_t m = escm;
            while (m) {
                const int kk = __ffs(m) - 1;
                m &= m - 1;
                const int i = threadIdx.x + SG_T * kk;
                const int64_t bit = (int64_t)R.ebase * 32 + ((int64_t)z * R.ey + G.y0) * G.ex + (i - G.ex);
                atomicOr(escbits + (bit >> 5), 1u << (bit & 31));
            }
            atomicOr(&regs[ri].has_esc, 1);
        }
        TS32 acc = ts32_identity();
        for (int c0 = wlo; c0 < whi; c0 += 32 * SG_L) {  // warp-uniform
            const LaneQ L = seg_lane_q(G, S, par, span_cap, c0 + SG_L * lane, whi, any_esc);
            TS32 t = lane_summary(L);
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {  // ordered tree: lane 0 ends with the chunk
                const TS32 o = ts32_shfl(t, off, false);
                if ((lane & (2 * off - 1)) == 0) t = ts32_combine(t, o);
            }
            acc = ts32_combine(acc, t);  // lane 0's value is the one used
        }
        if (lane == 0) {
            PieceRec2 pr;
            pr.len = (uint16_t)acc.len;
            pr.lead = (uint16_t)acc.lead;
            pr.trail = (uint16_t)acc.trail;
            pr.nesc = (uint16_t)acc.nesc;
            pr.bytes = (uint32_t)acc.bytes;
            pr.nz = (uint32_t)acc.nz;
            recs[seg_piece(R, z, G.band, warp)] = pr;
        }
    }
    if (chk32 && __any_sync(0xFFFFFFFFu, inexact) && lane == 0) atomicOr(&regs[ri].f32bad, 1);
}

// pass 2: recompute q, place and write every token byte (codec 1 / 2),
// escape values (codec 2), or the samples themselves (codec 3 / 0).  The
// warp's stream offset comes from its piece's exclusive prefix (PieceOff);
// lanes get theirs from one ordered warp scan per chunk, then write their
// samples' tokens sequentially.
template <typename T>
__global__ void __launch_bounds__(SG_T, 3) k_qemit(const T *__restrict__ vol, const EncParams *__restrict__ P,
                                                   const RegDev *__restrict__ regs,
                                                   const int32_t *__restrict__ item_reg,
                                                   const PieceOff *__restrict__ poffs, uint8_t *__restrict__ out,
                                                   int span_cap) {
    __shared__ RegDev R;
    const int64_t item = blockIdx.x;
    const int ri = __ldg(item_reg + item);
    coop_copy(&R, regs + ri);
    __syncthreads();
    const SegGeom G = seg_geom(R, item);
    const int64_t NX = P->NX, NY = P->NY, plane = NX * NY;
    const int codec = R.codec;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const T *base = vol + ((int64_t)(R.oz + G.z0) * NY + R.oy + G.y0 - 1) * NX + R.ox;  // halo row, plane z0
    if (codec == 0 || codec == 3) {  // verbatim: the samples in raster order
        for (int z = G.z0; z < G.z1; ++z, base += plane) {
            const int64_t s0 = R.s_off + ((int64_t)z * R.ey + G.y0) * G.ex - G.ex;  // stream index of slot 0
            for (int i = G.ex + threadIdx.x; i < G.span; i += SG_T) {
                const int row = seg_row(G, i);
                const T v = __ldg(base + (int64_t)row * NX + (i - row * G.ex));
                if (codec == 3) put_le(out + R.payload_off + 4 * (s0 + i), (float)v);
                else put_le(out + R.payload_off + 8 * (s0 + i), (double)v);
            }
        }
        return;
    }
    const SegSmem S = seg_smem(span_cap);
    const Quant Q = make_quant(R.e);
    seg_init(R, G, Q, true, base, NX, plane, S, span_cap);
    seg_issue(G, base, NX, seg_stage<T>(S, G.z0 & 1, span_cap));
    __syncthreads();
    const uint64_t vbase = R.payload_off + (uint64_t)((R.n_win + 7) >> 3);
    uint8_t *const tok = out + R.tok_start;
    const int wlo = warp * G.W, whi = min(wlo + G.W, G.span);
    const bool ends_window = R.last && G.band == R.nty - 1 && wlo < G.span && whi == G.span;
    uint32_t hist0 = 0u, hist1 = 0u;  // escape masks of the last two planes (by parity)
    bool unused = false;
    for (int z = G.z0; z < G.z1; ++z, base += plane) {
        const int par = z & 1;
        if (z + 1 < G.z1) seg_issue(G, base + plane, NX, seg_stage<T>(S, par ^ 1, span_cap));
        else asm volatile("cp.async.commit_group;\n" ::: "memory");
        const PieceOff po = poffs[seg_piece(R, z, G.band, warp)];
        seg_wait_prev();
        const uint32_t escm =
            seg_phase1<T, false>(G, Q, true, base, NX, S, par, span_cap, par ? hist1 : hist0, unused);
        if (par) hist1 = escm; else hist0 = escm;
        const bool any_esc = __syncthreads_or(escm != 0);
        // placement after (piece prefix) ++ r (r: this warp's samples so far):
        //   token offset = r.nz ? tok_off + r.bytes + run_bytes(carry + r.lead) : tok_off
        //   zero carry   = r.nz ? r.trail : carry + r.len
        TS32 r = ts32_identity();
        for (int c0 = wlo; c0 < whi; c0 += 32 * SG_L) {  // warp-uniform
            const int i0 = c0 + SG_L * lane;
            const LaneQ L = seg_lane_q(G, S, par, span_cap, i0, whi, any_esc);
            const TS32 t = lane_summary(L);
            TS32 inc = t;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const TS32 o = ts32_shfl(inc, off, true);
                if (lane >= off) inc = ts32_combine(o, inc);
            }
            TS32 ex = ts32_shfl(inc, 1, true);
            if (lane == 0) ex = ts32_identity();
            const TS32 pre = ts32_combine(r, ex);  // samples of this piece before the lane's
            if (t.nz || t.nesc) {
                int64_t off = pre.nz ? po.tok_off + pre.bytes + run_bytes(po.carry + pre.lead) : po.tok_off;
                int64_t zc = pre.nz ? (int64_t)pre.trail : po.carry + pre.len;  // zeros since the last literal
                int64_t nesc = po.esc_off + pre.nesc;
#pragma unroll
                for (int j = 0; j < SG_L; ++j) {
                    if (!((L.own >> j) & 1u)) continue;
                    const uint32_t z1v = L.z1[j];
                    if (z1v != 1u) {
                        uint8_t *p = tok + off;
                        uint8_t *e = put_varint32(put_run(p, zc), z1v);
                        off += e - p;
                        zc = 0;
                    } else {
                        ++zc;
                    }
                    if ((L.esc >> j) & 1u) {
                        const int i = i0 + j;
                        const int row = seg_row(G, i);
                        const double v = (double)__ldg(base + (int64_t)row * NX + (i - row * G.ex));
                        put_le(out + vbase + 8 * nesc, v);
                        ++nesc;
                    }
                }
            }
            r = ts32_combine(r, ts32_bcast(inc, 31));
        }
        // the window's final zero run, after its last sample
        if (ends_window && z == R.ez - 1 && lane == 0) {
            const int64_t off = r.nz ? po.tok_off + r.bytes + run_bytes(po.carry + r.lead) : po.tok_off;
            const int64_t fin = r.nz ? (int64_t)r.trail : po.carry + r.len;
            put_run(tok + off, fin);
        }
    }
}

// ------------------------------------------------------------------ host
struct EncPlan {
    std::vector<RegDev> regs;
    int64_t nitems = 0, npieces_total = 0, nchunks = 0, qtotal = 0, etotal = 0;
    bool portions = false;  // empty windows allowed (z-slab portions)
    bool segmode = false;   // single-read segment path (k_qseg / k_qemit)
    int span_cap = 0;       // segment path: max band-plane slots (multiple of 32)
    PieceRec2 *recs2 = nullptr;  // segment path: piece summaries (k_qseg)
    size_t ws_bytes = 0, keep_bytes = 0;
    // carved pointers
    EncParams *params;
    RegDev *d_regs;
    PieceRec *recs;
    PieceOff *poffs;
    TokSeg *chunk;
    CrcSeg *segs;
    uint32_t *seg_raw;
    int32_t *codec2;
    EncScalars *scal;
    int32_t *item_reg, *chunk_reg;
    uint32_t *qz, *escbits;
    // host-built item -> region and chunk -> region maps (uploaded with the
    // region records; shared by the per-thread plan cache)
    std::shared_ptr<const std::vector<int32_t>> hitem, hchunk;
};

static void host_maps(EncPlan &pl) {
    auto it = std::make_shared<std::vector<int32_t>>((size_t)pl.nitems + 1, 0);
    auto ch = std::make_shared<std::vector<int32_t>>((size_t)pl.nchunks + 1, 0);
    for (size_t r = 0; r < pl.regs.size(); ++r) {
        const RegDev &R = pl.regs[r];
        const int64_t nit = pl.segmode ? (int64_t)R.nty * R.nzc : (int64_t)R.ntx * R.nty * R.nzc;
        for (int64_t i = 0; i < nit; ++i) (*it)[R.item_base + i] = (int32_t)r;
        for (int64_t i = 0; i < R.nchunks; ++i) (*ch)[R.chunk_base + i] = (int32_t)r;
    }
    pl.hitem = it;
    pl.hchunk = ch;
}

static bool build_plan_uncached(const chr_region_t *h, int64_t nreg, EncPlan &pl) {
    pl.regs.resize(nreg);
    int64_t item = 0, piece = 0, chunk = 0;
    for (int64_t r = 0; r < nreg; ++r) {
        RegDev &R = pl.regs[r];
        std::memset(&R, 0, sizeof(R));
        R.ox = h[r].origin[0];
        R.oy = h[r].origin[1];
        R.oz = h[r].origin[2];
        R.ex = h[r].extent[0];
        R.ey = h[r].extent[1];
        R.ez = h[r].extent[2];
        if (R.ex < 1 || R.ey < 1 || R.ez < (pl.portions ? 0 : 1)) return false;
        R.e = h[r].error_bound;
        if (!(R.e >= 0.0) || !std::isfinite(R.e)) return false;
        R.mode = R.e == 0.0 ? 1 : 0;
        R.n = (int64_t)R.ex * R.ey * R.ez;
        R.ntx = (int32_t)ceil_div(R.ex, TX);
        R.nty = (int32_t)ceil_div(R.ey, TY);
        R.nzc = (int32_t)ceil_div(R.ez, ZC);
        R.qband = 0;
        R.rb = 0;
        R.qzch = ZC;
        if (R.ex <= QB_CAP / 2) {  // full-row bands: rb rows + the halo row fit one CTA's slots
            // balanced bands and plane chunks (a 33-row window is one band
            // of 33 rows, not 30 + 3; 33 planes one chunk, not 16 + 16 + 1)
            R.qband = 1;
            const int rbmax = std::max(1, std::min(R.ey, QB_CAP / R.ex - 1));
            R.nty = (int32_t)ceil_div(R.ey, rbmax);
            R.rb = (int32_t)ceil_div(R.ey, R.nty);
            R.nty = (int32_t)ceil_div(R.ey, R.rb);
            R.ntx = 1;
            if (R.ez > 0) {  // (an empty z-slab portion has no items)
                R.nzc = (int32_t)ceil_div(R.ez, QB_ZMAX);
                R.qzch = (int32_t)ceil_div(R.ez, R.nzc);
                R.nzc = (int32_t)ceil_div(R.ez, R.qzch);
            }
        }
        R.item_base = item;
        item += (int64_t)R.ntx * R.nty * R.nzc;
        R.piece_base = piece;
        R.npieces = ceil_div(R.n, TX);  // 64-sample pieces of the raster stream
        R.chunk_base = chunk;
        R.nchunks = ceil_div(R.npieces, CH);
        chunk += R.nchunks;
        piece += R.nchunks * CH;
        R.s_off = 0;
        R.n_win = R.n;
        R.zhalo = 0;
        R.last = 1;
        R.pre = tokseg_identity();
        R.q_base = pl.qtotal;
        pl.qtotal += (R.n + 3) & ~int64_t(3);  // 16-byte aligned token values per region (k_summarize2)
        R.ebase = pl.etotal;
        pl.etotal += ceil_div(R.n, 32) + 1;
        R.mask = h[r].mask;
        for (int a = 0; a < 3; ++a) {
            R.lo[a] = h[r].lo[a];
            R.hi[a] = h[r].hi[a];
        }
    }
    pl.nitems = item;
    pl.npieces_total = piece;
    pl.nchunks = chunk;
    return true;
}

// Segment-path geometry (k_qseg / k_qemit): bands of rb whole rows with
// (rb + 1) * ex <= SG_TARGET (at least one row: (1 + 1) * ex <= SG_SPAN),
// z-chunks of <= SG_ZMAX planes balanced over the window; a segment per
// (plane, band) in stream order; scan chunks of CH segments.  Returns false
// when a window is too wide for the path (the caller keeps the piece path).
static bool plan_segments(EncPlan &pl) {
    int64_t item = 0, seg = 0, chunk = 0, span_cap = 32;
    for (const RegDev &R : pl.regs)
        if (2 * (int64_t)R.ex > SG_SPAN) return false;
    for (RegDev &R : pl.regs) {
        R.rb = (int32_t)std::max<int64_t>(1, std::min<int64_t>(R.ey, SG_TARGET / R.ex - 1));
        R.ntx = 1;
        R.nty = (int32_t)ceil_div(R.ey, R.rb);
        R.nzc = (int32_t)std::max<int64_t>(1, ceil_div(R.ez, SG_ZMAX));
        R.zl = (int32_t)std::max<int64_t>(1, ceil_div(R.ez, R.nzc));
        R.nzc = (int32_t)std::max<int64_t>(1, ceil_div(R.ez, R.zl));
        R.qband = 0;
        R.item_base = item;
        item += (int64_t)R.nty * R.nzc;
        R.piece_base = seg;
        R.npieces = (int64_t)R.ez * R.nty * SG_NW;  // pieces: (plane, band, warp) in stream order
        R.chunk_base = chunk;
        R.nchunks = std::max<int64_t>(1, ceil_div(R.npieces, CH));
        chunk += R.nchunks;
        seg += R.nchunks * CH;
        span_cap = std::max<int64_t>(span_cap, (int64_t)(std::min(R.rb, R.ey) + 1) * R.ex);
    }
    pl.nitems = item;
    pl.npieces_total = seg;
    pl.nchunks = chunk;
    pl.span_cap = (int)((span_cap + 31) & ~int64_t(31));
    pl.qtotal = 0;  // no quantum intermediate
    pl.segmode = true;
    return true;
}

// SegSmem: D x 2 + U (padded int32, + lookahead) + escape flags x 2 (bytes)
// + staged input x 2 (elem bytes each)
static size_t seg_smem_bytes(int span_cap, size_t elem) {
    return 3 * sizeof(int32_t) * (size_t)(span_cap + span_cap / 8 + 16) + 2 * (size_t)(span_cap + 16) + 16 +
           2 * elem * (size_t)span_cap + 16;
}

// The pipeline asks for the workspace size and then compresses with the same
// region table: the host plan of the last table is kept per thread (the table
// is compared byte for byte, ~3 us, instead of rebuilt, ~25 us at 426 regions).
static bool build_plan(const chr_region_t *h, int64_t nreg, EncPlan &pl, bool allow_seg = true) {
    struct Cache {
        std::vector<chr_region_t> key;
        EncPlan plan;
        bool allow_seg = true;
        bool valid = false;
    };
    thread_local Cache C;
    // the piece path stays the default: the segment path reads the input once
    // less but issues ~1.5x the instructions; CHR_ENC_SEG=1
    allow_seg = allow_seg && getenv("CHR_ENC_SEG") != nullptr;
    if (pl.portions) {
        if (!build_plan_uncached(h, nreg, pl)) return false;
        host_maps(pl);
        return true;
    }
    if (C.valid && C.allow_seg == allow_seg && (int64_t)C.key.size() == nreg &&
        std::memcmp(C.key.data(), h, sizeof(chr_region_t) * (size_t)nreg) == 0) {
        pl = C.plan;
        return true;
    }
    C.valid = false;
    if (!build_plan_uncached(h, nreg, pl)) return false;
    if (allow_seg) plan_segments(pl);  // false (a window too wide): the piece path
    host_maps(pl);
    C.key.assign(h, h + nreg);
    C.plan = pl;
    C.allow_seg = allow_seg;
    C.valid = true;
    return true;
}

static void carve(EncPlan &pl, void *base, size_t cap) {
    WsCarver c{reinterpret_cast<char *>(base), 0, cap};
    const int64_t nreg = (int64_t)pl.regs.size();
    // what the CRC tail (crc_launch, k_finalize_*) reads comes first: a
    // caller overlapping that tail reuses the workspace past keep_bytes
    pl.params = c.take<EncParams>(1);
    pl.d_regs = c.take<RegDev>(nreg);
    pl.segs = c.take<CrcSeg>(nreg + 1);
    pl.seg_raw = c.take<uint32_t>(nreg + 1);
    pl.scal = c.take<EncScalars>(1);
    pl.keep_bytes = (c.off + 255) & ~size_t(255);
    pl.recs = c.take<PieceRec>(pl.segmode ? 0 : pl.npieces_total);
    pl.poffs = c.take<PieceOff>(pl.npieces_total);
    pl.chunk = c.take<TokSeg>(pl.nchunks);
    pl.codec2 = c.take<int32_t>(nreg);
    pl.item_reg = c.take<int32_t>(pl.nitems + 1);
    pl.chunk_reg = c.take<int32_t>(pl.nchunks + 1);
    pl.qz = c.take<uint32_t>(pl.qtotal + 1);
    if (pl.segmode) {
        pl.recs2 = c.take<PieceRec2>(pl.npieces_total);
    }
    pl.escbits = c.take<uint32_t>(pl.etotal + 2);
    pl.ws_bytes = ((c.off + 255) & ~size_t(255)) + 256;  // 256-aligned: callers carve past it
}

}  // namespace chr

using namespace chr;

extern "C" size_t chr_compress_workspace_size(const chr_region_t *h, int64_t nreg) {
    CHR_XFER_SCOPE;
    EncPlan pl;
    if (!h || nreg < 1 || !build_plan(h, nreg, pl)) return 0;
    carve(pl, nullptr, ~size_t(0));
    return pl.ws_bytes;
}

extern "C" uint64_t chr_compress_capacity(const chr_region_t *h, int64_t nreg, int m, int src_dtype) {
    CHR_XFER_SCOPE;
    (void)src_dtype;
    uint64_t cap = (uint64_t)kFileHeader + 4 + 8ull * m + 4 + 4;
    const int mb = (m + 7) / 8;
    for (int64_t r = 0; r < nreg; ++r) {
        const uint64_t n = (uint64_t)h[r].extent[0] * h[r].extent[1] * h[r].extent[2];
        cap += kRegionFixed + mb + kBlockHeader + 8 * n;
    }
    return cap;
}

extern "C" int chr_compress2(const void *d_vol, int dtype, int src_dtype, int64_t nx, int64_t ny, int64_t nz,
                             const double *spacing, int64_t bs, double vmin, double vmax, const double *h_cands,
                             int m, chr_region_t *h_regions, int64_t nreg, int write_file, int bound_mode,
                             double accuracy, void *d_ws, size_t ws_bytes, uint8_t *d_out, uint64_t out_cap,
                             uint64_t *h_out_nbytes, void *stream);

extern "C" int chr_compress(const void *d_vol, int dtype, int src_dtype, int64_t nx, int64_t ny,
                            int64_t nz, const double *spacing, int64_t bs, double vmin, double vmax,
                            const double *h_cands, int m, chr_region_t *h_regions, int64_t nreg,
                            int write_file, void *d_ws, size_t ws_bytes, uint8_t *d_out,
                            uint64_t out_cap, uint64_t *h_out_nbytes, void *stream) {
    CHR_XFER_SCOPE;
    return chr_compress2(d_vol, dtype, src_dtype, nx, ny, nz, spacing, bs, vmin, vmax, h_cands, m, h_regions, nreg,
                         write_file, 0, 1.0, d_ws, ws_bytes, d_out, out_cap, h_out_nbytes, stream);
}

static int compress_impl(const void *d_vol, int dtype, int src_dtype, int64_t nx, int64_t ny, int64_t nz,
                         const double *spacing, int64_t bs, double vmin, double vmax, const double *h_cands, int m,
                         chr_region_t *h_regions, int64_t nreg, int write_file, int bound_mode, double accuracy,
                         void *d_ws, size_t ws_bytes, uint8_t *d_out, uint64_t out_cap, uint64_t *h_out_nbytes,
                         Side *side, size_t *keep_bytes, void **d_regs_out, cudaStream_t st);

extern "C" int chr_compress2(const void *d_vol, int dtype, int src_dtype, int64_t nx, int64_t ny, int64_t nz,
                             const double *spacing, int64_t bs, double vmin, double vmax, const double *h_cands,
                             int m, chr_region_t *h_regions, int64_t nreg, int write_file, int bound_mode,
                             double accuracy, void *d_ws, size_t ws_bytes, uint8_t *d_out, uint64_t out_cap,
                             uint64_t *h_out_nbytes, void *stream) {
    CHR_XFER_SCOPE;
    return compress_impl(d_vol, dtype, src_dtype, nx, ny, nz, spacing, bs, vmin, vmax, h_cands, m, h_regions, nreg,
                         write_file, bound_mode, accuracy, d_ws, ws_bytes, d_out, out_cap, h_out_nbytes, nullptr,
                         nullptr, nullptr, (cudaStream_t)stream);
}

namespace chr {
int compress_with_side(const void *d_vol, int dtype, int src_dtype, int64_t nx, int64_t ny, int64_t nz,
                       const double *spacing, int64_t bs, double vmin, double vmax, const double *h_cands, int m,
                       chr_region_t *h_regions, int64_t nreg, void *d_ws, size_t ws_bytes, uint8_t *d_out,
                       uint64_t out_cap, uint64_t *h_out_nbytes, Side *side, size_t *keep_bytes, void **d_regs,
                       cudaStream_t st) {
    return compress_impl(d_vol, dtype, src_dtype, nx, ny, nz, spacing, bs, vmin, vmax, h_cands, m, h_regions, nreg, 1,
                         0, 1.0, d_ws, ws_bytes, d_out, out_cap, h_out_nbytes, side, keep_bytes, d_regs, st);
}

__global__ void k_crc_out(const RegDev *__restrict__ regs, int64_t nreg, uint32_t *__restrict__ crc) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < nreg) crc[r] = regs[r].crc;
}

int compress_crcs(const void *d_regs, int64_t nreg, uint32_t *d_crc, cudaStream_t st) {
    if (nreg < 1) return CHR_OK;
    CHR_PROF("k_crc_out", st);
    k_crc_out<<<(unsigned)ceil_div(nreg, 256), 256, 0, st>>>(reinterpret_cast<const RegDev *>(d_regs), nreg, d_crc);
    return cudaGetLastError() == cudaSuccess ? CHR_OK : CHR_E_CUDA;
}
}  // namespace chr

static int compress_impl(const void *d_vol, int dtype, int src_dtype, int64_t nx, int64_t ny, int64_t nz,
                         const double *spacing, int64_t bs, double vmin, double vmax, const double *h_cands, int m,
                         chr_region_t *h_regions, int64_t nreg, int write_file, int bound_mode, double accuracy,
                         void *d_ws, size_t ws_bytes, uint8_t *d_out, uint64_t out_cap, uint64_t *h_out_nbytes,
                         Side *side, size_t *keep_bytes, void **d_regs_out, cudaStream_t st) {
    if (bound_mode < 0 || bound_mode > 1 || !(accuracy > 0.0 && accuracy <= 1.0)) return CHR_E_PARAMETER;
    if (!d_vol || !h_regions || nreg < 1 || !d_out || !h_out_nbytes) return CHR_E_PARAMETER;
    if (dtype != CHR_F32 && dtype != CHR_F64) return CHR_E_PARAMETER;
    if (src_dtype != CHR_F32 && src_dtype != CHR_F64) return CHR_E_PARAMETER;
    if (write_file && (m < 1 || m > 64 || !h_cands || !spacing)) return CHR_E_PARAMETER;
    EncPlan pl;
    if (!build_plan(h_regions, nreg, pl)) return CHR_E_PARAMETER;
    for (const RegDev &R : pl.regs)
        if (R.ox < 0 || R.oy < 0 || R.oz < 0 || R.ox + R.ex > nx || R.oy + R.ey > ny || R.oz + R.ez > nz)
            return CHR_E_PARAMETER;
    carve(pl, d_ws, ws_bytes);
    if (!d_ws || pl.ws_bytes > ws_bytes) return CHR_E_WORKSPACE;
    const CrcTables *tabs = crc_tables_device();
    if (!tabs) return CHR_E_CUDA;

    EncParams hp;
    std::memset(&hp, 0, sizeof(hp));
    hp.NX = nx;
    hp.NY = ny;
    hp.NZ = nz;
    hp.nreg = nreg;
    hp.nitems = pl.nitems;
    hp.nchunks = pl.nchunks;
    hp.dtype = dtype;
    hp.src_dtype = src_dtype;
    hp.write_file = write_file ? 1 : 0;
    hp.m = write_file ? m : 0;
    for (int a = 0; a < 3; ++a) hp.spacing[a] = spacing ? spacing[a] : 1.0;
    hp.vmin = vmin;
    hp.vmax = vmax;
    hp.bs = bs;
    for (int i = 0; i < hp.m; ++i) hp.cands[i] = h_cands[i];
    hp.header_table = write_file ? (uint64_t)(kFileHeader + 4 + 8 * m + 4) +
                                       (uint64_t)nreg * (kRegionFixed + (m + 7) / 8)
                                 : 0;
    hp.bound_mode = bound_mode;
    hp.accuracy = accuracy;
    // capacity check against the worst case (verbatim f64 everywhere)
    if (out_cap < chr_compress_capacity(h_regions, nreg, m, src_dtype)) return CHR_E_PARAMETER;

    CHR_CUDA_TRY(h2d_multi({{pl.params, &hp, sizeof(hp)},
                            {pl.d_regs, pl.regs.data(), sizeof(RegDev) * nreg},
                            {pl.item_reg, pl.hitem->data(), sizeof(int32_t) * pl.hitem->size()},
                            {pl.chunk_reg, pl.hchunk->data(), sizeof(int32_t) * pl.hchunk->size()}},
                           st));
    CHR_CUDA_TRY(zero_async({{pl.scal, sizeof(EncScalars)},
                             {pl.seg_raw, sizeof(uint32_t) * (nreg + 1)},
                             {pl.escbits, sizeof(uint32_t) * (pl.etotal + 2)}},
                            st));

    const unsigned items = (unsigned)pl.nitems, chunks = (unsigned)pl.nchunks;
    if (pl.segmode) {
        const size_t smem = seg_smem_bytes(pl.span_cap, dtype == CHR_F32 ? 4 : 8);
        if (smem > 48 * 1024) {
            CHR_CUDA_TRY(cudaFuncSetAttribute(k_qseg<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CHR_CUDA_TRY(cudaFuncSetAttribute(k_qseg<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CHR_CUDA_TRY(cudaFuncSetAttribute(k_qemit<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CHR_CUDA_TRY(cudaFuncSetAttribute(k_qemit<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        }
        if (dtype == CHR_F32) {
            CHR_PROF("k_qseg<float>", st);
            k_qseg<float><<<items, SG_T, smem, st>>>((const float *)d_vol, pl.params, pl.d_regs, pl.item_reg,
                                                     pl.recs2, pl.escbits, pl.span_cap);
        } else {
            CHR_PROF("k_qseg<double>", st);
            k_qseg<double><<<items, SG_T, smem, st>>>((const double *)d_vol, pl.params, pl.d_regs, pl.item_reg,
                                                      pl.recs2, pl.escbits, pl.span_cap);
        }
        {
            CHR_PROF("k_scan_reduce", st);
            k_scan_reduce<<<chunks, 256, 0, st>>>(pl.params, pl.d_regs, pl.recs2, pl.chunk);
        }
    } else {
        if (dtype == CHR_F32) {
            CHR_PROF("k_quant<float>", st);
            k_quant<float><<<items, NW * 32, 0, st>>>((const float *)d_vol, pl.params, pl.d_regs, pl.item_reg,
                                                      pl.qz, pl.escbits);
            k_quant_band<float><<<items, QB_T, 0, st>>>((const float *)d_vol, pl.params, pl.d_regs, pl.item_reg,
                                                        pl.qz, pl.escbits);
        } else {
            CHR_PROF("k_quant<double>", st);
            k_quant<double><<<items, NW * 32, 0, st>>>((const double *)d_vol, pl.params, pl.d_regs, pl.item_reg,
                                                       pl.qz, pl.escbits);
            k_quant_band<double><<<items, QB_T, 0, st>>>((const double *)d_vol, pl.params, pl.d_regs,
                                                            pl.item_reg, pl.qz, pl.escbits);
        }
        {
            CHR_PROF("k_summarize", st);
            k_summarize2<<<chunks * CSPLIT, 256, 0, st>>>(pl.d_regs, pl.chunk_reg, pl.qz, pl.escbits, pl.recs);
        }
        {
            CHR_PROF("k_scan_reduce", st);
            k_scan_reduce<<<chunks, 256, 0, st>>>(pl.params, pl.d_regs, pl.recs, pl.chunk);
        }
    }
    {
        CHR_PROF("k_scan_regions", st);
        k_scan_regions<<<(unsigned)ceil_div(nreg, 4), 128, 0, st>>>(pl.params, pl.d_regs, pl.chunk,
                                                                    pl.codec2, pl.scal);
    }
    {
        CHR_PROF("k_layout", st);
        k_layout<<<1, 1024, 0, st>>>(pl.params, pl.d_regs, pl.segs, pl.scal);
    }
    if (pl.segmode) {
        const size_t smem = seg_smem_bytes(pl.span_cap, dtype == CHR_F32 ? 4 : 8);
        {
            CHR_PROF("k_scan_down", st);
            k_scan_down<<<chunks, 256, 0, st>>>(pl.params, pl.d_regs, pl.recs2, pl.chunk, pl.poffs);
        }
        if (dtype == CHR_F32) {
            CHR_PROF("k_qemit<float>", st);
            k_qemit<float><<<items, SG_T, smem, st>>>((const float *)d_vol, pl.params, pl.d_regs, pl.item_reg,
                                                      pl.poffs, d_out, pl.span_cap);
        } else {
            CHR_PROF("k_qemit<double>", st);
            k_qemit<double><<<items, SG_T, smem, st>>>((const double *)d_vol, pl.params, pl.d_regs, pl.item_reg,
                                                       pl.poffs, d_out, pl.span_cap);
        }
    } else {
        {
            CHR_PROF("k_scan_down", st);
            k_scan_down<<<chunks, 256, 0, st>>>(pl.params, pl.d_regs, pl.recs, pl.chunk, pl.poffs);
        }
        if (dtype == CHR_F32) {
            CHR_PROF("k_emit_q<float>", st);
            k_emit_q2<float><<<chunks * (unsigned)(CH / (E2_WARPS * 32)), E2_WARPS * 32, 0, st>>>((const float *)d_vol, pl.params, pl.d_regs,
                                                             pl.chunk_reg, pl.recs, pl.poffs, pl.qz, pl.escbits,
                                                             d_out);
        } else {
            CHR_PROF("k_emit_q<double>", st);
            k_emit_q2<double><<<chunks * (unsigned)(CH / (E2_WARPS * 32)), E2_WARPS * 32, 0, st>>>((const double *)d_vol, pl.params, pl.d_regs,
                                                              pl.chunk_reg, pl.recs, pl.poffs, pl.qz, pl.escbits,
                                                              d_out);
        }
    }
    {
        CHR_PROF("k_bitmap", st);
        k_bitmap<<<148, 256, 0, st>>>(pl.d_regs, pl.codec2, pl.scal, pl.escbits, d_out);
    }
    if (write_file)
        {
            CHR_PROF("k_write_table", st);
            k_write_table<<<(unsigned)ceil_div(nreg, 256), 256, 0, st>>>(pl.params, pl.d_regs, d_out);
        }
    CHR_CUDA_TRY(cudaGetLastError());
    // the host needs the layout (codecs, offsets, lengths: known since
    // k_layout), not the CRCs: with a side stream the CRC tail runs there
    EncScalars hs;
    if (side) CHR_CUDA_TRY(d2h_multi({{pl.regs.data(), pl.d_regs, sizeof(RegDev) * nreg}, {&hs, pl.scal, sizeof(hs)}}, st));
    cudaStream_t ct = st;
    if (side) {
        CHR_CUDA_TRY(cudaEventRecord(side->ev[0], st));
        CHR_CUDA_TRY(cudaStreamWaitEvent(side->st, side->ev[0], 0));
        ct = side->st;
    }
    // CRC segments: the superchunk total lives on the device; a persistent
    // grid strides over it (no host round trip)
    const int64_t nseg = nreg + (write_file ? 1 : 0);
    int rc = crc_launch(d_out, pl.segs, nseg, 0, pl.seg_raw, ct);
    if (rc) return rc;
    {
        CHR_PROF("k_finalize_regions", ct);
        k_finalize_regions<<<(unsigned)ceil_div(nreg, 4), 128, 0, ct>>>(pl.params, pl.d_regs, pl.seg_raw,
                                                                          tabs, pl.scal, d_out);
    }
    if (write_file)
    {
        CHR_PROF("k_finalize_file", ct);
            k_finalize_file<<<1, 1, 0, ct>>>(tabs, pl.scal, d_out);
    }
    CHR_CUDA_TRY(cudaGetLastError());
    if (side) {
        CHR_CUDA_TRY(cudaEventRecord(side->ev[1], side->st));
        if (keep_bytes) *keep_bytes = pl.keep_bytes;
        if (d_regs_out) *d_regs_out = pl.d_regs;
    } else {
        CHR_CUDA_TRY(d2h_multi({{pl.regs.data(), pl.d_regs, sizeof(RegDev) * nreg}, {&hs, pl.scal, sizeof(hs)}}, st));
    }
    CHR_CUDA_TRY(stream_sync(st));
    for (int64_t r = 0; r < nreg; ++r) {
        const RegDev &R = pl.regs[r];
        chr_region_t &o = h_regions[r];
        o.codec_id = R.codec;
        o.payload_crc = side ? 0u : R.crc;  // side: compress_crcs() after side->ev[1]
        o.block_offset = R.block_off;
        o.block_nbytes = kBlockHeader + (uint64_t)R.payload_len;
        o.n_escaped = (uint64_t)R.nesc;
    }
    *h_out_nbytes = hs.out_nbytes;
    return CHR_OK;
}

// ------------------------------------------------------------------ token-stream seam
// rle_varint_encode (kernels.py:198-296) on a device int64 array: the same
// summarize -> scan -> emit kernels as the archive path, on one "region"
// of n samples whose token values come from the caller's quanta.
namespace chr {
__global__ void k_q_to_tokens(const int64_t *__restrict__ q, int64_t n, uint32_t *__restrict__ qz,
                              int32_t *__restrict__ bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = q[i];
        if (v > (1ll << 30) || v < -(1ll << 30)) {  // |q| <= 2^30
            atomicOr(bad, 1);
            continue;
        }
        qz[i] = zz1_32((int32_t)v);
    }
}
__global__ void k_force_tokens(RegDev *__restrict__ R) {
    R->codec = 1;
    R->payload_off = 0;
    R->tok_start = 0;
    R->payload_len = R->tok_len;
}
}  // namespace chr

static chr_region_t rle_region(int64_t n) {
    chr_region_t h;
    std::memset(&h, 0, sizeof(h));
    h.extent[0] = (int32_t)n;
    h.extent[1] = 1;
    h.extent[2] = 1;
    h.error_bound = 1.0;
    return h;
}

extern "C" size_t chr_rle_encode_workspace_size(int64_t n) {
    CHR_XFER_SCOPE;
    if (n < 1 || n > INT32_MAX) return 256;
    const chr_region_t h = rle_region(n);
    EncPlan pl;
    if (!build_plan(&h, 1, pl, false)) return 256;
    carve(pl, nullptr, ~size_t(0));
    return pl.ws_bytes + 256;
}

extern "C" int chr_rle_encode(const int64_t *d_q, int64_t n, uint8_t *d_out, uint64_t out_cap, void *d_ws,
                              size_t ws_bytes, uint64_t *h_nbytes, void *stream) {
    CHR_XFER_SCOPE;
    if (!h_nbytes) return CHR_E_PARAMETER;
    if (n == 0) {
        *h_nbytes = 0;
        return CHR_OK;
    }
    if (!d_q || !d_out || n < 0 || n > INT32_MAX) return CHR_E_PARAMETER;
    if (out_cap < 5ull * (uint64_t)n + 16) return CHR_E_PARAMETER;
    cudaStream_t st = (cudaStream_t)stream;
    const chr_region_t h = rle_region(n);
    EncPlan pl;
    if (!build_plan(&h, 1, pl, false)) return CHR_E_PARAMETER;
    carve(pl, d_ws, ws_bytes);
    if (!d_ws || pl.ws_bytes + 256 > ws_bytes) return CHR_E_WORKSPACE;
    int32_t *d_bad = reinterpret_cast<int32_t *>(reinterpret_cast<char *>(d_ws) + pl.ws_bytes);
    EncParams hp;
    std::memset(&hp, 0, sizeof(hp));
    hp.NX = n;
    hp.NY = 1;
    hp.NZ = 1;
    hp.nreg = 1;
    hp.nitems = pl.nitems;
    hp.nchunks = pl.nchunks;
    hp.dtype = CHR_F64;
    hp.src_dtype = CHR_F64;
    CHR_CUDA_TRY(h2d(pl.params, &hp, sizeof(hp), st));
    CHR_CUDA_TRY(h2d(pl.d_regs, pl.regs.data(), sizeof(RegDev), st));
    CHR_CUDA_TRY(fill_async(pl.scal, 0, sizeof(EncScalars), st));
    CHR_CUDA_TRY(fill_async(pl.escbits, 0, sizeof(uint32_t) * (pl.etotal + 2), st));
    CHR_CUDA_TRY(fill_async(d_bad, 0, sizeof(int32_t), st));
    const unsigned chunks = (unsigned)pl.nchunks;
    k_tile_fill_map<<<1, 256, 0, st>>>(pl.d_regs, 1, pl.item_reg, pl.chunk_reg);
    {
        CHR_PROF("k_q_to_tokens", st);
        k_q_to_tokens<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 148 * 16), 256, 0, st>>>(d_q, n, pl.qz, d_bad);
    }
    {
        CHR_PROF("k_summarize", st);
        k_summarize2<<<chunks * CSPLIT, 256, 0, st>>>(pl.d_regs, pl.chunk_reg, pl.qz, pl.escbits, pl.recs);
    }
    k_scan_reduce<<<chunks, 256, 0, st>>>(pl.params, pl.d_regs, pl.recs, pl.chunk);
    k_scan_regions<<<1, 128, 0, st>>>(pl.params, pl.d_regs, pl.chunk, pl.codec2, pl.scal);
    k_force_tokens<<<1, 1, 0, st>>>(pl.d_regs);
    k_scan_down<<<chunks, 256, 0, st>>>(pl.params, pl.d_regs, pl.recs, pl.chunk, pl.poffs);
    {
        CHR_PROF("k_emit_q<double>", st);
        k_emit_q2<double><<<chunks * (unsigned)(CH / (E2_WARPS * 32)), E2_WARPS * 32, 0, st>>>(nullptr, pl.params, pl.d_regs, pl.chunk_reg, pl.recs, pl.poffs,
                                                 pl.qz, pl.escbits, d_out);
    }
    CHR_CUDA_TRY(cudaGetLastError());
    int32_t bad = 0;
    CHR_CUDA_TRY(d2h(&bad, d_bad, sizeof(bad), st));
    CHR_CUDA_TRY(d2h(pl.regs.data(), pl.d_regs, sizeof(RegDev), st));
    CHR_CUDA_TRY(stream_sync(st));
    if (bad) return CHR_E_PARAMETER;
    *h_nbytes = (uint64_t)pl.regs[0].tok_len;
    return CHR_OK;
}

// ------------------------------------------------------------------ z-slab protocol
// rank r encodes the planes [zs, ze) of every window (its
// "portion", a contiguous piece of the window's raster stream) from a local
// volume holding planes [z_base, z_base + nz_local) (zs - 1 and the block
// ghost plane included).  Phase 1 summarises each portion's stream (the
// token-size monoid); after an allgather of those summaries every rank knows
// each window's codec, length and layout and the summary of the stream
// before its own portion, writes its bytes at their final offsets (phase 2)
// and returns the raw CRC of its share of each payload (zeros elsewhere:
// CRC is linear over GF(2), so the shares XOR to the payload CRC).  Rank 0
// then writes the block headers and the trailer (phase 3).
static bool dist_plan(const chr_region_t *h, int64_t nreg, int64_t z_base, int64_t nz_local, int64_t zs,
                      int64_t ze, EncPlan &pl) {
    std::vector<chr_region_t> loc(h, h + nreg);
    std::vector<int64_t> pa(nreg), pb(nreg);
    for (int64_t r = 0; r < nreg; ++r) {
        const int64_t oz = h[r].origin[2], ez = h[r].extent[2];
        pa[r] = std::max(oz, zs);
        pb[r] = std::max(pa[r], std::min(oz + ez, ze));
        loc[r].origin[2] = (int32_t)(pa[r] - z_base);
        loc[r].extent[2] = (int32_t)(pb[r] - pa[r]);
        if (pb[r] > pa[r] && (pa[r] - (pa[r] > oz ? 1 : 0) < z_base || pb[r] > z_base + nz_local)) return false;
    }
    pl.portions = true;
    if (!build_plan(loc.data(), nreg, pl)) return false;
    for (int64_t r = 0; r < nreg; ++r) {
        RegDev &R = pl.regs[r];
        const int64_t oz = h[r].origin[2];
        R.s_off = (pa[r] - oz) * (int64_t)R.ex * R.ey;
        R.n_win = (int64_t)R.ex * R.ey * h[r].extent[2];
        R.zhalo = pa[r] > oz ? 1 : 0;
        R.last = pb[r] == oz + h[r].extent[2] ? 1 : 0;
    }
    return true;
}

extern "C" size_t chr_dcompress_workspace_size(const chr_region_t *h, int64_t nreg, int64_t z_base, int64_t nz_local,
                                               int64_t zs, int64_t ze) {
    CHR_XFER_SCOPE;
    EncPlan pl;
    if (!h || nreg < 1 || !dist_plan(h, nreg, z_base, nz_local, zs, ze, pl)) return 0;
    carve(pl, nullptr, ~size_t(0));
    // + CRC segments of this rank (<= 3 per region) and the header phase's tables
    return pl.ws_bytes + (sizeof(CrcSeg) + 8) * (size_t)(3 * nreg + 2) + sizeof(RegDev) * (size_t)nreg + 8192;
}

namespace chr {
__global__ void k_portion_agg(const RegDev *__restrict__ regs, int64_t nreg, const TokSeg *__restrict__ chunk_agg,
                              int dtype_f32, TokSeg *__restrict__ out) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= nreg) return;
    const RegDev &R = regs[r];
    TokSeg acc = tokseg_identity();
    for (int64_t c0 = 0; c0 < R.nchunks; c0 += 32) {
        const bool ok = c0 + lane < R.nchunks;
        TokSeg inc = ok ? chunk_agg[R.chunk_base + c0 + lane] : tokseg_identity();
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const TokSeg o = WarpSeg::shfl_up(inc, off);
            if (lane >= off) inc = tokseg_combine(o, inc);
        }
        TokSeg tot;
        tot.len = __shfl_sync(0xFFFFFFFFu, inc.len, 31);
        tot.lead = __shfl_sync(0xFFFFFFFFu, inc.lead, 31);
        tot.trail = __shfl_sync(0xFFFFFFFFu, inc.trail, 31);
        tot.bytes = __shfl_sync(0xFFFFFFFFu, inc.bytes, 31);
        tot.nesc = __shfl_sync(0xFFFFFFFFu, inc.nesc, 31);
        tot.nz = __shfl_sync(0xFFFFFFFFu, inc.nz, 31);
        tot.f32ok = __shfl_sync(0xFFFFFFFFu, inc.f32ok, 31);
        acc = tokseg_combine(acc, tot);
    }
    if (lane == 0) {
        acc.f32ok = dtype_f32 ? 1 : (R.f32bad == 0 ? 1 : 0);
        out[r] = acc;
    }
}
}  // namespace chr

static void dist_params(EncParams &hp, const EncPlan &pl, int64_t nx, int64_t ny, int64_t nz_local, int dtype,
                        int src_dtype, int write_file, const double *spacing, int64_t bs, double vmin, double vmax,
                        const double *h_cands, int m, int64_t nreg) {
    std::memset(&hp, 0, sizeof(hp));
    hp.NX = nx;
    hp.NY = ny;
    hp.NZ = nz_local;
    hp.nreg = nreg;
    hp.nitems = pl.nitems;
    hp.nchunks = pl.nchunks;
    hp.dtype = dtype;
    hp.src_dtype = src_dtype;
    hp.write_file = write_file;
    hp.m = m;
    hp.dist = 1;
    for (int a = 0; a < 3; ++a) hp.spacing[a] = spacing ? spacing[a] : 1.0;
    hp.vmin = vmin;
    hp.vmax = vmax;
    hp.bs = bs;
    for (int i = 0; i < m && i < 64; ++i) hp.cands[i] = h_cands[i];
    hp.header_table = (uint64_t)(kFileHeader + 4 + 8 * m + 4) + (uint64_t)nreg * (kRegionFixed + (m + 7) / 8);
    hp.bound_mode = 0;
    hp.accuracy = 1.0;
}

// phase 1: quantise this rank's portions and summarise their streams
extern "C" int chr_dcompress_local(const void *d_vol, int dtype, int src_dtype, int64_t nx, int64_t ny,
                                   int64_t nz_local, int64_t z_base, int64_t zs, int64_t ze,
                                   const chr_region_t *h_regions, int64_t nreg, void *d_ws, size_t ws_bytes,
                                   chr_portion_t *h_portions, void *stream) {
    CHR_XFER_SCOPE;
    if (!d_vol || !h_regions || nreg < 1 || !h_portions) return CHR_E_PARAMETER;
    if (dtype != CHR_F32 && dtype != CHR_F64) return CHR_E_PARAMETER;
    static_assert(sizeof(chr_portion_t) == sizeof(TokSeg), "chr_portion_t mirrors TokSeg");
    cudaStream_t st = (cudaStream_t)stream;
    EncPlan pl;
    if (!dist_plan(h_regions, nreg, z_base, nz_local, zs, ze, pl)) return CHR_E_PARAMETER;
    for (const RegDev &R : pl.regs)
        if (R.ox < 0 || R.oy < 0 || R.ox + R.ex > nx || R.oy + R.ey > ny) return CHR_E_PARAMETER;
    carve(pl, d_ws, ws_bytes);
    if (!d_ws || pl.ws_bytes > ws_bytes) return CHR_E_WORKSPACE;
    TokSeg *d_agg = reinterpret_cast<TokSeg *>(reinterpret_cast<char *>(d_ws) + pl.ws_bytes);
    EncParams hp;
    dist_params(hp, pl, nx, ny, nz_local, dtype, src_dtype, 0, nullptr, 1, 0, 0, nullptr, 0, nreg);
    CHR_CUDA_TRY(h2d(pl.params, &hp, sizeof(hp), st));
    CHR_CUDA_TRY(h2d(pl.d_regs, pl.regs.data(), sizeof(RegDev) * nreg, st));
    CHR_CUDA_TRY(fill_async(pl.escbits, 0, sizeof(uint32_t) * (pl.etotal + 2), st));
    const unsigned items = (unsigned)pl.nitems, chunks = (unsigned)pl.nchunks;
    k_tile_fill_map<<<(unsigned)nreg, 256, 0, st>>>(pl.d_regs, nreg, pl.item_reg, pl.chunk_reg);
    if (items) {
        CHR_PROF(dtype == CHR_F32 ? "k_quant<float>" : "k_quant<double>", st);
        if (dtype == CHR_F32)
            k_quant<float><<<items, NW * 32, 0, st>>>((const float *)d_vol, pl.params, pl.d_regs, pl.item_reg,
                                                      pl.qz, pl.escbits);
        if (dtype == CHR_F32)
            k_quant_band<float><<<items, QB_T, 0, st>>>((const float *)d_vol, pl.params, pl.d_regs, pl.item_reg,
                                                        pl.qz, pl.escbits);
        else
            k_quant<double><<<items, NW * 32, 0, st>>>((const double *)d_vol, pl.params, pl.d_regs, pl.item_reg,
                                                       pl.qz, pl.escbits);
        if (dtype != CHR_F32)
            k_quant_band<double><<<items, QB_T, 0, st>>>((const double *)d_vol, pl.params, pl.d_regs, pl.item_reg,
                                                         pl.qz, pl.escbits);
    }
    if (chunks) {
        {
            CHR_PROF("k_summarize", st);
            k_summarize2<<<chunks * CSPLIT, 256, 0, st>>>(pl.d_regs, pl.chunk_reg, pl.qz, pl.escbits, pl.recs);
        }
        k_scan_reduce<<<chunks, 256, 0, st>>>(pl.params, pl.d_regs, pl.recs, pl.chunk);
    }
    k_portion_agg<<<(unsigned)ceil_div(nreg, 4), 128, 0, st>>>(pl.d_regs, nreg, pl.chunk, dtype == CHR_F32, d_agg);
    CHR_CUDA_TRY(cudaGetLastError());
    CHR_CUDA_TRY(d2h(h_portions, d_agg, sizeof(TokSeg) * nreg, st));
    CHR_CUDA_TRY(stream_sync(st));
    return CHR_OK;
}

static TokSeg as_seg(const chr_portion_t &p) {
    TokSeg s;
    std::memcpy(&s, &p, sizeof(s));
    return s;
}

// phase 2: codec / layout from every rank's summaries, this rank's bytes at
// their final offsets, its raw CRC share of every payload
extern "C" int chr_dcompress_finish(const void *d_vol, int dtype, int src_dtype, int64_t nx, int64_t ny,
                                    int64_t nz_local, int64_t z_base, int64_t zs, int64_t ze, const double *spacing,
                                    int64_t bs, double vmin, double vmax, const double *h_cands, int m,
                                    chr_region_t *h_regions, int64_t nreg, const chr_portion_t *h_all, int nranks,
                                    int rank, void *d_ws, size_t ws_bytes, uint8_t *d_out, uint64_t out_cap,
                                    uint32_t *h_raw, uint64_t *h_file_nbytes, void *stream) {
    CHR_XFER_SCOPE;
    if (!d_vol || !h_regions || nreg < 1 || !h_all || nranks < 1 || rank < 0 || rank >= nranks || !d_out ||
        !h_raw || !h_file_nbytes || m < 1 || m > 64 || !h_cands)
        return CHR_E_PARAMETER;
    cudaStream_t st = (cudaStream_t)stream;
    EncPlan pl;
    if (!dist_plan(h_regions, nreg, z_base, nz_local, zs, ze, pl)) return CHR_E_PARAMETER;
    carve(pl, d_ws, ws_bytes);
    if (!d_ws || pl.ws_bytes > ws_bytes) return CHR_E_WORKSPACE;
    if (out_cap < chr_compress_capacity(h_regions, nreg, m, src_dtype)) return CHR_E_PARAMETER;
    // the device records keep phase 1's flags (has_esc, f32bad, maps)
    CHR_CUDA_TRY(d2h(pl.regs.data(), pl.d_regs, sizeof(RegDev) * nreg, st));
    CHR_CUDA_TRY(stream_sync(st));
    std::vector<int32_t> c2;
    for (int64_t r = 0; r < nreg; ++r) {
        RegDev &R = pl.regs[r];
        TokSeg tot = tokseg_identity(), pre = tokseg_identity();
        bool f32ok = true;
        for (int k = 0; k < nranks; ++k) {
            const TokSeg s = as_seg(h_all[(int64_t)k * nreg + r]);
            if (k < rank) pre = tokseg_combine(pre, s);
            tot = tokseg_combine(tot, s);
            f32ok = f32ok && s.f32ok;
        }
        const bool vf32 = src_dtype == CHR_F32 && (dtype == CHR_F32 || f32ok);
        const int64_t vlen = R.n_win * (vf32 ? 4 : 8);
        const int vcodec = vf32 ? 3 : 0;
        int codec;
        int64_t plen, tok = 0, nesc = 0;
        if (R.mode == 1) {
            codec = vcodec;
            plen = vlen;
        } else {
            tok = tokseg_stream_bytes(tot);
            nesc = tot.nesc;
            codec = nesc ? 2 : 1;
            plen = nesc ? ((R.n_win + 7) >> 3) + 8 * nesc + tok : tok;
            if (plen >= vlen) {
                codec = vcodec;
                plen = vlen;
            }
        }
        R.codec = codec;
        R.f32ok = f32ok;
        R.tok_len = tok;
        R.nesc = nesc;
        R.payload_len = plen;
        R.pre = pre;
        if (codec == 2 && R.n > 0) c2.push_back((int32_t)r);
    }
    const int write_file = 1;  // every rank lays out the whole file (header/table written by rank 0 in phase 3)
    EncParams hp;
    dist_params(hp, pl, nx, ny, nz_local, dtype, src_dtype, write_file, spacing, bs, vmin, vmax, h_cands, m, nreg);
    EncScalars hs0;
    std::memset(&hs0, 0, sizeof(hs0));
    hs0.n_codec2 = (int64_t)c2.size();
    CHR_CUDA_TRY(h2d(pl.params, &hp, sizeof(hp), st));
    CHR_CUDA_TRY(h2d(pl.d_regs, pl.regs.data(), sizeof(RegDev) * nreg, st));
    CHR_CUDA_TRY(h2d(pl.scal, &hs0, sizeof(hs0), st));
    if (!c2.empty())
        CHR_CUDA_TRY(h2d(pl.codec2, c2.data(), sizeof(int32_t) * c2.size(), st));
    const unsigned chunks = (unsigned)pl.nchunks;
    k_scan_regions<<<(unsigned)ceil_div(nreg, 4), 128, 0, st>>>(pl.params, pl.d_regs, pl.chunk, pl.codec2, pl.scal);
    k_layout<<<1, 1024, 0, st>>>(pl.params, pl.d_regs, pl.segs, pl.scal);
    if (chunks) {
        k_scan_down<<<chunks, 256, 0, st>>>(pl.params, pl.d_regs, pl.recs, pl.chunk, pl.poffs);
        CHR_PROF(dtype == CHR_F32 ? "k_emit_q<float>" : "k_emit_q<double>", st);
        if (dtype == CHR_F32)
            k_emit_q2<float><<<chunks * (unsigned)(CH / (E2_WARPS * 32)), E2_WARPS * 32, 0, st>>>((const float *)d_vol, pl.params, pl.d_regs, pl.chunk_reg,
                                                    pl.recs, pl.poffs, pl.qz, pl.escbits, d_out);
        else
            k_emit_q2<double><<<chunks * (unsigned)(CH / (E2_WARPS * 32)), E2_WARPS * 32, 0, st>>>((const double *)d_vol, pl.params, pl.d_regs, pl.chunk_reg,
                                                     pl.recs, pl.poffs, pl.qz, pl.escbits, d_out);
    }
    if (!c2.empty()) k_bitmap<<<148, 256, 0, st>>>(pl.d_regs, pl.codec2, pl.scal, pl.escbits, d_out);
    CHR_CUDA_TRY(cudaGetLastError());
    EncScalars hs;
    CHR_CUDA_TRY(d2h_multi({{pl.regs.data(), pl.d_regs, sizeof(RegDev) * nreg}, {&hs, pl.scal, sizeof(hs)}}, st));
    CHR_CUDA_TRY(stream_sync(st));
    // this rank's byte ranges inside every payload (+ the header/table on rank 0)
    std::vector<CrcSeg> segs;
    std::vector<int64_t> seg_reg;
    auto add = [&](uint64_t a, uint64_t b, int64_t r) {
        if (b <= a) return;
        CrcSeg sg;
        std::memset(&sg, 0, sizeof(sg));
        sg.begin = a;
        sg.end = b;
        segs.push_back(sg);
        seg_reg.push_back(r);
    };
    for (int64_t r = 0; r < nreg; ++r) {
        const RegDev &R = pl.regs[r];
        if (R.n == 0) continue;
        if (R.codec == 0 || R.codec == 3) {
            const int w = R.codec == 3 ? 4 : 8;
            add(R.payload_off + (uint64_t)(w * R.s_off), R.payload_off + (uint64_t)(w * (R.s_off + R.n)), r);
            continue;
        }
        const TokSeg mine = as_seg(h_all[(int64_t)rank * nreg + r]);
        const TokSeg upto = tokseg_combine(R.pre, mine);
        auto tok_off = [](const TokSeg &t) { return t.bytes + (t.nz ? run_bytes(t.lead) : 0); };
        const int64_t t0 = tok_off(R.pre);
        const int64_t t1 = R.last ? R.tok_len : tok_off(upto);
        add(R.tok_start + (uint64_t)t0, R.tok_start + (uint64_t)t1, r);
        if (R.codec == 2) {
            const uint64_t vbase = R.payload_off + (uint64_t)((R.n_win + 7) >> 3);
            add(vbase + 8ull * (uint64_t)R.pre.nesc, vbase + 8ull * (uint64_t)(R.pre.nesc + mine.nesc), r);
            add(R.payload_off + (uint64_t)(R.s_off >> 3), R.payload_off + (uint64_t)((R.s_off + R.n + 7) >> 3), r);
        }
    }
    for (int64_t r = 0; r <= nreg; ++r) h_raw[r] = 0;
    if (!segs.empty()) {
        const int64_t ns = (int64_t)segs.size();
        const int64_t total_sc = crc_plan_segments(segs.data(), ns);
        CrcSeg *d_segs = reinterpret_cast<CrcSeg *>(reinterpret_cast<char *>(d_ws) + pl.ws_bytes);
        uint32_t *d_sraw = reinterpret_cast<uint32_t *>(d_segs + ns);
        if (pl.ws_bytes + (size_t)ns * (sizeof(CrcSeg) + 4) + 64 > ws_bytes) return CHR_E_WORKSPACE;
        CHR_CUDA_TRY(h2d(d_segs, segs.data(), sizeof(CrcSeg) * ns, st));
        CHR_CUDA_TRY(fill_async(d_sraw, 0, sizeof(uint32_t) * ns, st));
        int rc = crc_launch(d_out, d_segs, ns, total_sc, d_sraw, st);
        if (rc) return rc;
        std::vector<uint32_t> sraw(ns);
        CHR_CUDA_TRY(d2h(sraw.data(), d_sraw, sizeof(uint32_t) * ns, st));
        CHR_CUDA_TRY(stream_sync(st));
        const CrcTables &H = crc_tables_hostref();
        for (int64_t i = 0; i < ns; ++i) {
            const int64_t r = seg_reg[i];
            const RegDev &R = pl.regs[r];
            const uint64_t pend = R.payload_off + (uint64_t)R.payload_len;
            h_raw[1 + r] ^= crc_shift(H.x2n, sraw[i], pend - segs[i].end);  // shift to the payload end
        }
    }
    for (int64_t r = 0; r < nreg; ++r) {
        const RegDev &R = pl.regs[r];
        chr_region_t &o = h_regions[r];
        o.codec_id = R.codec;
        o.block_offset = R.block_off;
        o.block_nbytes = kBlockHeader + (uint64_t)R.payload_len;
        o.n_escaped = (uint64_t)R.nesc;
    }
    *h_file_nbytes = hs.out_nbytes;
    return CHR_OK;
}

// phase 3 (rank 0): block headers with the combined payload CRCs, trailer
extern "C" int chr_dcompress_headers(int64_t nx, int64_t ny, int64_t nz, int src_dtype, const double *spacing,
                                     int64_t bs, double vmin, double vmax, const double *h_cands, int m,
                                     chr_region_t *h_regions, int64_t nreg, const uint32_t *h_raw_all, void *d_ws,
                                     size_t ws_bytes, uint8_t *d_out, void *stream) {
    CHR_XFER_SCOPE;
    if (!h_regions || nreg < 1 || !h_raw_all || !d_out || m < 1 || m > 64 || !h_cands) return CHR_E_PARAMETER;
    cudaStream_t st = (cudaStream_t)stream;
    EncPlan pl;
    pl.portions = true;
    if (!build_plan(h_regions, nreg, pl)) return CHR_E_PARAMETER;
    {  // only the small tables are needed here
        WsCarver c{reinterpret_cast<char *>(d_ws), 0, ws_bytes};
        pl.params = c.take<EncParams>(1);
        pl.d_regs = c.take<RegDev>(nreg);
        pl.segs = c.take<CrcSeg>(2);
        pl.seg_raw = c.take<uint32_t>(nreg + 1);
        pl.scal = c.take<EncScalars>(1);
        if (!d_ws || !c.ok) return CHR_E_WORKSPACE;
    }
    const CrcTables *tabs = crc_tables_device();
    if (!tabs) return CHR_E_CUDA;
    uint64_t body = 0;
    for (int64_t r = 0; r < nreg; ++r) {
        RegDev &R = pl.regs[r];
        R.codec = h_regions[r].codec_id;
        R.block_off = h_regions[r].block_offset;
        R.payload_off = R.block_off + kBlockHeader;
        R.payload_len = (int64_t)h_regions[r].block_nbytes - kBlockHeader;
        body = std::max<uint64_t>(body, R.block_off + h_regions[r].block_nbytes);
    }
    EncParams hp;
    dist_params(hp, pl, nx, ny, nz, CHR_F32, src_dtype, 1, spacing, bs, vmin, vmax, h_cands, m, nreg);
    EncScalars hs0;
    std::memset(&hs0, 0, sizeof(hs0));
    hs0.file_body = body;
    hs0.out_nbytes = body + 4;
    CHR_CUDA_TRY(h2d(pl.params, &hp, sizeof(hp), st));
    CHR_CUDA_TRY(h2d(pl.d_regs, pl.regs.data(), sizeof(RegDev) * nreg, st));
    CHR_CUDA_TRY(h2d(pl.scal, &hs0, sizeof(hs0), st));
    // file header + region table (global windows), then their raw CRC into
    // seg_raw[0]; seg_raw[1 + r] = payload raw CRCs (XOR of every rank's share)
    k_write_table<<<(unsigned)ceil_div(nreg, 256), 256, 0, st>>>(pl.params, pl.d_regs, d_out);
    CHR_CUDA_TRY(h2d(pl.seg_raw + 1, h_raw_all + 1, sizeof(uint32_t) * nreg, st));
    CHR_CUDA_TRY(fill_async(pl.seg_raw, 0, sizeof(uint32_t), st));
    CrcSeg hseg;
    std::memset(&hseg, 0, sizeof(hseg));
    hseg.begin = 0;
    hseg.end = hp.header_table;
    const int64_t hsc = crc_plan_segments(&hseg, 1);
    CHR_CUDA_TRY(h2d(pl.segs, &hseg, sizeof(hseg), st));
    {
        const int rc = crc_launch(d_out, pl.segs, 1, hsc, pl.seg_raw, st);
        if (rc) return rc;
    }
    k_finalize_regions<<<(unsigned)ceil_div(nreg, 4), 128, 0, st>>>(pl.params, pl.d_regs, pl.seg_raw, tabs, pl.scal,
                                                                      d_out);
    k_finalize_file<<<1, 1, 0, st>>>(tabs, pl.scal, d_out);
    CHR_CUDA_TRY(cudaGetLastError());
    CHR_CUDA_TRY(d2h(pl.regs.data(), pl.d_regs, sizeof(RegDev) * nreg, st));
    CHR_CUDA_TRY(stream_sync(st));
    for (int64_t r = 0; r < nreg; ++r) h_regions[r].payload_crc = pl.regs[r].crc;
    return CHR_OK;
}
