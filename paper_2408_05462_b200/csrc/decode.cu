// decode.cu -- step 4 of the hot path: selective reconstruction.
//
// Reference: codec.decompress (codec.py:146-229: CRC first, codec registry,
// escape bitmap + values), kernels.rle_varint_decode (kernels.py:299-345,
// with its 5 error cases), kernels.lorenzo_decode (kernels.py:131-166:
// u = 3D inclusive prefix of q, recon = u * 2e, escapes overwritten in
// raster order), chr_archive.request (chr_archive.py:226-274).
//
// Device pipeline for the selected regions:
//   k_crc_segments   payload CRCs (crc.cu), k_check compares with headers
//   k_esc_count      codec 2: escape count -> token stream start
//   k_tok_count      per 4 KiB byte chunk: samples produced by the tokens
//                    that END in the chunk (tokenised thread-locally: a
//                    token's start/previous token are found by reading
//                    back <= 11 bytes; a token follows a 0-valued token
//                    iff it is a run length)
//   k_tok_scan       per region: chunk sample offsets, count check
//   k_locate         per token: the decode segments starting inside it
//                    (byte offset + samples to skip)
//   k_esc_base       codec 2: escapes before every segment
//   k_lorenzo        one CTA per (region, row tile); marches z.  Per plane:
//                    parallel tokenise of the segment's bytes in shared
//                    memory -> q tile -> row prefix (warp scans) -> column
//                    prefix + carry from the row tile above (published
//                    per plane through global memory, a chain that is
//                    deadlock-free because tiles are taken in order from
//                    an atomic ticket) -> u = u(z-1) + S2 -> f64 recon.
//   k_verbatim       codec 0 / 3: widen to f64
// All integer work is int64 like the reference, so even CRC-valid
// hand-made streams decode bit-identically.
#include <algorithm>
#include <cstring>
#include <vector>

#include "chr_internal.cuh"

namespace chr {

constexpr int64_t DCB = 16384;    // bytes per token chunk
constexpr int DTHREADS = 256;
constexpr int DBYTES_T = DCB / DTHREADS;  // 16 bytes per thread
constexpr int DWIN = 16384;       // byte window of k_lorenzo (smem)

enum : uint32_t {
    EF_TRUNC = 1u << CHR_DEC_TRUNCATED,
    EF_LONG = 1u << CHR_DEC_VARINT_LONG,
    EF_MISSING = 1u << CHR_DEC_RUN_MISSING,
    EF_RANGE = 1u << CHR_DEC_RUN_RANGE,
    EF_TRAIL = 1u << CHR_DEC_TRAILING,
    EF_COUNT = 1u << CHR_DEC_COUNT,
    EF_CRC = 1u << CHR_DEC_CHECKSUM,
    EF_SHORTBM = 1u << CHR_DEC_SHORT_BITMAP,
    EF_SHORTESC = 1u << CHR_DEC_SHORT_ESCAPES,
    EF_CODEC = 1u << CHR_DEC_BAD_CODEC,
};

struct DecReg {
    uint64_t poff, plen;       // payload bytes in the blob
    int32_t codec, ex, ey, ez;
    double e;
    uint32_t crc;
    int32_t rows;              // row-tile height of k_lorenzo
    int64_t n;
    uint64_t out_off;
    int32_t nyt, pad;
    int64_t chunk_base, nchunks;   // token chunks (over the whole payload)
    int64_t seg_base, nseg;        // decode segments (nyt * ez)
    int64_t item_base;             // k_lorenzo tiles (nyt)
    int64_t carry_base;            // int64 elements of the carry history
    // fast (canonical-stream) path: 64x8x8 wavefront tiles, row-piece index
    int64_t abase;                 // 16-byte aligned chunk origin (blob-relative)
    int32_t ntx, tnx, tny, tnz;    // row pieces per row; wavefront tiles per axis
    int64_t tile_base, ntiles, rp_base, nrp;
    // device-computed
    uint64_t tok_start;            // absolute offset of the token stream
    int64_t nesc;
    uint32_t err;
    uint32_t slow;                 // non-canonical varints seen -> generic path
};

struct DecParams {
    int64_t nreg, nchunks, nitems, nseg;
    int32_t max_rows_ex;  // smem sizing
};

__device__ __forceinline__ int64_t find_dreg(const DecReg *__restrict__ r, int64_t n, int64_t key,
                                             int which) {
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        const int64_t b = which == 0 ? r[mid].chunk_base : (which == 1 ? r[mid].seg_base : r[mid].item_base);
        if (b <= key) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void k_check(DecReg *__restrict__ regs, int64_t nreg, const uint32_t *__restrict__ seg_raw,
                        const CrcTables *__restrict__ tabs, const uint8_t *__restrict__ blob) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nreg) return;
    DecReg &R = regs[r];
    const uint32_t crc = crc_finalize(tabs->x2n, seg_raw[r], R.plen);
    uint32_t err = 0;
    if (crc != R.crc) err |= EF_CRC;
    else if (R.codec < 0 || R.codec > 3) err |= EF_CODEC;
    R.tok_start = R.poff;
    R.nesc = 0;
    if (!err) {
        if (R.codec == 0 && R.plen < 8ull * (uint64_t)R.n) err |= EF_TRUNC;
        if (R.codec == 3 && R.plen < 4ull * (uint64_t)R.n) err |= EF_TRUNC;
        if (R.codec == 2 && R.plen < (uint64_t)((R.n + 7) >> 3)) err |= EF_SHORTBM;
    }
    R.err = err;
}

// codec 2: count escapes (popcount of the bitmap) -> token start
__global__ void __launch_bounds__(256) k_esc_count(DecReg *__restrict__ regs, int64_t nreg,
                                                   const uint8_t *__restrict__ blob) {
    const int64_t r = blockIdx.x;
    if (r >= nreg) return;
    DecReg &R = regs[r];
    if (R.codec != 2 || R.err) return;
    const int64_t nb = (R.n + 7) >> 3;
    int64_t cnt = 0;
    for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) {
        uint32_t v = blob[R.poff + b];
        if (b == nb - 1 && (R.n & 7)) v &= (1u << (R.n & 7)) - 1;  // unpackbits(count=n)
        cnt += __popc(v);
    }
    cnt = __reduce_add_sync(0xFFFFFFFFu, (unsigned)cnt);
    __shared__ int64_t ws[8];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int i = 0; i < 8; ++i) t += ws[i];
        const uint64_t start = R.poff + (uint64_t)nb + 8ull * (uint64_t)t;
        if (start > R.poff + R.plen) {
            R.err |= EF_SHORTESC;
        } else {
            R.nesc = t;
            R.tok_start = start;
        }
    }
}

// ------------------------------------------------------------------ tokens
// A token ends at a byte < 0x80.  For the token ending at byte `e` find its
// start (scanning back over continuation bytes, never before `lo`) and
// value; *bad set if longer than 5 bytes (kernels.py:316-317).
__device__ __forceinline__ int64_t tok_start_of(const uint8_t *__restrict__ b, int64_t e, int64_t lo,
                                                bool *bad) {
    int64_t s = e;
    while (s > lo && b[s - 1] >= 0x80) {
        --s;
        if (e - s >= 5) {
            *bad = true;
            return s;
        }
    }
    return s;
}

__device__ __forceinline__ uint64_t tok_value(const uint8_t *__restrict__ b, int64_t s, int64_t e) {
    uint64_t v = 0;
    for (int64_t i = s; i <= e; ++i) v |= (uint64_t)(b[i] & 0x7F) << (7 * (i - s));
    return v;
}

struct TokInfo {
    int64_t start;   // first byte (for a run length: the marker's first byte)
    int64_t count;   // samples produced
    int64_t value;   // literal quantum (if literal)
    int kind;        // 0 literal, 1 marker, 2 run length
};

// classify the token ending at e (stream bytes [lo, hi))
__device__ __forceinline__ TokInfo classify(const uint8_t *__restrict__ b, int64_t e, int64_t lo,
                                            uint32_t *err) {
    TokInfo t;
    bool bad = false;
    const int64_t s = tok_start_of(b, e, lo, &bad);
    if (bad) *err |= EF_LONG;
    const uint64_t v = tok_value(b, s, e);
    // previous token: value 0 => this one is a run length
    bool is_len = false;
    int64_t ps = s;
    if (s > lo) {
        bool pbad = false;
        ps = tok_start_of(b, s - 1, lo, &pbad);
        is_len = !pbad && tok_value(b, ps, s - 1) == 0;
    }
    if (is_len) {
        t.kind = 2;
        t.start = ps;
        t.count = (int64_t)v;
        t.value = 0;
        if (v == 0) *err |= EF_RANGE;
    } else if (v == 0) {
        t.kind = 1;
        t.start = s;
        t.count = 0;
        t.value = 0;
    } else {
        t.kind = 0;
        t.start = s;
        t.count = 1;
        const uint64_t zz = v - 1;
        t.value = (int64_t)(zz >> 1) ^ -(int64_t)(zz & 1);
    }
    return t;
}

__device__ __forceinline__ int64_t block_sum64(int64_t v) {
    __shared__ int64_t ws[32];
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, off);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    int64_t t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += ws[i];
    return t;
}

__device__ __forceinline__ int64_t block_excl64(int64_t v, int64_t *total) {
    __shared__ int64_t ws[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t inc = v;
    for (int off = 1; off < 32; off <<= 1) {
        const int64_t o = __shfl_up_sync(0xFFFFFFFFu, inc, off);
        if (lane >= off) inc += o;
    }
    __syncthreads();
    if (lane == 31) ws[warp] = inc;
    __syncthreads();
    int64_t pre = 0, tot = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
        if (i < warp) pre += ws[i];
        tot += ws[i];
    }
    if (total) *total = tot;
    return pre + inc - v;
}

// samples produced by the tokens ending in each 4 KiB chunk
__global__ void __launch_bounds__(DTHREADS) k_tok_count(DecReg *__restrict__ regs, int64_t nreg,
                                                        const uint8_t *__restrict__ blob,
                                                        int64_t *__restrict__ chunk_samples) {
    const int64_t c = blockIdx.x;
    __shared__ int64_t ri;
    if (threadIdx.x == 0) ri = find_dreg(regs, nreg, c, 0);
    __syncthreads();
    DecReg &R = regs[ri];
    int64_t cnt = 0;
    uint32_t err = 0;
    const bool active = (R.codec == 1 || R.codec == 2) && R.err == 0 && R.slow;
    if (!((R.codec == 1 || R.codec == 2) && R.slow)) return;  // fast regions: k_tok_fast
    if (active) {
        const int64_t lo = (int64_t)R.tok_start, hi = (int64_t)(R.poff + R.plen);
        const int64_t b0 = R.abase + (c - R.chunk_base) * DCB + threadIdx.x * DBYTES_T;
        for (int64_t e = max(b0, lo); e < min(b0 + DBYTES_T, hi); ++e) {
            if (blob[e] >= 0x80) {
                if (e == hi - 1) err |= EF_TRUNC;
                continue;
            }
            const TokInfo t = classify(blob, e, lo, &err);
            cnt += t.count;
            if (t.kind == 1 && e == hi - 1) err |= EF_MISSING;
        }
    }
    const int64_t tot = block_sum64(cnt);
    if (err) atomicOr(&R.err, err);
    if (threadIdx.x == 0) chunk_samples[c] = tot;
}

// per region: exclusive prefix of chunk samples, total must equal n
__global__ void k_tok_scan(DecReg *__restrict__ regs, int64_t nreg, int64_t *__restrict__ chunk_samples) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nreg) return;
    DecReg &R = regs[r];
    if (!((R.codec == 1 || R.codec == 2) && R.err == 0)) return;
    int64_t acc = 0;
    bool over = false;
    for (int64_t c = R.chunk_base; c < R.chunk_base + R.nchunks; ++c) {
        const int64_t v = chunk_samples[c];
        chunk_samples[c] = acc;
        acc += v;
        if (acc > R.n || v < 0) over = true;
    }
    if (over) R.err |= EF_RANGE;
    else if (acc < R.n) R.err |= EF_TRUNC;
    if (R.tok_start == R.poff + R.plen && R.n > 0) R.err |= EF_TRUNC;
}

// record, for every decode segment, the token (byte) it starts in
__global__ void __launch_bounds__(DTHREADS) k_locate(const DecReg *__restrict__ regs, int64_t nreg,
                                                     const uint8_t *__restrict__ blob,
                                                     const int64_t *__restrict__ chunk_start,
                                                     int64_t *__restrict__ seg_byte,
                                                     int64_t *__restrict__ seg_skip) {
    const int64_t c = blockIdx.x;
    __shared__ int64_t ri;
    if (threadIdx.x == 0) ri = find_dreg(regs, nreg, c, 0);
    __syncthreads();
    const DecReg &R = regs[ri];
    const bool active = (R.codec == 1 || R.codec == 2) && R.err == 0 && R.slow;
    if (!active) return;  // uniform across the block
    const int64_t lo = (int64_t)R.tok_start, hi = (int64_t)(R.poff + R.plen);
    const int64_t b0 = R.abase + (c - R.chunk_base) * DCB + threadIdx.x * DBYTES_T;
    uint32_t err = 0;
    int64_t cnt = 0;
    for (int64_t e = max(b0, lo); e < min(b0 + DBYTES_T, hi); ++e)
        if (blob[e] < 0x80) cnt += classify(blob, e, lo, &err).count;
    int64_t pos = chunk_start[c] + block_excl64(cnt, nullptr);
    const int64_t plane = (int64_t)R.ex * R.ey;
    const int64_t segl = (int64_t)R.rows * R.ex;
    for (int64_t e = max(b0, lo); e < min(b0 + DBYTES_T, hi); ++e) {
        if (blob[e] >= 0x80) continue;
        const TokInfo t = classify(blob, e, lo, &err);
        if (t.count <= 0) continue;
        const int64_t a = pos, b = pos + t.count;
        pos = b;
        // first segment start >= a
        int64_t z = a / plane, rem = a - z * plane;
        int64_t j = (rem + segl - 1) / segl;
        if (j >= R.nyt) {
            j = 0;
            ++z;
        }
        for (;;) {
            const int64_t s = z * plane + j * segl;
            if (s >= b || z >= R.ez) break;
            const int64_t k = R.seg_base + z * R.nyt + j;
            seg_byte[k] = t.start;
            seg_skip[k] = s - a;
            if (++j >= R.nyt) {
                j = 0;
                ++z;
            }
        }
    }
}

// codec 2: escapes before each segment
__global__ void k_esc_base(const DecReg *__restrict__ regs, int64_t nreg, const uint8_t *__restrict__ blob,
                           int64_t *__restrict__ esc_base) {
    const int64_t r = blockIdx.x;
    const DecReg &R = regs[r];
    if (R.codec != 2 || R.err || !R.slow) return;
    const int64_t plane = (int64_t)R.ex * R.ey, segl = (int64_t)R.rows * R.ex;
    // per-segment counts by the block, then a serial scan by thread 0
    for (int64_t k = threadIdx.x; k < R.nseg; k += blockDim.x) {
        const int64_t z = k / R.nyt, j = k % R.nyt;
        const int64_t s0 = z * plane + j * segl;
        const int64_t s1 = min(s0 + segl, (z + 1) * plane);
        int64_t cnt = 0;
        for (int64_t s = s0; s < s1; ++s) cnt += (blob[R.poff + (s >> 3)] >> (s & 7)) & 1;
        esc_base[R.seg_base + k] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t acc = 0;
        for (int64_t k = 0; k < R.nseg; ++k) {
            const int64_t v = esc_base[R.seg_base + k];
            esc_base[R.seg_base + k] = acc;
            acc += v;
        }
    }
}

__device__ __forceinline__ int64_t ld_acquire(const int64_t *p) {
    int64_t v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int64_t *p, int64_t v) {
    asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_acquire32(const int32_t *p) {
    int32_t v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release32(int32_t *p, int32_t v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// the chained 3D prefix decode (see header)
__global__ void __launch_bounds__(DTHREADS) k_lorenzo(const DecReg *__restrict__ regs, int64_t nreg,
                                                      const uint8_t *__restrict__ blob,
                                                      const int64_t *__restrict__ seg_byte,
                                                      const int64_t *__restrict__ seg_skip,
                                                      const int64_t *__restrict__ esc_base,
                                                      int64_t *__restrict__ carry,
                                                      int64_t *__restrict__ flags,
                                                      unsigned long long *__restrict__ ticket,
                                                      double *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ int64_t s_item;
    __shared__ int32_t s_prev_marker;
    __shared__ int64_t s_wpos;
    if (threadIdx.x == 0) s_item = (int64_t)atomicAdd(ticket, 1ull);
    __syncthreads();
    const int64_t item = s_item;
    const DecReg &R = regs[find_dreg(regs, nreg, item, 2)];
    if (!((R.codec == 1 || R.codec == 2) && R.err == 0 && R.slow)) return;
    const int yt = (int)(item - R.item_base);
    const int rows_full = R.rows;
    const int y0 = yt * rows_full;
    const int rows = min(rows_full, R.ey - y0);
    const int ex = R.ex;
    const int64_t seglen = (int64_t)rows * ex;
    int64_t *q = reinterpret_cast<int64_t *>(dsm);                    // [rows_full][ex]
    int64_t *up = q + (int64_t)rows_full * ex;                         // u at z-1
    uint8_t *win = reinterpret_cast<uint8_t *>(up + (int64_t)rows_full * ex);  // DWIN bytes
    const double twoe = 2.0 * R.e;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t hi = (int64_t)(R.poff + R.plen);
    const int64_t lo = (int64_t)R.tok_start;
    for (int64_t i = threadIdx.x; i < seglen; i += DTHREADS) up[i] = 0;
    int64_t *my_carry = carry + R.carry_base + (int64_t)yt * R.ez * ex;
    const int64_t *above = yt > 0 ? carry + R.carry_base + (int64_t)(yt - 1) * R.ez * ex : nullptr;
    int64_t *my_flag = flags + R.item_base + yt;
    const int64_t *above_flag = yt > 0 ? flags + R.item_base + yt - 1 : nullptr;
    const int64_t plane = (int64_t)ex * R.ey;

    for (int z = 0; z < R.ez; ++z) {
        const int64_t k = R.seg_base + (int64_t)z * R.nyt + yt;
        const int64_t sk = z * plane + (int64_t)y0 * ex;
        for (int64_t i = threadIdx.x; i < seglen; i += DTHREADS) q[i] = 0;
        // ---- tokenise [seg_byte[k], ...) until the segment is covered
        int64_t bstart = seg_byte[k];
        int64_t filled = -seg_skip[k];  // sample position of the next token
        if (threadIdx.x == 0) s_prev_marker = 0;
        __syncthreads();
        // bytes of this segment: up to the next segment's first token (+ one
        // run pair, <= 10 bytes, when the next segment starts inside a run)
        const int64_t seg_hi = (k + 1 < R.seg_base + R.nseg) ? min(hi, seg_byte[k + 1] + 16) : hi;
        while (filled < seglen && bstart < seg_hi) {
            const int64_t wlen = min((int64_t)DWIN, seg_hi - bstart);
            for (int64_t i = threadIdx.x; i < wlen; i += DTHREADS) win[i] = blob[bstart + i];
            __syncthreads();
            // window end: stop at the last end byte so no token straddles
            int64_t wend = wlen;
            if (bstart + wlen < hi) {
                while (wend > 0 && win[wend - 1] >= 0x80) --wend;
            }
            // per thread: a contiguous byte range; tokens end inside it
            const int64_t per = (wend + DTHREADS - 1) / DTHREADS;
            const int64_t e0 = threadIdx.x * per, e1 = min(e0 + per, wend);
            int64_t cnt = 0;
            int last_marker_here = -1;  // kind of the last token in my range
            for (int64_t e = e0; e < e1; ++e) {
                if (win[e] >= 0x80) continue;
                bool bad = false;
                const int64_t s = tok_start_of(win, e, 0, &bad);
                const uint64_t v = tok_value(win, s, e);
                bool is_len;
                if (s > 0) {
                    bool pb = false;
                    const int64_t ps = tok_start_of(win, s - 1, 0, &pb);
                    is_len = tok_value(win, ps, s - 1) == 0;
                } else {
                    is_len = s_prev_marker != 0;
                }
                cnt += is_len ? (int64_t)v : (v == 0 ? 0 : 1);
                last_marker_here = (!is_len && v == 0) ? 1 : 0;
            }
            int64_t total;
            int64_t pos = filled + block_excl64(cnt, &total);
            for (int64_t e = e0; e < e1; ++e) {
                if (win[e] >= 0x80) continue;
                bool bad = false;
                const int64_t s = tok_start_of(win, e, 0, &bad);
                const uint64_t v = tok_value(win, s, e);
                bool is_len;
                if (s > 0) {
                    bool pb = false;
                    const int64_t ps = tok_start_of(win, s - 1, 0, &pb);
                    is_len = tok_value(win, ps, s - 1) == 0;
                } else {
                    is_len = s_prev_marker != 0;
                }
                if (is_len) {
                    pos += (int64_t)v;
                } else if (v != 0) {
                    if (pos >= 0 && pos < seglen) {
                        const uint64_t zz = v - 1;
                        q[pos] = (int64_t)(zz >> 1) ^ -(int64_t)(zz & 1);
                    }
                    ++pos;
                }
            }
            // carry the marker state of the window's last token
            __syncthreads();
            if (e1 == wend && e0 < e1 && last_marker_here >= 0) s_prev_marker = last_marker_here;
            if (threadIdx.x == 0) s_wpos = filled + total;
            __syncthreads();
            filled = s_wpos;
            bstart += wend;
            if (wend == 0) break;  // malformed (checked earlier)
        }
        __syncthreads();
        // ---- row prefix along x: one warp per row
        for (int r = warp; r < rows; r += DTHREADS / 32) {
            int64_t run = 0;
            int64_t *row = q + (int64_t)r * ex;
            for (int x0 = 0; x0 < ex; x0 += 32) {
                const int x = x0 + lane;
                int64_t v = x < ex ? row[x] : 0;
                for (int off = 1; off < 32; off <<= 1) {
                    const int64_t o = __shfl_up_sync(0xFFFFFFFFu, v, off);
                    if (lane >= off) v += o;
                }
                v += run;
                if (x < ex) row[x] = v;
                run = __shfl_sync(0xFFFFFFFFu, v, 31);
            }
        }
        // ---- carry from the row tile above (same plane)
        if (yt > 0) {
            if (threadIdx.x == 0) {
                while (ld_acquire(above_flag) <= z) __nanosleep(64);
            }
        }
        __syncthreads();
        const int64_t *arow = above ? above + (int64_t)z * ex : nullptr;
        for (int x = threadIdx.x; x < ex; x += DTHREADS) {
            int64_t acc = arow ? __ldcg(arow + x) : 0;
            for (int r = 0; r < rows; ++r) {
                acc += q[(int64_t)r * ex + x];
                q[(int64_t)r * ex + x] = acc;
            }
            my_carry[(int64_t)z * ex + x] = acc;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            st_release(my_flag, z + 1);
        }
        // ---- u = u(z-1) + S2; recon
        double *o = out + R.out_off + sk;
        for (int64_t i = threadIdx.x; i < seglen; i += DTHREADS) {
            const int64_t u = up[i] + q[i];
            up[i] = u;
            o[i] = (double)u * twoe;
        }
        if (R.codec == 2 && R.nesc > 0) {
            __syncthreads();
            const uint8_t *bm = blob + R.poff;
            const double *ev = nullptr;
            (void)ev;
            for (int64_t i = threadIdx.x; i < seglen; i += DTHREADS) {
                const int64_t s = sk + i;
                if ((bm[s >> 3] >> (s & 7)) & 1) {
                    int64_t rank = esc_base[k];
                    for (int64_t t = sk; t < s; ++t) rank += (bm[t >> 3] >> (t & 7)) & 1;
                    double v;
                    uint8_t tmp[8];
                    const uint8_t *src = blob + R.poff + ((R.n + 7) >> 3) + 8 * rank;
                    for (int b = 0; b < 8; ++b) tmp[b] = src[b];
                    memcpy(&v, tmp, 8);
                    o[i] = v;
                }
            }
        }
        __syncthreads();
    }
}

__global__ void k_verbatim(const DecReg *__restrict__ regs, int64_t r0, const uint8_t *__restrict__ blob,
                           double *__restrict__ out) {
    const int64_t r = r0 + blockIdx.y;
    const DecReg &R = regs[r];
    if (!((R.codec == 0 || R.codec == 3) && R.err == 0)) return;
    const int w = R.codec == 3 ? 4 : 8;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < R.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t *src = blob + R.poff + (uint64_t)w * i;
        uint8_t b[8];
        for (int k = 0; k < w; ++k) b[k] = src[k];
        double v;
        if (w == 4) {
            float f;
            memcpy(&f, b, 4);
            v = (double)f;
        } else {
            memcpy(&v, b, 8);
        }
        out[R.out_off + i] = v;
    }
}

// ================================================================== fast path
// Canonical streams (every varint minimal, as the encoder writes them): a
// 0x00 byte is always a whole token (a zero-run marker) and a token is a run
// length iff the byte before it is 0x00.  A 0x00 end byte after a
// continuation byte (non-minimal varint) marks the region `slow` and the
// generic path above decodes it, so parity holds for any CRC-valid stream.

// ---- bit-parallel tokenizer over a 32-byte window {prev 16 | own 16}:
// bit j <-> byte j.  E = end bytes (< 0x80), Z = zero bytes (markers),
// C = ~E.  The run-length token after a marker at m ends at the first end
// byte >= m+1, found for all markers at once by a carry-propagating add:
//   Lend = (C + (Z << 1)) & ~C.
__device__ __forceinline__ uint32_t word_end4(uint32_t x) {
    return ((((~x) >> 7) & 0x01010101u) * 0x10204080u) >> 28;
}
__device__ __forceinline__ uint32_t word_zero4(uint32_t x) {
    const uint32_t nz = ((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x;  // high bit set iff byte != 0
    return ((((~nz) >> 7) & 0x01010101u) * 0x10204080u) >> 28;
}

struct UnitMasks {
    uint32_t lit;    // literal end bytes (own half, in range)
    uint32_t len;    // run-length end bytes (own half, in range)
    uint32_t E;      // end bytes (with virtual ends outside the stream)
    uint32_t err;
    bool noncanon;
};

// w[0..3]: previous 16 bytes, w[4..7]: own 16 bytes; bit 16 <-> offset u0.
// The stream is [lo, hi) (blob offsets).
__device__ __forceinline__ UnitMasks unit_masks(const uint32_t (&w)[8], int64_t u0, int64_t lo, int64_t hi) {
    uint32_t E = 0, Z = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        E |= word_end4(w[k]) << (4 * k);
        Z |= word_zero4(w[k]) << (4 * k);
    }
    const int64_t base = u0 - 16;
    const int64_t nlo = lo - base, nhi = hi - base;  // bits [nlo, nhi) are stream bytes
    const uint32_t lob = nlo <= 0 ? 0u : (nlo >= 32 ? 0xFFFFFFFFu : ((1u << nlo) - 1u));
    const uint32_t hib = nhi >= 32 ? 0u : (nhi <= 0 ? 0xFFFFFFFFu : ~((1u << nhi) - 1u));
    const uint32_t out = lob | hib;
    E |= out;
    Z &= ~out;
    const uint32_t C = ~E;
    const uint32_t mine = 0xFFFF0000u & ~out;
    UnitMasks m;
    m.err = 0;
    m.noncanon = (Z & (C << 1) & mine) != 0;            // 0x00 after a continuation byte
    if (Z & (Z << 1) & mine) m.err |= EF_RANGE;          // marker followed by marker: run of 0
    if (C & (C << 1) & (C << 2) & (C << 3) & (C << 4) & mine) m.err |= EF_LONG;
    if (nhi >= 17 && nhi <= 32) {                        // last stream byte is mine
        const uint32_t lb = 1u << (nhi - 1);
        if (C & lb) m.err |= EF_TRUNC;
        if (Z & lb) m.err |= EF_MISSING;
    }
    const uint32_t Lend = (C + (Z << 1)) & ~C;
    m.len = Lend & ~Z & mine;
    m.lit = E & ~Z & ~Lend & mine;
    m.E = E;
    return m;
}

// value of the token [s, e] (<= 5 bytes) at blob offset `p` (start byte):
// two aligned 32-bit loads, branch-free 7-bit gather
__device__ __forceinline__ uint64_t varint_at(const uint8_t *__restrict__ blob, int64_t p, int len) {
    const uint8_t *a = blob + (p & ~3ll);
    const uint32_t lo = __ldg(reinterpret_cast<const uint32_t *>(a));
    const uint32_t hi = __ldg(reinterpret_cast<const uint32_t *>(a) + 1);
    const uint64_t x = (((uint64_t)hi << 32) | lo) >> (8 * (p & 3));
    uint64_t v = (x & 0x7Full) | ((x >> 1) & (0x7Full << 7)) | ((x >> 2) & (0x7Full << 14)) |
                 ((x >> 3) & (0x7Full << 21)) | ((x >> 4) & (0x7Full << 28));
    return v & ((1ull << (7 * len)) - 1);
}

// value of the token ending at bit `e` of the 32-byte window at u0 - 16
__device__ __forceinline__ uint64_t unit_token_value(const uint8_t *__restrict__ blob, uint32_t E, int e, int64_t u0) {
    const uint32_t below = E & ((1u << e) - 1u);
    const int s = below ? 32 - __clz(below) : 0;
    return varint_at(blob, u0 - 16 + s, e - s + 1);
}

// value of the token ending at bit `e` of a byte window read through `rd`
template <typename RD>
__device__ __forceinline__ uint64_t token_value(uint32_t E, int e, RD rd) {
    const uint32_t below = E & ((1u << e) - 1u);
    const int s = below ? 32 - __clz(below) : 0;  // first byte after the previous end byte
    uint64_t v = 0;
    for (int k = s; k <= e; ++k) v |= (uint64_t)(rd(k) & 0x7Fu) << (7 * (k - s));
    return v;
}

__device__ __forceinline__ void load_units(const uint8_t *__restrict__ blob, int64_t u0, uint32_t (&w)[8]) {
    const uint4 cur = __ldg(reinterpret_cast<const uint4 *>(blob + u0));
    uint4 prv = make_uint4(0, 0, 0, 0);
    if (u0 >= 16) prv = __ldg(reinterpret_cast<const uint4 *>(blob + u0 - 16));
    w[0] = prv.x; w[1] = prv.y; w[2] = prv.z; w[3] = prv.w;
    w[4] = cur.x; w[5] = cur.y; w[6] = cur.z; w[7] = cur.w;
}

__device__ __forceinline__ void next_unit(const uint8_t *__restrict__ blob, int64_t u0, uint32_t (&w)[8]) {
    w[0] = w[4]; w[1] = w[5]; w[2] = w[6]; w[3] = w[7];
    const uint4 cur = __ldg(reinterpret_cast<const uint4 *>(blob + u0));
    w[4] = cur.x; w[5] = cur.y; w[6] = cur.z; w[7] = cur.w;
}

// samples produced by the tokens ending in one unit
__device__ __forceinline__ int64_t unit_count(const UnitMasks &m, const uint8_t *__restrict__ blob, int64_t u0) {
    int64_t c = __popc(m.lit);
    uint32_t L = m.len;
    while (L) {
        const int e = __ffs(L) - 1;
        L &= L - 1;
        c += (int64_t)unit_token_value(blob, m.E, e, u0);
    }
    return c;
}

// region of every chunk / tile (filled once per call; replaces per-CTA
// binary searches whose dependent loads dominated small CTAs)
__global__ void k_fill_maps(const DecReg *__restrict__ regs, int64_t nreg, int32_t *__restrict__ chunk_reg,
                            int32_t *__restrict__ tile_reg) {
    const int64_t r = blockIdx.x;
    if (r >= nreg) return;
    const DecReg &R = regs[r];
    for (int64_t i = threadIdx.x; i < R.nchunks; i += blockDim.x) chunk_reg[R.chunk_base + i] = (int32_t)r;
    for (int64_t i = threadIdx.x; i < R.ntiles; i += blockDim.x) tile_reg[R.tile_base + i] = (int32_t)r;
}

constexpr int UPT = (int)(DCB / (16 * DTHREADS));  // 16-byte units per thread

// tile order for k_lorenzo3d: all regions' tiles grouped by wavefront
// diagonal d = tx + ty + tz (every dependency of a tile lies on d - 1, so
// taking tiles in this order from a ticket cannot deadlock and keeps every
// region's wavefront advancing at once).  One thread per (diagonal, region)
// pair writes its tiles at pair_base.
__global__ void k_tile_order(const DecReg *__restrict__ regs, const int64_t *__restrict__ pair_base,
                             int64_t npairs, int64_t nreg, int32_t *__restrict__ order) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npairs) return;
    const int64_t d = i / nreg, r = i % nreg;
    const DecReg &R = regs[r];
    if (R.ntiles == 0) return;
    int64_t k = pair_base[i];
    const int nx = R.tnx, ny = R.tny, nz = R.tnz;
    for (int tz = max(0, (int)d - (nx - 1) - (ny - 1)); tz <= min(nz - 1, (int)d); ++tz) {
        const int rem = (int)d - tz;
        for (int ty = max(0, rem - (nx - 1)); ty <= min(ny - 1, rem); ++ty) {
            const int tx = rem - ty;
            order[k++] = (int32_t)(R.tile_base + ((int64_t)tz * ny + ty) * nx + tx);
        }
    }
}

// samples per chunk (fast path); flags non-canonical regions
__global__ void __launch_bounds__(DTHREADS) k_tok_fast(DecReg *__restrict__ regs, const int32_t *__restrict__ chunk_reg,
                                                       const uint8_t *__restrict__ blob,
                                                       int64_t *__restrict__ chunk_samples) {
    const int64_t c = blockIdx.x;
    DecReg &R = regs[chunk_reg[c]];
    if (!((R.codec == 1 || R.codec == 2) && R.err == 0)) {
        if (threadIdx.x == 0) chunk_samples[c] = 0;
        return;
    }
    const int64_t lo = (int64_t)R.tok_start, hi = (int64_t)(R.poff + R.plen);
    const int64_t ub = R.abase + (c - R.chunk_base) * DCB + (int64_t)threadIdx.x * UPT * 16;
    int64_t cnt = 0;
    uint32_t err = 0;
    bool nc = false;
    if (ub + UPT * 16 > lo && ub < hi) {
        uint32_t w[8];
        load_units(blob, ub, w);
#pragma unroll 1
        for (int u = 0; u < UPT; ++u) {
            const int64_t u0 = ub + 16 * u;
            if (u) next_unit(blob, u0, w);
            if (u0 + 16 > lo && u0 < hi) {
                const UnitMasks m = unit_masks(w, u0, lo, hi);
                err |= m.err;
                nc |= m.noncanon;
                cnt += unit_count(m, blob, u0);
            }
        }
    }
    const int64_t tot = block_sum64(cnt);
    if (err) atomicOr(&R.err, err);
    if (nc) atomicOr(&R.slow, 1u);
    if (threadIdx.x == 0) chunk_samples[c] = tot;
}

// row-piece index: for every 64-sample piece of every row, the byte of the
// token (marker for runs) holding its first sample and the samples to skip
__global__ void __launch_bounds__(DTHREADS) k_rp_locate(const DecReg *__restrict__ regs,
                                                        const int32_t *__restrict__ chunk_reg,
                                                        const uint8_t *__restrict__ blob,
                                                        const int64_t *__restrict__ chunk_start,
                                                        int64_t *__restrict__ rp_byte,
                                                        int64_t *__restrict__ rp_skip) {
    const int64_t c = blockIdx.x;
    const DecReg &R = regs[chunk_reg[c]];
    if (!((R.codec == 1 || R.codec == 2) && R.err == 0 && !R.slow)) return;
    const int64_t lo = (int64_t)R.tok_start, hi = (int64_t)(R.poff + R.plen);
    const int64_t ub = R.abase + (c - R.chunk_base) * DCB + (int64_t)threadIdx.x * UPT * 16;
    const bool mine = ub + UPT * 16 > lo && ub < hi;
    int64_t cnt = 0;
    uint32_t w[8];
    if (mine) {
        load_units(blob, ub, w);
#pragma unroll 1
        for (int u = 0; u < UPT; ++u) {
            const int64_t u0 = ub + 16 * u;
            if (u) next_unit(blob, u0, w);
            if (u0 + 16 > lo && u0 < hi) cnt += unit_count(unit_masks(w, u0, lo, hi), blob, u0);
        }
    }
    int64_t a = chunk_start[c] + block_excl64(cnt, nullptr);
    if (!mine || cnt == 0) return;
    const int64_t ex = R.ex;
    // first row-piece start >= a; nothing to do if it lies beyond the thread's samples
    int64_t row = a / ex;
    int64_t x = a - row * ex;
    {
        int64_t xs = (x + 63) & ~63ll, r2 = row;
        if (xs >= ex) {
            xs = 0;
            ++r2;
        }
        if (r2 * ex + xs >= a + cnt) return;
    }
    load_units(blob, ub, w);
#pragma unroll 1
    for (int u = 0; u < UPT; ++u) {
        const int64_t u0 = ub + 16 * u;
        if (u) next_unit(blob, u0, w);
        if (!(u0 + 16 > lo && u0 < hi)) continue;
        const UnitMasks m = unit_masks(w, u0, lo, hi);
        uint32_t T = m.lit | m.len;
        while (T) {
            const int e = __ffs(T) - 1;
            T &= T - 1;
            const bool isl = (m.len >> e) & 1u;
            int64_t tc = 1, sbyte;
            const uint32_t below = m.E & ((1u << e) - 1u);
            const int s = below ? 32 - __clz(below) : 0;
            if (isl) {
                tc = (int64_t)unit_token_value(blob, m.E, e, u0);
                sbyte = u0 - 16 + s - 1;  // the marker
            } else {
                sbyte = u0 - 16 + s;
            }
            if ((x & 63) == 0 || tc > 1) {
                int64_t xs = (x + 63) & ~63ll, r2 = row;
                if (xs >= ex) {
                    xs = 0;
                    ++r2;
                }
                int64_t pp = r2 * ex + xs;
                while (pp < a + tc) {
                    const int64_t k = R.rp_base + r2 * R.ntx + (xs >> 6);
                    rp_byte[k] = sbyte;
                    rp_skip[k] = pp - a;
                    xs += 64;
                    if (xs >= ex) {
                        xs = 0;
                        ++r2;
                    }
                    pp = r2 * ex + xs;
                }
            }
            a += tc;
            x += tc;
            if (x >= ex) {
                if (x < 2 * ex) {
                    x -= ex;
                    ++row;
                } else {
                    row += x / ex;
                    x %= ex;
                }
            }
        }
    }
}

// codec 2: escapes before every row piece (one CTA per region)
__global__ void __launch_bounds__(256) k_esc_rp(const DecReg *__restrict__ regs, const uint8_t *__restrict__ blob,
                                                int64_t *__restrict__ esc_rp) {
    const DecReg &R = regs[blockIdx.x];
    if (R.codec != 2 || R.err || R.slow) return;
    const uint8_t *bm = blob + R.poff;
    int64_t carry = 0;
    for (int64_t p0 = 0; p0 < R.nrp; p0 += 256) {
        const int64_t p = p0 + threadIdx.x;
        int64_t cnt = 0;
        if (p < R.nrp) {
            const int64_t row = p / R.ntx, xt = p % R.ntx;
            const int64_t s0 = row * R.ex + xt * 64, s1 = s0 + min((int64_t)64, (int64_t)R.ex - xt * 64);
            for (int64_t s = s0; s < s1; ++s) cnt += (bm[s >> 3] >> (s & 7)) & 1;
        }
        int64_t total;
        const int64_t ex = block_excl64(cnt, &total);
        if (p < R.nrp) esc_rp[R.rp_base + p] = carry + ex;
        carry += total;
        __syncthreads();
    }
}

__device__ __forceinline__ int64_t ld_cg64(const int64_t *p) { return __ldcg(p); }

// the 3D wavefront: one CTA per tile of <= 65 x 9 x 9 samples (64/8/8 plus
// the region's trailing ghost sample in the last tile of each axis), taken in
// wavefront-diagonal order from an atomic ticket; waits for the x-, y- and
// z-neighbour's published faces.
constexpr int TXM = 65, TYM = 9, TZM = 9;          // tile capacity
constexpr int FXN = (TZM + 1) * (TYM + 1);         // S(x1-1, y0-1..y1-1, z0-1..z1-1)
constexpr int FYN = (TZM + 1) * TXM;               // S(x0..x1-1, y1-1, z0-1..z1-1)
constexpr int FZN = TYM * TXM;                     // S(x0..x1-1, y0..y1-1, z1-1)
constexpr int FACE_N = FXN + FYN + FZN;
constexpr int SEGW = 11;                           // row segments per warp (81 / 8)
constexpr int UNITS_W = 256;                       // units per warp (>= 11 * 22)

__device__ __forceinline__ int tile_lo(int t, int step) { return t * step; }
__device__ __forceinline__ int tile_hi(int t, int nt, int step, int ext) { return t == nt - 1 ? ext : (t + 1) * step; }

__global__ void __launch_bounds__(256) k_lorenzo3d(const DecReg *__restrict__ regs,
                                                   const int32_t *__restrict__ tile_reg,
                                                   const uint8_t *__restrict__ blob,
                                                   const int64_t *__restrict__ rp_byte,
                                                   const int64_t *__restrict__ rp_skip,
                                                   const int64_t *__restrict__ esc_rp,
                                                   int64_t *__restrict__ faces, int32_t *__restrict__ tflag,
                                                   unsigned long long *__restrict__ ticket,
                                                   const int32_t *__restrict__ order,
                                                   double *__restrict__ out) {
    extern __shared__ __align__(16) int64_t dyn_s[];  // S[TZM][TYM][TXM]
    int64_t(*S)[TYM][TXM] = reinterpret_cast<int64_t(*)[TYM][TXM]>(dyn_s);
    __shared__ int64_t Fx[TZM + 1][TYM + 1];
    __shared__ int64_t Fy[TZM + 1][TXM];
    __shared__ int64_t Fz[TYM][TXM];
    __shared__ int64_t Ayz[TZM][TYM];
    __shared__ int64_t ucnt[8][UNITS_W];
    __shared__ int64_t sg_lo[8][SEGW], sg_hi[8][SEGW], sg_ub[8][SEGW], sg_skip[8][SEGW];
    __shared__ int32_t sg_base[8][SEGW + 1];
    __shared__ int64_t s_item;
    if (threadIdx.x == 0) s_item = order[atomicAdd(ticket, 1ull)];
    __syncthreads();
    const int64_t tile = s_item;
    const DecReg &R = regs[tile_reg[tile]];
    if (!((R.codec == 1 || R.codec == 2) && R.err == 0 && !R.slow)) return;
    const int64_t local = tile - R.tile_base;
    const int tx = (int)(local % R.tnx);
    const int64_t l2 = local / R.tnx;
    const int ty = (int)(l2 % R.tny), tz = (int)(l2 / R.tny);
    const int x0 = tile_lo(tx, 64), x1 = tile_hi(tx, R.tnx, 64, R.ex);
    const int y0 = tile_lo(ty, 8), y1 = tile_hi(ty, R.tny, 8, R.ey);
    const int z0 = tile_lo(tz, 8), z1 = tile_hi(tz, R.tnz, 8, R.ez);
    const int nxv = x1 - x0, nyv = y1 - y0, nzv = z1 - z0;
    const int nrs = nyv * nzv;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t hi = (int64_t)(R.poff + R.plen);
    const int64_t rp_end = R.rp_base + R.nrp;
    const int64_t nrows = (int64_t)R.ey * R.ez;

    int64_t *Sf = &S[0][0][0];
    for (int i = threadIdx.x; i < TZM * TYM * TXM; i += 256) Sf[i] = 0;
    // ---- 1. tokens -> q.  Warp w owns row segments rs = w, w+8, ... (rs = zz*nyv + yy);
    //         its units (16 aligned bytes) are spread over all 32 lanes.
    const int nseg = nrs > warp ? (nrs - warp + 7) >> 3 : 0;
    {
        int nun = 0;
        if (lane < nseg) {
            const int rs = warp + 8 * lane, zz = rs / nyv, yy = rs - zz * nyv;
            const int64_t row = (int64_t)(z0 + zz) * R.ey + (y0 + yy);
            const int64_t p = R.rp_base + row * R.ntx + (x0 >> 6);
            const int64_t b0 = rp_byte[p];
            const int64_t pe = x1 < R.ex ? R.rp_base + row * R.ntx + (x1 >> 6)
                                         : (row + 1 < nrows ? R.rp_base + (row + 1) * R.ntx : rp_end);
            const int64_t b1 = pe < rp_end ? min(hi, rp_byte[pe] + 11) : hi;
            const int64_t ub = R.abase + ((b0 - R.abase) & ~15ll);
            sg_lo[warp][lane] = b0;
            sg_hi[warp][lane] = b1;
            sg_ub[warp][lane] = ub;
            sg_skip[warp][lane] = rp_skip[p];
            nun = (int)((b1 - ub + 15) >> 4);
        }
        int inc = nun;
        for (int off = 1; off < 32; off <<= 1) {
            const int o = __shfl_up_sync(0xFFFFFFFFu, inc, off);
            if (lane >= off) inc += o;
        }
        if (lane < nseg) sg_base[warp][lane] = inc - nun;
        if (lane == 31) sg_base[warp][nseg] = inc;
    }
    __syncwarp();
    const int U = nseg ? sg_base[warp][nseg] : 0;
    for (int g = lane; g < U; g += 32) {
        int i = 0;
        while (i + 1 < nseg && sg_base[warp][i + 1] <= g) ++i;
        const int64_t u0 = sg_ub[warp][i] + 16 * (int64_t)(g - sg_base[warp][i]);
        uint32_t w[8];
        load_units(blob, u0, w);
        const UnitMasks m = unit_masks(w, u0, sg_lo[warp][i], sg_hi[warp][i]);
        ucnt[warp][g] = unit_count(m, blob, u0);
    }
    __syncwarp();
    if (lane < nseg) {  // exclusive scan of the segment's unit counts, minus the skip
        int64_t acc = -sg_skip[warp][lane];
        for (int g = sg_base[warp][lane]; g < sg_base[warp][lane + 1]; ++g) {
            const int64_t t = ucnt[warp][g];
            ucnt[warp][g] = acc;
            acc += t;
        }
    }
    __syncwarp();
    __syncthreads();  // S zeroed
    for (int g = lane; g < U; g += 32) {
        int i = 0;
        while (i + 1 < nseg && sg_base[warp][i + 1] <= g) ++i;
        int64_t at = ucnt[warp][g];
        if (at >= nxv) continue;
        const int rs = warp + 8 * i, zz = rs / nyv, yy = rs - zz * nyv;
        const int64_t u0 = sg_ub[warp][i] + 16 * (int64_t)(g - sg_base[warp][i]);
        uint32_t w[8];
        load_units(blob, u0, w);
        const UnitMasks m = unit_masks(w, u0, sg_lo[warp][i], sg_hi[warp][i]);
        uint32_t T = m.lit | m.len;
        int64_t *srow = &S[zz][yy][0];
        while (T && at < nxv) {
            const int e = __ffs(T) - 1;
            T &= T - 1;
            uint64_t v;
            if ((m.E >> (e - 1)) & 1u) {  // one-byte token (the common case)
                v = __ldg(blob + u0 - 16 + e) & 0x7Fu;
            } else {
                v = unit_token_value(blob, m.E, e, u0);
            }
            if ((m.len >> e) & 1u) {
                at += (int64_t)v;
            } else {
                if (at >= 0) {
                    const uint64_t zz2 = v - 1;
                    srow[at] = (int64_t)(zz2 >> 1) ^ -(int64_t)(zz2 & 1);
                }
                ++at;
            }
        }
    }
    __syncthreads();
    // ---- 2. local 3D prefix: x (warp per row: x = lane, lane+32, 64), y, z
    int zz2 = warp / nyv, yy2 = warp - zz2 * nyv;
    for (int r = warp; r < nrs; r += 8) {
        const int zz = zz2, yy = yy2;
        yy2 += 8;
        while (yy2 >= nyv) {
            yy2 -= nyv;
            ++zz2;
        }
        int64_t *row = &S[zz][yy][0];
        int64_t a = row[lane], b = row[lane + 32];
        for (int off = 1; off < 32; off <<= 1) {
            const int64_t oa = __shfl_up_sync(0xFFFFFFFFu, a, off);
            const int64_t ob = __shfl_up_sync(0xFFFFFFFFu, b, off);
            if (lane >= off) {
                a += oa;
                b += ob;
            }
        }
        b += __shfl_sync(0xFFFFFFFFu, a, 31);
        const int64_t tot = __shfl_sync(0xFFFFFFFFu, b, 31);
        row[lane] = a;
        row[lane + 32] = b;
        if (lane == 0) row[64] += tot;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nzv * TXM; t += 256) {
        const int zz = t / TXM, x = t - zz * TXM;
        int64_t acc = 0;
        for (int yy = 0; yy < nyv; ++yy) {
            acc += S[zz][yy][x];
            S[zz][yy][x] = acc;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nyv * TXM; t += 256) {
        const int yy = t / TXM, x = t - yy * TXM;
        int64_t acc = 0;
        for (int zz = 0; zz < nzv; ++zz) {
            acc += S[zz][yy][x];
            S[zz][yy][x] = acc;
        }
    }
    // ---- 3. neighbour faces
    const int64_t nb_x = tx > 0 ? tile - 1 : -1;
    const int64_t nb_y = ty > 0 ? tile - R.tnx : -1;
    const int64_t nb_z = tz > 0 ? tile - (int64_t)R.tnx * R.tny : -1;
    if (threadIdx.x == 0) {
        if (nb_x >= 0) while (ld_acquire32(tflag + nb_x) == 0) __nanosleep(20);
        if (nb_y >= 0) while (ld_acquire32(tflag + nb_y) == 0) __nanosleep(20);
        if (nb_z >= 0) while (ld_acquire32(tflag + nb_z) == 0) __nanosleep(20);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < FXN; i += 256) (&Fx[0][0])[i] = nb_x >= 0 ? ld_cg64(faces + nb_x * FACE_N + i) : 0;
    for (int i = threadIdx.x; i < FYN; i += 256)
        (&Fy[0][0])[i] = nb_y >= 0 ? ld_cg64(faces + nb_y * FACE_N + FXN + i) : 0;
    for (int i = threadIdx.x; i < FZN; i += 256)
        (&Fz[0][0])[i] = nb_z >= 0 ? ld_cg64(faces + nb_z * FACE_N + FXN + FYN + i) : 0;
    __syncthreads();
    for (int i = threadIdx.x; i < TZM * TYM; i += 256) {
        const int zz = i / TYM, yy = i - zz * TYM;
        Ayz[zz][yy] = Fx[zz + 1][yy + 1] - Fx[zz + 1][0] - Fx[0][yy + 1] + Fx[0][0];
    }
    __syncthreads();
    // ---- 4. S = T + A(y,z) + [Fy(x,z) - Fy(x,z0-1)] + Fz(x,y)
    {
        int zz = warp / nyv, yy = warp - zz * nyv;
        for (int r = warp; r < nrs; r += 8) {
            const int64_t a = Ayz[zz][yy];
            for (int x = lane; x < nxv; x += 32) S[zz][yy][x] += a + (Fy[zz + 1][x] - Fy[0][x]) + Fz[yy][x];
            yy += 8;
            while (yy >= nyv) {
                yy -= nyv;
                ++zz;
            }
        }
    }
    __syncthreads();
    // ---- 5. publish this tile's high faces (consumers index with their own extents)
    int64_t *my = faces + tile * FACE_N;
    const int xl = nxv - 1;
    for (int i = threadIdx.x; i < FXN; i += 256) {
        const int zp = i / (TYM + 1), yp = i - zp * (TYM + 1);
        if (zp > nzv || yp > nyv) continue;
        int64_t v;
        if (zp == 0) v = yp == 0 ? Fy[0][xl] : Fz[yp - 1][xl];
        else if (yp == 0) v = Fy[zp][xl];
        else v = S[zp - 1][yp - 1][xl];
        my[i] = v;
    }
    for (int i = threadIdx.x; i < FYN; i += 256) {
        const int zp = i / TXM, x = i - zp * TXM;
        if (zp > nzv || x >= nxv) continue;
        my[FXN + i] = zp == 0 ? Fz[nyv - 1][x] : S[zp - 1][nyv - 1][x];
    }
    for (int i = threadIdx.x; i < FZN; i += 256) {
        const int yy = i / TXM, x = i - yy * TXM;
        if (yy >= nyv || x >= nxv) continue;
        my[FXN + FYN + i] = S[nzv - 1][yy][x];
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release32(tflag + tile, 1);
    // ---- 6. reconstruction (escapes overwritten in raster order)
    const double twoe = 2.0 * R.e;
    const bool esc = R.codec == 2 && R.nesc > 0;
    const uint8_t *bm = blob + R.poff;
    const uint8_t *ev = blob + R.poff + ((R.n + 7) >> 3);
    int zz3 = warp / nyv, yy3 = warp - zz3 * nyv;
    for (int r = warp; r < nrs; r += 8) {
        const int zz = zz3, yy = yy3;
        yy3 += 8;
        while (yy3 >= nyv) {
            yy3 -= nyv;
            ++zz3;
        }
        const int64_t rowi = (int64_t)(z0 + zz) * R.ey + (y0 + yy);
        const int64_t srow = rowi * R.ex + x0;
        double *o = out + R.out_off + srow;
        uint64_t em = 0;
        uint32_t em64 = 0;
        int64_t ebase = 0;
        if (esc) {
            const int sh = (int)(srow & 7);
            const int64_t byte0 = srow >> 3, nbm = (R.n + 7) >> 3;
            uint32_t bt = 0;
            if (lane < 10 && byte0 + lane < nbm) bt = bm[byte0 + lane];
            uint64_t lo64 = 0;
            for (int k = 0; k < 8; ++k) lo64 |= (uint64_t)__shfl_sync(0xFFFFFFFFu, bt, k) << (8 * k);
            const uint64_t b8 = __shfl_sync(0xFFFFFFFFu, bt, 8), b9 = __shfl_sync(0xFFFFFFFFu, bt, 9);
            const uint64_t hi16 = b8 | (b9 << 8);
            em = sh ? (lo64 >> sh) | (hi16 << (64 - sh)) : lo64;
            em64 = (uint32_t)((hi16 >> sh) & 1u);
            if (nxv < 64) em &= (1ull << nxv) - 1;
            if (nxv < 65) em64 = 0;
            ebase = esc_rp[R.rp_base + rowi * R.ntx + (x0 >> 6)];
        }
        for (int x = lane; x < nxv; x += 32) {
            double v = (double)S[zz][yy][x] * twoe;
            if (esc) {
                const bool isesc = x < 64 ? ((em >> x) & 1) : em64;
                if (isesc) {
                    const int64_t rank = ebase + (x < 64 ? __popcll((long long)(em & ((1ull << x) - 1)))
                                                         : __popcll((long long)em));
                    uint8_t tmp[8];
                    for (int k = 0; k < 8; ++k) tmp[k] = ev[8 * rank + k];
                    memcpy(&v, tmp, 8);
                }
            }
            o[x] = v;
        }
    }
}

// ------------------------------------------------------------------ host
struct DecPlan {
    std::vector<DecReg> regs;
    int64_t nchunks = 0, nseg = 0, nitems = 0, ncarry = 0, ntiles = 0, nrp = 0;
    int max_rows_ex = 0;
    size_t ws = 0;
    DecReg *d_regs;
    CrcSeg *segs;
    uint32_t *seg_raw;
    int64_t *chunk_samples, *seg_byte, *seg_skip, *esc_base, *carry, *flags;
    int64_t *rp_byte, *rp_skip, *esc_rp, *faces;
    int32_t *tflag, *chunk_reg, *tile_reg, *order;
    int64_t *pair_base;
    std::vector<int64_t> h_pair_base;
    int64_t ndiag = 0;
    unsigned long long *ticket, *ticket3;
};

static int dec_rows_for(int ex) {
    // q tile + u(z-1) tile (int64) must fit next to the byte window
    const int64_t budget = 180 * 1024 - DWIN;
    int rows = (int)std::min<int64_t>(8, budget / (16ll * ex));
    return rows < 1 ? 0 : rows;
}

static bool dec_build(const chr_dec_region_t *h, int64_t n, uintptr_t blob, DecPlan &pl) {
    pl.regs.resize(n);
    int64_t chunk = 0, seg = 0, item = 0, carry = 0, tile = 0, rp = 0;
    for (int64_t i = 0; i < n; ++i) {
        DecReg &R = pl.regs[i];
        std::memset(&R, 0, sizeof(R));
        R.poff = h[i].payload_offset;
        R.plen = h[i].payload_nbytes;
        R.codec = h[i].codec_id;
        R.ex = h[i].dims[0];
        R.ey = h[i].dims[1];
        R.ez = h[i].dims[2];
        if (R.ex < 1 || R.ey < 1 || R.ez < 1) return false;
        R.e = h[i].error_bound;
        R.crc = h[i].crc;
        R.n = (int64_t)R.ex * R.ey * R.ez;
        R.out_off = h[i].out_offset;
        R.rows = dec_rows_for(R.ex);
        if (R.rows < 1) return false;
        R.nyt = (int32_t)ceil_div(R.ey, R.rows);
        // chunks: 4 KiB over [16-aligned(poff), poff + plen)
        R.abase = (int64_t)(((blob + R.poff) & ~(uintptr_t)15) - blob);
        R.chunk_base = chunk;
        R.nchunks = std::max<int64_t>(1, ceil_div((int64_t)(R.poff + R.plen) - R.abase, DCB));
        chunk += R.nchunks;
        R.seg_base = seg;
        R.item_base = item;
        R.carry_base = carry;
        R.ntx = (int32_t)ceil_div(R.ex, 64);
        // tiles of 64 / 8 / 8 samples; the last one of each axis absorbs the
        // trailing sample of 32k+1 extents (<= 65 / 9 / 9)
        R.tnx = (int32_t)std::max<int64_t>(1, ceil_div(R.ex - 1, 64));
        R.tny = (int32_t)std::max<int64_t>(1, ceil_div(R.ey - 1, 8));
        R.tnz = (int32_t)std::max<int64_t>(1, ceil_div(R.ez - 1, 8));
        R.tile_base = tile;
        R.rp_base = rp;
        if (R.codec == 1 || R.codec == 2) {
            R.nseg = (int64_t)R.nyt * R.ez;
            seg += R.nseg;
            item += R.nyt;
            carry += (int64_t)R.nyt * R.ez * R.ex;
            pl.max_rows_ex = std::max(pl.max_rows_ex, R.rows * R.ex);
            R.ntiles = (int64_t)R.tnx * R.tny * R.tnz;
            tile += R.ntiles;
            R.nrp = (int64_t)R.ntx * R.ey * R.ez;
            rp += R.nrp;
        }
    }
    pl.nchunks = chunk;
    pl.nseg = seg;
    pl.nitems = item;
    pl.ncarry = carry;
    pl.ntiles = tile;
    pl.nrp = rp;
    // tiles per (diagonal, region) -> exclusive bases in diagonal-major order
    int64_t D = 0;
    for (const DecReg &R : pl.regs)
        if (R.ntiles) D = std::max<int64_t>(D, (int64_t)R.tnx + R.tny + R.tnz - 2);
    pl.ndiag = pl.ntiles ? D + 1 : 0;
    std::vector<int64_t> cnt((size_t)(pl.ndiag * n) + 1, 0);  // [r][d]
    std::vector<int64_t> diff((size_t)pl.ndiag + 2);
    for (int64_t i = 0; i < n; ++i) {
        const DecReg &R = pl.regs[i];
        if (!R.ntiles) continue;
        std::fill(diff.begin(), diff.end(), 0);
        for (int tz = 0; tz < R.tnz; ++tz)
            for (int ty = 0; ty < R.tny; ++ty) {
                diff[ty + tz] += 1;
                diff[ty + tz + R.tnx] -= 1;
            }
        int64_t run = 0;
        for (int64_t d = 0; d < pl.ndiag; ++d) {
            run += diff[d];
            cnt[i * pl.ndiag + d] = run;
        }
    }
    pl.h_pair_base.assign((size_t)(pl.ndiag * n) + 1, 0);
    int64_t acc = 0;
    for (int64_t d = 0; d < pl.ndiag; ++d)
        for (int64_t i = 0; i < n; ++i) {
            pl.h_pair_base[d * n + i] = acc;
            acc += cnt[i * pl.ndiag + d];
        }
    return true;
}

static void dec_carve(DecPlan &pl, void *base, size_t cap) {
    WsCarver c{reinterpret_cast<char *>(base), 0, cap};
    const int64_t n = (int64_t)pl.regs.size();
    pl.d_regs = c.take<DecReg>(n);
    pl.segs = c.take<CrcSeg>(n);
    pl.seg_raw = c.take<uint32_t>(n);
    pl.chunk_samples = c.take<int64_t>(pl.nchunks);
    pl.seg_byte = c.take<int64_t>(pl.nseg + 1);
    pl.seg_skip = c.take<int64_t>(pl.nseg + 1);
    pl.esc_base = c.take<int64_t>(pl.nseg + 1);
    pl.carry = c.take<int64_t>(pl.ncarry + 1);
    pl.flags = c.take<int64_t>(pl.nitems + 1);
    pl.rp_byte = c.take<int64_t>(pl.nrp + 1);
    pl.rp_skip = c.take<int64_t>(pl.nrp + 1);
    pl.esc_rp = c.take<int64_t>(pl.nrp + 1);
    pl.faces = c.take<int64_t>((size_t)pl.ntiles * FACE_N + 1);
    pl.tflag = c.take<int32_t>(pl.ntiles + 1);
    pl.chunk_reg = c.take<int32_t>(pl.nchunks + 1);
    pl.tile_reg = c.take<int32_t>(pl.ntiles + 1);
    pl.order = c.take<int32_t>(pl.ntiles + 1);
    pl.pair_base = c.take<int64_t>(pl.h_pair_base.size() + 1);
    pl.ticket = c.take<unsigned long long>(1);
    pl.ticket3 = c.take<unsigned long long>(1);
    pl.ws = c.off + 256;
}

}  // namespace chr

using namespace chr;

extern "C" size_t chr_decode_workspace_size(const chr_dec_region_t *h, int64_t n) {
    DecPlan pl;
    if (!h || n < 1 || !dec_build(h, n, 0, pl)) return 256;
    dec_carve(pl, nullptr, ~size_t(0));
    return pl.ws;
}

extern "C" int chr_decode_regions(const uint8_t *d_blob, const chr_dec_region_t *h, int64_t n,
                                  double *d_out, void *d_ws, size_t ws_bytes, int32_t *h_status,
                                  void *stream) {
    if (n == 0) return CHR_OK;
    if (!d_blob || !h || n < 0 || !d_out) return CHR_E_PARAMETER;
    cudaStream_t st = (cudaStream_t)stream;
    DecPlan pl;
    if (!dec_build(h, n, (uintptr_t)d_blob, pl)) return CHR_E_PARAMETER;
    dec_carve(pl, d_ws, ws_bytes);
    if (!d_ws || pl.ws > ws_bytes) return CHR_E_WORKSPACE;
    const CrcTables *tabs = crc_tables_device();
    if (!tabs) return CHR_E_CUDA;
    std::vector<CrcSeg> segs(n);
    for (int64_t i = 0; i < n; ++i) {
        segs[i].begin = pl.regs[i].poff;
        segs[i].end = pl.regs[i].poff + pl.regs[i].plen;
    }
    const int64_t total_sc = crc_plan_segments(segs.data(), n);
    CHR_CUDA_TRY(cudaMemcpyAsync(pl.d_regs, pl.regs.data(), sizeof(DecReg) * n, cudaMemcpyHostToDevice, st));
    CHR_CUDA_TRY(cudaMemcpyAsync(pl.segs, segs.data(), sizeof(CrcSeg) * n, cudaMemcpyHostToDevice, st));
    CHR_CUDA_TRY(cudaMemsetAsync(pl.seg_raw, 0, sizeof(uint32_t) * n, st));
    CHR_CUDA_TRY(cudaMemsetAsync(pl.flags, 0, sizeof(int64_t) * (pl.nitems + 1), st));
    CHR_CUDA_TRY(cudaMemsetAsync(pl.ticket, 0, sizeof(unsigned long long), st));
    CHR_CUDA_TRY(cudaMemsetAsync(pl.ticket3, 0, sizeof(unsigned long long), st));
    CHR_CUDA_TRY(cudaMemsetAsync(pl.tflag, 0, sizeof(int32_t) * (pl.ntiles + 1), st));
    int rc = crc_launch(d_blob, pl.segs, n, total_sc, pl.seg_raw, st);
    if (rc) return rc;
    {
        CHR_PROF("k_check", st);
        k_check<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(pl.d_regs, n, pl.seg_raw, tabs, d_blob);
    }
    {
        CHR_PROF("k_esc_count", st);
        k_esc_count<<<(unsigned)n, 256, 0, st>>>(pl.d_regs, n, d_blob);
    }
    {
        CHR_PROF("k_fill_maps", st);
        k_fill_maps<<<(unsigned)n, 256, 0, st>>>(pl.d_regs, n, pl.chunk_reg, pl.tile_reg);
    }
    {
        CHR_PROF("k_tok_fast", st);
        k_tok_fast<<<(unsigned)pl.nchunks, DTHREADS, 0, st>>>(pl.d_regs, pl.chunk_reg, d_blob, pl.chunk_samples);
    }
    {
        CHR_PROF("k_tok_count", st);
        k_tok_count<<<(unsigned)pl.nchunks, DTHREADS, 0, st>>>(pl.d_regs, n, d_blob, pl.chunk_samples);
    }
    {
        CHR_PROF("k_tok_scan", st);
        k_tok_scan<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(pl.d_regs, n, pl.chunk_samples);
    }
    {
        CHR_PROF("k_rp_locate", st);
        k_rp_locate<<<(unsigned)pl.nchunks, DTHREADS, 0, st>>>(pl.d_regs, pl.chunk_reg, d_blob, pl.chunk_samples,
                                                               pl.rp_byte, pl.rp_skip);
    }
    {
        CHR_PROF("k_locate", st);
        k_locate<<<(unsigned)pl.nchunks, DTHREADS, 0, st>>>(pl.d_regs, n, d_blob, pl.chunk_samples,
                                                            pl.seg_byte, pl.seg_skip);
    }
    {
        CHR_PROF("k_esc_rp", st);
        k_esc_rp<<<(unsigned)n, 256, 0, st>>>(pl.d_regs, d_blob, pl.esc_rp);
    }
    {
        CHR_PROF("k_esc_base", st);
        k_esc_base<<<(unsigned)n, 256, 0, st>>>(pl.d_regs, n, d_blob, pl.esc_base);
    }
    if (pl.ntiles > 0) {
        const int64_t npairs = pl.ndiag * n;
        CHR_CUDA_TRY(cudaMemcpyAsync(pl.pair_base, pl.h_pair_base.data(), sizeof(int64_t) * npairs,
                                     cudaMemcpyHostToDevice, st));
        {
            CHR_PROF("k_tile_order", st);
            k_tile_order<<<(unsigned)ceil_div(npairs, 256), 256, 0, st>>>(pl.d_regs, pl.pair_base, npairs, n, pl.order);
        }
        const int smem3 = (int)(sizeof(int64_t) * TZM * TYM * TXM);
        CHR_CUDA_TRY(cudaFuncSetAttribute(k_lorenzo3d, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3));
        CHR_PROF("k_lorenzo3d", st);
        k_lorenzo3d<<<(unsigned)pl.ntiles, 256, smem3, st>>>(pl.d_regs, pl.tile_reg, d_blob, pl.rp_byte, pl.rp_skip, pl.esc_rp,
                                                         pl.faces, pl.tflag, pl.ticket3, pl.order, d_out);
    }
    if (pl.nitems > 0) {
        const size_t smem = (size_t)pl.max_rows_ex * 16 + DWIN;
        CHR_CUDA_TRY(cudaFuncSetAttribute(k_lorenzo, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        {
            CHR_PROF("k_lorenzo", st);
            k_lorenzo<<<(unsigned)pl.nitems, DTHREADS, smem, st>>>(pl.d_regs, n, d_blob, pl.seg_byte,
                                                                   pl.seg_skip, pl.esc_base, pl.carry,
                                                                   pl.flags, pl.ticket, d_out);
        }
    }
    for (int64_t r0 = 0; r0 < n; r0 += 65535) {
        dim3 g(64, (unsigned)std::min<int64_t>(65535, n - r0));
        {
            CHR_PROF("k_verbatim", st);
            k_verbatim<<<g, 256, 0, st>>>(pl.d_regs, r0, d_blob, d_out);
        }
    }
    CHR_CUDA_TRY(cudaGetLastError());
    CHR_CUDA_TRY(cudaMemcpyAsync(pl.regs.data(), pl.d_regs, sizeof(DecReg) * n, cudaMemcpyDeviceToHost, st));
    CHR_CUDA_TRY(cudaStreamSynchronize(st));
    int status = CHR_OK;
    for (int64_t i = 0; i < n; ++i) {
        const uint32_t err = pl.regs[i].err;
        int code = CHR_DEC_OK;
        if (err) {
            code = __builtin_ctz(err);
            if (err & EF_CRC) code = CHR_DEC_CHECKSUM;
            else if (err & EF_CODEC) code = CHR_DEC_BAD_CODEC;
            if (status == CHR_OK) status = code == CHR_DEC_BAD_CODEC ? CHR_E_UNSUPPORTED_CODEC : CHR_E_CORRUPT;
        }
        if (h_status) h_status[i] = code;
    }
    return status;
}
