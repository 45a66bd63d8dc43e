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

constexpr int64_t DCB = 4096;     // bytes per token chunk
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
    // device-computed
    uint64_t tok_start;            // absolute offset of the token stream
    int64_t nesc;
    uint32_t err;
    uint32_t pad2;
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
    const bool active = (R.codec == 1 || R.codec == 2) && R.err == 0;
    if (active) {
        const int64_t lo = (int64_t)R.tok_start, hi = (int64_t)(R.poff + R.plen);
        const int64_t b0 = (int64_t)R.poff + (c - R.chunk_base) * DCB + threadIdx.x * DBYTES_T;
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
    const bool active = (R.codec == 1 || R.codec == 2) && R.err == 0;
    if (!active) return;  // uniform across the block
    const int64_t lo = (int64_t)R.tok_start, hi = (int64_t)(R.poff + R.plen);
    const int64_t b0 = (int64_t)R.poff + (c - R.chunk_base) * DCB + threadIdx.x * DBYTES_T;
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
    if (R.codec != 2 || R.err) return;
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
    if (!((R.codec == 1 || R.codec == 2) && R.err == 0)) return;
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

// ------------------------------------------------------------------ host
struct DecPlan {
    std::vector<DecReg> regs;
    int64_t nchunks = 0, nseg = 0, nitems = 0, ncarry = 0;
    int max_rows_ex = 0;
    size_t ws = 0;
    DecReg *d_regs;
    CrcSeg *segs;
    uint32_t *seg_raw;
    int64_t *chunk_samples, *seg_byte, *seg_skip, *esc_base, *carry, *flags;
    unsigned long long *ticket;
};

static int dec_rows_for(int ex) {
    // q tile + u(z-1) tile (int64) must fit next to the byte window
    const int64_t budget = 180 * 1024 - DWIN;
    int rows = (int)std::min<int64_t>(8, budget / (16ll * ex));
    return rows < 1 ? 0 : rows;
}

static bool dec_build(const chr_dec_region_t *h, int64_t n, DecPlan &pl) {
    pl.regs.resize(n);
    int64_t chunk = 0, seg = 0, item = 0, carry = 0;
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
        R.chunk_base = chunk;
        R.nchunks = std::max<int64_t>(1, ceil_div((int64_t)R.plen, DCB));
        chunk += R.nchunks;
        R.seg_base = seg;
        R.item_base = item;
        R.carry_base = carry;
        if (R.codec == 1 || R.codec == 2) {
            R.nseg = (int64_t)R.nyt * R.ez;
            seg += R.nseg;
            item += R.nyt;
            carry += (int64_t)R.nyt * R.ez * R.ex;
            pl.max_rows_ex = std::max(pl.max_rows_ex, R.rows * R.ex);
        }
    }
    pl.nchunks = chunk;
    pl.nseg = seg;
    pl.nitems = item;
    pl.ncarry = carry;
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
    pl.ticket = c.take<unsigned long long>(1);
    pl.ws = c.off + 256;
}

}  // namespace chr

using namespace chr;

extern "C" size_t chr_decode_workspace_size(const chr_dec_region_t *h, int64_t n) {
    DecPlan pl;
    if (!h || n < 1 || !dec_build(h, n, pl)) return 256;
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
    if (!dec_build(h, n, pl)) return CHR_E_PARAMETER;
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
        CHR_PROF("k_tok_count", st);
        k_tok_count<<<(unsigned)pl.nchunks, DTHREADS, 0, st>>>(pl.d_regs, n, d_blob, pl.chunk_samples);
    }
    {
        CHR_PROF("k_tok_scan", st);
        k_tok_scan<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(pl.d_regs, n, pl.chunk_samples);
    }
    {
        CHR_PROF("k_locate", st);
        k_locate<<<(unsigned)pl.nchunks, DTHREADS, 0, st>>>(pl.d_regs, n, d_blob, pl.chunk_samples,
                                                            pl.seg_byte, pl.seg_skip);
    }
    {
        CHR_PROF("k_esc_base", st);
        k_esc_base<<<(unsigned)n, 256, 0, st>>>(pl.d_regs, n, d_blob, pl.esc_base);
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
