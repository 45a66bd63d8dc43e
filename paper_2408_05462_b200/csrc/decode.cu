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
#include <memory>
#include <cstdio>
#include <cstdlib>
#include <cmath>
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
    // fast (canonical-stream) path: band tiles (full rows x bty rows x btz planes)
    int64_t abase;                 // 16-byte aligned chunk origin (blob-relative)
    int32_t tnx, tny, tnz;         // tiles per axis (tnx = 1, tny = bands, tnz = chunks)
    int32_t doff, pad2;            // step offset of the region's wavefront (host tile order, dec_build)
    int32_t bty, btz, rs;          // band rows, chunk planes, smem row stride
    int64_t tile_base, ntiles;
    int64_t sp_base;               // segment index: ez * tny entries
    int64_t face_base, face_n;     // int64 faces per tile: ex * (btz + 1 + bty)
    int64_t mask_off;              // inside-mask words (v >= iso), plane-linear bits (optional output)
    int32_t pw, pad3;              // mask words per plane
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

// per-region checks that need no payload pass (the CRC is k_crc_flag's, on
// the side stream: decoding proceeds and the call's status reports a
// mismatch first, as decompress() raises it before decoding, codec.py:220)
__global__ void k_check(DecReg *__restrict__ regs, int64_t nreg) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nreg) return;
    DecReg &R = regs[r];
    uint32_t err = 0;
    if (R.codec < 0 || R.codec > 3) err |= EF_CODEC;
    R.tok_start = R.poff;
    R.nesc = 0;
    if (!err) {
        if (R.codec == 0 && R.plen < 8ull * (uint64_t)R.n) err |= EF_TRUNC;
        if (R.codec == 3 && R.plen < 4ull * (uint64_t)R.n) err |= EF_TRUNC;
        if (R.codec == 2 && R.plen < (uint64_t)((R.n + 7) >> 3)) err |= EF_SHORTBM;
    }
    R.err = err;
}

// payload CRC vs the expected one: the host's (R.crc) or, with `hdr`, the
// block header's last four bytes (just before the payload).  Writes only
// crc_bad, which no decode kernel reads (R.err stays the decoders' own).
__global__ void k_crc_flag(const DecReg *__restrict__ regs, int64_t nreg, const uint32_t *__restrict__ seg_raw,
                           const CrcTables *__restrict__ tabs, const uint8_t *__restrict__ blob, int hdr,
                           int32_t *__restrict__ crc_bad) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nreg) return;
    const DecReg &R = regs[r];
    const uint32_t crc = crc_finalize(tabs->x2n, seg_raw[r], R.plen);
    uint32_t want = R.crc;
    if (hdr) {
        const uint8_t *p = blob + R.poff - 4;
        want = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
    }
    crc_bad[r] = crc != want ? 1 : 0;
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
__global__ void k_tok_scan(DecReg *__restrict__ regs, int64_t nreg, int64_t *__restrict__ chunk_samples,
                           int slow_pass) {
    // CTA per region: blockDim chunk counts per step (a region can span
    // thousands of 4 KiB chunks; a warp-wide scan left a long serial chain)
    const int64_t r = blockIdx.x;
    if (r >= nreg) return;
    DecReg &R = regs[r];
    if (!((R.codec == 1 || R.codec == 2) && R.err == 0)) return;
    if ((R.slow != 0) != (slow_pass != 0)) return;  // pass 0: band regions, pass 1: generic
    int64_t acc = 0;
    int over = 0;
    for (int64_t c0 = 0; c0 < R.nchunks; c0 += blockDim.x) {
        const int64_t c = R.chunk_base + c0 + threadIdx.x;
        const bool ok = c0 + threadIdx.x < R.nchunks;
        const int64_t v = ok ? chunk_samples[c] : 0;
        int64_t tot;
        const int64_t ex = block_excl64(v, &tot);
        if (ok) chunk_samples[c] = acc + ex;
        if (ok && (acc + ex + v > R.n || v < 0)) over = 1;
        acc += tot;
    }
    over = __syncthreads_or(over);
    if (threadIdx.x != 0) return;
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
__device__ __forceinline__ int32_t ld_relaxed32(const int32_t *p) {
    int32_t v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// spin on a tile flag with relaxed loads (an acquire load invalidates the
// SM's L1 on every poll), then one acquire load orders the reads after it
__device__ __forceinline__ void wait_flag(const int32_t *p, int32_t v) {
    while (ld_relaxed32(p) != v) __nanosleep(20);
    (void)ld_acquire32(p);
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
// end / zero bits of 16 bytes (4 words)
__device__ __forceinline__ void ez16(const uint32_t *w, uint32_t &E, uint32_t &Z) {
    E = 0;
    Z = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        E |= word_end4(w[k]) << (4 * k);
        Z |= word_zero4(w[k]) << (4 * k);
    }
}

// from the raw end / zero bits of the 32-byte window (consecutive units of
// a thread pass their own half on as the next unit's context half)
__device__ __forceinline__ UnitMasks unit_masks_ez(uint32_t E, uint32_t Z, int64_t u0, int64_t lo, int64_t hi) {
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

__device__ __forceinline__ UnitMasks unit_masks(const uint32_t (&w)[8], int64_t u0, int64_t lo, int64_t hi) {
    uint32_t E0, Z0, E1, Z1;
    ez16(w, E0, Z0);
    ez16(w + 4, E1, Z1);
    return unit_masks_ez(E0 | (E1 << 16), Z0 | (Z1 << 16), u0, lo, hi);
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

constexpr int UPT = (int)(DCB / (16 * DTHREADS));  // 16-byte units per thread

// samples per chunk (fast path); flags non-canonical regions
__global__ void __launch_bounds__(DTHREADS) k_tok_fast(DecReg *__restrict__ regs, const int32_t *__restrict__ chunk_reg,
                                                       const uint8_t *__restrict__ blob,
                                                       int64_t *__restrict__ chunk_samples,
                                                       int64_t *__restrict__ thr_cnt,
                                                       int32_t *__restrict__ any_slow) {
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
        uint32_t Ec, Zc;  // raw end / zero bits of the context half
        ez16(w, Ec, Zc);
#pragma unroll 1
        for (int u = 0; u < UPT; ++u) {
            const int64_t u0 = ub + 16 * u;
            if (u) next_unit(blob, u0, w);
            uint32_t Eo, Zo;
            ez16(w + 4, Eo, Zo);
            const uint32_t Ew = Ec | (Eo << 16), Zw = Zc | (Zo << 16);
            Ec = Eo;
            Zc = Zo;
            if (u0 + 16 > lo && u0 < hi) {
                const UnitMasks m = unit_masks_ez(Ew, Zw, u0, lo, hi);
                err |= m.err;
                nc |= m.noncanon;
                cnt += unit_count(m, blob, u0);
            }
        }
    }
    thr_cnt[c * DTHREADS + threadIdx.x] = cnt;
    const int64_t tot = block_sum64(cnt);
    if (err) atomicOr(&R.err, err);
    if (nc) {
        atomicOr(&R.slow, 1u);
        atomicOr(any_slow, 1);
    }
    if (threadIdx.x == 0) chunk_samples[c] = tot;
}

// segment index of the band path: for every (plane z, band b) of a region
// the byte of the token (marker for runs) holding sample (z*ey + b*bty)*ex
// and the samples of that token before it.  Per-thread sample counts come
// from k_tok_fast; only threads whose samples contain a segment start walk
// their tokens again.
__global__ void __launch_bounds__(DTHREADS) k_seg_locate(const DecReg *__restrict__ regs,
                                                         const int32_t *__restrict__ chunk_reg,
                                                         const uint8_t *__restrict__ blob,
                                                         const int64_t *__restrict__ chunk_start,
                                                         const int64_t *__restrict__ thr_cnt,
                                                         int64_t *__restrict__ sp_byte,
                                                         int64_t *__restrict__ sp_skip,
                                                         int64_t *__restrict__ pos64) {
    const int64_t c = blockIdx.x;
    const DecReg &R = regs[chunk_reg[c]];
    if (!((R.codec == 1 || R.codec == 2) && R.err == 0 && !R.slow)) return;
    const int64_t cnt = thr_cnt[c * DTHREADS + threadIdx.x];
    int64_t a = chunk_start[c] + block_excl64(cnt, nullptr);
    pos64[c * DTHREADS + threadIdx.x] = a;  // first sample of the tokens ending in this 64-byte group
    if (cnt == 0) return;
    const int64_t ex = R.ex, plane = ex * R.ey, band = ex * R.bty, nb = R.tny;
    int64_t z, b;
    if (a < (1ll << 32) && plane < (1ll << 31)) {  // 32-bit divisions (a 64-bit one is a long software routine)
        const uint32_t a32 = (uint32_t)a, p32 = (uint32_t)plane, b32 = (uint32_t)band;
        const uint32_t zz = a32 / p32;
        z = zz;
        b = (a32 - zz * p32 + b32 - 1) / b32;
    } else {
        z = a / plane;
        b = (a - z * plane + band - 1) / band;
    }
    if (b >= nb) {
        b = 0;
        ++z;
    }
    int64_t s = z * plane + b * band;  // first segment start >= a
    const int64_t a_end = a + cnt;
    if (s >= a_end) return;
    const int64_t lo = (int64_t)R.tok_start, hi = (int64_t)(R.poff + R.plen);
    const int64_t ub = R.abase + (c - R.chunk_base) * DCB + (int64_t)threadIdx.x * UPT * 16;
    uint32_t w[8];
    load_units(blob, ub, w);
    uint32_t Ec, Zc;  // raw end / zero bits of the context half
    ez16(w, Ec, Zc);
#pragma unroll 1
    for (int u = 0; u < UPT; ++u) {
        const int64_t u0 = ub + 16 * u;
        if (u) next_unit(blob, u0, w);
        uint32_t Eo, Zo;
        ez16(w + 4, Eo, Zo);
        const uint32_t Ew = Ec | (Eo << 16), Zw = Zc | (Zo << 16);
        Ec = Eo;
        Zc = Zo;
        if (!(u0 + 16 > lo && u0 < hi)) continue;
        const UnitMasks m = unit_masks_ez(Ew, Zw, u0, lo, hi);
        if (m.len == 0) {  // literals only: one sample per token, starts found by rank
            const int n = __popc(m.lit);
            while (s < a + n) {
                const int e = (int)__fns(m.lit, 0, (int)(s - a) + 1);
                const uint32_t below = m.E & ((1u << e) - 1u);
                const int sb = below ? 32 - __clz(below) : 0;
                const int64_t k = R.sp_base + z * nb + b;
                sp_byte[k] = u0 - 16 + sb;
                sp_skip[k] = 0;
                if (++b >= nb) {
                    b = 0;
                    ++z;
                }
                s = z * plane + b * band;
            }
            a += n;
            if (s >= a_end) return;
            continue;
        }
        uint32_t T = m.lit | m.len;
        while (T) {
            const int e = __ffs(T) - 1;
            T &= T - 1;
            const uint32_t below = m.E & ((1u << e) - 1u);
            const int sb = below ? 32 - __clz(below) : 0;
            int64_t tc = 1, sbyte = u0 - 16 + sb;
            if ((m.len >> e) & 1u) {
                tc = (int64_t)unit_token_value(blob, m.E, e, u0);
                sbyte -= 1;  // the marker
            }
            while (s < a + tc) {
                const int64_t k = R.sp_base + z * nb + b;
                sp_byte[k] = sbyte;
                sp_skip[k] = s - a;
                if (++b >= nb) {
                    b = 0;
                    ++z;
                }
                s = z * plane + b * band;
            }
            a += tc;
        }
        if (s >= a_end) return;  // no segment start left in this thread's samples
    }
}

// codec 2 (band path): escapes before every segment (one CTA per region)
__global__ void __launch_bounds__(256) k_esc_seg(const DecReg *__restrict__ regs, const uint8_t *__restrict__ blob,
                                                 int64_t *__restrict__ esc_sp) {
    const DecReg &R = regs[blockIdx.x];
    if (R.codec != 2 || R.err || R.slow || R.nesc == 0) return;
    const uint8_t *bm = blob + R.poff;
    const int64_t plane = (int64_t)R.ex * R.ey, band = (int64_t)R.ex * R.bty, nb = R.tny;
    const int64_t nsp = (int64_t)R.ez * nb;
    int64_t carry = 0;
    for (int64_t k0 = 0; k0 < nsp; k0 += 256) {
        const int64_t k = k0 + threadIdx.x;
        int64_t cnt = 0;
        if (k < nsp) {
            const int64_t z = k / nb, b = k - z * nb;
            const int64_t s0 = z * plane + b * band, s1 = b + 1 < nb ? s0 + band : (z + 1) * plane;
            int64_t s = s0;
            for (; s < s1 && (s & 7); ++s) cnt += (bm[s >> 3] >> (s & 7)) & 1;
            for (; s + 8 <= s1; s += 8) cnt += __popc(bm[s >> 3]);
            for (; s < s1; ++s) cnt += (bm[s >> 3] >> (s & 7)) & 1;
        }
        int64_t total;
        const int64_t ex = block_excl64(cnt, &total);
        if (k < nsp) esc_sp[R.sp_base + k] = carry + ex;
        carry += total;
    }
}

// ---- band tiles.  A tile is (full rows x, a band of bty rows y, a chunk of
// btz planes z) of one region in SMB bytes of shared memory (int32).
// Tile-local prefixes along x (rows are whole), y and z give T; then
//   u(x,y,z) = T + [Fy(x,z) - Fy(x,z0-1)] + Fz(x,y)
// with Fy = last row of the band above (planes z0-1..z1-1) and Fz = last
// plane of the chunk before.  All int64 (modular like the reference's
// cumsum), so every canonical stream decodes exactly.  Tiles wait only on
// those two neighbours, both on the previous wavefront diagonal b + c, so
// taking tiles in diagonal order from a ticket cannot deadlock; a tile
// publishes its own faces right after the wait (a few adds per column)
// and only then writes its samples, so a chain hop costs one face update.
// The tile holds q and its x / y prefixes as int32: those sums stay inside
// one plane segment of the tile, so int32 is exact when the segment's sum |q|
// < 2^31 (k_band checks it right after tokenising; a segment at or above it
// -- rare, only from extreme quanta -- sends its region to the int64 pass via
// k_asum_check).  The z prefix, the faces (u at tile boundaries) and u =
// prefix + faces are int64, exact like the reference's int64 cumsum.
using BV = int32_t;
// Dynamic shared memory per band tile (int32 pass): the int32 tile and, for
// a region with more than one band, its dF (btz x ex int64) behind it.  The
// largest budget that keeps 3 CTAs per SM next to the ~3 KB of segment
// tables (72 KB: 18432 int32 samples without dF).  Measured at c3 with a
// fixed 12 KB dF array beside the tile: 10240 samples -> 1.167 ms, 12288 ->
// 1.118, 14336 -> 1.100, 15360 -> 1.077, 16384 -> 1.284 (2 CTAs/SM).
#ifndef CHR_BAND_SMEM
#define CHR_BAND_SMEM 73728
#endif
constexpr int64_t SMB = CHR_BAND_SMEM;
#ifndef CHR_KBT
#define CHR_KBT 384
#endif
constexpr int KBT = CHR_KBT, KBW = KBT / 32;  // k_band threads / warps per CTA    // dF entries (btz * ex) when a tile has a band above
constexpr int BSEGM = 64;    // planes per tile

__device__ __forceinline__ int seg_of(const int32_t *base, int nseg, int g) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (base[mid] <= g) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// ---- band tokenizer: 24-byte windows {8 look-back | 16 own} held in six
// registers; bit j <-> byte j, own bytes are bits 8..23.  Canonical streams
// (validated by k_tok_fast) only, so no error checks here.
struct Win24 {
    uint32_t w[6];
    uint32_t E, lit, len;  // end bytes; literal / run-length token ends (own)
};

// the window from its 8 context bytes (prv) and 16 own bytes (cur) at u0
__device__ __forceinline__ Win24 win24_of(uint2 prv, uint4 cur, int64_t u0, int64_t lo, int64_t hi) {
    Win24 W;
    W.w[0] = prv.x; W.w[1] = prv.y;
    W.w[2] = cur.x; W.w[3] = cur.y; W.w[4] = cur.z; W.w[5] = cur.w;
    uint32_t E = 0, Z = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        E |= word_end4(W.w[k]) << (4 * k);
        Z |= word_zero4(W.w[k]) << (4 * k);
    }
    const int64_t nlo = lo - (u0 - 8), nhi = hi - (u0 - 8);  // bits [nlo, nhi) are stream bytes
    const uint32_t lob = nlo <= 0 ? 0u : (nlo >= 24 ? 0xFFFFFFu : ((1u << nlo) - 1u));
    const uint32_t hib = nhi >= 24 ? 0u : (nhi <= 0 ? 0xFFFFFFu : (0xFFFFFFu & ~((1u << nhi) - 1u)));
    const uint32_t out = lob | hib;
    E = (E | out) & 0xFFFFFFu;
    Z &= ~out & 0xFFFFFFu;
    const uint32_t C = ~E & 0xFFFFFFu;
    const uint32_t Lend = (C + (Z << 1)) & ~C;
    const uint32_t own = 0xFFFF00u & ~out;
    W.E = E;
    W.len = Lend & ~Z & own;
    W.lit = E & ~Z & ~Lend & own;
    return W;
}

__device__ __forceinline__ uint32_t win_byte(const Win24 &W, int j) {  // j static after unrolling
    return (W.w[j >> 2] >> (8 * (j & 3))) & 0xFFu;
}

// samples of the tokens ending in the unit's own bytes
__device__ __forceinline__ int64_t win24_count(const Win24 &W) {
    int64_t c = __popc(W.lit);
    uint32_t Lm = W.len;
    while (Lm) {
        const int e = __ffs(Lm) - 1;
        Lm &= Lm - 1;
        const uint32_t below = W.E & ((1u << e) - 1u);
        const int s = 32 - __clz(below);
        uint64_t v = 0;
#pragma unroll
        for (int j = 3; j < 24; ++j)  // static byte positions; token bytes are s..e
            if (j >= s && j <= e) v |= (uint64_t)(win_byte(W, j) & 0x7Fu) << (7 * (j - s));
        c += (int64_t)v;
    }
    return c;
}

// one unit -> literals into the plane `q` (positions count samples from the
// segment start; PAD planes have row stride ex + 1).  Branch-free over the 16
// own positions: H holds the LEB128 payload of bytes e-4..e, so the token
// ending at e has value H >> 7 (5 - len).  Only for positions below -2^30
// (a segment starting deep inside a zero run) or a 5-byte token in the
// warp, in the int64 pass (the int32 pass sends such regions there).
template <bool PAD, typename QV>
__device__ __forceinline__ int64_t band_scatter_unit64(const Win24 &W, int64_t at64, int L, int ex, uint64_t M,
                                                     QV *__restrict__ q) {
    int64_t at = at64;
    int idx = (int)at, x = 0;
    if (PAD && at >= 0) {
        const int row = (int)(((uint64_t)at * M) >> 32);
        x = (int)at - row * ex;
        idx = row * (ex + 1) + x;
    }
    uint64_t H = 0;
#pragma unroll
    for (int j = 3; j < 8; ++j) H = (H >> 7) | ((uint64_t)(win_byte(W, j) & 0x7Fu) << 28);
#pragma unroll
    for (int e = 8; e < 24; ++e) {
        H = (H >> 7) | ((uint64_t)(win_byte(W, e) & 0x7Fu) << 28);
        const bool lit = (W.lit >> e) & 1u, run = (W.len >> e) & 1u;
        if (!(lit | run)) continue;
        const uint32_t below = W.E & ((1u << e) - 1u);
        const int len = e - (32 - __clz(below)) + 1;
        const uint64_t v = H >> (7 * (5 - len));
        if (lit) {
            const uint64_t zz = v - 1;
            if ((uint64_t)at < (uint64_t)L) {
                q[idx] = (QV)((int64_t)(zz >> 1) ^ -(int64_t)(zz & 1));
            }
            ++at;
            ++idx;
            if (PAD && ++x == ex) {
                x = 0;
                ++idx;
            }
        } else {
            at += (int64_t)v;
            idx = (int)min(at, (int64_t)L);
            if (PAD && at >= 0 && at < L) {
                const int row = (int)(((uint64_t)at * M) >> 32);
                x = (int)at - row * ex;
                idx = row * (ex + 1) + x;
            }
        }
    }
    return at;
}

// 32-bit path: tokens <= 4 bytes (H = payload of bytes e-3..e in 28 bits),
// positions in int32 (clamped to 2^30 past L: every position that matters
// is < L <= SMB / 4 and a segment starts at -skip >= -2^30).  Returns the
// position after the unit's tokens.
template <bool PAD, typename QV>
__device__ __forceinline__ int band_scatter_unit32(const Win24 &W, int at, int L, int ex, uint64_t M,
                                                   QV *__restrict__ q, uint32_t &asum) {
    uint32_t H = 0;
    const uint32_t qs = (uint32_t)__cvta_generic_to_shared(q);
#pragma unroll
    for (int j = 4; j < 8; ++j) H = (H >> 7) | ((win_byte(W, j) & 0x7Fu) << 21);
#pragma unroll
    for (int e = 8; e < 24; ++e) {
        H = (H >> 7) | ((win_byte(W, e) & 0x7Fu) << 21);
        const bool lit = (W.lit >> e) & 1u, run = (W.len >> e) & 1u;
        const uint32_t below = W.E & ((1u << e) - 1u);
        const int len = e - (32 - __clz(below)) + 1;
        const uint32_t v = H >> (7 * (4 - len));
        if (lit && (unsigned)at < (unsigned)L) {
            const uint32_t zz = v - 1u;
            const int idx = PAD ? at + (int)(((uint64_t)(unsigned)at * M) >> 32) : at;
            const int32_t qv = (int32_t)((zz >> 1) ^ (0u - (zz & 1u)));
            if (sizeof(QV) == 4) {  // a shared-window store from the hoisted 32-bit address
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(qs + 4u * (uint32_t)idx), "r"(qv) : "memory");
            } else {
                q[idx] = (QV)qv;
            }
            asum += v >> 1;  // |q| (v = zigzag + 1)
        }
        // positions past L only need to stay past L: clamping at 2^30 keeps
        // at + v (< 2^28 here) inside int32
        at = min(at + (lit ? 1 : (run ? (int)v : 0)), 1 << 30);
    }
    return at;
}

// QV = int64_t: tokens of any width.  QV = int32_t (the fast pass): a unit
// with a 5-byte token or a position below -2^30 in the warp flags its region
// for the int64 pass (`wide_out`) and is skipped; otherwise the stored
// literals' |q| add to `asum` (<= 2^31 over a 64-byte group: at most 2^25
// per byte).
template <bool PAD, typename QV>
__device__ __forceinline__ int64_t band_scatter_unit(const Win24 &W, int64_t at, int L, int ex, uint64_t M,
                                                     QV *__restrict__ q, bool active, uint32_t &asum,
                                                     bool &wide_out) {
    const uint32_t C = ~W.E & 0xFFFFFFu;
    const bool long5 = active && ((C << 1) & (C << 2) & (C << 3) & (C << 4) & (W.lit | W.len)) != 0;
    const bool wide = active && (long5 || at < -(1ll << 30));
    if (sizeof(QV) == 4) {
        if (__any_sync(0xFFFFFFFFu, wide)) {
            wide_out |= wide;
            return at;  // the region is decoded again by the int64 pass
        }
        return active ? (int64_t)band_scatter_unit32<PAD, QV>(W, (int)at, L, ex, M, q, asum) : at;
    }
    uint32_t unused = 0;
    if (__any_sync(0xFFFFFFFFu, wide)) {
        return active ? band_scatter_unit64<PAD, QV>(W, at, L, ex, M, q) : at;
    }
    return active ? (int64_t)band_scatter_unit32<PAD, QV>(W, (int)at, L, ex, M, q, unused) : at;
}

// QV = int32_t: the fast pass (checks the tile's sum |q|); QV = int64_t: the
// pass over the regions some int32 tile could not hold (asum_reg >= 2^31)
#ifdef CHR_BAND_TRACE
// diagnostic build only: per tile (smid, start, after scatter, after x/y
// prefix, band-above face in, chunk-before face in, published, end) in ns
__device__ unsigned long long *g_band_trace;
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define BAND_TR(k)                                                                      \
    do {                                                                                \
        if (g_band_trace && sizeof(QV) == 4 && tid == 0) g_band_trace[tile * 8 + (k)] = gtime(); \
    } while (0)
#else
#define BAND_TR(k) \
    do {           \
    } while (0)
#endif

template <typename QV>
__global__ void __launch_bounds__(KBT) k_band(const DecReg *__restrict__ regs, const int32_t *__restrict__ tile_reg,
                                              const uint8_t *__restrict__ blob,
                                              const int64_t *__restrict__ sp_byte,
                                              const int64_t *__restrict__ sp_skip,
                                              const int64_t *__restrict__ esc_sp, const int64_t *__restrict__ pos64,
                                              int64_t *__restrict__ faces,
                                              int32_t *__restrict__ tflag, unsigned long long *__restrict__ ticket,
                                              const int32_t *__restrict__ order, double *__restrict__ out,
                                              uint32_t *__restrict__ mask, double iso,
                                              unsigned long long *__restrict__ asum_reg) {
    extern __shared__ __align__(16) unsigned char kb_raw[];
    QV *const Q = reinterpret_cast<QV *>(kb_raw);  // [nzv][nyv][rs]
    __shared__ int64_t s_lo[BSEGM], s_hi[BSEGM], s_ub[BSEGM], s_off[BSEGM];
    __shared__ int32_t s_base[BSEGM + 1];
    __shared__ int64_t s_tile, s_zero;
    __shared__ unsigned long long s_asum[BSEGM];  // sum |q| per plane segment
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_tile = order[atomicAdd(ticket, 1ull)];
        s_zero = 0;
    }
    __syncthreads();
    const int64_t tile = s_tile;
    const DecReg &R = regs[tile_reg[tile]];
    if (!((R.codec == 1 || R.codec == 2) && R.err == 0 && !R.slow)) return;
    if (sizeof(QV) == 8 && asum_reg[tile_reg[tile]] < (1ull << 31)) return;  // done by the int32 pass
    const int nb = R.tny, ex = R.ex, ey = R.ey, rs = R.rs, bty = R.bty, btz = R.btz;
    const int64_t local = tile - R.tile_base;
    const int b = (int)(local % nb), c = (int)(local / nb);
    const int y0 = b * bty, z0 = c * btz;
    const int nyv = min(bty, ey - y0), nzv = min(btz, R.ez - z0);
    const int L = nyv * ex;       // samples per plane segment
    const int PL = nyv * rs;      // smem words per plane
    const int64_t hi = (int64_t)(R.poff + R.plen);
    const int64_t sp_end = R.sp_base + (int64_t)R.ez * nb;
#ifdef CHR_BAND_TRACE
    if (g_band_trace && sizeof(QV) == 4 && tid == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_band_trace[tile * 8] = smid;
    }
#endif
    BAND_TR(1);

    for (int i = tid; i < nzv * PL; i += KBT) Q[i] = 0;
    if (tid < BSEGM) s_asum[tid] = 0;
    // ---- segments (one per plane) and the 64-byte token groups they cover.
    //      Group g (bytes [G, G+64) from the chunk origin) has its first sample
    //      in pos64 (k_seg_locate), so a thread walks one group without a count
    //      pass; the group holding the segment's first byte starts at -skip.
    if (warp == 0) {
        int ng[2] = {0, 0};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = lane + 32 * h;
            if (j < nzv) {
                const int64_t k = R.sp_base + (int64_t)(z0 + j) * nb + b;
                const int64_t b0 = sp_byte[k];
                const int64_t b1 = k + 1 < sp_end ? min(hi, sp_byte[k + 1] + 11) : hi;
                const int64_t g0 = (b0 - R.abase) >> 6, g1 = (b1 - 1 - R.abase) >> 6;
                s_lo[j] = b0;
                s_hi[j] = b1;
                s_ub[j] = g0;
                s_off[j] = sp_skip[k];
                ng[h] = (int)(g1 - g0 + 1);
            }
        }
        int i0 = ng[0];  // lane owns j = lane and lane + 32: scan in two halves
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int o = __shfl_up_sync(0xFFFFFFFFu, i0, off);
            if (lane >= off) i0 += o;
        }
        const int tot0 = __shfl_sync(0xFFFFFFFFu, i0, 31);
        int i1 = ng[1];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int o = __shfl_up_sync(0xFFFFFFFFu, i1, off);
            if (lane >= off) i1 += o;
        }
        const int tot1 = __shfl_sync(0xFFFFFFFFu, i1, 31);
        if (lane < nzv) s_base[lane] = i0 - ng[0];
        if (lane + 32 < nzv) s_base[lane + 32] = tot0 + i1 - ng[1];
        if (lane == 0) s_base[nzv] = tot0 + tot1;
    }
    __syncthreads();
    const int U = s_base[nzv];
    const uint64_t M = ((1ull << 32) + (uint64_t)ex - 1) / (uint64_t)ex;  // row = (at * M) >> 32
    const int64_t gbase = R.chunk_base * DTHREADS;  // pos64 index of the region's first group
    bool wide = false;  // a token the int32 pass does not take (5 bytes / deep negative start)
    for (int g0 = warp * 32; g0 < U; g0 += KBT) {  // warp-uniform bounds (the unit walk votes)
        uint32_t asum = 0;  // sum |q| of the literals this thread stores (segment j; <= 2^31)
        const int gi = g0 + lane;
        const bool own = gi < U;
        int j = 0;
        int64_t G = 0, at = L;
        uint4 cur = make_uint4(0, 0, 0, 0);  // the unit's 16 bytes, loaded one unit ahead
        uint2 prv = make_uint2(0, 0);        // the 8 bytes before it
        int64_t slo = 0, shi = 0;
        if (own) {
            j = seg_of(s_base, nzv, gi);
            const int64_t grp = s_ub[j] + (gi - s_base[j]);
            G = R.abase + grp * 64;
            slo = s_lo[j];
            shi = s_hi[j];
            cur = __ldg(reinterpret_cast<const uint4 *>(blob + G));  // G < shi: inside the file
            if (G >= 8) prv = __ldg(reinterpret_cast<const uint2 *>(blob + G - 8));
            const int64_t segstart = ((int64_t)(z0 + j) * ey + y0) * ex;
            at = G <= slo ? -s_off[j] : __ldg(pos64 + gbase + grp) - segstart;
        }
        QV *q = Q + j * PL;
#pragma unroll 1
        for (int u = 0; u < 4; ++u) {
            const int64_t u0 = G + 16 * u;
            const bool act = own && at < L && u0 + 16 > slo && u0 < shi;
            uint4 nxt = make_uint4(0, 0, 0, 0);
            if (own && u < 3 && u0 + 16 < shi) nxt = __ldg(reinterpret_cast<const uint4 *>(blob + u0 + 16));
            if (__any_sync(0xFFFFFFFFu, act)) {
                Win24 W;
                if (act) W = win24_of(prv, cur, u0, slo, shi);
                at = rs == ex ? band_scatter_unit<false, QV>(W, at, L, ex, M, q, act, asum, wide)
                              : band_scatter_unit<true, QV>(W, at, L, ex, M, q, act, asum, wide);
            }
            prv = make_uint2(cur.z, cur.w);
            cur = nxt;
        }
        if (sizeof(QV) == 4) {
            // one shared atomic per warp when its lanes' groups are in one
            // segment and their sum fits 32 bits (the usual case)
            const int j0 = __shfl_sync(0xFFFFFFFFu, j, 0);
            if (__all_sync(0xFFFFFFFFu, (j == j0 || !own) && asum < (1u << 26))) {
                const uint32_t tot = __reduce_add_sync(0xFFFFFFFFu, asum);
                if (lane == 0 && tot) atomicAdd(&s_asum[j0], (unsigned long long)tot);
            } else if (asum) {
                atomicAdd(&s_asum[j], (unsigned long long)asum);
            }
        }
    }
    if (sizeof(QV) == 4 && wide) atomicMax(&s_asum[0], 1ull << 31);
    __syncthreads();
    BAND_TR(2);
    // The x / y prefixes stay inside one plane segment, so int32 holds them
    // exactly when the segment's sum |q| < 2^31 (the z prefix is summed in
    // int64 below).  Otherwise the region is decoded again by the int64 pass
    // (this tile still publishes its faces so the region's chain completes).
    if (sizeof(QV) == 4 && warp == 0) {
        unsigned long long mx = 0;
        for (int j = lane; j < nzv; j += 32) mx = max(mx, s_asum[j]);
#pragma unroll
        for (int off = 16; off; off >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, off));
        if (lane == 0 && mx >= (1ull << 31)) atomicMax(asum_reg + tile_reg[tile], mx);
    }
    // ---- x-prefix (rows are whole)
    const int rows = nzv * nyv;
    if (rows >= 64) {
        for (int r = tid; r < rows; r += KBT) {
            QV *p = Q + r * rs;
            QV acc = 0;
            for (int xx = 0; xx < ex; ++xx) {
                acc += p[xx];
                p[xx] = acc;
            }
        }
    } else {
        for (int r = warp; r < rows; r += KBW) {
            QV *p = Q + r * rs;
            QV carry = 0;
            for (int x0 = 0; x0 < ex; x0 += 32) {
                const int xx = x0 + lane;
                QV v = xx < ex ? p[xx] : 0;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const QV o = __shfl_up_sync(0xFFFFFFFFu, v, off);
                    if (lane >= off) v += o;
                }
                v += carry;
                if (xx < ex) p[xx] = v;
                carry = __shfl_sync(0xFFFFFFFFu, v, 31);
            }
        }
    }
    __syncthreads();
    // ---- y-prefix (columns (plane, x))
    auto split = [&](int t, int &hi_, int &lo_) {  // t = hi_ * ex + lo_
        hi_ = (int)(((uint64_t)t * M) >> 32);
        lo_ = t - hi_ * ex;
    };
    for (int t = tid; t < ex * nzv; t += KBT) {
        int j, xx;
        split(t, j, xx);
        QV *p = Q + j * PL + xx;
        QV acc = 0;
        for (int yy = 0; yy < nyv; ++yy) {
            acc += p[yy * rs];
            p[yy * rs] = acc;
        }
    }
    // ---- the z prefix runs in int64 inside the face / reconstruction loops
    const bool pad = rs != ex;
    // ---- band above (same chunk): its inclusive faces give dF(z, x) = Fy(z) - Fy(z0 - 1)
    // Face record of a tile: [Fy' (btz+1) x ex | I (bty x ex)] with
    // Fy' = u(row y1-1, planes z0-1..z1-1) and I = u(plane z1-1); flag 2 =
    // published.
    const int64_t fn = R.face_n;
    const int64_t io = (int64_t)(btz + 1) * ex;
    // [nzv][ex] behind the tile (band_shape budgets both when a band below exists)
    int64_t *dF = reinterpret_cast<int64_t *>(kb_raw + (((size_t)nzv * PL * sizeof(QV) + 15) & ~size_t(15)));
    int64_t *myF = faces + R.face_base + local * fn;
    BAND_TR(3);
    if (b > 0) {
#ifndef CHR_BAND_NOWAIT
        if (tid == 0)
            wait_flag(tflag + tile - 1, 2);
#endif
        __syncthreads();
        BAND_TR(4);
        const int64_t *Fy = faces + R.face_base + (local - 1) * fn;
        for (int t = tid; t < ex * nzv; t += KBT) dF[t] = __ldcg(Fy + ex + t) - __ldcg(Fy + (t - (t / ex) * ex));
    }
    __syncthreads();
    auto qidx = [&](int t, int &xx) {
        int yy = 0;
        xx = t;
        if (pad || b > 0) split(t, yy, xx);
        return pad ? yy * rs + xx : t;
    };
    // a tile publishes only what its successors read: Fy' (last row, every
    // plane) when a band below exists, I (last plane) when a chunk follows
    const bool need_fy = b + 1 < nb, need_i = c + 1 < R.tnz;
    auto publish_col = [&](int t, int64_t fz) {
        int xx;
        const int qi = qidx(t, xx);
        int64_t acc = 0;  // z prefix of the column
        if (need_fy && t >= L - ex) {  // last row (xx is the column only when split ran)
            const int xl = t - (L - ex);
            myF[xl] = fz;
            for (int j = 0; j < nzv; ++j) {
                acc += Q[j * PL + qi];
                myF[(j + 1) * ex + xl] = acc + (b > 0 ? dF[j * ex + xl] : 0) + fz;
            }
        } else {
            for (int j = 0; j < nzv; ++j) acc += Q[j * PL + qi];
        }
        if (need_i) myF[io + t] = acc + (b > 0 ? dF[(nzv - 1) * ex + xx] : 0) + fz;
    };
    const double twoe = 2.0 * R.e;
    const int64_t zstride = (int64_t)ex * ey;
    double *obase = out + R.out_off + ((int64_t)z0 * ey + y0) * ex;
    auto recon_col = [&](int t, int64_t fz) {
        int xx;
        const QV *p = Q + qidx(t, xx);
        double *o = obase + t;
        int64_t acc = fz;
        if (b > 0) {
            const int64_t *d = dF + xx;
            for (int j = 0; j < nzv; ++j) {
                acc += p[j * PL];
                __stcs(o + j * zstride, (double)(acc + d[j * ex]) * twoe);
            }
        } else {
            for (int j = 0; j < nzv; ++j) {
                acc += p[j * PL];
                __stcs(o + j * zstride, (double)acc * twoe);
            }
        }
    };
    auto release = [&](int f) {  // the barrier orders all face stores before thread 0's fence + flag
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            st_release32(tflag + tile, f);
        }
    };
    // ---- chunk before (same band): its inclusive faces give the carry Fz
    const int64_t *Ip = faces + R.face_base + (local - nb) * fn + io;
#ifndef CHR_BAND_NOWAIT
    if (c > 0 && tid == 0)
        wait_flag(tflag + tile - nb, 2);
#endif
    __syncthreads();
    BAND_TR(5);
    constexpr int FU = 4;  // columns per thread per round: all face loads first
    const int tpub = need_i ? 0 : (need_fy ? L - ex : L);  // columns whose faces are read
    for (int t0 = tpub + tid; t0 < L; t0 += KBT * FU) {
        int64_t fzv[FU];
#pragma unroll
        for (int k = 0; k < FU; ++k) {
            const int t = t0 + KBT * k;
            fzv[k] = (c > 0 && t < L) ? __ldcg(Ip + t) : 0;
        }
#pragma unroll
        for (int k = 0; k < FU; ++k) {
            const int t = t0 + KBT * k;
            if (t < L) publish_col(t, fzv[k]);
        }
    }
    if (need_fy || need_i) release(2);  // (no successor waits on a tile that publishes nothing)
    BAND_TR(6);
    if (!mask) {
        for (int t = tid; t < L; t += KBT) recon_col(t, c > 0 ? __ldcg(Ip + t) : 0);
    } else {
        // the same reconstruction in warp-uniform 32-column steps, each plane's
        // inside bits (v >= iso) ballot-packed into the mask (plane-linear bit
        // y * ex + x; words shared with the band above/below are ORed)
        uint32_t *mp = mask + R.mask_off;
        const int64_t bit0 = (int64_t)y0 * ex;
        for (int t0 = warp * 32; t0 < L; t0 += KBT) {
            const int t = t0 + lane;
            const bool act = t < L;
            int xx = 0, qi = 0;
            int64_t fz = 0;
            if (act) {
                qi = qidx(t, xx);
                fz = c > 0 ? __ldcg(Ip + t) : 0;
            }
            const int64_t wb = bit0 + t0;
            const int sh = (int)(wb & 31);
            const int64_t pw = R.pw;
            uint32_t *w = mp + (wb >> 5) + (int64_t)z0 * pw;
            // inactive lanes read valid shared words (index 0) and store nothing
            const QV *qp = Q + qi;
            const int64_t *dp = dF + xx;
            double *op = obase + t;
            int64_t acc = fz;  // z prefix
            if (nb == 1) {  // one band (most windows): no band above, this warp owns its mask words
                for (int j = 0; j < nzv; ++j, w += pw, qp += PL, op += zstride) {
                    acc += *qp;
                    const double v = (double)acc * twoe;
                    if (act) __stcs(op, v);
                    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, act && v >= iso);
                    if (lane == 0) *w = bal;
                }
                continue;
            }
            const int dstep = b > 0 ? ex : 0;
            if (b == 0) dp = &s_zero;
            for (int j = 0; j < nzv; ++j, w += pw, qp += PL, dp += dstep, op += zstride) {
                acc += *qp;
                const double v = (double)(acc + *dp) * twoe;
                if (act) __stcs(op, v);
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, act && v >= iso);
                if (lane == 0) {
                    if (nb == 1) {  // whole planes: this warp owns the word
                        *w = bal;
                    } else if (bal) {  // band edges share words with the band above / below
                        atomicOr(w, bal << sh);
                        if (sh && (bal >> (32 - sh))) atomicOr(w + 1, bal >> (32 - sh));
                    }
                }
            }
        }
    }
    BAND_TR(7);
    // ---- codec 2: escaped samples keep their f64 value (raster order rank)
    if (R.codec == 2 && R.nesc > 0) {
        __syncthreads();
        const uint8_t *bm = blob + R.poff;
        const uint8_t *ev = bm + ((R.n + 7) >> 3);
        const uint32_t lt = (1u << lane) - 1u;
        for (int j = warp; j < nzv; j += KBW) {
            int64_t rank = esc_sp[R.sp_base + (int64_t)(z0 + j) * nb + b];
            const int64_t s0 = ((int64_t)(z0 + j) * ey + y0) * ex;
            for (int p0 = 0; p0 < L; p0 += 32) {
                const int p = p0 + lane;
                const int64_t s = s0 + p;
                const bool bit = p < L && ((bm[s >> 3] >> (s & 7)) & 1);
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, bit);
                if (bit) {
                    const uint8_t *src = ev + 8 * (rank + __popc(bal & lt));
                    uint64_t bits = 0;
                    for (int k = 0; k < 8; ++k) bits |= (uint64_t)src[k] << (8 * k);
                    const double v = __longlong_as_double((long long)bits);
                    obase[j * zstride + p] = v;
                    if (mask) {  // the escaped value decides its inside bit
                        const int64_t pb = (int64_t)y0 * ex + p;
                        uint32_t *w = mask + R.mask_off + (int64_t)(z0 + j) * R.pw + (pb >> 5);
                        if (v >= iso) atomicOr(w, 1u << (pb & 31));
                        else atomicAnd(w, ~(1u << (pb & 31)));
                    }
                }
                rank += __popc(bal);
            }
        }
    }
}

// regions with a tile whose sum |q| reached 2^31 (its int32 prefixes may
// have wrapped): k_band<int64_t> decodes them again, overwriting the output
__global__ void k_asum_check(const DecReg *__restrict__ regs, int64_t nreg,
                             const unsigned long long *__restrict__ asum, int32_t *__restrict__ any_redo) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nreg) return;
    const DecReg &R = regs[r];
    if ((R.codec == 1 || R.codec == 2) && !R.slow && R.err == 0 && asum[r] >= (1ull << 31)) *any_redo = 1;
}

// inside-mask words of the regions the int64 pass redoes (its band edges OR
// into words the int32 pass already wrote)
__global__ void k_mask_clear(const DecReg *__restrict__ regs, int64_t nreg, const unsigned long long *__restrict__ asum,
                             uint32_t *__restrict__ mask) {
    for (int64_t r = blockIdx.y; r < nreg; r += gridDim.y) {
        if (asum[r] < (1ull << 31)) continue;
        const DecReg &R = regs[r];
        const int64_t nw = (int64_t)R.pw * R.ez;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += (int64_t)gridDim.x * blockDim.x)
            mask[R.mask_off + i] = 0;
    }
}

// inside masks of the regions k_band did not reconstruct (verbatim codecs,
// generic path), from their f64 windows: warp per 32-bit word
__global__ void __launch_bounds__(256) k_mask_rest(const DecReg *__restrict__ regs, int64_t r0,
                                                   const double *__restrict__ out, uint32_t *__restrict__ mask,
                                                   double iso) {
    const DecReg &R = regs[r0 + blockIdx.y];
    const bool band = (R.codec == 1 || R.codec == 2) && !R.slow;
    if (band || R.err) return;
    const int lane = threadIdx.x & 31;
    const int64_t plane = (int64_t)R.ex * R.ey, words = (int64_t)R.pw * R.ez;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < words;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t z = w / R.pw, t = (w - z * R.pw) * 32 + lane;
        const bool in = t < plane && out[R.out_off + z * plane + t] >= iso;
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, in);
        if (lane == 0) mask[R.mask_off + w] = bal;
    }
}

// ------------------------------------------------------------------ host
struct DecPlan {
    std::vector<DecReg> regs;
    int64_t nchunks = 0, nseg = 0, nitems = 0, ncarry = 0, ntiles = 0, nsp = 0, nface = 0, nmask = 0;
    int max_rows_ex = 0;
    size_t ws = 0;
    DecReg *d_regs;
    CrcSeg *segs;
    uint32_t *seg_raw;
    int32_t *crc_bad;
    int64_t *chunk_samples, *seg_byte, *seg_skip, *esc_base, *carry, *flags;
    int64_t *sp_byte, *sp_skip, *esc_sp, *thr_cnt, *pos64;
    int64_t *faces;
    unsigned long long *asum;  // per region: max tile sum |q| >= 2^31 (else 0)
    int32_t *tflag, *chunk_reg, *tile_reg, *order;
    int64_t ndiag = 0;
    // host-built [chunk -> region | tile -> region | tile order], uploaded with
    // the region records (built once per region table, shared by the cache)
    std::shared_ptr<const std::vector<int32_t>> hmaps;
    int32_t *maps;
    unsigned long long *ticket, *ticket3;
    int32_t *any_slow;
    bool host_slow = false;  // some region needs the generic path whatever the stream
};

static int dec_rows_for(int ex) {
    // q tile + u(z-1) tile (int64) must fit next to the byte window
    const int64_t budget = 180 * 1024 - DWIN;
    int rows = (int)std::min<int64_t>(8, budget / (16ll * ex));
    return rows < 1 ? 0 : rows;
}

// band tile shape of a region: rows padded to an odd smem stride; whole
// planes per tile when they fit, otherwise bands x chunks balanced so the
// wavefront (bands + chunks) stays short
static bool band_shape(DecReg &R) {
    const int rs = R.ex | 1;
    const int64_t rowb = 4ll * rs;  // int32 bytes per tile row
    if (rowb > SMB) return false;
    const int64_t K = SMB / rowb;   // rows (y * z) per tile when no dF is needed
    int bty = 0, btz = 0;
    if ((int64_t)R.ey * R.ez <= K && R.ez <= BSEGM) {
        bty = R.ey;
        btz = R.ez;
    } else {
        // the tiles of a region form a (band, chunk) grid whose dependency
        // chains are tny + tnz - 1 hops long (band above, chunk before): pick
        // the shape with the shortest chain, then the fewest tiles
        int64_t best_chain = INT64_MAX, best_tiles = INT64_MAX;
        for (int tz = 1; tz <= (int)std::min<int64_t>({(int64_t)R.ez, K, (int64_t)BSEGM}); ++tz) {  // chunk depth
            int64_t ty2 = std::min<int64_t>(R.ey, K / tz);  // widest band for it
            if (ty2 < R.ey) {  // bands below exist: their dF (tz x ex int64) shares the budget
                ty2 = std::min<int64_t>(R.ey, (SMB - 8ll * tz * R.ex) / (rowb * tz));
                if (ty2 < 1) continue;
            }
            const int64_t ny = ceil_div(R.ey, ty2), nz = ceil_div(R.ez, tz);
            const int64_t chain = ny + nz - 1, tiles = ny * nz;
            if (chain < best_chain || (chain == best_chain && tiles < best_tiles)) {
                best_chain = chain;
                best_tiles = tiles;
                bty = (int)ty2;
                btz = tz;
            }
        }
        if (bty < 1) return false;
        // the same grid with balanced bands and chunks (33 + 32 rows, not 40 + 25)
        bty = (int)ceil_div(R.ey, ceil_div(R.ey, bty));
        btz = (int)ceil_div(R.ez, ceil_div(R.ez, btz));
    }
    R.rs = rs;
    R.bty = bty;
    R.btz = btz;
    R.tnx = 1;
    R.tny = (int32_t)ceil_div(R.ey, bty);
    R.tnz = (int32_t)ceil_div(R.ez, btz);
    R.face_n = (int64_t)R.ex * (btz + 1 + bty);
    return true;
}

static bool dec_build(const chr_dec_region_t *h, int64_t n, uintptr_t blob, DecPlan &pl) {
    pl.regs.resize(n);
    int64_t chunk = 0, seg = 0, item = 0, carry = 0, tile = 0, sp = 0, face = 0;
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
        R.pw = (int32_t)ceil_div((int64_t)R.ex * R.ey, 32);
        R.mask_off = pl.nmask;
        pl.nmask += (int64_t)R.pw * R.ez;
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
        R.tile_base = tile;
        R.sp_base = sp;
        R.face_base = face;
        if (R.codec == 1 || R.codec == 2) {
            R.nseg = (int64_t)R.nyt * R.ez;
            seg += R.nseg;
            item += R.nyt;
            carry += (int64_t)R.nyt * R.ez * R.ex;
            pl.max_rows_ex = std::max(pl.max_rows_ex, R.rows * R.ex);
            if (!band_shape(R)) {
                R.slow = 1;  // rows wider than a band tile: generic path
                pl.host_slow = true;
            } else {
                R.ntiles = (int64_t)R.tny * R.tnz;
                tile += R.ntiles;
                sp += (int64_t)R.ez * R.tny;
                face += R.ntiles * R.face_n;
            }
        }
    }
    pl.nchunks = chunk;
    pl.nseg = seg;
    pl.nitems = item;
    pl.ncarry = carry;
    pl.ntiles = tile;
    pl.nsp = sp;
    pl.nface = face;
    // tiles per (step, region) -> exclusive bases in step-major order
    int64_t D = 0;
    for (const DecReg &R : pl.regs)
        if (R.ntiles) D = std::max<int64_t>(D, (int64_t)R.tny + R.tnz - 2);
    pl.ndiag = pl.ntiles ? D + 1 : 0;
    for (int64_t i = 0; i < n; ++i) {
        DecReg &R = pl.regs[i];
        if (R.ntiles) R.doff = (int32_t)(D - (R.tny + R.tnz - 2));
    }
    // chunk / tile -> region maps and the critical-path tile order (step d of
    // a region's wavefront = band + chunk + doff; every region ends on the last
    // step; a tile's two predecessors lie on step d - 1, so taking tiles in
    // this order from a ticket cannot deadlock)
    auto m = std::make_shared<std::vector<int32_t>>((size_t)(pl.nchunks + 2 * pl.ntiles + 3), 0);
    int32_t *creg = m->data(), *treg = creg + pl.nchunks + 1, *ord = treg + pl.ntiles + 1;
    for (int64_t r = 0; r < n; ++r) {
        const DecReg &R = pl.regs[r];
        for (int64_t i = 0; i < R.nchunks; ++i) creg[R.chunk_base + i] = (int32_t)r;
        for (int64_t i = 0; i < R.ntiles; ++i) treg[R.tile_base + i] = (int32_t)r;
    }
    int64_t k = 0;
    for (int64_t d = 0; d < pl.ndiag; ++d)
        for (int64_t r = 0; r < n; ++r) {
            const DecReg &R = pl.regs[r];
            if (!R.ntiles) continue;
            const int64_t dl = d - R.doff;
            if (dl < 0) continue;
            for (int64_t tz = std::max<int64_t>(0, dl - (R.tny - 1)); tz <= std::min<int64_t>(R.tnz - 1, dl); ++tz)
                ord[k++] = (int32_t)(R.tile_base + tz * R.tny + (dl - tz));
        }
    if (k != pl.ntiles) return false;
    pl.hmaps = m;
    return true;
}

// The host plan of the last table this thread built (chr_decode_workspace_size
// is normally followed by the decode of the same table): reused when the
// table bytes and the blob's 16-byte alignment match.
struct DecPlanCache {
    std::vector<chr_dec_region_t> key;
    uintptr_t align = ~uintptr_t(0);
    bool ok = false;
    DecPlan plan;
};

static bool dec_build_cached(const chr_dec_region_t *h, int64_t n, uintptr_t blob, DecPlan &pl) {
    thread_local DecPlanCache C;
    const uintptr_t al = blob & 15;
    if (C.align == al && (int64_t)C.key.size() == n && std::memcmp(C.key.data(), h, sizeof(*h) * n) == 0) {
        if (!C.ok) return false;
        pl = C.plan;
        return true;
    }
    C.key.assign(h, h + n);
    C.align = al;
    C.plan = DecPlan();
    C.ok = dec_build(h, n, al, C.plan);  // offsets are relative to the blob: only the alignment matters
    if (C.ok) pl = C.plan;
    return C.ok;
}

static void dec_carve(DecPlan &pl, void *base, size_t cap) {
    WsCarver c{reinterpret_cast<char *>(base), 0, cap};
    const int64_t n = (int64_t)pl.regs.size();
    pl.d_regs = c.take<DecReg>(n);
    pl.segs = c.take<CrcSeg>(n);
    pl.seg_raw = c.take<uint32_t>(2 * n);  // + crc_bad (one zero range)
    pl.crc_bad = base ? reinterpret_cast<int32_t *>(pl.seg_raw + n) : nullptr;
    pl.chunk_samples = c.take<int64_t>(pl.nchunks);
    pl.seg_byte = c.take<int64_t>(pl.nseg + 1);
    pl.seg_skip = c.take<int64_t>(pl.nseg + 1);
    pl.esc_base = c.take<int64_t>(pl.nseg + 1);
    pl.carry = c.take<int64_t>(pl.ncarry + 1);
    pl.flags = c.take<int64_t>(pl.nitems + 1);
    pl.sp_byte = c.take<int64_t>(pl.nsp + 1);
    pl.sp_skip = c.take<int64_t>(pl.nsp + 1);
    pl.esc_sp = c.take<int64_t>(pl.nsp + 1);
    pl.thr_cnt = c.take<int64_t>(pl.nchunks * DTHREADS + 1);
    pl.pos64 = c.take<int64_t>(pl.nchunks * DTHREADS + 1);
    pl.faces = c.take<int64_t>(pl.nface + 1);
    pl.asum = c.take<unsigned long long>(pl.regs.size() + 1);
    pl.tflag = c.take<int32_t>(pl.ntiles + 1);
    pl.maps = c.take<int32_t>(pl.nchunks + 2 * pl.ntiles + 3);  // layout of hmaps
    pl.chunk_reg = pl.maps;
    pl.tile_reg = base ? pl.maps + pl.nchunks + 1 : nullptr;
    pl.order = base ? pl.tile_reg + pl.ntiles + 1 : nullptr;
    pl.ticket = c.take<unsigned long long>(1);
    pl.ticket3 = c.take<unsigned long long>(1);
    pl.any_slow = c.take<int32_t>(2);  // [0] generic path needed, [1] int64 band pass needed
    pl.ws = ((c.off + 255) & ~size_t(255)) + 256;
}

}  // namespace chr

using namespace chr;

extern "C" size_t chr_decode_workspace_size(const chr_dec_region_t *h, int64_t n) {
    CHR_XFER_SCOPE;
    DecPlan pl;
    if (!h || n < 1 || !dec_build_cached(h, n, 0, pl)) return 256;
    dec_carve(pl, nullptr, ~size_t(0));
    return pl.ws;
}

static int decode_impl(const uint8_t *d_blob, const chr_dec_region_t *h, int64_t n, double *d_out, void *d_ws,
                       size_t ws_bytes, int32_t *h_status, double iso, uint32_t *d_mask, void *stream,
                       int crc_hdr = 0);

extern "C" int chr_decode_regions(const uint8_t *d_blob, const chr_dec_region_t *h, int64_t n,
                                  double *d_out, void *d_ws, size_t ws_bytes, int32_t *h_status,
                                  void *stream) {
    CHR_XFER_SCOPE;
    return decode_impl(d_blob, h, n, d_out, d_ws, ws_bytes, h_status, 0.0, nullptr, stream);
}

extern "C" uint64_t chr_mask_words(const int32_t *h_dims, int64_t n) {
    CHR_XFER_SCOPE;
    uint64_t w = 0;
    for (int64_t i = 0; i < n; ++i)
        w += (uint64_t)ceil_div((int64_t)h_dims[3 * i] * h_dims[3 * i + 1], 32) * (uint64_t)h_dims[3 * i + 2];
    return w;
}

extern "C" int chr_decode_regions_mask(const uint8_t *d_blob, const chr_dec_region_t *h, int64_t n, double *d_out,
                                       void *d_ws, size_t ws_bytes, int32_t *h_status, double iso,
                                       uint32_t *d_mask, void *stream) {
    CHR_XFER_SCOPE;
    if (!d_mask) return CHR_E_PARAMETER;
    return decode_impl(d_blob, h, n, d_out, d_ws, ws_bytes, h_status, iso, d_mask, stream);
}

namespace chr {
int decode_mask_hdrcrc(const uint8_t *d_blob, const chr_dec_region_t *h, int64_t n, double *d_out, void *d_ws,
                       size_t ws_bytes, int32_t *h_status, double iso, uint32_t *d_mask, cudaStream_t st) {
    return decode_impl(d_blob, h, n, d_out, d_ws, ws_bytes, h_status, iso, d_mask, st, 1);
}
}  // namespace chr

static int decode_impl(const uint8_t *d_blob, const chr_dec_region_t *h, int64_t n, double *d_out, void *d_ws,
                       size_t ws_bytes, int32_t *h_status, double iso, uint32_t *d_mask, void *stream,
                       int crc_hdr) {
    if (n == 0) return CHR_OK;
    if (!d_blob || !h || n < 0 || !d_out) return CHR_E_PARAMETER;
    cudaStream_t st = (cudaStream_t)stream;
    DecPlan pl;
    if (!dec_build_cached(h, n, (uintptr_t)d_blob, pl)) return CHR_E_PARAMETER;
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
    CHR_CUDA_TRY(h2d_multi({{pl.d_regs, pl.regs.data(), sizeof(DecReg) * n},
                            {pl.segs, segs.data(), sizeof(CrcSeg) * n},
                            {pl.maps, pl.hmaps->data(), sizeof(int32_t) * pl.hmaps->size()}},
                           st));
    CHR_CUDA_TRY(zero_async({{pl.seg_raw, 2 * sizeof(uint32_t) * n},  // + crc_bad
                             {pl.flags, sizeof(int64_t) * (pl.nitems + 1)},
                             {pl.ticket, sizeof(unsigned long long)},
                             {pl.ticket3, sizeof(unsigned long long)},
                             {pl.any_slow, 2 * sizeof(int32_t)},
                             {pl.asum, sizeof(unsigned long long) * (size_t)(n + 1)},
                             {d_mask, d_mask ? sizeof(uint32_t) * (pl.nmask + 8) : 0},
                             {pl.tflag, sizeof(int32_t) * (pl.ntiles + 1)}},
                            st));
    {
        CHR_PROF("k_check", st);
        k_check<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(pl.d_regs, n);
    }
    // payload CRCs: on the side stream (overlapping the decode), joined
    // before the status read-back
    Side *side = side_stream();
    cudaStream_t ct = st;
    if (side) {
        CHR_CUDA_TRY(cudaEventRecord(side->ev[2], st));
        CHR_CUDA_TRY(cudaStreamWaitEvent(side->st, side->ev[2], 0));
        ct = side->st;
    }
    static const int crc_ctas = [] {  // side-stream CRC grid (it shares the SMs with the tokenizer passes)
        const char *e = std::getenv("CHR_CRC_CTAS");
        return e ? std::atoi(e) : 148 * 4;
    }();
    int rc = crc_launch(d_blob, pl.segs, n, total_sc, pl.seg_raw, ct, side ? crc_ctas : 0);
    if (rc) return rc;
    {
        CHR_PROF("k_crc_flag", ct);
        k_crc_flag<<<(unsigned)ceil_div(n, 128), 128, 0, ct>>>(pl.d_regs, n, pl.seg_raw, tabs, d_blob, crc_hdr,
                                                               pl.crc_bad);
    }
    CHR_CUDA_TRY(cudaGetLastError());
    if (side) CHR_CUDA_TRY(cudaEventRecord(side->ev[3], side->st));
    {
        CHR_PROF("k_esc_count", st);
        k_esc_count<<<(unsigned)n, 256, 0, st>>>(pl.d_regs, n, d_blob);
    }
    {
        CHR_PROF("k_tok_fast", st);
        k_tok_fast<<<(unsigned)pl.nchunks, DTHREADS, 0, st>>>(pl.d_regs, pl.chunk_reg, d_blob, pl.chunk_samples,
                                                              pl.thr_cnt, pl.any_slow);
    }
    {
        CHR_PROF("k_tok_scan", st);
        k_tok_scan<<<(unsigned)n, 512, 0, st>>>(pl.d_regs, n, pl.chunk_samples, 0);
    }
    // ---- band path (canonical streams)
    if (pl.ntiles > 0) {
        {
            CHR_PROF("k_seg_locate", st);
            k_seg_locate<<<(unsigned)pl.nchunks, DTHREADS, 0, st>>>(pl.d_regs, pl.chunk_reg, d_blob,
                                                                    pl.chunk_samples, pl.thr_cnt, pl.sp_byte,
                                                                    pl.sp_skip, pl.pos64);
        }
        {
            CHR_PROF("k_esc_seg", st);
            k_esc_seg<<<(unsigned)n, 256, 0, st>>>(pl.d_regs, d_blob, pl.esc_sp);
        }
        const int smem = (int)SMB;
        CHR_CUDA_TRY(cudaFuncSetAttribute(k_band<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
#ifdef CHR_BAND_TRACE
        unsigned long long *d_tr = nullptr;
        const char *trf = std::getenv("CHR_BAND_TRACE_FILE");
        if (trf) {
            CHR_CUDA_TRY(cudaMalloc(&d_tr, sizeof(unsigned long long) * 8 * (size_t)pl.ntiles));
            CHR_CUDA_TRY(cudaMemcpyToSymbol(g_band_trace, &d_tr, sizeof(d_tr)));
        }
#endif
        {
            CHR_PROF("k_band", st);
            k_band<int32_t><<<(unsigned)pl.ntiles, KBT, smem, st>>>(
                pl.d_regs, pl.tile_reg, d_blob, pl.sp_byte, pl.sp_skip, pl.esc_sp, pl.pos64, pl.faces, pl.tflag,
                pl.ticket3, pl.order, d_out, d_mask, iso, pl.asum);
        }
#ifdef CHR_BAND_TRACE
        if (d_tr) {
            std::vector<unsigned long long> h((size_t)8 * pl.ntiles);
            CHR_CUDA_TRY(cudaStreamSynchronize(st));
            CHR_CUDA_TRY(cudaMemcpy(h.data(), d_tr, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
            unsigned long long *z = nullptr;
            CHR_CUDA_TRY(cudaMemcpyToSymbol(g_band_trace, &z, sizeof(z)));
            cudaFree(d_tr);
            if (FILE *f = std::fopen(trf, "wb")) {
                std::fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
                std::fclose(f);
            }
        }
#endif
        {
            CHR_PROF("k_asum_check", st);
            k_asum_check<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(pl.d_regs, n, pl.asum, pl.any_slow + 1);
        }
    }
    // ---- generic path (non-canonical streams, rows wider than a band tile)
    //      and the int64 band pass: skipped unless some region needs them
    //      (one 8-byte read-back)
    int32_t h_flags[2] = {0, 0};
    CHR_CUDA_TRY(d2h(h_flags, pl.any_slow, sizeof(h_flags), st));
    CHR_CUDA_TRY(stream_sync(st));
    if (h_flags[1] && pl.ntiles > 0) {  // int64 tiles for the regions an int32 tile could not hold
        CHR_CUDA_TRY(zero_async({{pl.tflag, sizeof(int32_t) * (pl.ntiles + 1)}, {pl.ticket3, sizeof(unsigned long long)}},
                                st));
        if (d_mask) {
            CHR_PROF("k_mask_clear", st);
            k_mask_clear<<<dim3(16, (unsigned)std::min<int64_t>(n, 1024)), 256, 0, st>>>(pl.d_regs, n, pl.asum, d_mask);
        }
        const int smem = (int)(2 * SMB);  // int64 tile + dF
        CHR_CUDA_TRY(cudaFuncSetAttribute(k_band<int64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        CHR_PROF("k_band64", st);
        k_band<int64_t><<<(unsigned)pl.ntiles, KBT, smem, st>>>(
            pl.d_regs, pl.tile_reg, d_blob, pl.sp_byte, pl.sp_skip, pl.esc_sp, pl.pos64, pl.faces, pl.tflag,
            pl.ticket3, pl.order, d_out, d_mask, iso, pl.asum);
    }
    if (pl.host_slow || h_flags[0]) {
        {
            CHR_PROF("k_tok_count", st);
            k_tok_count<<<(unsigned)pl.nchunks, DTHREADS, 0, st>>>(pl.d_regs, n, d_blob, pl.chunk_samples);
        }
        {
            CHR_PROF("k_tok_scan", st);
            k_tok_scan<<<(unsigned)n, 512, 0, st>>>(pl.d_regs, n, pl.chunk_samples, 1);
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
    }
    for (int64_t r0 = 0; r0 < n; r0 += 65535) {
        dim3 g(64, (unsigned)std::min<int64_t>(65535, n - r0));
        {
            CHR_PROF("k_verbatim", st);
            k_verbatim<<<g, 256, 0, st>>>(pl.d_regs, r0, d_blob, d_out);
        }
    }
    if (d_mask)  // regions k_band did not reconstruct
        for (int64_t r0 = 0; r0 < n; r0 += 65535) {
            dim3 g(16, (unsigned)std::min<int64_t>(65535, n - r0));
            CHR_PROF("k_mask_rest", st);
            k_mask_rest<<<g, 256, 0, st>>>(pl.d_regs, r0, d_out, d_mask, iso);
        }
    CHR_CUDA_TRY(cudaGetLastError());
    if (side) CHR_CUDA_TRY(cudaStreamWaitEvent(st, side->ev[3], 0));
    std::vector<int32_t> crc_bad((size_t)n);
    CHR_CUDA_TRY(d2h_multi({{pl.regs.data(), pl.d_regs, sizeof(DecReg) * n},
                            {crc_bad.data(), pl.crc_bad, sizeof(int32_t) * n}}, st));
    CHR_CUDA_TRY(stream_sync(st));
    int status = CHR_OK;
    for (int64_t i = 0; i < n; ++i) {
        const uint32_t err = pl.regs[i].err | (crc_bad[i] ? (uint32_t)EF_CRC : 0u);
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
