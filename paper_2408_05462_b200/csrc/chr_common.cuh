// chr_common.cuh -- shared device/host helpers for libchr (sm_100a).
//
// * CRC-32/IEEE algebra (zlib.crc32 semantics, codec.py:132) expressed as
//   GF(2) linear maps so a payload can be checksummed by many threads and
//   recombined: raw(A||B) = S(raw(A), |B|) ^ raw(B), with S(c, n) the
//   multiplication by x^(8n) mod P.
// * the token-size monoid of the zigzag/LEB128/zero-run stream
//   (kernels.py:198-234): lets every 64-sample row piece be summarised
//   independently and scanned into exact byte offsets.
// * the quantiser of kernels.py:58-74 (ties-to-odd via the 1.5*2^52
//   shift, escape test), with a proven branch-free fast path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/chr.h"

#if defined(__CUDA_ARCH__)
#define CHR_HD __host__ __device__ __forceinline__
#else
#define CHR_HD inline
#endif

#define CHR_CUDA_TRY(expr)                                   \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) return CHR_E_CUDA;            \
    } while (0)

namespace chr {

constexpr uint32_t kCrcPoly = 0xEDB88320u;  // reflected CRC-32/IEEE
constexpr int kBlockHeader = 34;             // codec.py:41  "<B3IdBQI"
constexpr int kFileHeader = 63;              // chr_archive.py:50
constexpr int kRegionFixed = 85;             // chr_archive.py:51

// ---------------------------------------------------------------- bits
CHR_HD int clz64(uint64_t v) {
#if defined(__CUDA_ARCH__)
    return __clzll((long long)v);
#else
    return v ? __builtin_clzll(v) : 64;
#endif
}

// bytes of the LEB128 encoding of u (the encoder's `while u >= 0x80` loop)
CHR_HD int varint_len(uint64_t u) {
    const int bits = 64 - clz64(u | 1);
    return (bits + 6) / 7;
}

// bytes of the token(s) encoding a zero run of length L (kernels.py:205-218):
// nothing for L == 0, literal 0x01 for L == 1, else 0x00 + LEB128(L)
CHR_HD int64_t run_bytes(int64_t L) {
    return L <= 0 ? 0 : (L == 1 ? 1 : 1 + varint_len((uint64_t)L));
}

CHR_HD uint64_t zigzag1(int64_t v) {  // zigzag(v) + 1
    return (((uint64_t)v << 1) ^ (uint64_t)(v >> 63)) + 1;
}

// ---------------------------------------------------------------- CRC
// multiplication of two reflected polynomials mod P (zlib multmodp)
CHR_HD uint32_t gf2_mul(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
    // branch-free on the device (lanes of a warp never diverge on the bits)
    uint32_t p = 0;
#pragma unroll
    for (int i = 31; i >= 0; --i) {
        p ^= b & (0u - ((a >> i) & 1u));
        b = (b >> 1) ^ (kCrcPoly & (0u - (b & 1u)));
    }
    return p;
#else
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ kCrcPoly : b >> 1;
    }
    return p;
#endif
}

// x^(2^k) mod P for k = 0..63 (zlib x2n_table); filled by crc_tables_init
struct CrcTables {
    uint32_t x2n[64];
    uint32_t t[4][256];      // slice-by-4: F(v) = v * x^32 mod P, per byte lane
    uint32_t g[4][256];      // G(v) = v * x^1024 mod P, per byte lane
    uint32_t xw[33];         // x^(32 k) mod P, k = 0..32 (word shifts)
};

// x^(8 n) mod P using the x2n table (zlib x2nmodp(n, 3))
CHR_HD uint32_t x8n(const uint32_t *x2n, uint64_t n) {
    uint32_t p = 1u << 31;  // x^0
    int k = 3;
    while (n) {
        if (n & 1) p = gf2_mul(x2n[k & 63], p);
        n >>= 1;
        ++k;
    }
    return p;
}

// S(c, n): shift a raw CRC across n further (zero-contribution) bytes
CHR_HD uint32_t crc_shift(const uint32_t *x2n, uint32_t c, uint64_t n) {
    return n ? gf2_mul(x8n(x2n, n), c) : c;
}

// raw CRC (init 0, no final xor) continued over bytes
CHR_HD uint32_t crc_raw_bytes(const uint32_t *t0, uint32_t c, const uint8_t *p, int64_t n) {
    for (int64_t i = 0; i < n; ++i) c = t0[(c ^ p[i]) & 0xFF] ^ (c >> 8);
    return c;
}

// finalised zlib crc32 from the raw CRC of n bytes
CHR_HD uint32_t crc_finalize(const uint32_t *x2n, uint32_t raw, uint64_t n) {
    return crc_shift(x2n, 0xFFFFFFFFu, n) ^ raw ^ 0xFFFFFFFFu;
}

void crc_tables_host(CrcTables *t);           // builds all tables on the host
const CrcTables *crc_tables_device();         // device copy (initialised once)
const CrcTables &crc_tables_hostref();

// ---------------------------------------------------------------- monoid
// Summary of a contiguous piece of one region's quantum stream, enough to
// place every token byte (kernels.py:198-234).  The run preceding the
// first literal and the run after the last are left open (lead / trail)
// so pieces compose associatively:
//   A.B: bytes = A.bytes + B.bytes + run_bytes(A.trail + B.lead)  (both nz)
struct TokSeg {
    int64_t len;    // samples
    int64_t lead;   // zeros before the first nonzero (== len if none)
    int64_t trail;  // zeros after the last nonzero (== len if none)
    int64_t bytes;  // literal tokens + runs between literals
    int64_t nesc;   // escaped samples
    int32_t nz;     // piece holds a nonzero quantum
    int32_t f32ok;  // every sample is exactly representable in f32
};

CHR_HD TokSeg tokseg_identity() {
    TokSeg s;
    s.len = s.lead = s.trail = s.bytes = s.nesc = 0;
    s.nz = 0;
    s.f32ok = 1;
    return s;
}

CHR_HD TokSeg tokseg_combine(const TokSeg &a, const TokSeg &b) {
    TokSeg r;
    r.len = a.len + b.len;
    r.nesc = a.nesc + b.nesc;
    r.f32ok = a.f32ok & b.f32ok;
    if (!a.nz) {
        r.nz = b.nz;
        r.lead = a.len + b.lead;
        r.trail = b.nz ? b.trail : r.len;
        r.bytes = b.bytes;
    } else if (!b.nz) {
        r.nz = 1;
        r.lead = a.lead;
        r.trail = a.trail + b.len;
        r.bytes = a.bytes;
    } else {
        r.nz = 1;
        r.lead = a.lead;
        r.trail = b.trail;
        r.bytes = a.bytes + b.bytes + run_bytes(a.trail + b.lead);
    }
    return r;
}

// total token bytes of a complete stream with summary s
CHR_HD int64_t tokseg_stream_bytes(const TokSeg &s) {
    return s.nz ? s.bytes + run_bytes(s.lead) + run_bytes(s.trail) : run_bytes(s.len);
}

// 8-byte per-row-piece record written by the count pass (64 samples)
struct PieceRec {
    uint16_t bytes;   // literal + internal run bytes (<= 64*5)
    uint8_t lead, trail, nesc, vcount, flags, pad;  // flags: 1 = nz, 2 = not f32-exact
};

CHR_HD TokSeg piece_to_seg(const PieceRec &p) {
    TokSeg s;
    s.len = p.vcount;
    s.lead = p.lead;
    s.trail = p.trail;
    s.bytes = p.bytes;
    s.nesc = p.nesc;
    s.nz = p.flags & 1;
    s.f32ok = (p.flags & 2) ? 0 : 1;
    return s;
}

// 16-byte record of a wider stream piece (segment encoder: <= 65535 samples)
struct PieceRec2 {
    uint16_t len, lead, trail, nesc;
    uint32_t bytes;   // literal + internal run bytes
    uint32_t nz;
};

CHR_HD TokSeg piece_to_seg(const PieceRec2 &p) {
    TokSeg s;
    s.len = p.len;
    s.lead = p.lead;
    s.trail = p.trail;
    s.bytes = p.bytes;
    s.nesc = p.nesc;
    s.nz = (int32_t)p.nz;
    s.f32ok = 1;
    return s;
}

// where piece j starts: exclusive-prefix consequences
struct PieceOff {
    int64_t tok_off;  // token bytes owned by earlier pieces of the region
    int64_t carry;    // zeros since the last nonzero (or stream start)
    int64_t esc_off;  // escaped samples before the piece
};

// ---------------------------------------------------------------- quantiser
constexpr double kRoundShift = 6755399441055744.0;  // 1.5 * 2^52, kernels.py:18
constexpr double kEscapeUmax = 134217728.0;         // 2^27,        kernels.py:22
// fast-path margin: |d| < 1/2 - 2^-20 and |qf| < 2^27 prove "not escaped"
// (rounding of qf, uf*2e and the subtraction stays below 2^-24 relative;
// see DESIGN.md "quantiser fast path").  Only valid for e >= 2^-1000.
constexpr double kTieMargin = 0.5 - 9.5367431640625e-07;

struct Quant {
    double e, twoe, inv;
    int fast;  // e >= 2^-1000
};

CHR_HD Quant make_quant(double e) {
    Quant q;
    q.e = e;
    q.twoe = 2.0 * e;
    q.inv = 1.0 / q.twoe;
    q.fast = e >= 9.332636185032189e-302;  // 2^-1000
    return q;
}

#if defined(__CUDACC__)
// kernels.py:58-74 bit-exactly; returns the lattice value u (0 if escaped)
__device__ __forceinline__ int32_t quantize(const Quant &Q, double v, bool &esc) {
    const double qf = __dmul_rn(v, Q.inv);
    const double t = __dadd_rn(qf, kRoundShift);
    double uf = __dadd_rn(t, -kRoundShift);
    const double d = __dadd_rn(qf, -uf);
    if (Q.fast && fabs(qf) < kEscapeUmax && fabs(d) < kTieMargin) {
        esc = false;
        return __double2loint(t);  // uf as two's complement in t's low word
    }
    if (d == 0.5)
        uf = __dadd_rn(uf, 1.0);
    else if (d == -0.5)
        uf = __dadd_rn(uf, -1.0);
    if (fabs(uf) > kEscapeUmax || fabs(__dadd_rn(__dmul_rn(uf, Q.twoe), -v)) > Q.e) {
        esc = true;
        return 0;
    }
    esc = false;
    return (int32_t)(long long)uf;
}
#endif

}  // namespace chr
