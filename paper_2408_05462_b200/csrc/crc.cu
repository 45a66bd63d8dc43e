// crc.cu -- CRC-32/IEEE (zlib.crc32) of many byte segments at HBM speed.
//
// Reference uses: codec.py:132 (payload checksum), codec.py:220-226
// (verification in decompress), chr_archive.py:338 / 351-356 (whole-file
// trailer).  zlib's byte-serial loop is replaced by a lane-interleaved
// word formulation: lane l of a warp owns words l, l+32, l+64, ... of a
// superchunk and keeps B = G(B) ^ w (G = multiply by x^1024 mod P, four
// 256-entry table lookups); the lane's share of the superchunk CRC is then
// B * x^(32 (W - last)) and the superchunk CRC is the XOR over lanes.
// Superchunk CRCs are shifted to the segment end and XOR-accumulated, so
// any number of warps can work on one segment.  Loads are 128-byte
// coalesced 32-bit words.
#include <algorithm>
#include <mutex>
#include <vector>

#include "chr_common.cuh"
#include "chr_internal.cuh"

namespace chr {

static CrcTables g_host_tables;
constexpr int kMaxDevices = 64;
static CrcTables *g_dev_tables[kMaxDevices] = {};  // per CUDA device (cudaGetDevice)
static std::once_flag g_host_once;
static std::mutex g_dev_mu;

void crc_tables_host(CrcTables *t) {
    // byte table (zlib make_crc_table)
    for (uint32_t n = 0; n < 256; ++n) {
        uint32_t c = n;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kCrcPoly : c >> 1;
        t->t[0][n] = c;
    }
    for (uint32_t n = 0; n < 256; ++n)
        for (int k = 1; k < 4; ++k)
            t->t[k][n] = (t->t[k - 1][n] >> 8) ^ t->t[0][t->t[k - 1][n] & 0xFF];
    // x^(2^k) mod P by repeated squaring, starting from x^1 = 0x40000000
    uint32_t p = 1u << 30;
    for (int k = 0; k < 64; ++k) {
        t->x2n[k] = p;
        p = gf2_mul(p, p);
    }
    const uint32_t x1024 = x8n(t->x2n, 128);
    for (int k = 0; k < 4; ++k)
        for (uint32_t n = 0; n < 256; ++n) t->g[k][n] = gf2_mul(x1024, n << (8 * k));
    for (int k = 0; k < 33; ++k) t->xw[k] = x8n(t->x2n, 4ull * k);
}

const CrcTables &crc_tables_hostref() {
    std::call_once(g_host_once, [] { crc_tables_host(&g_host_tables); });
    return g_host_tables;
}

const CrcTables *crc_tables_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (!g_dev_tables[dev]) {
        const CrcTables &h = crc_tables_hostref();
        CrcTables *d = nullptr;
        if (cudaMalloc(&d, sizeof(CrcTables)) != cudaSuccess) return nullptr;
        if (cudaMemcpy(d, &h, sizeof(CrcTables), cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaFree(d);
            return nullptr;
        }
        g_dev_tables[dev] = d;
    }
    return g_dev_tables[dev];
}

// x^(8n) mod P computed by a whole warp (one bit of n per lane, then a
// shuffle product tree); every lane returns the result
// G tables replicated 8x (word idx * 8 + (lane & 7)): random byte indices of
// 32 lanes then spread over all 32 banks (~2-way instead of ~4-way conflicts)
__device__ __forceinline__ uint32_t apply_g(const uint32_t *g, uint32_t v, int r) {
    return g[((v & 0xFF) << 3) + r] ^ g[2048 + (((v >> 8) & 0xFF) << 3) + r] ^
           g[4096 + (((v >> 16) & 0xFF) << 3) + r] ^ g[6144 + ((v >> 24) << 3) + r];
}

constexpr int kCrcSmemSegs = 1024;
#ifndef CHR_CRC_UNROLL
#define CHR_CRC_UNROLL 16
#endif
constexpr int kCrcUnroll = CHR_CRC_UNROLL;
// one warp per superchunk (kCrcScWords words); seg_raw[s] ^= contribution
__global__ void __launch_bounds__(256) k_crc_segments(const uint8_t *__restrict__ buf,
                                                      const CrcSeg *__restrict__ segs, int64_t nseg,
                                                      const CrcTables *__restrict__ tabs,
                                                      uint32_t *__restrict__ seg_raw) {
    __shared__ uint32_t g[4 * 256 * 8];
    __shared__ uint32_t t0[256];
    __shared__ uint32_t x2n[64];
    __shared__ uint32_t xw[33];
    __shared__ int64_t s_scb[kCrcSmemSegs];  // segment first superchunks (when few segments)
    const bool seg_smem = nseg <= kCrcSmemSegs;
    if (seg_smem)
        for (int64_t i = threadIdx.x; i < nseg; i += blockDim.x) s_scb[i] = segs[i].sc_base;
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) g[i] = tabs->g[i >> 11][(i >> 3) & 255];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) t0[i] = tabs->t[0][i];
    if (threadIdx.x < 64) x2n[threadIdx.x] = tabs->x2n[threadIdx.x];
    if (threadIdx.x < 33) xw[threadIdx.x] = tabs->xw[threadIdx.x];
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int64_t total_sc = segs[nseg - 1].sc_base + segs[nseg - 1].n_sc;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t sc = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); sc < total_sc;
         sc += warps) {
        // segment of this superchunk (segments sorted by sc_base)
        int64_t lo = 0, hi = nseg - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if ((seg_smem ? s_scb[mid] : segs[mid].sc_base) <= sc) lo = mid; else hi = mid - 1;
        }
        const CrcSeg S = segs[lo];
        const uint64_t a = S.begin, b = S.end;
        // word alignment on ABSOLUTE addresses (the buffer may be unaligned)
        const uint64_t base = (uint64_t)(uintptr_t)buf;
        const uint64_t a4 = ((base + a + 3) & ~3ull) - base, b4 = ((base + b) & ~3ull) - base;
        const int64_t isc = sc - S.sc_base;
        uint32_t contrib = 0;
        if (a4 < b4) {
            const uint64_t W = (b4 - a4) >> 2;
            const uint64_t w0 = (uint64_t)isc * kCrcScWords;
            const uint64_t w1 = min(W, w0 + kCrcScWords);
            const uint32_t *wp = reinterpret_cast<const uint32_t *>(buf + a4);
            uint32_t B = 0;
            int64_t last = -1;
            uint64_t i = w0 + lane;
            // kCrcUnroll words per lane loaded before any is folded: the fold is a
            // dependent chain of shared lookups, so the loads must be in flight together
            for (; i + 32 * (kCrcUnroll - 1) < w1; i += 32 * kCrcUnroll) {
                uint32_t w[kCrcUnroll];
#pragma unroll
                for (int j = 0; j < kCrcUnroll; ++j) w[j] = __ldg(wp + i + 32 * j);
#pragma unroll
                for (int j = 0; j < kCrcUnroll; ++j) B = apply_g(g, B, lane & 7) ^ w[j];
                last = (int64_t)(i + 32 * (kCrcUnroll - 1) - w0);
            }
            for (; i < w1; i += 32) {
                B = apply_g(g, B, lane & 7) ^ __ldg(wp + i);
                last = (int64_t)(i - w0);
            }
            const int64_t Ws = (int64_t)(w1 - w0);
            uint32_t part = last >= 0 ? gf2_mul(xw[Ws - last], B) : 0;
#pragma unroll
            for (int off = 16; off; off >>= 1) part ^= __shfl_xor_sync(0xFFFFFFFFu, part, off);
            // shift to the segment end
            const uint64_t after = b - (a4 + 4 * w1);
            const uint32_t m = warp_x8n(x2n, after);
            contrib = gf2_mul(m, part);
            if (isc == 0 && lane == 0) {
                uint32_t h = crc_raw_bytes(t0, 0, buf + a, (int64_t)(a4 - a));
                contrib ^= crc_shift(x2n, h, b - a4);
                contrib ^= crc_raw_bytes(t0, 0, buf + b4, (int64_t)(b - b4));
            }
        } else if (lane == 0) {
            contrib = crc_raw_bytes(t0, 0, buf + a, (int64_t)(b - a));
        }
        if (lane == 0 && contrib) atomicXor(seg_raw + lo, contrib);
    }
}

// number of superchunks of a segment and their prefix (host side)
int64_t crc_plan_segments(CrcSeg *segs, int64_t nseg) {
    int64_t base = 0;
    for (int64_t s = 0; s < nseg; ++s) {
        segs[s].sc_base = base;
        segs[s].n_sc = crc_num_superchunks(segs[s].begin, segs[s].end);
        base += segs[s].n_sc;
    }
    return base;
}

int crc_launch(const uint8_t *d_buf, const CrcSeg *d_segs, int64_t nseg, int64_t total_sc,
               uint32_t *d_seg_raw, cudaStream_t st, int64_t max_blocks) {
    const CrcTables *tabs = crc_tables_device();
    if (!tabs) return CHR_E_CUDA;
    if (nseg <= 0) return CHR_OK;
    // total_sc <= 0: unknown on the host (lives on the device) -> persistent grid
    const int64_t warps_needed = total_sc > 0 ? total_sc : 148 * 128;
    int64_t blocks = (warps_needed + 7) / 8;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (max_blocks > 0 && blocks > max_blocks) blocks = max_blocks;
    if (blocks < 1) blocks = 1;
    {
        CHR_PROF("k_crc_segments", st);
        k_crc_segments<<<(unsigned)blocks, 256, 0, st>>>(d_buf, d_segs, nseg, tabs, d_seg_raw);
    }
    return cudaGetLastError() == cudaSuccess ? CHR_OK : CHR_E_CUDA;
}

}  // namespace chr

using namespace chr;

extern "C" size_t chr_crc32_workspace_size(uint64_t) {
    CHR_XFER_SCOPE; return 256; }

extern "C" int chr_crc32(const uint8_t *d_buf, uint64_t n, void *d_ws, size_t ws_bytes,
                         uint32_t *h_crc, void *stream) {
    CHR_XFER_SCOPE;
    if (!h_crc || (!d_buf && n)) return CHR_E_PARAMETER;
    if (ws_bytes < 256 || !d_ws) return CHR_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    const CrcTables &H = crc_tables_hostref();
    if (n == 0) {
        *h_crc = 0;
        return CHR_OK;
    }
    CrcSeg seg;
    seg.begin = 0;
    seg.end = n;
    crc_plan_segments(&seg, 1);
    CrcSeg *d_seg = reinterpret_cast<CrcSeg *>(d_ws);
    uint32_t *d_raw = reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(d_ws) + 128);
    CHR_CUDA_TRY(h2d(d_seg, &seg, sizeof(seg), st));
    CHR_CUDA_TRY(fill_async(d_raw, 0, 4, st));
    int rc = crc_launch(d_buf, d_seg, 1, seg.n_sc, d_raw, st);
    if (rc) return rc;
    uint32_t raw = 0;
    CHR_CUDA_TRY(d2h(&raw, d_raw, 4, st));
    CHR_CUDA_TRY(stream_sync(st));
    *h_crc = crc_finalize(H.x2n, raw, n);
    return CHR_OK;
}

extern "C" size_t chr_crc32_segments_workspace_size(int64_t n) {
    CHR_XFER_SCOPE;
    return n < 1 ? 256 : (size_t)(n + 1) * (sizeof(CrcSeg) + sizeof(uint32_t)) + 512;
}

// CRC-32 of n byte ranges [begin, end) of one device buffer, one launch:
// h_raw (may be NULL) = the raw register (init 0, no final xor; linear, so
// shares of disjoint ranges XOR after shifting), h_crc (may be NULL) =
// zlib.crc32 of each range.  Synchronises.
extern "C" int chr_crc32_segments(const uint8_t *d_buf, const uint64_t *h_ranges, int64_t n, void *d_ws,
                                  size_t ws_bytes, uint32_t *h_raw, uint32_t *h_crc, void *stream) {
    CHR_XFER_SCOPE;
    if (n < 0 || (n && (!h_ranges || !d_buf))) return CHR_E_PARAMETER;
    if (n == 0) return CHR_OK;
    if (!d_ws || ws_bytes < chr_crc32_segments_workspace_size(n)) return CHR_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    const CrcTables &H = crc_tables_hostref();
    std::vector<CrcSeg> segs((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        segs[i].begin = h_ranges[2 * i];
        segs[i].end = std::max(h_ranges[2 * i], h_ranges[2 * i + 1]);
    }
    const int64_t total_sc = crc_plan_segments(segs.data(), n);
    CrcSeg *d_seg = reinterpret_cast<CrcSeg *>(d_ws);
    uint32_t *d_raw = reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(d_ws) +
                                                   ((sizeof(CrcSeg) * (size_t)n + 255) & ~size_t(255)));
    CHR_CUDA_TRY(h2d(d_seg, segs.data(), sizeof(CrcSeg) * (size_t)n, st));
    CHR_CUDA_TRY(fill_async(d_raw, 0, 4 * (size_t)n, st));
    int rc = crc_launch(d_buf, d_seg, n, total_sc, d_raw, st);
    if (rc) return rc;
    std::vector<uint32_t> raw((size_t)n);
    CHR_CUDA_TRY(d2h(raw.data(), d_raw, 4 * (size_t)n, st));
    CHR_CUDA_TRY(stream_sync(st));
    for (int64_t i = 0; i < n; ++i) {
        if (h_raw) h_raw[i] = raw[i];
        if (h_crc) h_crc[i] = segs[i].end > segs[i].begin ? crc_finalize(H.x2n, raw[i], segs[i].end - segs[i].begin) : 0;
    }
    return CHR_OK;
}

// raw register of a range shifted by `len` more bytes (zeros) after it: the
// share of a range inside a longer buffer (chr_crc32_segments' raw values)
extern "C" uint32_t chr_crc32_shift(uint32_t raw, uint64_t len) {
    CHR_XFER_SCOPE;
    return crc_shift(crc_tables_hostref().x2n, raw, len);
}

// h_out[i] = chr_crc32_shift(h_raw[i], h_len[i]) for n values (host)
extern "C" void chr_crc32_shift_many(const uint32_t *h_raw, const uint64_t *h_len, int64_t n, uint32_t *h_out) {
    CHR_XFER_SCOPE;
    const CrcTables &H = crc_tables_hostref();
    for (int64_t i = 0; i < n; ++i) h_out[i] = crc_shift(H.x2n, h_raw[i], h_len[i]);
}

extern "C" uint32_t chr_crc32_combine(uint32_t crc1, uint32_t crc2, uint64_t len2) {
    CHR_XFER_SCOPE;
    const CrcTables &H = crc_tables_hostref();
    return crc_shift(H.x2n, crc1, len2) ^ crc2;
}
