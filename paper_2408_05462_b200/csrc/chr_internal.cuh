// chr_internal.cuh -- declarations shared between libchr translation units.
#pragma once

#include <initializer_list>
#include <utility>

#include "chr_common.cuh"

namespace chr {

// ------------------------------------------------------------------ CRC
constexpr int64_t kCrcScWords = 8192;  // words per superchunk (32 KiB): the per-superchunk lane combine + shift (~1600 instr/lane) amortised over 256 words/lane

struct CrcSeg {
    uint64_t begin, end;  // byte range
    int64_t sc_base;      // first superchunk id
    int64_t n_sc;         // superchunks
};

// superchunks needed for bytes [a, b) whatever the buffer's alignment
// (one spare word covers the alignment slack; empty superchunks add 0)
CHR_HD int64_t crc_num_superchunks(uint64_t a, uint64_t b) {
    const uint64_t Wmax = b > a ? (b - a) / 4 + 1 : 0;
    return Wmax ? (int64_t)((Wmax + kCrcScWords - 1) / kCrcScWords) : 1;
}

int64_t crc_plan_segments(CrcSeg *segs, int64_t nseg);
// max_blocks > 0 caps the grid (a CRC overlapping other kernels on a side stream)
int crc_launch(const uint8_t *d_buf, const CrcSeg *d_segs, int64_t nseg, int64_t total_sc,
               uint32_t *d_seg_raw, cudaStream_t st, int64_t max_blocks = 0);
__global__ void k_crc_segments(const uint8_t *__restrict__ buf, const CrcSeg *__restrict__ segs,
                               int64_t nseg, const CrcTables *__restrict__ tabs,
                               uint32_t *__restrict__ seg_raw);

// ------------------------------------------------------------------ profiling
// RAII: counts a launch; when chr_prof_enable(1), records CUDA events on the
// launching stream around it (prof.cu)
class ProfScope {
  public:
    ProfScope(const char *name, cudaStream_t st);
    ~ProfScope();

  private:
    const char *name_;
    cudaStream_t st_;
    cudaEvent_t a_;
};
#define CHR_PROF_CAT2(a, b) a##b
#define CHR_PROF_CAT(a, b) CHR_PROF_CAT2(a, b)
#define CHR_PROF(name, st) ::chr::ProfScope CHR_PROF_CAT(_chr_prof_, __LINE__)(name, st)

// ------------------------------------------------------------------ transfers
// small host<->device copies without the copy engines (xfer.cu): h2d is
// staged in a pinned ring and pulled by a kernel; d2h is pushed by a kernel
// and delivered at the next stream_sync of the stream.  Every extern "C"
// function that calls d2h holds an XferScope.
cudaError_t h2d(void *dst, const void *src, size_t n, cudaStream_t st);
cudaError_t d2h(void *dst, const void *src, size_t n, cudaStream_t st);
const void *d2h_view(const void *src, size_t n, cudaStream_t st, cudaError_t *err);  // zero-copy read-back
cudaError_t stream_sync(cudaStream_t st);
cudaError_t fill_async(void *dst, int v, size_t n, cudaStream_t st);   // cudaMemsetAsync as a kernel
constexpr int kFillMax = 8;
struct Xfer {
    void *dst;
    const void *src;
    size_t n;
};
cudaError_t h2d_multi(std::initializer_list<Xfer> xs, cudaStream_t st);  // one pull launch
cudaError_t d2h_multi(std::initializer_list<Xfer> xs, cudaStream_t st);  // one push launch
cudaError_t zero_async(std::initializer_list<std::pair<void *, size_t>> ranges, cudaStream_t st);  // one launch
cudaError_t copy_async(void *dst, const void *src, size_t n, cudaStream_t st);  // kernel copy, UVA pointers
class XferScope {
  public:
    XferScope();
    ~XferScope();

  private:
    size_t mark_;
};
#define CHR_XFER_SCOPE ::chr::XferScope CHR_PROF_CAT(_chr_xfer_, __LINE__)

// ------------------------------------------------------------------ side stream
// Per host thread and device: a second (non-blocking) stream and events for
// work that overlaps the caller's stream inside one library call -- the
// payload CRC-32s, which nothing on the caller's stream reads until the
// call's final status.  nullptr when CHR_NO_SIDE=1 (serial A/B runs) or on
// a CUDA error; callers then run everything on their own stream.
struct Side {
    cudaStream_t st = nullptr;
    cudaEvent_t ev[4] = {};
};
Side *side_stream();

// compress with the CRC tail (payload CRCs, block headers, file trailer) on
// `side` (encode.cu): returns after the host knows the layout; the archive
// is complete once side->ev[1] fires.  The control arrays the tail reads are
// carved first in the workspace (`keep_bytes`), so a caller may reuse the
// rest of the workspace right away.  compress_crcs() then copies the
// finished payload CRCs into a device array (after side->ev[1]).
int compress_with_side(const void *d_vol, int dtype, int src_dtype, int64_t nx, int64_t ny, int64_t nz,
                       const double *spacing, int64_t bs, double vmin, double vmax, const double *h_cands, int m,
                       chr_region_t *h_regions, int64_t nreg, void *d_ws, size_t ws_bytes, uint8_t *d_out,
                       uint64_t out_cap, uint64_t *h_out_nbytes, Side *side, size_t *keep_bytes, void **d_regs,
                       cudaStream_t st);
int compress_crcs(const void *d_regs, int64_t nreg, uint32_t *d_crc, cudaStream_t st);
// chr_decode_regions_mask with the expected payload CRCs read from the block
// headers in d_blob (the pipeline: the host has not seen them yet)
int decode_mask_hdrcrc(const uint8_t *d_blob, const chr_dec_region_t *h, int64_t n, double *d_out, void *d_ws,
                       size_t ws_bytes, int32_t *h_status, double iso, uint32_t *d_mask, cudaStream_t st);

// ------------------------------------------------------------------ workspace
struct WsCarver {
    char *base;
    size_t off, cap;
    bool ok = true;
    template <typename T>
    T *take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T *p = reinterpret_cast<T *>(base ? base + off : nullptr);
        off += count * sizeof(T);
        if (off > cap) ok = false;
        return p;
    }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

#if defined(__CUDACC__)
// x^(8n) mod P with the 61 factors spread over the lanes of a warp (all
// lanes call; every lane gets the product)
__device__ __forceinline__ uint32_t warp_x8n(const uint32_t *x2n, uint64_t n) {
    const int lane = threadIdx.x & 31;
    uint32_t p = 1u << 31;
    if ((n >> lane) & 1) p = x2n[lane + 3];
    if (lane + 32 < 61 && ((n >> (lane + 32)) & 1)) p = gf2_mul(p, x2n[lane + 35]);
#pragma unroll
    for (int off = 16; off; off >>= 1) p = gf2_mul(p, __shfl_xor_sync(0xFFFFFFFFu, p, off));
    return p;
}


// copy a struct from global to shared memory with all threads (parallel
// 4-byte loads instead of one thread's serialised copy); caller syncs
template <typename S>
__device__ __forceinline__ void coop_copy(S *dst, const S *src) {
    static_assert(sizeof(S) % 4 == 0, "4-byte multiple");
    const uint32_t *a = reinterpret_cast<const uint32_t *>(src);
    uint32_t *b = reinterpret_cast<uint32_t *>(dst);
    for (int i = threadIdx.x; i < (int)(sizeof(S) / 4); i += blockDim.x) b[i] = __ldg(a + i);
}
#endif

}  // namespace chr
