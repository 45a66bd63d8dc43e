// readchr.cu -- SURVEY 8(f1): read_chr validation on the device
// (chr_archive.read_chr, chr_archive.py:343-407; FORMAT.md).
//
// The file is already in HBM (the caller uploaded it, or it is the output of
// chr_compress).  One pass: the whole-file CRC-32 (the segmented CRC kernel
// of crc.cu) and, on the same stream, a thread per region record that parses
// the table entry and the 34-byte block header it points at and applies the
// reference's per-region checks (payload inside the file, block length ==
// table length).  One device->host copy returns the parsed table; the host
// raises the reference's exception for the first failing check in file
// order.
#include <cstring>

#include "chr_internal.cuh"

namespace chr {

constexpr uint64_t kFileHdr = 63;  // "<4sH3I3dBIdd"
constexpr uint64_t kRecFixed = 85;  // "<I3I3I3I3IBddQQ"
constexpr uint64_t kBlkHdr = 34;    // "<B3IdBQI"

template <typename T>
__device__ __forceinline__ T ldu(const uint8_t *p) {  // unaligned little-endian load
    T v;
    uint8_t *d = reinterpret_cast<uint8_t *>(&v);
#pragma unroll
    for (int i = 0; i < (int)sizeof(T); ++i) d[i] = __ldg(p + i);
    return v;
}

__global__ void k_read_table(const uint8_t *__restrict__ f, uint64_t nbytes, uint64_t table0, int m, int64_t nreg,
                             chr_table_entry_t *__restrict__ out) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nreg) return;
    const int mb = (m + 7) / 8;
    const uint8_t *p = f + table0 + (uint64_t)r * (kRecFixed + mb);
    chr_table_entry_t E;
    memset(&E, 0, sizeof(E));
    E.region_id = ldu<uint32_t>(p);
    for (int a = 0; a < 3; ++a) {
        E.region.lo[a] = (int32_t)ldu<uint32_t>(p + 4 + 4 * a);
        E.region.hi[a] = (int32_t)ldu<uint32_t>(p + 16 + 4 * a);
        E.region.origin[a] = (int32_t)ldu<uint32_t>(p + 28 + 4 * a);
        E.region.extent[a] = (int32_t)ldu<uint32_t>(p + 40 + 4 * a);
    }
    E.bound_mode = p[52];
    E.accuracy = ldu<double>(p + 53);
    E.region.error_bound = ldu<double>(p + 61);
    const uint64_t poff = ldu<uint64_t>(p + 69), plen = ldu<uint64_t>(p + 77);
    E.region.block_offset = poff;
    E.region.block_nbytes = plen;
    uint64_t mask = 0;
    for (int i = 0; i < mb && i < 8; ++i) mask |= (uint64_t)p[kRecFixed + i] << (8 * i);
    E.region.mask = mask;
    // chr_archive.py:377-386 in order
    if (poff + plen > nbytes - 4 || poff + plen < poff) {
        E.status = CHR_READ_PAYLOAD_PAST_END;
    } else if (poff + kBlkHdr > nbytes) {
        E.status = CHR_READ_BLOCK_HEADER_TRUNCATED;
    } else {
        const uint8_t *b = f + poff;
        E.region.codec_id = b[0];
        for (int a = 0; a < 3; ++a) E.block_dims[a] = ldu<uint32_t>(b + 1 + 4 * a);
        E.block_error_bound = ldu<double>(b + 13);
        E.block_dtype = b[21];
        E.payload_len = ldu<uint64_t>(b + 22);
        E.region.payload_crc = ldu<uint32_t>(b + 30);
        const uint64_t avail = nbytes - (poff + kBlkHdr);
        if (E.payload_len > avail) E.status = CHR_READ_PAYLOAD_TRUNCATED;
        else if (kBlkHdr + E.payload_len != plen) E.status = CHR_READ_LENGTH_MISMATCH;
        else E.status = 0;
    }
    out[r] = E;
}

}  // namespace chr

using namespace chr;

extern "C" int chr_read_header(const uint8_t *d_file, uint64_t nbytes, chr_file_info_t *h_info, void *stream) {
    CHR_XFER_SCOPE;
    if (!h_info || (!d_file && nbytes)) return CHR_E_PARAMETER;
    std::memset(h_info, 0, sizeof(*h_info));
    if (nbytes < kFileHdr + 4) {
        h_info->error = CHR_READ_TOO_SHORT;
        return CHR_OK;
    }
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t hdr[kFileHdr + 4];
    CHR_CUDA_TRY(d2h(hdr, d_file, kFileHdr + 4, st));
    CHR_CUDA_TRY(stream_sync(st));
    std::memcpy(h_info->magic, hdr, 4);
    if (std::memcmp(hdr, "CHR1", 4) != 0) {
        h_info->error = CHR_READ_BAD_MAGIC;
        return CHR_OK;
    }
    uint16_t ver;
    std::memcpy(&ver, hdr + 4, 2);
    h_info->version = ver;
    for (int a = 0; a < 3; ++a) std::memcpy(&h_info->dims[a], hdr + 6 + 4 * a, 4);
    for (int a = 0; a < 3; ++a) std::memcpy(&h_info->spacing[a], hdr + 18 + 8 * a, 8);
    h_info->dtype = hdr[42];
    std::memcpy(&h_info->block_size, hdr + 43, 4);
    std::memcpy(&h_info->vmin, hdr + 47, 8);
    std::memcpy(&h_info->vmax, hdr + 55, 8);
    std::memcpy(&h_info->m, hdr + 63, 4);
    const uint64_t rpos = kFileHdr + 4 + 8ull * h_info->m;
    if (rpos + 4 <= nbytes) {
        uint32_t nreg = 0;
        CHR_CUDA_TRY(d2h(&nreg, d_file + rpos, 4, st));
        CHR_CUDA_TRY(stream_sync(st));
        h_info->n_regions = nreg;
    } else {
        h_info->error = CHR_READ_TABLE_PAST_END;
    }
    const uint64_t tab_end = rpos + 4 + (uint64_t)h_info->n_regions * (kRecFixed + (h_info->m + 7) / 8);
    h_info->table_nbytes = tab_end;
    if (!h_info->error && tab_end > nbytes) h_info->error = CHR_READ_TABLE_PAST_END;
    uint32_t stored;
    CHR_CUDA_TRY(d2h(&stored, d_file + nbytes - 4, 4, st));
    CHR_CUDA_TRY(stream_sync(st));
    h_info->stored_crc = stored;
    return CHR_OK;
}

extern "C" size_t chr_read_workspace_size(uint64_t nbytes, int64_t n_regions) {
    CHR_XFER_SCOPE;
    (void)nbytes;
    return 256 + (size_t)n_regions * sizeof(chr_table_entry_t) + 256;
}

extern "C" int chr_read_archive(const uint8_t *d_file, uint64_t nbytes, chr_file_info_t *h_info, double *h_cands,
                                chr_table_entry_t *h_entries, void *d_ws, size_t ws_bytes, void *stream) {
    CHR_XFER_SCOPE;
    if (!h_info || !d_file || nbytes < kFileHdr + 4) return CHR_E_PARAMETER;
    const int64_t nreg = h_info->n_regions;
    if (!d_ws || ws_bytes < chr_read_workspace_size(nbytes, nreg)) return CHR_E_WORKSPACE;
    if (nreg && !h_entries) return CHR_E_PARAMETER;
    cudaStream_t st = (cudaStream_t)stream;
    const CrcTables &H = crc_tables_hostref();
    // whole-file CRC (everything before the trailer)
    CrcSeg seg;
    seg.begin = 0;
    seg.end = nbytes - 4;
    crc_plan_segments(&seg, 1);
    char *ws = reinterpret_cast<char *>(d_ws);
    CrcSeg *d_seg = reinterpret_cast<CrcSeg *>(ws);
    uint32_t *d_raw = reinterpret_cast<uint32_t *>(ws + 128);
    chr_table_entry_t *d_ent = reinterpret_cast<chr_table_entry_t *>(ws + 256);
    CHR_CUDA_TRY(h2d(d_seg, &seg, sizeof(seg), st));
    CHR_CUDA_TRY(fill_async(d_raw, 0, 4, st));
    {
        CHR_PROF("k_crc_segments", st);
        const int rc = crc_launch(d_file, d_seg, 1, seg.n_sc, d_raw, st);
        if (rc) return rc;
    }
    const bool table_ok = h_info->table_nbytes <= nbytes && !h_info->error;
    if (table_ok && nreg) {
        CHR_PROF("k_read_table", st);
        k_read_table<<<(unsigned)ceil_div(nreg, 128), 128, 0, st>>>(d_file, nbytes, h_info->table_nbytes -
                                                                   (uint64_t)nreg * (kRecFixed + (h_info->m + 7) / 8),
                                                                   (int)h_info->m, nreg, d_ent);
        CHR_CUDA_TRY(cudaGetLastError());
        CHR_CUDA_TRY(d2h(h_entries, d_ent, nreg * sizeof(chr_table_entry_t), st));
    }
    if (h_cands && h_info->m && kFileHdr + 4 + 8ull * h_info->m <= nbytes)
        CHR_CUDA_TRY(d2h(h_cands, d_file + kFileHdr + 4, 8ull * h_info->m, st));
    uint32_t raw = 0;
    CHR_CUDA_TRY(d2h(&raw, d_raw, 4, st));
    CHR_CUDA_TRY(stream_sync(st));
    h_info->actual_crc = crc_finalize(H.x2n, raw, nbytes - 4);
    return CHR_OK;
}
