/*
 * chr.h -- C ABI of libchr.so, the B200 (sm_100a) implementation of the
 * CHR hot path of arXiv 2408.05462 (reference package `isochr`).
 *
 * The reference is pure Python + numba; its plug points are the kernel
 * seam (isochr/kernels.py, switched by backend.USE_NUMBA, backend.py:19-42),
 * the codec plugin (build_chr(codec=...), chr_archive.py:142; register_codec,
 * codec.py:207-211) and the public API (isochr/__init__.py:9-86).  A
 * Python host binds this ABI with ctypes (paper_2408_05462_b200/_abi.py,
 * INTEGRATION.md) and keeps the reference call signatures.
 *
 * Conventions
 *  - every device buffer is caller-allocated (e.g. a torch tensor) and
 *    passed as a raw pointer; host buffers are plain C arrays;
 *  - temporary device memory comes from a caller workspace whose size is
 *    returned by the matching *_workspace_size() query; the library keeps
 *    no allocations between calls and no mutable global state beyond
 *    constant tables initialised once under a mutex;
 *  - `stream` is a cudaStream_t (0 = legacy default stream);
 *  - functions return a chr_status_t; calls that produce host-visible
 *    results synchronise `stream` before returning.
 *
 * Volume layout: x fastest ("Fortran ravel" of the [x, y, z] grid), the
 * layout of Volume.values (volume.py:35-93) and of raw files (load_raw).
 */
#ifndef CHR_H_
#define CHR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: the Python host maps them onto isochr.errors classes */
typedef enum {
    CHR_OK = 0,
    CHR_E_PARAMETER = 1,       /* ParameterError            (errors.py:8)  */
    CHR_E_NONFINITE = 2,       /* NonFiniteSampleError      (errors.py:12) */
    CHR_E_CORRUPT = 3,         /* CorruptPayloadError       (errors.py:34) */
    CHR_E_UNSUPPORTED_CODEC = 4, /* UnsupportedCodecError  (errors.py:38) */
    CHR_E_CUDA = 5,            /* CUDA runtime failure */
    CHR_E_WORKSPACE = 6        /* workspace too small */
} chr_status_t;

/* per-region corruption subcodes written by chr_decode_regions
 * (kernels.py:299-345, codec.py:146-229) */
enum {
    CHR_DEC_OK = 0,
    CHR_DEC_TRUNCATED = 1,
    CHR_DEC_VARINT_LONG = 2,
    CHR_DEC_RUN_MISSING = 3,
    CHR_DEC_RUN_RANGE = 4,
    CHR_DEC_TRAILING = 5,
    CHR_DEC_COUNT = 6,
    CHR_DEC_CHECKSUM = 7,
    CHR_DEC_SHORT_BITMAP = 8,
    CHR_DEC_SHORT_ESCAPES = 9,
    CHR_DEC_BAD_CODEC = 10
};

/* dtype tags (volume.py:18, FORMAT.md) */
enum { CHR_F32 = 0, CHR_F64 = 1 };

/* One region of the archive (ArchiveRegion, chr_archive.py:54-75 and the
 * FORMAT.md region record).  Filled in two steps: chr_plan() writes the
 * geometry, mask and error bound; chr_compress() writes codec, offsets,
 * lengths and CRC. */
typedef struct {
    int32_t lo[3];             /* block span lo (bx, by, bz), inclusive */
    int32_t hi[3];             /* block span hi, inclusive */
    int32_t origin[3];         /* sample origin */
    int32_t extent[3];         /* sample extent incl. high ghost planes */
    uint64_t mask;             /* relevance bitmask: bit ci <-> candidate ci */
    double error_bound;        /* absolute bound (bound.py:150-219) */
    int32_t codec_id;          /* 0 verbatim f64, 1 lorenzo, 2 lorenzo+esc, 3 verbatim f32 */
    uint32_t payload_crc;      /* zlib.crc32(payload) */
    uint64_t block_offset;     /* absolute file offset of the CompressedBlock */
    uint64_t block_nbytes;     /* 34 + payload length (CompressedBlock.nbytes) */
    uint64_t n_escaped;        /* escaped samples (codec 2) */
} chr_region_t;

/* A region to decode (codec.decompress on one CompressedBlock whose
 * header the host has parsed, codec.py:146-229). */
typedef struct {
    uint64_t payload_offset;   /* byte offset of the payload in the blob */
    uint64_t payload_nbytes;
    int32_t codec_id;
    int32_t dims[3];           /* ex, ey, ez */
    double error_bound;        /* from the block header */
    uint32_t crc;              /* from the block header */
    uint32_t _pad;
    uint64_t out_offset;       /* element offset of this window in the f64 output */
} chr_dec_region_t;

/* A grid to contour (marching_cubes on one window, isosurf.py:183-204). */
typedef struct {
    uint64_t grid_offset;      /* element offset of the f64 window (x fastest) */
    int32_t dims[3];           /* samples per axis, each >= 2 */
    int32_t zoff;              /* lattice z of grid plane 0 (0 for a whole window; a z-slab
                                  portion grid sets its plane offset in the region window) */
    double origin[3];          /* world origin of lattice point (0,0,0) of the region window */
    double spacing[3];
} chr_mc_grid_t;

/* ---------------------------------------------------------------- */
/* library info                                                     */
int chr_abi_version(void);
const char *chr_status_string(int status);

/* ---------------------------------------------------------------- */
/* 1. block decomposition + min/max index (blocking.py:64-127) and the
 *    strict accuracy-1 distance reduction (bound.py:150-219 with
 *    kernels.min_abs_distance, kernels.py:417-425) in ONE streaming pass.
 *
 * d_vol: nx*ny*nz samples (dtype CHR_F32 or CHR_F64).  h_cands: m <= 64
 * strictly increasing finite candidates.  Writes, per block
 * (block_id = bx + nbx*(by + nby*bz)): d_block_stats[3*id+0..2] =
 * (vmin, vmax, dmin) with dmin = min over the window of min_k |s-k|.
 * d_first_nonfinite[0] = first flat index of a NaN/Inf sample, or -1.
 * Asynchronous. */
int chr_stats(const void *d_vol, int dtype, int64_t nx, int64_t ny, int64_t nz,
              int64_t block_size, const double *h_cands, int m,
              double *d_block_stats, int64_t *d_first_nonfinite, void *stream);

/* number of blocks of the decomposition (blocking.block_grid_shape) */
int64_t chr_num_blocks(int64_t nx, int64_t ny, int64_t nz, int64_t block_size);

/* 2. host planning: relevance masks, greedy merge (blocking.py:130-193)
 *    and per-region strict bounds.  h_block_stats is the D2H copy of
 *    chr_stats' output.  h_regions needs chr_num_blocks() entries;
 *    *n_regions receives the region count (region_id = index). */
int chr_plan(const double *h_block_stats, int64_t nx, int64_t ny, int64_t nz,
             int64_t block_size, const double *h_cands, int m, double vmin, double vmax,
             double loose_fraction, double safety_factor,
             chr_region_t *h_regions, int64_t *n_regions);

/* 2b. merge_regions (blocking.py:130-193) over caller-supplied keys: one
 *     integer per block (block_id order; equal integers = equal relevance
 *     keys, i.e. the IsoIndex.relevance_key frozensets the caller holds).
 *     h_spans receives 6 int32 per region (lo x,y,z, hi x,y,z, inclusive) in
 *     region_id order and needs 6*nbx*nby*nbz entries.  Host only. */
int chr_merge_keys(const uint64_t *h_keys, int64_t nbx, int64_t nby, int64_t nbz, int32_t *h_spans,
                   int64_t *n_regions);

/* 1b. Volume.value_range + the finite check (volume.py:54-78) of n samples
 *     on the device: h_range = (min, max) of the finite samples,
 *     *h_first_nonfinite = first flat index of a NaN/Inf or -1.  Workspace:
 *     24 bytes.  Synchronises. */
int chr_value_range(const void *d_vol, int dtype, int64_t n, void *d_workspace, size_t workspace_bytes,
                    double *h_range, int64_t *h_first_nonfinite, void *stream);

/* 3. compress all regions into a complete .chr file on the device
 *    (codec.compress per region, codec.py:91-143; write_chr layout,
 *    chr_archive.py:297-340).  Regions come from chr_plan or from the
 *    caller (codec.compress on one array = one region covering it).
 *    With write_file == 0 only the CompressedBlocks are written, each at
 *    its block_offset starting from 0 (no file header/table/trailer).
 *    Fills codec/offset/length/crc of h_regions and *h_out_nbytes
 *    (file or blob size).  Synchronises the stream. */
size_t chr_compress_workspace_size(const chr_region_t *h_regions, int64_t n_regions);
uint64_t chr_compress_capacity(const chr_region_t *h_regions, int64_t n_regions, int m,
                               int source_dtype);
int chr_compress(const void *d_vol, int dtype, int source_dtype, int64_t nx, int64_t ny,
                 int64_t nz, const double *spacing, int64_t block_size, double vmin,
                 double vmax, const double *h_cands, int m, chr_region_t *h_regions,
                 int64_t n_regions, int write_file, void *d_workspace, size_t workspace_bytes,
                 uint8_t *d_out, uint64_t out_capacity, uint64_t *h_out_nbytes, void *stream);

/* 4. selective reconstruction: decode the given blocks of d_blob into
 *    f64 windows (x fastest) at d_out + out_offset.  h_status[i]
 *    receives a CHR_DEC_* code per region.  Returns CHR_E_CORRUPT /
 *    CHR_E_UNSUPPORTED_CODEC if any region failed (the host raises for
 *    the first failing region in request order).  Synchronises. */
size_t chr_decode_workspace_size(const chr_dec_region_t *h_regs, int64_t n);
int chr_decode_regions(const uint8_t *d_blob, const chr_dec_region_t *h_regs, int64_t n,
                       double *d_out, void *d_workspace, size_t workspace_bytes,
                       int32_t *h_status, void *stream);

/* 5. marching cubes, count -> scan -> emit (kernels.py:428-524,
 *    isosurf.py:183-225).  Grids are meshed in order and concatenated
 *    with merge_meshes semantics (vertex ids offset by the vertices of
 *    the previous grids).  chr_mc_count fills per-grid triangle/vertex
 *    counts (h_ntri/h_nvert may be NULL) and the totals; chr_mc_emit
 *    (same workspace, untouched in between) writes d_verts (nv x 3 f64,
 *    world coordinates) and d_tris (nt x 3 int32). */
size_t chr_mc_workspace_size(const chr_mc_grid_t *h_grids, int64_t n);
int chr_mc_count(const double *d_grids, const chr_mc_grid_t *h_grids, int64_t n, double k,
                 void *d_workspace, size_t workspace_bytes, int64_t *h_ntri, int64_t *h_nvert,
                 int64_t *h_total_tri, int64_t *h_total_vert, void *stream);
int chr_mc_emit(const double *d_grids, const chr_mc_grid_t *h_grids, int64_t n, double k,
                void *d_workspace, size_t workspace_bytes, double *d_verts, int32_t *d_tris,
                void *stream);

/*    chr_mc_emit plus every vertex's canonical edge (grid-local
 *    ((z * ny + y) * nx + x) * 3 + axis) in d_vedge (nv int64): the z-slab
 *    request matches the vertices of a plane two ranks share by it. */
int chr_mc_emit_edges(const double *d_grids, const chr_mc_grid_t *h_grids, int64_t n, double k,
                      void *d_workspace, size_t workspace_bytes, double *d_verts, int32_t *d_tris,
                      int64_t *d_vedge, void *stream);

/* 6. per-cell case codes of one grid (isosurf.case_field, isosurf.py:77-88
 *    when binary_order != 0; Bourke order of mc_extract otherwise). */
int chr_case_codes(const double *d_grid, int64_t nx, int64_t ny, int64_t nz, double k,
                   int binary_order, uint8_t *d_codes, void *stream);

/* 7. CRC-32/IEEE (zlib.crc32) of a device buffer; combine operator. */
size_t chr_crc32_workspace_size(uint64_t n);
int chr_crc32(const uint8_t *d_buf, uint64_t n, void *d_workspace, size_t workspace_bytes,
              uint32_t *h_crc, void *stream);
uint32_t chr_crc32_combine(uint32_t crc1, uint32_t crc2, uint64_t len2);
/*    n byte ranges [begin, end) (h_ranges: 2n u64) of one buffer in one
 *    launch: h_raw = raw registers (init 0, no final xor; shares of disjoint
 *    ranges XOR after chr_crc32_shift), h_crc = zlib.crc32 per range (either
 *    may be NULL).  Synchronises. */
size_t chr_crc32_segments_workspace_size(int64_t n);
int chr_crc32_segments(const uint8_t *d_buf, const uint64_t *h_ranges, int64_t n, void *d_workspace,
                       size_t workspace_bytes, uint32_t *h_raw, uint32_t *h_crc, void *stream);
uint32_t chr_crc32_shift(uint32_t raw, uint64_t len);
void chr_crc32_shift_many(const uint32_t *h_raw, const uint64_t *h_len, int64_t n, uint32_t *h_out);

/* 8. kernel seam (isochr/kernels.py) on single windows */
int chr_min_abs_distance(const double *d_flat, int64_t n, double k, double *h_out,
                         void *d_workspace, size_t workspace_bytes, void *stream);
int chr_lorenzo_encode(const double *d_flat, int64_t nx, int64_t ny, int64_t nz, double e,
                       int64_t *d_q, uint8_t *d_escaped, void *stream);
/* rle_varint_encode (kernels.py:198-296, signature kernels.py:292-296):
 * quanta |q| <= 2^30 -> LEB128 token stream (zero runs >= 2 packed),
 * *h_nbytes receives its length; out_cap >= 5n + 16.  Synchronises.
 * (rle_varint_decode and lorenzo_decode are served by chr_decode_regions
 * on a codec-1 stream, see the Python shims.) */
size_t chr_rle_encode_workspace_size(int64_t n);
int chr_rle_encode(const int64_t *d_q, int64_t n, uint8_t *d_out, uint64_t out_cap, void *d_workspace,
                   size_t workspace_bytes, uint64_t *h_nbytes, void *stream);

/* 10. z-slab multi-GPU protocol.  Rank r holds volume planes
 *     [z_base, z_base + nz_local) (global z) and encodes planes [zs, ze) of
 *     every window: its portion, a contiguous piece of the window's raster
 *     stream.  Phase 1 (chr_dcompress_local) summarises each portion's
 *     stream; after an allgather of the nreg summaries of every rank,
 *     phase 2 (chr_dcompress_finish, h_all = [nranks][nreg]) writes this
 *     rank's bytes at their final file offsets into a zeroed d_out and
 *     returns h_raw[1 + r] = raw CRC (init 0, no final xor) of its share of
 *     payload r.  Rank 0 then calls chr_dcompress_headers with the XOR of
 *     every rank's h_raw to write the file header, region table, block
 *     headers and trailer.  Slices of all ranks OR together into the file
 *     that chr_compress writes on one GPU.  The workspace must persist
 *     from phase 1 to phase 2. */
typedef struct {              /* token-stream summary of a portion (a monoid) */
    int64_t len;              /* samples */
    int64_t lead, trail;      /* zero samples before the first / after the last nonzero */
    int64_t bytes;            /* literal tokens + runs between them */
    int64_t nesc;             /* escaped samples */
    int32_t nz, f32ok;        /* any nonzero quantum; every sample f32-exact */
} chr_portion_t;
size_t chr_dcompress_workspace_size(const chr_region_t *h_regions, int64_t n_regions, int64_t z_base,
                                    int64_t nz_local, int64_t zs, int64_t ze);
int chr_dcompress_local(const void *d_vol, int dtype, int source_dtype, int64_t nx, int64_t ny, int64_t nz_local,
                        int64_t z_base, int64_t zs, int64_t ze, const chr_region_t *h_regions, int64_t n_regions,
                        void *d_workspace, size_t workspace_bytes, chr_portion_t *h_portions, void *stream);
int chr_dcompress_finish(const void *d_vol, int dtype, int source_dtype, int64_t nx, int64_t ny, int64_t nz_local,
                         int64_t z_base, int64_t zs, int64_t ze, const double *spacing, int64_t block_size,
                         double vmin, double vmax, const double *h_cands, int m, chr_region_t *h_regions,
                         int64_t n_regions, const chr_portion_t *h_all, int nranks, int rank, void *d_workspace,
                         size_t workspace_bytes, uint8_t *d_out, uint64_t out_cap, uint32_t *h_raw,
                         uint64_t *h_file_nbytes, void *stream);
int chr_dcompress_headers(int64_t nx, int64_t ny, int64_t nz, int source_dtype, const double *spacing,
                          int64_t block_size, double vmin, double vmax, const double *h_cands, int m,
                          chr_region_t *h_regions, int64_t n_regions, const uint32_t *h_raw_all,
                          void *d_workspace, size_t workspace_bytes, uint8_t *d_out, void *stream);

/* 10b. z-slab request: finish n portions decoded with e = 1/2 (u_local as
 *     exact integers in f64) in place: u = u_local + carry plane (int64 at
 *     d_carry + carry_offset, ex*ey entries; carry_offset < 0: none), then
 *     recon = u * 2e with the region's bound e.  Workspace: 48 * n bytes. */
int chr_portion_finish(double *d_windows, const uint64_t *h_out_offset, const int64_t *h_plane,
                       const int64_t *h_nplanes, const int64_t *h_carry_offset, const double *h_error_bound,
                       int64_t n, const int64_t *d_carry, void *d_workspace, size_t workspace_bytes, void *stream);

/*     n segments (h_table: 4 u64 each = dst offset, src offset, length,
 *     source 0 / 1) from d_src0 / d_src1 into d_dst in one launch (the
 *     z-slab request's re-framed token streams and packed planes); elem = 1:
 *     byte copies; elem = 8: int64 elements ADDED into d_dst (segments may
 *     share a destination; z-carry sums).  Workspace: 32 * n bytes. */
int chr_copy_segments(void *d_dst, const void *d_src0, const void *d_src1, const uint64_t *h_table, int64_t n,
                      int elem, void *d_workspace, size_t workspace_bytes, void *stream);

/*     z-slab request, vertex bookkeeping: h_grids = ng x 6 int64 (vertex
 *     base, vertex end, halo limit, top-plane edge id, key base, id base).
 *     chr_slab_classify: per vertex flags (1 dropped halo-plane x/y vertex,
 *     2 exported top-plane x/y vertex) + key, per-grid (dropped, exported)
 *     counts in h_counts (2 ng u64; synchronises).  chr_slab_gid: global id
 *     = id base + inclusive kept count - 1.  Workspace: 64 ng + 512 bytes. */
int chr_slab_classify(const int64_t *d_vedge, int64_t nv, const int64_t *h_grids, int ng, int8_t *d_flags,
                      int64_t *d_key, uint64_t *h_counts, void *d_workspace, size_t workspace_bytes, void *stream);
int chr_slab_gid(const int64_t *d_kept_incl, int64_t nv, const int64_t *h_grids, int ng, int64_t *d_gid,
                 void *d_workspace, size_t workspace_bytes, void *stream);

/* 13. SURVEY 8(f2): accuracy < 1 and paper_edges bounds.  For every pair
 *     (window [ox,oy,oz,ex,ey,ez], candidate k) the n-th smallest of the
 *     pair's distances (mode 0 strict_vertices: |s-k| over the window;
 *     mode 1 paper_edges: k-s0, s1-k of straddling edges), n = max(1, 1 +
 *     floor((1 - accuracy) |D|)) (bound.py:117-219); h_value = -1 when D is
 *     empty.  chr_compress2 also records the bound mode and accuracy in the
 *     region table. */
size_t chr_select_workspace_size(int64_t n_pairs);
int chr_select_distances(const void *d_vol, int dtype, int64_t nx, int64_t ny, int64_t nz, const int32_t *h_windows,
                         const double *h_k, int64_t n_pairs, double accuracy, int mode, void *d_workspace,
                         size_t workspace_bytes, double *h_value, int64_t *h_count, int64_t *h_n, void *stream);
int chr_compress2(const void *d_vol, int dtype, int source_dtype, int64_t nx, int64_t ny, int64_t nz,
                  const double *spacing, int64_t block_size, double vmin, double vmax, const double *h_cands, int m,
                  chr_region_t *h_regions, int64_t n_regions, int write_file, int bound_mode, double accuracy,
                  void *d_workspace, size_t workspace_bytes, uint8_t *d_out, uint64_t out_cap,
                  uint64_t *h_out_nbytes, void *stream);

/* 12. fused request + extract: the decoder also writes each window's
 *     inside mask (bit y*nx + x of plane z's ceil(nx*ny/32) words is
 *     v >= iso; windows back to back, chr_mask_words() words in all) and
 *     the marching cubes passes read those masks instead of recomputing
 *     them from the f64 windows (same grids, same order). */
uint64_t chr_mask_words(const int32_t *h_dims, int64_t n);
int chr_decode_regions_mask(const uint8_t *d_blob, const chr_dec_region_t *h_regions, int64_t n,
                            double *d_out, void *d_workspace, size_t workspace_bytes, int32_t *h_status,
                            double iso, uint32_t *d_masks, void *stream);
int chr_mc_count_masked(const double *d_grids, const chr_mc_grid_t *h_grids, int64_t n, double k,
                        const uint32_t *d_masks, void *d_workspace, size_t workspace_bytes, int64_t *h_ntri,
                        int64_t *h_nvert, int64_t *h_total_tri, int64_t *h_total_vert, void *stream);
int chr_mc_emit_masked(const double *d_grids, const chr_mc_grid_t *h_grids, int64_t n, double k,
                       const uint32_t *d_masks, void *d_workspace, size_t workspace_bytes, double *d_verts,
                       int32_t *d_tris, void *stream);

/* 11. bulk copy by a small grid through UVA (pinned host <-> device):
 *     keeps the copy engines free for the library's own small copies when
 *     a caller pipelines its inputs/outputs.  16-byte aligned pointers. */
int chr_sm_copy(void *dst, const void *src, uint64_t nbytes, int ctas, void *stream);
/*     the same for small copies at any alignment (the library's own small
 *     transfers use this path internally by default) */
int chr_copy(void *dst, const void *src, uint64_t nbytes, void *stream);
/*     the library's own small host<->device transfers (plans, sizes, status):
 *     dma = 0 (default) by kernels through a pinned mapped ring, so they never
 *     queue behind a caller's bulk copies on the copy engines; dma = 1 on the
 *     copy engines (cheaper when the caller keeps them idle).  Process-wide;
 *     returns the previous mode.  Env CHR_XFER=dma sets 1 at load. */
int chr_set_xfer_mode(int dma);

/* 14. SURVEY 8(f3): stitch + verify_topology on the device.
 *     chr_stitch replaces chr_archive.stitch (chr_archive.py:277-294): the
 *     request windows (f64, each at window_offset samples into d_windows)
 *     are written into d_out (nx*ny*nz f64, x fastest, prefilled by the
 *     caller with the fill value), each sample by its owner -- the window
 *     with the lowest (z, y, x) origin among those covering it.  block_lo /
 *     block_hi: the region's block span (FORMAT.md record fields).
 *     chr_topology_compare replaces the case-code comparison of
 *     verify_topology (isosurf.py:91-114): number of cells whose binary
 *     case codes differ between a and b at k, and the smallest differing
 *     cell index (x fastest over the (nx-1)(ny-1)(nz-1) cells; -1 if none).
 *     Workspace: 16 bytes. */
typedef struct {
    uint64_t window_offset;
    int32_t origin[3];
    int32_t extent[3];
    int32_t block_lo[3];
    int32_t block_hi[3];
} chr_stitch_t;

size_t chr_stitch_workspace_size(int64_t n_windows, int64_t nx, int64_t ny, int64_t nz, int64_t bs);
int chr_stitch(const double *d_windows, const chr_stitch_t *h_windows, int64_t n, int64_t nx, int64_t ny,
               int64_t nz, int64_t bs, void *d_workspace, size_t workspace_bytes, double *d_out, void *stream);
int chr_topology_compare(const void *d_a, int dtype_a, const void *d_b, int dtype_b, int64_t nx, int64_t ny,
                         int64_t nz, double k, void *d_workspace, size_t workspace_bytes, uint64_t *h_ndiff,
                         int64_t *h_first, void *stream);

/* 15. SURVEY 8(f1): read_chr on the device (chr_archive.py:343-407).
 *     Step 1, chr_read_header: the fixed header, m, the region count and
 *     the stored trailer CRC (small device->host copies); sets
 *     info.error for a short file / bad magic / a table past the end.
 *     Step 2, chr_read_archive: whole-file CRC-32 and one thread per region
 *     record parsing the table entry + the 34-byte block header it points
 *     at, with the reference's checks (status per entry); the candidates
 *     and the table come back in one synchronised copy.  The caller raises
 *     the reference's exceptions in its order: too short, magic, CRC,
 *     version, then the first region with a nonzero status. */
enum {
    CHR_READ_OK = 0,
    CHR_READ_TOO_SHORT = 1,
    CHR_READ_BAD_MAGIC = 2,
    CHR_READ_TABLE_PAST_END = 3,
    CHR_READ_PAYLOAD_PAST_END = 4,       /* poffset + plen > len(file) - 4 */
    CHR_READ_BLOCK_HEADER_TRUNCATED = 5, /* < 34 bytes at poffset */
    CHR_READ_PAYLOAD_TRUNCATED = 6,      /* block header length past the file */
    CHR_READ_LENGTH_MISMATCH = 7         /* 34 + payload length != table length */
};

typedef struct {
    char magic[4];
    uint32_t version;
    uint32_t dims[3];
    double spacing[3];
    uint32_t dtype;
    uint32_t block_size;
    double vmin, vmax;
    uint32_t m;
    uint32_t n_regions;
    uint64_t table_nbytes;     /* header_table_nbytes: first byte after the table */
    uint32_t stored_crc, actual_crc;
    int32_t error;             /* CHR_READ_* found by chr_read_header */
    int32_t _pad;
} chr_file_info_t;

typedef struct {
    chr_region_t region;       /* geometry, mask (first 64 candidates), table error bound,
                                  block offset/length; codec id + payload CRC from the block header */
    uint32_t region_id;
    int32_t status;            /* CHR_READ_* */
    uint32_t bound_mode;
    uint32_t block_dtype;
    double accuracy;
    uint32_t block_dims[3];
    uint32_t _pad;
    double block_error_bound;
    uint64_t payload_len;
} chr_table_entry_t;

int chr_read_header(const uint8_t *d_file, uint64_t nbytes, chr_file_info_t *h_info, void *stream);
size_t chr_read_workspace_size(uint64_t nbytes, int64_t n_regions);
int chr_read_archive(const uint8_t *d_file, uint64_t nbytes, chr_file_info_t *h_info, double *h_cands,
                     chr_table_entry_t *h_entries, void *d_workspace, size_t workspace_bytes, void *stream);

/* 16. request(k) tables from a region table, host only (chr_archive.py:249-259):
 *     regions whose mask has bit k_index (all when k_index < 0) as decode and
 *     marching tables with back-to-back windows; returns the count (-1 on a
 *     bad argument).  Output arrays need n entries. */
int64_t chr_request_tables(const chr_region_t *h_regions, int64_t n, int k_index, const double *spacing,
                           chr_dec_region_t *h_dec, chr_mc_grid_t *h_mc, int64_t *h_sel,
                           uint64_t *h_total_samples);

/* 17. the whole step in one call (stats -> plan -> compress -> request(k) ->
 *     decode + inside masks -> marching cubes), results identical to the
 *     separate entry points; no host round trips in between.  Strict bound,
 *     accuracy 1, out_of_range="error".  The archive goes to d_archive, the
 *     mesh to d_verts / d_tris (capacities in vertices / triangles), the f64
 *     windows and masks stay in the workspace at the offsets reported.
 *     CHR_E_WORKSPACE: grow to ws_needed / archive_needed / n_tri / n_vert
 *     and call again.  stage_events (may be NULL): 4 cudaEvent_t recorded at
 *     the start, after compress, after decode and after the mesh. */
typedef struct {
    int64_t n_regions, n_selected;
    uint64_t archive_nbytes, archive_needed;
    int64_t n_tri, n_vert;
    uint64_t window_samples;     /* f64 samples of the selected windows */
    uint64_t windows_offset;     /* byte offsets in the workspace */
    uint64_t masks_offset;
    uint64_t ws_needed;
    int64_t first_nonfinite;     /* CHR_E_NONFINITE: flat index */
    double vmin, vmax;
} chr_pipeline_result_t;

/* called (host thread, between compress and request) with the archive size:
 * lets a caller start copying the archive out while the rest runs */
typedef void (*chr_after_compress_fn)(uint64_t archive_nbytes, void *user);

int chr_pipeline(const void *d_vol, int dtype, int src_dtype, int64_t nx, int64_t ny, int64_t nz,
                 const double *spacing, int64_t block_size, const double *h_cands, int m, double loose_fraction,
                 double safety_factor, int k_index, void *d_workspace, size_t workspace_bytes, uint8_t *d_archive,
                 uint64_t archive_cap, double *d_verts, int64_t verts_cap, int32_t *d_tris, int64_t tris_cap,
                 chr_region_t *h_regions, void *const *stage_events, chr_after_compress_fn after_compress,
                 void *user, chr_pipeline_result_t *h_res, void *stream);

/* 9. instrumentation: launch counter and opt-in per-kernel CUDA-event
 *    timing on the launching stream ("name count total_ms" lines). */
void chr_prof_enable(int on);
long long chr_launch_count(void);
int chr_prof_report(char *buf, size_t cap);
int chr_prof_timeline(char *buf, size_t cap);
void chr_prof_mark(const char *name, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* CHR_H_ */
