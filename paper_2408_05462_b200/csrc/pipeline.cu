// pipeline.cu -- the whole hot path in one call: stats -> plan -> compress
// -> request(k) -> decode (+ inside masks) -> marching cubes count/emit.
//
// The steps and their results are exactly those of the separate entry points
// (chr_stats, chr_plan, chr_compress2, chr_request_tables,
// chr_decode_regions_mask, chr_mc_count_masked, chr_mc_emit_masked); doing
// them from one host function removes the interpreter round trips between
// them (an in-transit consumer runs this per time step).  Phases reuse one
// caller workspace: block stats, then the encoder's workspace, then the f64
// windows + masks followed by the decoder's / marching cubes' workspace.
// When a buffer is too small the call returns CHR_E_WORKSPACE with the
// sizes it needs (the caller grows them and calls again).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <vector>

#include "chr_internal.cuh"

using namespace chr;

extern "C" int chr_pipeline(const void *d_vol, int dtype, int src_dtype, int64_t nx, int64_t ny, int64_t nz,
                            const double *spacing, int64_t bs, const double *h_cands, int m, double loose_fraction,
                            double safety_factor, int k_index, void *d_ws, size_t ws_bytes, uint8_t *d_archive,
                            uint64_t archive_cap, double *d_verts, int64_t verts_cap, int32_t *d_tris,
                            int64_t tris_cap, chr_region_t *h_regions, void *const *stage_events,
                            chr_after_compress_fn after_compress, void *user, chr_pipeline_result_t *h_res,
                            void *stream) {
    CHR_XFER_SCOPE;
    // CHR_TRACE_HOST=1: host-side phase times of the call on stderr (diagnostics)
    static const bool trace = [] {
        const char *e = std::getenv("CHR_TRACE_HOST");
        return e && e[0] == '1';
    }();
    auto t_start = std::chrono::steady_clock::now();
    auto tmark = [&](const char *what) {
        if (!trace) return;
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_start).count();
        std::fprintf(stderr, "chr_pipeline %8.1f us  %s\n", us, what);
    };
    if (!d_vol || !h_cands || !h_regions || !h_res || !spacing) return CHR_E_PARAMETER;
    if (m < 1 || m > 64 || k_index < 0 || k_index >= m) return CHR_E_PARAMETER;
    std::memset(h_res, 0, sizeof(*h_res));
    h_res->first_nonfinite = -1;
    cudaStream_t st = (cudaStream_t)stream;
    auto mark = [&](int i) -> cudaError_t {
        return (stage_events && stage_events[i]) ? cudaEventRecord((cudaEvent_t)stage_events[i], st) : cudaSuccess;
    };
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    char *ws = reinterpret_cast<char *>(d_ws);
    CHR_CUDA_TRY(mark(0));

    // ---- stats (block extrema + distances), then the host plan
    const int64_t nb = chr_num_blocks(nx, ny, nz, bs);
    if (nb < 1) return CHR_E_PARAMETER;
    const size_t stats_bytes = al((size_t)nb * 3 * sizeof(double)) + 256;
    if (!d_ws || ws_bytes < stats_bytes) {
        h_res->ws_needed = stats_bytes;
        return CHR_E_WORKSPACE;
    }
    double *d_stats = reinterpret_cast<double *>(ws);
    int64_t *d_bad = reinterpret_cast<int64_t *>(ws + al((size_t)nb * 3 * sizeof(double)));
    int rc = chr_stats(d_vol, dtype, nx, ny, nz, bs, h_cands, m, d_stats, d_bad, stream);
    if (rc) return rc;
    // the block stats are read straight from the pinned transfer ring (no
    // copy-out: 786 KB at c3); they are consumed by the plan below, before
    // the next transfer reuses the ring
    std::vector<double> hs_copy;
    const double *hs = nullptr;
    int64_t bad = -1;
    cudaError_t ve = cudaSuccess;
    const size_t sbytes = al((size_t)nb * 3 * sizeof(double)) + sizeof(int64_t);  // stats, then d_bad
    const void *view = d2h_view(d_stats, sbytes, st, &ve);
    CHR_CUDA_TRY(ve);
    if (!view) {
        hs_copy.resize((size_t)nb * 3);
        CHR_CUDA_TRY(d2h_multi({{hs_copy.data(), d_stats, hs_copy.size() * sizeof(double)}, {&bad, d_bad, sizeof(bad)}},
                               st));
    }
    tmark("stats launched");
    CHR_CUDA_TRY(stream_sync(st));
    tmark("stats synced");
    if (view) {
        hs = reinterpret_cast<const double *>(view);
        std::memcpy(&bad, reinterpret_cast<const char *>(view) + (sbytes - sizeof(int64_t)), sizeof(bad));
    } else {
        hs = hs_copy.data();
    }
    if (bad >= 0) {
        h_res->first_nonfinite = bad;
        return CHR_E_NONFINITE;
    }
    double vmin = INFINITY, vmax = -INFINITY;
    for (int64_t b = 0; b < nb; ++b) {
        vmin = std::min(vmin, hs[3 * b]);
        vmax = std::max(vmax, hs[3 * b + 1]);
    }
    h_res->vmin = vmin;
    h_res->vmax = vmax;
    for (int i = 0; i < m; ++i)
        if (!(vmin <= h_cands[i] && h_cands[i] <= vmax)) return CHR_E_PARAMETER;  // out_of_range="error"
    tmark("value range");
    int64_t nreg = 0;
    rc = chr_plan(hs, nx, ny, nz, bs, h_cands, m, vmin, vmax, loose_fraction, safety_factor, h_regions, &nreg);
    if (rc) return rc;
    h_res->n_regions = nreg;
    tmark("plan");

    // ---- compress into the caller's archive buffer
    const size_t cws = chr_compress_workspace_size(h_regions, nreg);
    const uint64_t cap = chr_compress_capacity(h_regions, nreg, m, src_dtype);
    h_res->archive_needed = cap;
    tmark("compress sizes");
    if (cws == 0) return CHR_E_PARAMETER;
    if (ws_bytes < cws || archive_cap < cap || !d_archive) {
        h_res->ws_needed = std::max(cws, stats_bytes);
        return CHR_E_WORKSPACE;
    }
    // The CRC tail of the compress (payload CRCs, block headers, trailer)
    // runs on a side stream, overlapping the request; the decoder takes the
    // expected payload CRCs from the block headers and joins the side stream
    // before its status read-back.  The tail's control arrays stay at the
    // front of the workspace (keep), the windows start after them.
    Side *side = side_stream();
    uint64_t nbytes = 0;
    size_t keep = 0;
    void *enc_regs = nullptr;
    if (side) {
        rc = compress_with_side(d_vol, dtype, src_dtype, nx, ny, nz, spacing, bs, vmin, vmax, h_cands, m, h_regions,
                                nreg, d_ws, ws_bytes, d_archive, archive_cap, &nbytes, side, &keep, &enc_regs, st);
    } else {
        rc = chr_compress2(d_vol, dtype, src_dtype, nx, ny, nz, spacing, bs, vmin, vmax, h_cands, m, h_regions, nreg,
                           1, 0, 1.0, d_ws, ws_bytes, d_archive, archive_cap, &nbytes, stream);
    }
    if (rc) return rc;
    tmark("compress returned");
    h_res->archive_nbytes = nbytes;
    CHR_CUDA_TRY(mark(1));
    if (after_compress) {  // e.g. start the archive's device->host copy: the archive must be final
        if (side) CHR_CUDA_TRY(cudaStreamWaitEvent(st, side->ev[1], 0));
        after_compress(nbytes, user);
    }
    // the finished payload CRCs go back into h_regions at the next sync
    const size_t crc_off = al(keep), pre = side ? al(crc_off + sizeof(uint32_t) * (size_t)(nreg + 1)) : 0;
    uint32_t *d_crc = reinterpret_cast<uint32_t *>(ws + crc_off);
    std::vector<uint32_t> hcrc(side ? (size_t)nreg : 0);
    auto fetch_crcs = [&]() -> int {  // after the decoder joined the side stream (or after waiting here)
        if (!side) return CHR_OK;
        int r2 = compress_crcs(enc_regs, nreg, d_crc, st);
        if (r2) return r2;
        return d2h(hcrc.data(), d_crc, sizeof(uint32_t) * (size_t)nreg, st) == cudaSuccess ? CHR_OK : CHR_E_CUDA;
    };
    auto store_crcs = [&]() {
        for (int64_t r = 0; r < (int64_t)hcrc.size(); ++r) h_regions[r].payload_crc = hcrc[r];
    };

    // ---- request(k): decode the selected windows (+ inside masks)
    std::vector<chr_dec_region_t> dec((size_t)nreg);
    std::vector<chr_mc_grid_t> mcg((size_t)nreg);
    std::vector<int64_t> sel((size_t)nreg);
    uint64_t total = 0;
    const int64_t ns = chr_request_tables(h_regions, nreg, k_index, spacing, dec.data(), mcg.data(), sel.data(), &total);
    if (ns < 0) return CHR_E_PARAMETER;
    h_res->n_selected = ns;
    h_res->window_samples = total;
    if (ns == 0) {
        if (side) CHR_CUDA_TRY(cudaStreamWaitEvent(st, side->ev[1], 0));
        rc = fetch_crcs();
        if (rc) return rc;
        CHR_CUDA_TRY(stream_sync(st));
        store_crcs();
        CHR_CUDA_TRY(mark(2));
        CHR_CUDA_TRY(mark(3));
        return CHR_OK;
    }
    std::vector<int32_t> dims3((size_t)ns * 3);
    for (int64_t i = 0; i < ns; ++i)
        for (int a = 0; a < 3; ++a) dims3[3 * i + a] = dec[i].dims[a];
    const uint64_t mw = chr_mask_words(dims3.data(), ns);
    const size_t win_bytes = al(total * sizeof(double) + 16), mask_bytes = al((mw + 8) * sizeof(uint32_t));
    const size_t dws = chr_decode_workspace_size(dec.data(), ns), mws = chr_mc_workspace_size(mcg.data(), ns);
    const size_t need = pre + win_bytes + mask_bytes + std::max(dws, mws);
    if (ws_bytes < need) {
        h_res->ws_needed = std::max(need, cws);
        return CHR_E_WORKSPACE;
    }
    double *d_win = reinterpret_cast<double *>(ws + pre);
    uint32_t *d_masks = reinterpret_cast<uint32_t *>(ws + pre + win_bytes);
    char *tail = ws + pre + win_bytes + mask_bytes;
    const size_t tail_bytes = ws_bytes - pre - win_bytes - mask_bytes;
    h_res->windows_offset = pre;
    h_res->masks_offset = pre + win_bytes;
    std::vector<int32_t> status((size_t)ns);
    const double iso = h_cands[k_index];
    rc = decode_mask_hdrcrc(d_archive, dec.data(), ns, d_win, tail, tail_bytes, status.data(), iso, d_masks, st);
    if (rc) return rc;
    CHR_CUDA_TRY(mark(2));
    if (side) CHR_CUDA_TRY(cudaStreamWaitEvent(st, side->ev[1], 0));  // (the decoder already joined it)
    rc = fetch_crcs();  // delivered by the marching-cubes count's sync
    if (rc) return rc;

    // ---- marching cubes on the windows (masks from the decoder)
    int64_t ntri = 0, nvert = 0;
    rc = chr_mc_count_masked(d_win, mcg.data(), ns, iso, d_masks, tail, tail_bytes, nullptr, nullptr, &ntri, &nvert,
                             stream);
    if (rc) return rc;
    store_crcs();
    h_res->n_tri = ntri;
    h_res->n_vert = nvert;
    if (ntri > tris_cap || nvert > verts_cap || (ntri && (!d_tris || !d_verts))) {
        h_res->ws_needed = need;
        return CHR_E_WORKSPACE;  // caller grows the mesh buffers (n_tri / n_vert are set)
    }
    rc = chr_mc_emit_masked(d_win, mcg.data(), ns, iso, d_masks, tail, tail_bytes, d_verts, d_tris, stream);
    if (rc) return rc;
    CHR_CUDA_TRY(mark(3));
    return CHR_OK;
}
