// plan.cpp -- step 2 (host): span index, greedy region merge, strict bounds.
//
// Reference: blocking.py:114-127 (build_index: relevant iff
// vmin <= k <= vmax), blocking.py:130-193 (merge_regions: scan z, y, x;
// grow +x, then whole rows +y, then whole slabs +z while unclaimed and
// same key), bound.py:150-219 + chr_archive.py:168 (strict, accuracy 1).
//
// Bound closed form (exact, by monotonicity of f64 rounding):
//   e = fl(dm * sf)                      if the region serves a candidate
//   e = min(loose, fl(dm * sf))          otherwise
// with dm = min over the region's blocks of the per-block dmin from
// chr_stats.  A served candidate at distance 0 gives e == 0 (lossless),
// exactly like region_bound's early return.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/chr.h"

namespace {

// Greedy same-key box merge (blocking.py:130-193): scan z, y, x; from each
// unclaimed seed grow +x, then whole rows +y, then whole slabs +z while
// the blocks are unclaimed and carry the seed's key.  `emit(lo, hi)` is
// called per region in creation order (= region_id).
template <typename Emit>
void greedy_merge(const uint64_t *key, int64_t nbx, int64_t nby, int64_t nbz, Emit emit) {
    const int64_t nb = nbx * nby * nbz;
    auto id = [&](int64_t x, int64_t y, int64_t z) { return x + nbx * (y + nby * z); };
    std::vector<uint8_t> claimed(nb, 0);
    for (int64_t bz = 0; bz < nbz; ++bz)
        for (int64_t by = 0; by < nby; ++by)
            for (int64_t bx = 0; bx < nbx; ++bx) {
                if (claimed[id(bx, by, bz)]) continue;
                const uint64_t k = key[id(bx, by, bz)];
                auto free_same = [&](int64_t x, int64_t y, int64_t z) {
                    return !claimed[id(x, y, z)] && key[id(x, y, z)] == k;
                };
                int64_t hx = bx, hy = by, hz = bz;
                while (hx + 1 < nbx && free_same(hx + 1, by, bz)) ++hx;
                for (;;) {
                    if (hy + 1 >= nby) break;
                    bool ok = true;
                    for (int64_t x = bx; x <= hx && ok; ++x) ok = free_same(x, hy + 1, bz);
                    if (!ok) break;
                    ++hy;
                }
                for (;;) {
                    if (hz + 1 >= nbz) break;
                    bool ok = true;
                    for (int64_t y = by; y <= hy && ok; ++y)
                        for (int64_t x = bx; x <= hx && ok; ++x) ok = free_same(x, y, hz + 1);
                    if (!ok) break;
                    ++hz;
                }
                for (int64_t z = bz; z <= hz; ++z)
                    for (int64_t y = by; y <= hy; ++y)
                        for (int64_t x = bx; x <= hx; ++x) claimed[id(x, y, z)] = 1;
                const int64_t lo[3] = {bx, by, bz}, hi[3] = {hx, hy, hz};
                emit(lo, hi, k);
            }
}

}  // namespace

// merge_regions over caller-supplied keys (one integer per block, equal
// integers = equal relevance keys): block spans, 6 int32 per region
// (lo x, y, z, hi x, y, z), in region_id order.  h_spans needs
// nbx*nby*nbz * 6 entries.
extern "C" int chr_merge_keys(const uint64_t *h_keys, int64_t nbx, int64_t nby, int64_t nbz, int32_t *h_spans,
                              int64_t *n_regions) {
    if (!h_keys || !h_spans || !n_regions || nbx < 1 || nby < 1 || nbz < 1) return CHR_E_PARAMETER;
    int64_t nreg = 0;
    greedy_merge(h_keys, nbx, nby, nbz, [&](const int64_t *lo, const int64_t *hi, uint64_t) {
        int32_t *o = h_spans + 6 * nreg++;
        for (int a = 0; a < 3; ++a) {
            o[a] = (int32_t)lo[a];
            o[3 + a] = (int32_t)hi[a];
        }
    });
    *n_regions = nreg;
    return CHR_OK;
}

extern "C" int chr_plan(const double *h_stats, int64_t nx, int64_t ny, int64_t nz, int64_t bs,
                        const double *h_cands, int m, double vmin, double vmax,
                        double loose_fraction, double sf, chr_region_t *h_regions,
                        int64_t *n_regions) {
    if (!h_stats || !h_cands || !h_regions || !n_regions) return CHR_E_PARAMETER;
    if (bs < 2 || nx < 2 || ny < 2 || nz < 2 || m < 1 || m > 64) return CHR_E_PARAMETER;
    for (int i = 0; i < m; ++i) {
        if (!std::isfinite(h_cands[i])) return CHR_E_PARAMETER;
        if (i && !(h_cands[i] > h_cands[i - 1])) return CHR_E_PARAMETER;
    }
    if (!(loose_fraction > 0.0) || !(sf > 0.0 && sf < 1.0)) return CHR_E_PARAMETER;
    const int64_t nbx = (nx - 1 + bs - 1) / bs, nby = (ny - 1 + bs - 1) / bs,
                  nbz = (nz - 1 + bs - 1) / bs;
    const int64_t nb = nbx * nby * nbz;
    std::vector<uint64_t> key(nb);
    for (int64_t b = 0; b < nb; ++b) {
        const double lo = h_stats[3 * b], hi = h_stats[3 * b + 1];
        uint64_t k = 0;
        for (int ci = 0; ci < m; ++ci)
            if (lo <= h_cands[ci] && h_cands[ci] <= hi) k |= 1ull << ci;
        key[b] = k;
    }
    auto id = [&](int64_t x, int64_t y, int64_t z) { return x + nbx * (y + nby * z); };
    auto win = [bs](int64_t bc, int64_t n, int64_t *lo, int64_t *ext) {
        *lo = bc * bs;
        *ext = std::min((bc + 1) * bs, n - 1) - *lo + 1;
    };
    const double loose = loose_fraction * (vmax - vmin);
    int64_t nreg = 0;
    greedy_merge(key.data(), nbx, nby, nbz, [&](const int64_t *blo, const int64_t *bhi, uint64_t k) {
        double dm = INFINITY;
        for (int64_t z = blo[2]; z <= bhi[2]; ++z)
            for (int64_t y = blo[1]; y <= bhi[1]; ++y)
                for (int64_t x = blo[0]; x <= bhi[0]; ++x) dm = std::min(dm, h_stats[3 * id(x, y, z) + 2]);
        chr_region_t &R = h_regions[nreg++];
        std::memset(&R, 0, sizeof(R));
        const int64_t dims[3] = {nx, ny, nz};
        for (int a = 0; a < 3; ++a) {
            int64_t olo, elo, ohi, ehi;
            win(blo[a], dims[a], &olo, &elo);
            win(bhi[a], dims[a], &ohi, &ehi);
            R.lo[a] = (int32_t)blo[a];
            R.hi[a] = (int32_t)bhi[a];
            R.origin[a] = (int32_t)olo;
            R.extent[a] = (int32_t)(ohi + ehi - olo);
        }
        R.mask = k;
        double e = dm * sf;
        if (k == 0 && loose < e) e = loose;
        R.error_bound = e;
        R.codec_id = -1;
    });
    *n_regions = nreg;
    return CHR_OK;
}
