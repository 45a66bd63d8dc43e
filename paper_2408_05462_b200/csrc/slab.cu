// slab.cu -- the z-slab request: finishing a rank's portion
// of a region window.  A portion's tokens are decoded with e = 1/2, so the
// decoder writes u_local (the 3D inclusive prefix of the portion's quanta,
// an exact integer in f64); the true u adds the z-carry plane C (u at the
// plane before the portion: the sum of the earlier portions' last-plane
// u_local, all-gathered), and recon = u * 2e exactly as the single-GPU
// decoder computes it (kernels.py:131-166: recon = u * 2e after the prefix).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "chr_internal.cuh"

namespace chr {

struct PortionDev {
    uint64_t out_offset;   // first sample of the portion in the windows buffer
    int64_t plane;         // samples per plane (ex * ey)
    int64_t nplanes;
    int64_t carry_offset;  // int64 carry plane in d_carry, -1: none (first portion)
    double twoe;
};

__global__ void __launch_bounds__(256) k_portion_finish(double *__restrict__ w, const PortionDev *__restrict__ tab,
                                                        int64_t n, const int64_t *__restrict__ carry) {
    for (int64_t p = blockIdx.y; p < n; p += gridDim.y) {
        const PortionDev P = tab[p];
        const int64_t cnt = P.plane * P.nplanes;
        double *o = w + P.out_offset;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
            int64_t u = __double2ll_rn(o[i]);
            if (P.carry_offset >= 0) u += __ldg(carry + P.carry_offset + i % P.plane);
            o[i] = __dmul_rn((double)u, P.twoe);
        }
    }
}

}  // namespace chr

using namespace chr;

extern "C" int chr_portion_finish(double *d_windows, const uint64_t *h_out_offset, const int64_t *h_plane,
                                  const int64_t *h_nplanes, const int64_t *h_carry_offset, const double *h_error_bound,
                                  int64_t n, const int64_t *d_carry, void *d_ws, size_t ws_bytes, void *stream) {
    CHR_XFER_SCOPE;
    if (n == 0) return CHR_OK;
    if (!d_windows || n < 0 || !h_out_offset || !h_plane || !h_nplanes || !h_carry_offset || !h_error_bound)
        return CHR_E_PARAMETER;
    if (!d_ws || ws_bytes < sizeof(PortionDev) * (size_t)n) return CHR_E_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    std::vector<PortionDev> t((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        if (h_plane[i] < 1 || h_nplanes[i] < 0 || (h_carry_offset[i] >= 0 && !d_carry)) return CHR_E_PARAMETER;
        t[i].out_offset = h_out_offset[i];
        t[i].plane = h_plane[i];
        t[i].nplanes = h_nplanes[i];
        t[i].carry_offset = h_carry_offset[i];
        t[i].twoe = 2.0 * h_error_bound[i];
    }
    PortionDev *d_tab = reinterpret_cast<PortionDev *>(d_ws);
    CHR_CUDA_TRY(h2d(d_tab, t.data(), sizeof(PortionDev) * (size_t)n, st));
    {
        CHR_PROF("k_portion_finish", st);
        k_portion_finish<<<dim3(64, (unsigned)std::min<int64_t>(n, 65535)), 256, 0, st>>>(d_windows, d_tab, n, d_carry);
    }
    return cudaGetLastError() == cudaSuccess ? CHR_OK : CHR_E_CUDA;
}
