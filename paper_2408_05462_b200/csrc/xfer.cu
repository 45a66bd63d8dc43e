// xfer.cu -- the library's small host<->device transfers without the copy
// engines.  A caller pipelining bulk transfers (hundreds of MB on the DMA
// engines, other streams) would otherwise hold every small plan/size copy
// of the library behind them in the engines' queues.  Small transfers go
// through a thread-local pinned, mapped ring instead: host->device copies
// are staged there and pulled by a tiny kernel on the caller's stream;
// device->host copies are pushed into it by a kernel and delivered to the
// destination at the next chr::stream_sync() of that stream.  Transfers
// above kXferBig keep cudaMemcpyAsync.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "chr_internal.cuh"

namespace chr {

namespace {
constexpr size_t kXferBig = 4u << 20;

struct Pending {
    const uint8_t *src;
    void *dst;
    size_t n;
    cudaStream_t st;
};

struct Ring {
    uint8_t *buf = nullptr;
    size_t cap = 0, head = 0;
    std::vector<Pending> pend;
    std::vector<cudaStream_t> users;  // streams with ring traffic since the last reset
};

thread_local Ring g_ring;

__global__ void k_xfer(const uint8_t *__restrict__ src, uint8_t *__restrict__ dst, size_t n) {
    const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
    if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
        const size_t n16 = n >> 4;
        for (size_t i = i0; i < n16; i += stride)
            reinterpret_cast<uint4 *>(dst)[i] = reinterpret_cast<const uint4 *>(src)[i];
        for (size_t i = (n16 << 4) + i0; i < n; i += stride) dst[i] = src[i];
    } else {
        for (size_t i = i0; i < n; i += stride) dst[i] = src[i];
    }
}

// small copies through the copy engines (1) or by kernels (0): a caller that
// keeps the engines busy with bulk transfers wants kernels (the default);
// CHR_XFER=dma / chr_set_xfer_mode(1) for callers that do not
int g_xfer_dma = [] {
    const char *e = std::getenv("CHR_XFER");
    return e && std::strcmp(e, "dma") == 0 ? 1 : 0;
}();

cudaError_t launch_xfer(const void *src, void *dst, size_t n, cudaStream_t st) {
    if (g_xfer_dma) return cudaMemcpyAsync(dst, src, n, cudaMemcpyDefault, st);
    const unsigned blocks = (unsigned)std::min<size_t>(64, (n + 4095) / 4096 + 1);
    CHR_PROF("k_xfer", st);
    k_xfer<<<blocks, 256, 0, st>>>((const uint8_t *)src, (uint8_t *)dst, n);
    return cudaGetLastError();
}

void deliver(cudaStream_t st) {
    Ring &R = g_ring;
    size_t k = 0;
    for (const Pending &p : R.pend) {
        if (p.st == st) std::memcpy(p.dst, p.src, p.n);
        else R.pend[k++] = p;
    }
    R.pend.resize(k);
}

cudaError_t reserve(size_t n, cudaStream_t st, uint8_t **out) {
    Ring &R = g_ring;
    n = (n + 255) & ~size_t(255);
    if (R.head + n > R.cap) {  // wait for every stream using the ring, then reuse (or grow) it
        for (cudaStream_t s : R.users) {
            const cudaError_t e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) return e;
            deliver(s);
        }
        R.users.clear();
        R.head = 0;
        if (n > R.cap) {
            if (R.buf) cudaFreeHost(R.buf);
            R.buf = nullptr;
            R.cap = std::max({n, R.cap * 2, size_t(8) << 20});
            const cudaError_t e = cudaHostAlloc(reinterpret_cast<void **>(&R.buf), R.cap,
                                                cudaHostAllocMapped | cudaHostAllocPortable);
            if (e != cudaSuccess) {
                R.cap = 0;
                return e;
            }
        }
    }
    *out = R.buf + R.head;
    R.head += n;
    if (std::find(R.users.begin(), R.users.end(), st) == R.users.end()) R.users.push_back(st);
    return cudaSuccess;
}
}  // namespace

namespace {
struct CopySet {
    const uint8_t *src[kFillMax];
    uint8_t *dst[kFillMax];
    size_t n[kFillMax];
};

__global__ void k_xfer_multi(CopySet set) {
    const uint8_t *src = set.src[blockIdx.y];
    uint8_t *dst = set.dst[blockIdx.y];
    const size_t n = set.n[blockIdx.y];
    const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
    if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
        const size_t n16 = n >> 4;
        for (size_t i = i0; i < n16; i += stride)
            reinterpret_cast<uint4 *>(dst)[i] = reinterpret_cast<const uint4 *>(src)[i];
        for (size_t i = (n16 << 4) + i0; i < n; i += stride) dst[i] = src[i];
    } else {
        for (size_t i = i0; i < n; i += stride) dst[i] = src[i];
    }
}

cudaError_t launch_multi(const CopySet &set, int count, size_t most, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    if (g_xfer_dma) {
        for (int i = 0; i < count; ++i) {
            const cudaError_t e = cudaMemcpyAsync(set.dst[i], set.src[i], set.n[i], cudaMemcpyDefault, st);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    const unsigned bx = (unsigned)std::min<size_t>(64, (most + 4095) / 4096 + 1);
    CHR_PROF("k_xfer", st);
    k_xfer_multi<<<dim3(bx, count), 256, 0, st>>>(set);
    return cudaGetLastError();
}
}  // namespace

// several small host->device copies staged in the ring and pulled by one launch
cudaError_t h2d_multi(std::initializer_list<Xfer> xs, cudaStream_t st) {
    CopySet set;
    int count = 0;
    size_t most = 0;
    for (const Xfer &x : xs) {
        if (x.n == 0) continue;
        if (x.n > kXferBig || count == kFillMax) {
            const cudaError_t e = h2d(x.dst, x.src, x.n, st);
            if (e != cudaSuccess) return e;
            continue;
        }
        uint8_t *p = nullptr;
        const cudaError_t e = reserve(x.n, st, &p);
        if (e != cudaSuccess) return e;
        std::memcpy(p, x.src, x.n);
        set.src[count] = p;
        set.dst[count] = (uint8_t *)x.dst;
        set.n[count] = x.n;
        most = std::max(most, x.n);
        ++count;
    }
    return launch_multi(set, count, most, st);
}

// several small device->host copies pushed by one launch, delivered at stream_sync
cudaError_t d2h_multi(std::initializer_list<Xfer> xs, cudaStream_t st) {
    CopySet set;
    int count = 0;
    size_t most = 0;
    for (const Xfer &x : xs) {
        if (x.n == 0) continue;
        if (x.n > kXferBig || count == kFillMax) {
            const cudaError_t e = d2h(x.dst, x.src, x.n, st);
            if (e != cudaSuccess) return e;
            continue;
        }
        uint8_t *p = nullptr;
        const cudaError_t e = reserve(x.n, st, &p);
        if (e != cudaSuccess) return e;
        set.src[count] = (const uint8_t *)x.src;
        set.dst[count] = p;
        set.n[count] = x.n;
        most = std::max(most, x.n);
        g_ring.pend.push_back({p, x.dst, x.n, st});
        ++count;
    }
    return launch_multi(set, count, most, st);
}

cudaError_t h2d(void *dst, const void *src, size_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    if (n > kXferBig) return cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st);
    uint8_t *p = nullptr;
    cudaError_t e = reserve(n, st, &p);
    if (e != cudaSuccess) return e;
    std::memcpy(p, src, n);
    return launch_xfer(p, dst, n, st);
}

// device -> host into the pinned ring without the copy-out at stream_sync:
// the returned pointer is readable after the next stream_sync(st) and valid
// until the next transfer of this thread (nullptr: too large for the ring)
const void *d2h_view(const void *src, size_t n, cudaStream_t st, cudaError_t *err) {
    *err = cudaSuccess;
    if (n == 0 || n > kXferBig) return nullptr;
    uint8_t *p = nullptr;
    *err = reserve(n, st, &p);
    if (*err != cudaSuccess) return nullptr;
    *err = launch_xfer(src, p, n, st);
    return *err == cudaSuccess ? p : nullptr;
}

cudaError_t d2h(void *dst, const void *src, size_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    if (n > kXferBig) return cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st);
    uint8_t *p = nullptr;
    cudaError_t e = reserve(n, st, &p);
    if (e != cudaSuccess) return e;
    e = launch_xfer(src, p, n, st);
    if (e == cudaSuccess) g_ring.pend.push_back({p, dst, n, st});
    return e;
}

namespace {
__global__ void k_fill(uint8_t *__restrict__ dst, int v, size_t n) {
    const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
    const uint32_t w = 0x01010101u * (uint32_t)(v & 0xFF);
    if (((uintptr_t)dst & 15) == 0) {
        const size_t n16 = n >> 4;
        for (size_t i = i0; i < n16; i += stride) reinterpret_cast<uint4 *>(dst)[i] = make_uint4(w, w, w, w);
        for (size_t i = (n16 << 4) + i0; i < n; i += stride) dst[i] = (uint8_t)v;
    } else {
        for (size_t i = i0; i < n; i += stride) dst[i] = (uint8_t)v;
    }
}
}  // namespace

// cudaMemsetAsync as a kernel (no copy engine)
cudaError_t fill_async(void *dst, int v, size_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)std::min<size_t>(1184, (n + 16383) / 16384 + 1);
    CHR_PROF("k_fill", st);
    k_fill<<<blocks, 256, 0, st>>>((uint8_t *)dst, v, n);
    return cudaGetLastError();
}

namespace {
struct FillSet {
    uint8_t *ptr[kFillMax];
    size_t n[kFillMax];
    int count;
};

// one launch zero-fills up to kFillMax ranges: blockIdx.y picks the range
__global__ void k_fill_multi(FillSet set) {
    uint8_t *dst = set.ptr[blockIdx.y];
    const size_t n = set.n[blockIdx.y];
    const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
    if (((uintptr_t)dst & 15) == 0) {
        const size_t n16 = n >> 4;
        for (size_t i = i0; i < n16; i += stride) reinterpret_cast<uint4 *>(dst)[i] = make_uint4(0, 0, 0, 0);
        for (size_t i = (n16 << 4) + i0; i < n; i += stride) dst[i] = 0;
    } else {
        for (size_t i = i0; i < n; i += stride) dst[i] = 0;
    }
}
}  // namespace

cudaError_t zero_async(std::initializer_list<std::pair<void *, size_t>> ranges, cudaStream_t st) {
    FillSet set;
    set.count = 0;
    size_t most = 0;
    for (const auto &r : ranges) {
        if (!r.first || r.second == 0) continue;
        if (set.count == kFillMax) return cudaErrorInvalidValue;
        set.ptr[set.count] = (uint8_t *)r.first;
        set.n[set.count] = r.second;
        most = std::max(most, r.second);
        ++set.count;
    }
    if (set.count == 0) return cudaSuccess;
    const unsigned bx = (unsigned)std::min<size_t>(1184, (most + 16383) / 16384 + 1);
    CHR_PROF("k_fill", st);
    k_fill_multi<<<dim3(bx, set.count), 256, 0, st>>>(set);
    return cudaGetLastError();
}

// device-accessible pointers (device or mapped pinned host), any alignment
cudaError_t copy_async(void *dst, const void *src, size_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    return launch_xfer(src, dst, n, st);
}

cudaError_t stream_sync(cudaStream_t st) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    Ring &R = g_ring;
    deliver(st);
    if (R.users.size() == 1 && R.users[0] == st) {  // nothing else in flight in the ring
        R.users.clear();
        R.head = 0;
    }
    return cudaSuccess;
}

Side *side_stream() {
    static const bool off = [] {
        const char *e = std::getenv("CHR_NO_SIDE");
        return e && e[0] == '1';
    }();
    if (off) return nullptr;
    constexpr int kMaxDev = 64;
    thread_local Side sides[kMaxDev];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
    Side &S = sides[dev];
    if (!S.st) {
        if (cudaStreamCreateWithFlags(&S.st, cudaStreamNonBlocking) != cudaSuccess) {
            S.st = nullptr;
            return nullptr;
        }
        for (cudaEvent_t &e : S.ev)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    }
    return &S;
}

XferScope::XferScope() : mark_(g_ring.pend.size()) {}
XferScope::~XferScope() {  // undelivered copies of this call (an error path) must not outlive its buffers
    if (g_ring.pend.size() > mark_) g_ring.pend.resize(mark_);
}

}  // namespace chr

using namespace chr;

// copy between device-accessible pointers (device memory or pinned host
// memory) with a kernel on `stream`: no copy engine, any alignment
extern "C" int chr_set_xfer_mode(int dma) {
    const int old = g_xfer_dma;
    g_xfer_dma = dma ? 1 : 0;
    return old;
}

extern "C" int chr_copy(void *dst, const void *src, uint64_t nbytes, void *stream) {
    if (nbytes && (!dst || !src)) return CHR_E_PARAMETER;
    return copy_async(dst, src, nbytes, (cudaStream_t)stream) == cudaSuccess ? CHR_OK : CHR_E_CUDA;
}
