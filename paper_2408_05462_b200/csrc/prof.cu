// prof.cu -- opt-in per-kernel timing with CUDA events on the launching
// stream, plus a launch counter.  Used by bench.py to report the dominant
// kernel's duration (roofline) and the number of kernels launched.
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "chr_internal.cuh"

namespace chr {

namespace {
std::mutex g_mu;
bool g_on = false;
long long g_launches = 0;
struct Rec {
    const char *name;
    cudaEvent_t a, b;
};
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t take_event() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

ProfScope::ProfScope(const char *name, cudaStream_t st) : name_(name), st_(st), a_(nullptr) {
    std::lock_guard<std::mutex> lk(g_mu);
    ++g_launches;
    if (g_on) {
        a_ = take_event();
        cudaEventRecord(a_, st_);
    }
}

// CHR_DEBUG_SYNC=1: synchronise after every profiled launch and name the
// kernel that failed (debugging only: serialises the library)
static const bool g_debug_sync = [] {
    const char *e = std::getenv("CHR_DEBUG_SYNC");
    return e && e[0] == '1';
}();

ProfScope::~ProfScope() {
    if (g_debug_sync) {
        const cudaError_t e = cudaStreamSynchronize(st_);
        const cudaError_t l = cudaGetLastError();
        if (e != cudaSuccess || l != cudaSuccess)
            std::fprintf(stderr, "chr: %s failed: %s / %s\n", name_, cudaGetErrorString(e), cudaGetErrorString(l));
    }
    if (!a_) return;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaEvent_t b = take_event();
    cudaEventRecord(b, st_);
    g_recs.push_back({name_, a_, b});
}

}  // namespace chr

using namespace chr;

extern "C" void chr_prof_enable(int on) {
    CHR_XFER_SCOPE;
    std::lock_guard<std::mutex> lk(g_mu);
    g_on = on != 0;
}

extern "C" long long chr_launch_count(void) {
    CHR_XFER_SCOPE;
    std::lock_guard<std::mutex> lk(g_mu);
    return g_launches;
}

// "name count total_ms\n" per kernel name since the last report; clears.
extern "C" int chr_prof_report(char *buf, size_t cap) {
    CHR_XFER_SCOPE;
    std::lock_guard<std::mutex> lk(g_mu);
    std::map<std::string, std::pair<long long, double>> agg;
    for (const Rec &r : g_recs) {
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        auto &x = agg[r.name];
        x.first += 1;
        x.second += ms;
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_recs.clear();
    std::string s;
    for (auto &kv : agg) {
        char line[256];
        snprintf(line, sizeof(line), "%s %lld %.6f\n", kv.first.c_str(), kv.second.first, kv.second.second);
        s += line;
    }
    if (buf && cap) {
        const size_t n = std::min(cap - 1, s.size());
        memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    return (int)s.size();
}

// "name start_ms end_ms\n" per recorded launch (relative to the first
// record's start), in launch order; clears like chr_prof_report.
extern "C" int chr_prof_timeline(char *buf, size_t cap) {
    CHR_XFER_SCOPE;
    std::lock_guard<std::mutex> lk(g_mu);
    std::string s;
    cudaEvent_t t0 = g_recs.empty() ? nullptr : g_recs.front().a;
    for (const Rec &r : g_recs) {
        cudaEventSynchronize(r.b);
        float a = 0.f, b = 0.f;
        cudaEventElapsedTime(&a, t0, r.a);
        cudaEventElapsedTime(&b, t0, r.b);
        char line[256];
        snprintf(line, sizeof(line), "%s %.4f %.4f\n", r.name, a, b);
        s += line;
    }
    for (const Rec &r : g_recs) {
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_recs.clear();
    if (buf && cap) {
        const size_t n = std::min(cap - 1, s.size());
        memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    return (int)s.size();
}

// a named zero-length record on the stream (host-side phase marks in the
// timeline; not counted as a launch).  The name must outlive the report.
extern "C" void chr_prof_mark(const char *name, void *stream) {
    CHR_XFER_SCOPE;
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_on) return;
    static std::map<std::string, std::string> names;  // stable storage
    const char *nm = names.emplace(name, std::string("@") + name).first->second.c_str();
    cudaEvent_t a = take_event(), b = take_event();
    cudaEventRecord(a, (cudaStream_t)stream);
    cudaEventRecord(b, (cudaStream_t)stream);
    g_recs.push_back({nm, a, b});
}
