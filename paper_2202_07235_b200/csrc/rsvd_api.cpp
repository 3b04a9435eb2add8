// rsvd_api.cpp -- status plumbing of the C ABI (thread-local last-error string, CUDA error mapping).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rsvd.h"

namespace rsvd {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

rsvd_status fail(rsvd_status st, const std::string &msg) {
    g_last_error = msg;
    return st;
}

rsvd_status cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return RSVD_OK;
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return RSVD_ERR_CUDA;
}

// ------------------------------------------------------------------ launch counter / kernel timing
static std::atomic<long long> g_launches{0};
void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

struct TimedSpan { cudaEvent_t a, b; int kind; };
static std::mutex g_tmu;
static bool g_timing = false;
static std::vector<cudaEvent_t> g_pool;
static std::vector<TimedSpan> g_spans;

bool timing_enabled() {
    std::lock_guard<std::mutex> g(g_tmu);
    return g_timing;
}

cudaEvent_t timing_event(cudaStream_t s) {
    cudaEvent_t e = nullptr;
    {
        std::lock_guard<std::mutex> g(g_tmu);
        if (!g_pool.empty()) { e = g_pool.back(); g_pool.pop_back(); }
    }
    if (!e && cudaEventCreate(&e) != cudaSuccess) return nullptr;
    cudaEventRecord(e, s);
    return e;
}

void timing_span(cudaEvent_t a, cudaEvent_t b, int kind) {
    if (!a || !b) return;
    std::lock_guard<std::mutex> g(g_tmu);
    g_spans.push_back({a, b, kind});
}

}  // namespace rsvd

extern "C" int64_t rsvd_launch_count(void) { return rsvd::g_launches.load(); }

extern "C" void rsvd_timing_enable(int32_t on) {
    std::lock_guard<std::mutex> g(rsvd::g_tmu);
    rsvd::g_timing = on != 0;
}

extern "C" rsvd_status rsvd_timing_read(double *ms, int64_t *count, int32_t nkinds) {
    using namespace rsvd;
    std::vector<TimedSpan> spans;
    {
        std::lock_guard<std::mutex> g(g_tmu);
        spans.swap(g_spans);
    }
    for (int i = 0; i < nkinds; ++i) { if (ms) ms[i] = 0.0; if (count) count[i] = 0; }
    rsvd_status st = RSVD_OK;
    std::vector<cudaEvent_t> done;
    for (const auto &sp : spans) {
        float t = 0.f;
        cudaError_t e = cudaEventSynchronize(sp.b);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&t, sp.a, sp.b);
        if (e != cudaSuccess) st = cuda_check(e, "timing read");
        if (sp.kind >= 0 && sp.kind < nkinds) {
            if (ms) ms[sp.kind] += t;
            if (count) count[sp.kind] += 1;
        }
        done.push_back(sp.a);
        done.push_back(sp.b);
    }
    std::sort(done.begin(), done.end());
    done.erase(std::unique(done.begin(), done.end()), done.end());
    std::lock_guard<std::mutex> g(g_tmu);
    for (auto e : done) g_pool.push_back(e);
    return st;
}

extern "C" const char *rsvd_last_error(void) { return rsvd::g_last_error.c_str(); }
extern "C" int32_t rsvd_abi_version(void) { return 6; }
