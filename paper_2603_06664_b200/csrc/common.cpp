// common.cpp -- error message storage, launch accounting, device queries.
#include "common.hpp"

#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <algorithm>
#include <vector>

namespace spx {

namespace {
thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }
const std::string& last_error() { return g_last_error; }

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SPX_PDL");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

namespace {
constexpr int64_t kSpanSlots = 8192;
unsigned long long* g_spans = nullptr;  // [slots][2]
int64_t g_span_next = 0;
}  // namespace

bool span_tracing() {
    static const bool on = [] {
        const char* e = std::getenv("SPX_SPAN_TRACE");
        return e && std::atoi(e) == 1;
    }();
    return on;
}

unsigned long long* span_slot() {
    if (!span_tracing()) return nullptr;
    if (!g_spans) {
        SPX_CUDA(cudaMalloc(&g_spans, kSpanSlots * 2 * sizeof(unsigned long long)));
        std::vector<unsigned long long> init(kSpanSlots * 2);
        for (int64_t i = 0; i < kSpanSlots; ++i) {
            init[2 * i] = ~0ull;
            init[2 * i + 1] = 0;
        }
        SPX_CUDA(cudaMemcpy(g_spans, init.data(), init.size() * 8, cudaMemcpyHostToDevice));
    }
    if (g_span_next >= kSpanSlots) return nullptr;
    return g_spans + 2 * (g_span_next++);
}

int64_t span_count() { return g_span_next; }

void span_dump(uint64_t* out, int64_t n) {
    if (!g_spans) return;
    SPX_CUDA(cudaDeviceSynchronize());
    SPX_CUDA(cudaMemcpy(out, g_spans, static_cast<size_t>(std::min(n, g_span_next)) * 16,
                        cudaMemcpyDeviceToHost));
}

int device_sm_count(int device) {
    static std::mutex mu;
    static std::map<int, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(device);
    if (it != cache.end()) return it->second;
    int sms = 0;
    SPX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    cache[device] = sms;
    return sms;
}

}  // namespace spx
