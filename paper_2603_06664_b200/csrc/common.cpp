// common.cpp -- error message storage, launch accounting, device queries.
#include "common.hpp"

#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>

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
