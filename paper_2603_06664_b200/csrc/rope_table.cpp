// rope_table.cpp -- see rope_table.hpp. Angle at position m, pair j of a band with p pairs is
// m * base^(-j/p) (proj/src/rope.cpp:55-57), stored as interleaved (cos, sin).
#include "rope_table.hpp"

#include <cmath>
#include <string>

#include "common.hpp"

namespace spx {

BandSplit BandSplit::defaults_for(int64_t head_dim) {
    const int64_t pairs = head_dim / 2;
    const int64_t spatial = pairs / 3;
    return BandSplit{pairs - 2 * spatial, spatial, spatial};
}

RopeTable::RopeTable(int64_t max_frames, int64_t max_h, int64_t max_w, int64_t head_dim,
                     double base, const BandSplit& split)
    : max_pos_{max_frames, max_h, max_w}, head_dim_(head_dim), base_(base), split_(split) {
    require(head_dim >= 2 && head_dim % 2 == 0, SPX_ERR_CONFIG,
            "head_dim must be even and >= 2, got " + std::to_string(head_dim));
    require(split.temporal >= 0 && split.height >= 0 && split.width >= 0 &&
                split.total() == head_dim / 2,
            SPX_ERR_CONFIG,
            "band split (" + std::to_string(split.temporal) + ", " +
                std::to_string(split.height) + ", " + std::to_string(split.width) +
                ") must sum to D/2 = " + std::to_string(head_dim / 2));
    require(max_frames >= 1 && max_h >= 1 && max_w >= 1, SPX_ERR_CONFIG,
            "table extents must be >= 1");
    require(base > 0.0, SPX_ERR_CONFIG, "frequency base must be positive");
    for (int band = 0; band < 3; ++band) {
        const int64_t p = pairs(band);
        std::vector<double>& out = data_[band];
        out.resize(static_cast<size_t>(max_pos_[band] * p * 2));
        for (int64_t j = 0; j < p; ++j) {
            const double freq = std::pow(base, -static_cast<double>(j) / static_cast<double>(p));
            for (int64_t m = 0; m < max_pos_[band]; ++m) {
                const double angle = static_cast<double>(m) * freq;
                out[static_cast<size_t>((m * p + j) * 2)] = std::cos(angle);
                out[static_cast<size_t>((m * p + j) * 2 + 1)] = std::sin(angle);
            }
        }
    }
}

RopeTable::~RopeTable() {
    for (auto& kv : device_) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(kv.first);
        for (auto* p : kv.second.band) cudaFree(p);
        cudaSetDevice(prev);
    }
}

const DeviceRopeTable& RopeTable::on_device(int device) const {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = device_.find(device);
    if (it != device_.end()) return it->second;
    int prev = 0;
    SPX_CUDA(cudaGetDevice(&prev));
    SPX_CUDA(cudaSetDevice(device));
    DeviceRopeTable t;
    for (int band = 0; band < 3; ++band) {
        const size_t n = static_cast<size_t>(max_pos_[band] * pairs(band));
        std::vector<float2> host(n > 0 ? n : 1);
        for (size_t i = 0; i < n; ++i)
            host[i] = make_float2(static_cast<float>(data_[band][2 * i]),
                                  static_cast<float>(data_[band][2 * i + 1]));
        SPX_CUDA(cudaMalloc(&t.band[band], host.size() * sizeof(float2)));
        SPX_CUDA(cudaMemcpy(t.band[band], host.data(), host.size() * sizeof(float2),
                            cudaMemcpyHostToDevice));
    }
    // a pageable H2D copy may return before its DMA lands and the engine streams are
    // non-blocking: the table is complete before any kernel (which may read it before its
    // griddepcontrol.wait, RopeLaunch::tab_constant) can be enqueued
    SPX_CUDA(cudaDeviceSynchronize());
    SPX_CUDA(cudaSetDevice(prev));
    return device_.emplace(device, t).first->second;
}

}  // namespace spx
