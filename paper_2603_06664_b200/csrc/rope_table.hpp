// rope_table.hpp -- the precomputed 3-D RoPE table (reference: RopeFrequencyTable /
// precompute_frequencies, proj/include/spattn/rope.hpp:52-99, proj/src/rope.cpp:21-64).
// Host copy in fp64 (bit-identical to the reference), device copies in fp32 per GPU.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <vector>

namespace spx {

struct BandSplit {
    int64_t temporal = 0, height = 0, width = 0;
    int64_t total() const { return temporal + height + width; }
    static BandSplit defaults_for(int64_t head_dim);  // rope.cpp:15-19
};

struct DeviceRopeTable {
    float2* band[3] = {nullptr, nullptr, nullptr};
};

class RopeTable {
  public:
    RopeTable(int64_t max_frames, int64_t max_h, int64_t max_w, int64_t head_dim, double base,
              const BandSplit& split);
    ~RopeTable();
    RopeTable(const RopeTable&) = delete;
    RopeTable& operator=(const RopeTable&) = delete;

    int64_t max_pos(int band) const { return max_pos_[band]; }
    int64_t pairs(int band) const {
        return band == 0 ? split_.temporal : band == 1 ? split_.height : split_.width;
    }
    const BandSplit& split() const { return split_; }
    int64_t head_dim() const { return head_dim_; }
    double base() const { return base_; }
    double cos_at(int band, int64_t pos, int64_t pair) const {
        return data_[band][static_cast<size_t>((pos * pairs(band) + pair) * 2)];
    }
    double sin_at(int band, int64_t pos, int64_t pair) const {
        return data_[band][static_cast<size_t>((pos * pairs(band) + pair) * 2 + 1)];
    }
    // fp32 table on `device` (uploaded on first use; synchronous)
    const DeviceRopeTable& on_device(int device) const;

  private:
    int64_t max_pos_[3];
    int64_t head_dim_;
    double base_;
    BandSplit split_;
    std::vector<double> data_[3];
    mutable std::mutex mu_;
    mutable std::map<int, DeviceRopeTable> device_;
};

}  // namespace spx
