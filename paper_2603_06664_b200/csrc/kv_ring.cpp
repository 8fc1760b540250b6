// kv_ring.cpp -- see kv_ring.hpp.
#include "kv_ring.hpp"

#include <string>

#include "common.hpp"

namespace spx {

FrameRing::FrameRing(int64_t capacity_frames, int64_t window_frames)
    : capacity_(capacity_frames), window_(window_frames) {
    require(capacity_frames >= 1, SPX_ERR_CONFIG, "kv ring capacity must be >= 1 frame");
    require(window_frames < 0 || window_frames >= 1, SPX_ERR_CONFIG,
            "window_frames must be >= 1 when set");
    require(window_frames < 0 || window_frames <= capacity_frames, SPX_ERR_CONFIG,
            "window_frames exceeds the ring capacity");
}

int64_t FrameRing::update(int64_t block_index, int64_t num_frames) {
    require(num_frames >= 1, SPX_ERR_ALIGNMENT, "a block must hold at least one frame");
    // re-denoising the same block: its previous frames are dropped, then re-appended
    while (!frames_.empty() && frames_.back().block_index == block_index) frames_.pop_back();
    const int64_t after = cached_frames() + num_frames;
    const int64_t survivors = window_ < 0 ? after : (after < window_ ? after : window_);
    require(survivors <= capacity_, SPX_ERR_RANGE,
            "kv ring capacity of " + std::to_string(capacity_) + " frames exceeded (" +
                std::to_string(survivors) + " frames would be visible)");
    const int64_t first = frames_.empty() ? 0 : (frames_.back().slot + 1) % capacity_;
    for (int64_t f = 0; f < num_frames; ++f)
        frames_.push_back(Frame{block_index, (first + f) % capacity_});
    if (window_ >= 0) {
        while (cached_frames() > window_) frames_.pop_front();
    }
    return first;
}

int64_t FrameRing::oldest_block_index() const {
    require(!frames_.empty(), SPX_ERR_EMPTY_CACHE, "oldest_block_index() on an empty cache");
    return frames_.front().block_index;
}

std::vector<std::pair<int64_t, int64_t>> FrameRing::segments() const {
    std::vector<std::pair<int64_t, int64_t>> out;
    for (const Frame& f : frames_) {
        if (!out.empty() && out.back().first + out.back().second == f.slot) {
            ++out.back().second;
        } else {
            out.emplace_back(f.slot, 1);
        }
    }
    return out;
}

std::vector<std::pair<int64_t, int64_t>> FrameRing::frames() const {
    std::vector<std::pair<int64_t, int64_t>> out;
    for (const Frame& f : frames_) out.emplace_back(f.block_index, f.slot);
    return out;
}

void KvRingStorage::allocate() {
    int prev = 0;
    SPX_CUDA(cudaGetDevice(&prev));
    SPX_CUDA(cudaSetDevice(device));
    const size_t bytes = static_cast<size_t>(rows() * row_elems()) * sizeof(__nv_bfloat16);
    SPX_CUDA(cudaMalloc(&k, bytes));
    SPX_CUDA(cudaMalloc(&v, bytes));
    SPX_CUDA(cudaMemset(k, 0, bytes));
    SPX_CUDA(cudaMemset(v, 0, bytes));
    SPX_CUDA(cudaSetDevice(prev));
}

void KvRingStorage::release() {
    if (!k && !v) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaFree(k);
    cudaFree(v);
    cudaSetDevice(prev);
    k = v = nullptr;
}

}  // namespace spx
