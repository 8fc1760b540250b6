// kv_ring.hpp -- rolling KV cache as a device ring of frame slots (reference: KvCache,
// proj/include/spattn/kv_cache.hpp:16-50, proj/src/kv_cache.cpp:18-67).
//
// Bookkeeping is a deque of (block_index, slot) in chronological order; a new frame takes
// the slot after the newest one (mod capacity), so the cached frames always occupy a
// contiguous arc of the ring -> at most two row segments for the attention kernel, and no
// copy on read. update() mirrors the reference order exactly: drop trailing frames of the
// same block, append, then evict from the front while more than `window` frames remain.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <deque>
#include <utility>
#include <vector>

namespace spx {

class FrameRing {
  public:
    FrameRing() = default;
    FrameRing(int64_t capacity_frames, int64_t window_frames /* <0 unlimited */);

    // returns the slot of the first appended frame
    int64_t update(int64_t block_index, int64_t num_frames);
    int64_t cached_frames() const { return static_cast<int64_t>(frames_.size()); }
    int64_t oldest_block_index() const;
    int64_t capacity() const { return capacity_; }
    int64_t window() const { return window_; }
    // chronological slot runs: (first_slot, num_frames), at most 2
    std::vector<std::pair<int64_t, int64_t>> segments() const;
    std::vector<std::pair<int64_t, int64_t>> frames() const;  // (block, slot)

  private:
    struct Frame {
        int64_t block_index;
        int64_t slot;
    };
    int64_t capacity_ = 0;
    int64_t window_ = -1;
    std::deque<Frame> frames_;
};

// Device storage for one ring: k and v, each [capacity_frames * tokens_per_frame][H][D] bf16.
struct KvRingStorage {
    int device = 0;
    int64_t tokens_per_frame = 0;
    int64_t capacity_frames = 0;
    int64_t heads = 0;
    int64_t head_dim = 0;
    __nv_bfloat16* k = nullptr;
    __nv_bfloat16* v = nullptr;
    int64_t row_elems() const { return heads * head_dim; }
    int64_t rows() const { return capacity_frames * tokens_per_frame; }
    void allocate();  // zero-filled (masked tail rows are finite)
    void release();
};

}  // namespace spx
