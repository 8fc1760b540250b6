// spx_adapter.hpp -- the reference-side C++ adapter: spattn::-shaped
// functions over the C ABI of libspx.so (include/spx.h), so that code written against the
// reference (/root/reference/proj, namespace spattn) calls the B200 path. fp64 Tensor4 in and
// out; the device computes in bf16 / fp32 (include/spx.h). Header-only; a maintainer adds it
// under proj/include/spattn/ and links libspx.so + cudart.
// integration/adapter_check.cpp compiles it against the reference headers and sources.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "spattn/errors.hpp"
#include "spattn/generator.hpp"
#include "spattn/rope.hpp"
#include "spattn/sp_attention.hpp"
#include "spattn/tensor.hpp"
#include "spx.h"

namespace spattn::spx_adapter {

// spx_status -> the reference exception taxonomy (errors.hpp:8-36)
inline void check(spx_status s) {
    if (s == SPX_OK) return;
    const std::string m = spx_last_error();
    switch (s) {
        case SPX_ERR_SHAPE: throw ShapeError(m);
        case SPX_ERR_PARTITION: throw PartitionError(m);
        case SPX_ERR_CONFIG: throw ConfigError(m);
        case SPX_ERR_RANGE: throw RangeError(m);
        case SPX_ERR_ALIGNMENT: throw AlignmentError(m);
        case SPX_ERR_EMPTY_CACHE: throw EmptyCacheError(m);
        case SPX_ERR_COLLECTIVE: throw CollectiveError(m);
        default: throw std::runtime_error(std::string(spx_status_name(s)) + ": " + m);
    }
}

inline double bf16_to_double(uint16_t b) {
    const uint32_t u = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

struct DeviceBuf {  // bf16 staging of a Tensor4 (or n elements)
    void* p = nullptr;
    size_t n = 0;
    explicit DeviceBuf(const Tensor4& t) : n(static_cast<size_t>(t.numel())) {
        std::vector<uint16_t> h(n);
        check(spx_f64_to_bf16(t.data(), h.data(), static_cast<int64_t>(n)));
        if (cudaMalloc(&p, n * 2) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
        cudaMemcpy(p, h.data(), n * 2, cudaMemcpyHostToDevice);
    }
    explicit DeviceBuf(size_t count) : n(count) {
        if (cudaMalloc(&p, n * 2) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
    }
    ~DeviceBuf() { cudaFree(p); }
    DeviceBuf(const DeviceBuf&) = delete;
    DeviceBuf& operator=(const DeviceBuf&) = delete;
    Tensor4 download(Shape4 s) const {
        std::vector<uint16_t> h(n);
        cudaMemcpy(h.data(), p, n * 2, cudaMemcpyDeviceToHost);
        std::vector<double> d(n);
        for (size_t i = 0; i < n; ++i) d[i] = bf16_to_double(h[i]);
        return Tensor4(s, std::move(d));
    }
};

// an spx_rope_table owned by a unique_ptr (precompute_frequencies, rope.cpp:21-64)
using TablePtr = std::unique_ptr<spx_rope_table, void (*)(spx_rope_table*)>;
inline TablePtr precompute_frequencies(std::int64_t max_frames, std::int64_t max_h,
                                       std::int64_t max_w, std::int64_t head_dim, double base,
                                       const BandSplit& split) {
    const int64_t sp[3] = {split.temporal, split.height, split.width};
    spx_rope_table* t = nullptr;
    check(spx_rope_table_create(max_frames, max_h, max_w, head_dim, base, sp, &t));
    return TablePtr(t, spx_rope_table_destroy);
}

// global_time_index (rope.cpp:66-70)
inline std::int64_t global_time_index(std::int64_t i_local, std::int64_t rank, std::int64_t local_len,
                                      std::int64_t grid_hw, std::int64_t start_frame) {
    return spx_global_time_index(i_local, rank, local_len, grid_hw, start_frame);
}

// replaces apply_rope_causal_local (rope.cpp:145-164)
inline Tensor4 apply_rope_causal_local(const Tensor4& x, const GridSpec& g, spx_rope_table* table,
                                       std::int64_t start, std::int64_t rank, std::int64_t world) {
    DeviceBuf in(x), out(static_cast<size_t>(x.numel()));
    const int64_t grid[3] = {g.frames, g.height, g.width};
    const Shape4& s = x.shape();
    check(spx_rope_apply_causal_local(table, in.p, out.p, s.batch, s.seq, s.heads, s.head_dim, grid,
                                      start, rank, world, nullptr, 0.f, nullptr));
    return out.download(s);
}

// replaces scaled_dot_product_attention (tensor.cpp:161-209)
inline Tensor4 scaled_dot_product_attention(const Tensor4& q, const Tensor4& k, const Tensor4& v) {
    DeviceBuf dq(q), dk(k), dv(v), o(static_cast<size_t>(q.numel()));
    const Shape4& s = q.shape();
    check(spx_attention(dq.p, dk.p, dv.p, o.p, s.batch, s.seq, k.shape().seq, s.heads, s.head_dim,
                        nullptr));
    return o.download(s);
}

// replaces project_tokens (sp_attention.cpp:51-75)
inline Tensor4 project_tokens(const Tensor4& x, const Matrix& w) {
    DeviceBuf dx(x), dw(Tensor4(Shape4{1, w.rows, 1, w.cols}, w.w));
    DeviceBuf y(static_cast<size_t>(x.shape().batch * x.shape().seq * w.rows));
    const Shape4& s = x.shape();
    check(spx_project_tokens(dx.p, dw.p, y.p, s.batch * s.seq, s.heads * s.head_dim, w.rows, nullptr));
    return y.download(s);
}

// GenerationConfig (generator.hpp:14-42) -> spx_engine_config
inline spx_engine_config engine_config(const GenerationConfig& cfg) {
    spx_engine_config c;
    spx_engine_config_defaults(&c);
    c.frames = cfg.grid_per_block.frames;
    c.grid_h = cfg.grid_per_block.height;
    c.grid_w = cfg.grid_per_block.width;
    c.num_blocks = cfg.num_blocks;
    c.layers = cfg.layers;
    c.denoise_steps = cfg.denoise_steps;
    c.batch = cfg.batch;
    c.heads = cfg.heads;
    c.head_dim = cfg.head_dim;
    c.window_frames = cfg.window_frames ? *cfg.window_frames : -1;
    c.rope_base = cfg.rope_base;
    if (cfg.band_split) {
        c.band_split[0] = cfg.band_split->temporal;
        c.band_split[1] = cfg.band_split->height;
        c.band_split[2] = cfg.band_split->width;
    }
    c.seed = cfg.seed;
    c.force_start_frame_zero = cfg.force_start_frame_zero ? 1 : 0;
    const AblationFlags& a = cfg.variant.ablation;
    c.ablation = (a.use_fused_all_to_all ? SPX_ABLATION_FUSED_ALL_TO_ALL : 0) |
                 (a.use_local_rope ? SPX_ABLATION_LOCAL_ROPE : 0) |
                 (a.use_precomputed_freqs ? SPX_ABLATION_PRECOMPUTED_FREQS : 0);
    return c;
}

// GenerationConfig::validate + the device constraints (generator.cpp:7-38)
inline void validate(const GenerationConfig& cfg) {
    const spx_engine_config c = engine_config(cfg);
    check(spx_engine_config_validate(&c, cfg.world_size));
}

// generate(cfg) (generator.cpp:50-147) on the device: P ranks of a LOCAL world on the current
// GPU, the seeded reference weights and noise rounded to bf16; block outputs as fp64
inline std::vector<Tensor4> generate(const GenerationConfig& cfg) {
    const spx_engine_config c = engine_config(cfg);
    spx_world* world = nullptr;
    check(spx_world_create_local(cfg.world_size, nullptr, &world));
    std::unique_ptr<spx_world, void (*)(spx_world*)> w(world, spx_world_destroy);
    spx_engine* eng = nullptr;
    check(spx_engine_create(world, &c, &eng));
    std::unique_ptr<spx_engine, void (*)(spx_engine*)> e(eng, spx_engine_destroy);
    check(spx_engine_seed_weights(eng));
    const int64_t L = cfg.block_len(), per = L * cfg.heads * cfg.head_dim;
    std::vector<uint16_t> out(static_cast<size_t>(cfg.num_blocks * per));
    check(spx_engine_generate(eng, out.data()));
    std::vector<Tensor4> blocks;
    for (int64_t b = 0; b < cfg.num_blocks; ++b) {
        std::vector<double> d(static_cast<size_t>(per));
        for (int64_t i = 0; i < per; ++i) d[static_cast<size_t>(i)] = bf16_to_double(out[static_cast<size_t>(b * per + i)]);
        blocks.emplace_back(Shape4{1, L, cfg.heads, cfg.head_dim}, std::move(d));
    }
    return blocks;
}

}  // namespace spattn::spx_adapter
