// api.cpp -- the extern "C" boundary (include/spx.h). Each entry validates like the reference
// function it replaces, converts spx::Error into a status code, and launches on the caller's
// stream. No exception crosses this file.
#include <map>
#include <tuple>
#include <mutex>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/spx.h"
#include "common.hpp"
#include "engine.hpp"
#include "exchange_plan.hpp"
#include "host_rng.hpp"
#include "kernels.hpp"
#include "kv_ring.hpp"
#include "rope_table.hpp"
#include "world.hpp"

namespace spx {
const std::string& last_error();
}

using namespace spx;

struct spx_rope_table {
    std::unique_ptr<RopeTable> t;
};

struct spx_kv_ring {
    FrameRing book;
    KvRingStorage st;
};

struct spx_world {
    std::unique_ptr<World> w;
};

struct spx_engine {
    std::unique_ptr<Engine> e;
};

namespace {

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

int current_device() {
    int d = 0;
    SPX_CUDA(cudaGetDevice(&d));
    return d;
}

void require_ptr(const void* p, const char* what) {
    require(p != nullptr, SPX_ERR_CONFIG, std::string(what) + " is NULL");
}

// apply_rope_causal_local checks (proj/src/rope.cpp:145-164) then rotate_rows (:86-94)
void validate_rope(const RopeTable& t, int64_t local_len, int64_t head_dim, const int64_t grid[3],
                   int64_t start_frame, int64_t rank, int64_t world) {
    require(grid[0] >= 1 && grid[1] >= 1 && grid[2] >= 1, SPX_ERR_SHAPE,
            "grid extents must be >= 1");
    const int64_t full = grid[0] * grid[1] * grid[2];
    require(world >= 1 && full % world == 0, SPX_ERR_PARTITION,
            "sequence length " + std::to_string(full) + " not divisible by world size " +
                std::to_string(world));
    require(local_len == full / world, SPX_ERR_SHAPE,
            "local sequence length " + std::to_string(local_len) + " does not equal L/P = " +
                std::to_string(full / world));
    require(rank >= 0 && rank < world, SPX_ERR_PARTITION,
            "rank " + std::to_string(rank) + " out of range for world size " +
                std::to_string(world));
    require(t.split().total() == head_dim / 2, SPX_ERR_SHAPE,
            "table pairs " + std::to_string(t.split().total()) + " do not match head_dim " +
                std::to_string(head_dim));
    require(start_frame >= 0 && start_frame + grid[0] <= t.max_pos(0), SPX_ERR_RANGE,
            "block frames [" + std::to_string(start_frame) + ", " +
                std::to_string(start_frame + grid[0]) + ") exceed table max_frames " +
                std::to_string(t.max_pos(0)));
    require(grid[1] <= t.max_pos(1) && grid[2] <= t.max_pos(2), SPX_ERR_RANGE,
            "grid exceeds table spatial extents");
}

spx_status rope_apply_impl(const spx_rope_table* table, const void* x, void* y, int64_t batch,
                           int64_t local_len, int64_t heads, int64_t head_dim,
                           const int64_t grid[3], int64_t start_frame, int64_t rank,
                           int64_t world, const void* norm_weight, float norm_eps,
                           void* stream) {
    return guarded([&] {
        require_ptr(table, "table");
        require_ptr(grid, "grid");
        require(batch >= 1 && heads >= 1 && head_dim >= 2 && head_dim % 2 == 0, SPX_ERR_SHAPE,
                "all extents must be >= 1 and head_dim even");
        validate_rope(*table->t, local_len, head_dim, grid, start_frame, rank, world);
        require_ptr(x, "x");
        require_ptr(y, "y");
        RopeLaunch rl{};
        rl.in = static_cast<const bf16*>(x);
        rl.in_row_stride = heads * head_dim;
        rl.rows = batch * local_len;
        rl.rows_per_batch = local_len;
        rl.heads = static_cast<int>(heads);
        rl.head_dim = static_cast<int>(head_dim);
        rl.groups = 1;
        rl.has_kv = 0;
        rl.row_offset = rank * local_len;
        rl.hw = grid[1] * grid[2];
        rl.grid_w = grid[2];
        rl.start_frame = start_frame;
        const DeviceRopeTable& dt = table->t->on_device(current_device());
        for (int b = 0; b < 3; ++b) {
            rl.tab[b] = dt.band[b];
            rl.pairs[b] = static_cast<int>(table->t->pairs(b));
        }
        if (norm_weight) {
            rl.norm = 1;
            rl.norm_w_q = static_cast<const bf16*>(norm_weight);
            rl.norm_w_k = static_cast<const bf16*>(norm_weight);
            rl.norm_eps = norm_eps;
        }
        rl.dst.q[0] = static_cast<bf16*>(y);
        rl.dst.copies = 1;
        rl.dst_row_stride = heads * head_dim;
        rope_run(rl, as_stream(stream));
    });
}

}  // namespace

extern "C" {

int spx_abi_version(void) { return SPX_ABI_VERSION; }

const char* spx_last_error(void) { return spx::last_error().c_str(); }

const char* spx_status_name(int s) {
    switch (s) {
        case SPX_OK: return "OK";
        case SPX_ERR_SHAPE: return "ShapeError";
        case SPX_ERR_PARTITION: return "PartitionError";
        case SPX_ERR_CONFIG: return "ConfigError";
        case SPX_ERR_RANGE: return "RangeError";
        case SPX_ERR_ALIGNMENT: return "AlignmentError";
        case SPX_ERR_EMPTY_CACHE: return "EmptyCacheError";
        case SPX_ERR_COLLECTIVE: return "CollectiveError";
        case SPX_ERR_CUDA: return "CudaError";
        case SPX_ERR_NCCL: return "NcclError";
        case SPX_ERR_UNSUPPORTED: return "UnsupportedError";
        default: return "UnknownError";
    }
}

int64_t spx_launch_count(void) { return spx::launch_count(); }

spx_status spx_device_info(int device, int32_t out[4]) {
    return guarded([&] {
        require_ptr(out, "out");
        int n = 0;
        SPX_CUDA(cudaGetDeviceCount(&n));
        require(device >= 0 && device < n, SPX_ERR_CONFIG, "no such device");
        cudaDeviceProp prop{};
        SPX_CUDA(cudaGetDeviceProperties(&prop, device));
        out[0] = prop.multiProcessorCount;
        out[1] = prop.major;
        out[2] = prop.minor;
        out[3] = n;
    });
}

// ---- host RNG -------------------------------------------------------------------------
uint64_t spx_derive_seed(uint64_t base, uint64_t a, uint64_t b, uint64_t c) {
    return spx::derive_seed(base, a, b, c);
}

spx_status spx_block_noise(uint64_t seed, int64_t block, int64_t step, int64_t n,
                           int64_t head_dim, double* out) {
    return guarded([&] {
        require_ptr(out, "out");
        require(n >= 0 && head_dim >= 1, SPX_ERR_SHAPE, "bad noise size");
        fill_noise(spx::derive_seed(seed, 0x10, static_cast<uint64_t>(block),
                                    static_cast<uint64_t>(step)),
                   n, head_dim, out);
    });
}

spx_status spx_layer_weights(uint64_t seed, int64_t layer, int64_t model_dim, double* wq,
                             double* wk, double* wv, double* wo) {
    return guarded([&] {
        require(model_dim >= 1, SPX_ERR_SHAPE, "model_dim must be >= 1");
        const uint64_t base = spx::derive_seed(seed, 0x20, static_cast<uint64_t>(layer));
        double* outs[4] = {wq, wk, wv, wo};
        for (int m = 0; m < 4; ++m) {
            if (outs[m]) fill_matrix(spx::derive_seed(base, 11 + m), model_dim, model_dim, outs[m]);
        }
    });
}

spx_status spx_f64_to_bf16(const double* in, uint16_t* out, int64_t n) {
    return guarded([&] {
        require(n == 0 || (in && out), SPX_ERR_CONFIG, "null buffer");
        for (int64_t i = 0; i < n; ++i) out[i] = f64_to_bf16(in[i]);
    });
}

// ---- RoPE ---------------------------------------------------------------------------------
spx_status spx_band_split_defaults(int64_t head_dim, int64_t out_split[3]) {
    return guarded([&] {
        require_ptr(out_split, "out_split");
        const BandSplit s = BandSplit::defaults_for(head_dim);
        out_split[0] = s.temporal;
        out_split[1] = s.height;
        out_split[2] = s.width;
    });
}

spx_status spx_rope_table_create(int64_t max_frames, int64_t max_h, int64_t max_w,
                                 int64_t head_dim, double base, const int64_t* split,
                                 spx_rope_table** out) {
    return guarded([&] {
        require_ptr(out, "out");
        *out = nullptr;
        const BandSplit s = split ? BandSplit{split[0], split[1], split[2]}
                                  : BandSplit::defaults_for(head_dim);
        auto t = std::make_unique<spx_rope_table>();
        t->t = std::make_unique<RopeTable>(max_frames, max_h, max_w, head_dim, base, s);
        *out = t.release();
    });
}

void spx_rope_table_destroy(spx_rope_table* table) { delete table; }

spx_status spx_rope_table_info(const spx_rope_table* table, int64_t out[7]) {
    return guarded([&] {
        require_ptr(table, "table");
        require_ptr(out, "out");
        for (int b = 0; b < 3; ++b) {
            out[b] = table->t->max_pos(b);
            out[3 + b] = table->t->pairs(b);
        }
        out[6] = table->t->head_dim();
    });
}

spx_status spx_rope_table_at(const spx_rope_table* table, int32_t band, int64_t pos,
                             int64_t pair, double* cos_out, double* sin_out) {
    return guarded([&] {
        require_ptr(table, "table");
        require(band >= 0 && band < 3, SPX_ERR_RANGE, "band out of range");
        require(pos >= 0 && pos < table->t->max_pos(band), SPX_ERR_RANGE, "position out of range");
        require(pair >= 0 && pair < table->t->pairs(band), SPX_ERR_RANGE, "pair out of range");
        if (cos_out) *cos_out = table->t->cos_at(band, pos, pair);
        if (sin_out) *sin_out = table->t->sin_at(band, pos, pair);
    });
}

int64_t spx_global_time_index(int64_t i_local, int64_t rank, int64_t local_len, int64_t grid_hw,
                              int64_t start_frame) {
    const int64_t i_global = rank * local_len + i_local;
    return start_frame + i_global / grid_hw;
}

spx_status spx_rope_positions(const int64_t grid[3], int64_t start_frame, int64_t rank,
                              int64_t world_size, int32_t* t, int32_t* h, int32_t* w,
                              void* stream) {
    return guarded([&] {
        require_ptr(grid, "grid");
        require(grid[0] >= 1 && grid[1] >= 1 && grid[2] >= 1, SPX_ERR_SHAPE,
                "grid extents must be >= 1");
        const int64_t full = grid[0] * grid[1] * grid[2];
        require(world_size >= 1 && full % world_size == 0, SPX_ERR_PARTITION,
                "sequence length not divisible by world size");
        require(rank >= 0 && rank < world_size, SPX_ERR_PARTITION, "rank out of range");
        require(t && h && w, SPX_ERR_CONFIG, "null output");
        const int64_t local = full / world_size;
        rope_positions_run(local, rank * local, grid[1] * grid[2], grid[2], start_frame, t, h, w,
                           as_stream(stream));
    });
}

spx_status spx_rope_apply_causal_local(const spx_rope_table* table, const void* x, void* y,
                                       int64_t batch, int64_t local_len, int64_t heads,
                                       int64_t head_dim, const int64_t grid[3],
                                       int64_t start_frame, int64_t rank, int64_t world_size,
                                       const void* norm_weight, float norm_eps, void* stream) {
    return rope_apply_impl(table, x, y, batch, local_len, heads, head_dim, grid, start_frame,
                           rank, world_size, norm_weight, norm_eps, stream);
}

spx_status spx_rope_apply_global(const spx_rope_table* table, const void* x, void* y,
                                 int64_t batch, int64_t seq_len, int64_t heads, int64_t head_dim,
                                 const int64_t grid[3], int64_t start_frame, void* stream) {
    if (grid && grid[0] >= 1 && grid[1] >= 1 && grid[2] >= 1 &&
        seq_len != grid[0] * grid[1] * grid[2]) {
        spx::set_last_error("sequence length " + std::to_string(seq_len) +
                            " does not equal F*H_g*W_g = " +
                            std::to_string(grid[0] * grid[1] * grid[2]));
        return SPX_ERR_SHAPE;
    }
    return rope_apply_impl(table, x, y, batch, seq_len, heads, head_dim, grid, start_frame, 0, 1,
                           nullptr, 0.0f, stream);
}

// ---- dense ops ------------------------------------------------------------------------------
spx_status spx_project_tokens_ex(const void* x, const void* w, void* y, int64_t tokens,
                                 int64_t c_in, int64_t c_out, const float* bias, int32_t epilogue,
                                 const void* residual, const float* gate, void* stream) {
    return guarded([&] {
        require(x && w && y, SPX_ERR_CONFIG, "null buffer");
        require(tokens >= 1 && c_in >= 1 && c_out >= 1, SPX_ERR_SHAPE, "empty projection");
        require(c_in % 64 == 0 && c_out % 32 == 0, SPX_ERR_UNSUPPORTED,
                "tcgen05 projection needs c_in % 64 == 0 and c_out % 32 == 0");
        require(epilogue == 0 || epilogue == 1 || epilogue == 3, SPX_ERR_CONFIG,
                "epilogue: 0 plain, 1 residual + gate, 3 GELU(tanh)");
        require(epilogue != 1 || residual, SPX_ERR_CONFIG, "residual epilogue needs a residual");
        GemmOperands o{};
        o.a = static_cast<const bf16*>(x);
        o.a_row_stride = c_in;
        o.a_group_stride = tokens * c_in;
        o.groups = 1;
        o.k_inner = static_cast<int>(c_in);
        o.b = static_cast<const bf16*>(w);
        o.b_row_stride = c_in;
        o.out = static_cast<bf16*>(y);
        o.out_row_stride = c_out;
        o.M = static_cast<int>(tokens);
        o.N = static_cast<int>(c_out);
        o.K = static_cast<int>(c_in);
        o.bias = bias;
        o.epi_mode = epilogue;
        o.residual = static_cast<const bf16*>(residual);
        o.residual_row_stride = c_out;
        o.gate = gate;
        GemmPlan plan;
        gemm_plan(&plan, o, device_sm_count(current_device()));
        gemm_run(plan, as_stream(stream));
    });
}

spx_status spx_project_tokens(const void* x, const void* w, void* y, int64_t tokens,
                              int64_t c_in, int64_t c_out, void* stream) {
    return spx_project_tokens_ex(x, w, y, tokens, c_in, c_out, nullptr, 0, nullptr, nullptr, stream);
}

namespace {
// one attention launch with stream-ordered scratch for the split-KV partials
void attention_oneshot(spx::AttnOperands a, cudaStream_t st) {
    using namespace spx;
    int dev = 0;
    SPX_CUDA(cudaGetDevice(&dev));
    const int sms = device_sm_count(dev);
    const size_t ws = attn_workspace_bytes(a, attn_max_splits(a, sms));
    if (ws > 0) {
        // cached per (device, stream): the kernel re-arms its own counters, so the buffer
        // is zeroed only when it is (re)allocated; growth waits for the stream first
        static std::mutex mu;
        static std::map<std::pair<int, cudaStream_t>, std::pair<void*, size_t>> cache;
        static std::map<std::pair<int, cudaStream_t>, std::tuple<int64_t, int64_t, size_t>> last_shape;
        std::lock_guard<std::mutex> lock(mu);
        auto& slot = cache[{dev, st}];
        if (slot.second < ws) {
            if (slot.first) {
                SPX_CUDA(cudaStreamSynchronize(st));
                SPX_CUDA(cudaFree(slot.first));
            }
            slot = {nullptr, 0};
            SPX_CUDA(cudaMalloc(&slot.first, ws));
            SPX_CUDA(cudaMemset(slot.first, 0, ws));
            slot.second = ws;
        }
        a.workspace = slot.first;
        a.workspace_bytes = slot.second;
        // the split counters sit at the front of the workspace, sized by this call's tiles; a
        // previous call of another shape may have left partials (not re-armed counters) there,
        // so they are zeroed whenever the shape changes (a launch re-arms its own counters)
        const auto shape = std::make_tuple(static_cast<int64_t>(a.sq), static_cast<int64_t>(a.heads), ws);
        auto& prev = last_shape[{dev, st}];
        if (prev != shape) {
            const size_t rows = static_cast<size_t>((ceil_div(static_cast<int64_t>(a.sq), 128) + 1) & ~1) * 128;
            const size_t ctr = (rows / 128 * a.heads * sizeof(int) + 255) / 256 * 256;
            SPX_CUDA(cudaMemsetAsync(slot.first, 0, std::min(ctr, slot.second), st));
            prev = shape;
        }
    }
    AttnPlan plan;
    attn_plan(&plan, a, sms);
    attn_run(plan, st);
}
}  // namespace

spx_status spx_attention(const void* q, const void* k, const void* v, void* o, int64_t batch,
                         int64_t sq, int64_t skv, int64_t heads, int64_t head_dim, void* stream) {
    return guarded([&] {
        require(q && k && v && o, SPX_ERR_CONFIG, "null buffer");
        require(sq >= 1 && heads >= 1 && batch >= 1, SPX_ERR_SHAPE, "empty attention");
        require(skv >= 1, SPX_ERR_EMPTY_CACHE, "attention over an empty key/value set");
        AttnOperands a{};
        a.q = static_cast<const bf16*>(q);
        a.q_rows = sq;
        a.k = static_cast<const bf16*>(k);
        a.v = static_cast<const bf16*>(v);
        a.kv_rows = skv;
        a.batch = static_cast<int>(batch);
        a.heads = static_cast<int>(heads);
        a.head_dim = static_cast<int>(head_dim);
        a.sq = static_cast<int>(sq);
        a.seg_start[0] = 0;
        a.seg_len[0] = static_cast<int>(skv);
        a.num_segs = 1;
        a.out_base[0] = static_cast<bf16*>(o);
        a.rows_per_chunk = static_cast<int>(sq);
        a.out_row_stride = heads * head_dim;
        attention_oneshot(a, as_stream(stream));
    });
}

// ---- KV ring --------------------------------------------------------------------------------
spx_status spx_kv_ring_create(int device, int64_t tokens_per_frame, int64_t window_frames,
                              int64_t capacity_frames, int64_t heads, int64_t head_dim,
                              spx_kv_ring** out) {
    return guarded([&] {
        require_ptr(out, "out");
        *out = nullptr;
        require(tokens_per_frame >= 1, SPX_ERR_CONFIG, "tokens_per_frame must be >= 1");
        require(window_frames < 0 || window_frames >= 1, SPX_ERR_CONFIG,
                "window_frames must be >= 1 when set");
        require(heads >= 1 && head_dim >= 1, SPX_ERR_SHAPE, "bad head shape");
        int64_t cap = capacity_frames;
        if (cap <= 0) cap = window_frames > 0 ? window_frames : 64;
        auto r = std::make_unique<spx_kv_ring>();
        r->book = FrameRing(cap, window_frames);
        r->st.device = device;
        r->st.tokens_per_frame = tokens_per_frame;
        r->st.capacity_frames = cap;
        r->st.heads = heads;
        r->st.head_dim = head_dim;
        r->st.allocate();
        *out = r.release();
    });
}

void spx_kv_ring_destroy(spx_kv_ring* ring) {
    if (!ring) return;
    ring->st.release();
    delete ring;
}

spx_status spx_kv_ring_update(spx_kv_ring* ring, int64_t block_index, const void* k_block,
                              const void* v_block, int64_t seq_len, void* stream) {
    return guarded([&] {
        require_ptr(ring, "ring");
        require(k_block && v_block, SPX_ERR_CONFIG, "null block");
        const int64_t tpf = ring->st.tokens_per_frame;
        require(seq_len >= 1 && seq_len % tpf == 0, SPX_ERR_ALIGNMENT,
                "block length " + std::to_string(seq_len) +
                    " is not a whole number of frames of " + std::to_string(tpf) + " tokens");
        const int64_t frames = seq_len / tpf;
        const int64_t first = ring->book.update(block_index, frames);
        const size_t frame_bytes = static_cast<size_t>(tpf * ring->st.row_elems()) * sizeof(bf16);
        const int64_t cap = ring->st.capacity_frames;
        for (int64_t f = 0; f < frames; ++f) {
            const int64_t slot = (first + f) % cap;
            SPX_CUDA(cudaMemcpyAsync(
                reinterpret_cast<uint8_t*>(ring->st.k) + slot * frame_bytes,
                static_cast<const uint8_t*>(k_block) + f * frame_bytes, frame_bytes,
                cudaMemcpyDeviceToDevice, as_stream(stream)));
            SPX_CUDA(cudaMemcpyAsync(
                reinterpret_cast<uint8_t*>(ring->st.v) + slot * frame_bytes,
                static_cast<const uint8_t*>(v_block) + f * frame_bytes, frame_bytes,
                cudaMemcpyDeviceToDevice, as_stream(stream)));
        }
    });
}

spx_status spx_kv_ring_read(const spx_kv_ring* ring, void* k_out, void* v_out, void* stream) {
    return guarded([&] {
        require_ptr(ring, "ring");
        require(ring->book.cached_frames() > 0, SPX_ERR_EMPTY_CACHE, "read() on an empty cache");
        const size_t frame_bytes =
            static_cast<size_t>(ring->st.tokens_per_frame * ring->st.row_elems()) * sizeof(bf16);
        size_t off = 0;
        for (const auto& seg : ring->book.segments()) {
            const size_t bytes = static_cast<size_t>(seg.second) * frame_bytes;
            if (k_out)
                SPX_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(k_out) + off,
                                         reinterpret_cast<uint8_t*>(ring->st.k) +
                                             seg.first * frame_bytes,
                                         bytes, cudaMemcpyDeviceToDevice, as_stream(stream)));
            if (v_out)
                SPX_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(v_out) + off,
                                         reinterpret_cast<uint8_t*>(ring->st.v) +
                                             seg.first * frame_bytes,
                                         bytes, cudaMemcpyDeviceToDevice, as_stream(stream)));
            off += bytes;
        }
    });
}

spx_status spx_kv_ring_info(const spx_kv_ring* ring, int64_t out[4]) {
    return guarded([&] {
        require_ptr(ring, "ring");
        require_ptr(out, "out");
        out[0] = ring->book.cached_frames();
        out[1] = out[0] * ring->st.tokens_per_frame;
        out[2] = out[0] > 0 ? ring->book.oldest_block_index() : -1;
        out[3] = ring->st.capacity_frames;
    });
}

spx_status spx_kv_ring_attention(const spx_kv_ring* ring, const void* q, void* o, int64_t sq,
                                 void* stream) {
    return guarded([&] {
        require_ptr(ring, "ring");
        require(q && o, SPX_ERR_CONFIG, "null buffer");
        require(ring->book.cached_frames() > 0, SPX_ERR_EMPTY_CACHE,
                "attention over an empty cache");
        auto segs = ring->book.segments();
        AttnOperands a{};
        a.q = static_cast<const bf16*>(q);
        a.q_rows = sq;
        a.k = ring->st.k;
        a.v = ring->st.v;
        a.kv_rows = ring->st.rows();
        a.batch = 1;
        a.heads = static_cast<int>(ring->st.heads);
        a.head_dim = static_cast<int>(ring->st.head_dim);
        a.sq = static_cast<int>(sq);
        a.num_segs = static_cast<int>(segs.size());
        for (size_t s = 0; s < segs.size() && s < 2; ++s) {
            a.seg_start[s] = static_cast<int>(segs[s].first * ring->st.tokens_per_frame);
            a.seg_len[s] = static_cast<int>(segs[s].second * ring->st.tokens_per_frame);
        }
        a.out_base[0] = static_cast<bf16*>(o);
        a.rows_per_chunk = static_cast<int>(sq);
        a.out_row_stride = ring->st.row_elems();
        attention_oneshot(a, as_stream(stream));
    });
}

// ---- world ----------------------------------------------------------------------------------
spx_status spx_world_create_local(int world_size, const int* devices, spx_world** out) {
    return guarded([&] {
        require_ptr(out, "out");
        *out = nullptr;
        auto w = std::make_unique<spx_world>();
        w->w = std::make_unique<World>(world_size, devices);
        *out = w.release();
    });
}

spx_status spx_nccl_get_unique_id(uint8_t out_id[128]) {
    return guarded([&] {
        require_ptr(out_id, "out_id");
        nccl_unique_id(out_id);
    });
}

spx_status spx_world_create_nccl(int rank, int world_size, const uint8_t id[128], int device,
                                 spx_world** out) {
    return guarded([&] {
        require_ptr(out, "out");
        require_ptr(id, "id");
        *out = nullptr;
        auto w = std::make_unique<spx_world>();
        w->w = std::make_unique<World>(rank, world_size, id, device);
        *out = w.release();
    });
}

spx_status spx_world_create_peer(int rank, int world_size, int device, spx_world** out) {
    return guarded([&] {
        require_ptr(out, "out");
        *out = nullptr;
        auto w = std::make_unique<spx_world>();
        w->w = std::make_unique<World>(rank, world_size, device);
        *out = w.release();
    });
}

void spx_world_destroy(spx_world* world) { delete world; }

spx_status spx_world_info(const spx_world* world, int32_t out[4]) {
    return guarded([&] {
        require_ptr(world, "world");
        require_ptr(out, "out");
        out[0] = world->w->size();
        out[1] = world->w->num_local();
        out[2] = world->w->first_rank();
        out[3] = world->w->transport();
    });
}

spx_status spx_world_stream(const spx_world* world, int local_rank, void** stream_out) {
    return guarded([&] {
        require_ptr(world, "world");
        require_ptr(stream_out, "stream_out");
        require(local_rank >= 0 && local_rank < world->w->num_local(), SPX_ERR_COLLECTIVE,
                "local rank out of range");
        *stream_out = world->w->local(local_rank).stream;
    });
}

spx_status spx_world_synchronize(spx_world* world) {
    return guarded([&] {
        require_ptr(world, "world");
        world->w->synchronize();
    });
}

spx_status spx_world_stats(const spx_world* world, spx_comm_stats* out) {
    return guarded([&] {
        require_ptr(world, "world");
        require_ptr(out, "out");
        *out = world->w->stats();
    });
}

spx_status spx_world_reset_stats(spx_world* world) {
    return guarded([&] {
        require_ptr(world, "world");
        world->w->reset_stats();
    });
}

spx_status spx_world_reserve(spx_world* world, int64_t bytes) {
    return guarded([&] {
        require_ptr(world, "world");
        require(bytes >= 0, SPX_ERR_CONFIG, "bytes must be >= 0");
        world->w->reserve(static_cast<size_t>(bytes));
    });
}

spx_status spx_all_to_all(spx_world* world, void* const* in, void* const* out,
                          const int64_t shape[4], int32_t elem_bytes, int32_t scatter_axis,
                          int32_t gather_axis) {
    return guarded([&] {
        require_ptr(world, "world");
        require(in && out && shape, SPX_ERR_CONFIG, "null argument");
        world->w->all_to_all(in, out, shape, elem_bytes, scatter_axis, gather_axis);
    });
}

spx_status spx_fused_all_to_all(spx_world* world, void* const* q_in, void* const* k_in,
                                void* const* v_in, void* const* q_out, void* const* k_out,
                                void* const* v_out, const int64_t shape[4], int32_t elem_bytes,
                                int32_t scatter_axis, int32_t gather_axis) {
    return guarded([&] {
        require_ptr(world, "world");
        require(q_in && k_in && v_in && q_out && k_out && v_out && shape, SPX_ERR_CONFIG,
                "null argument");
        void* const* const ins[3] = {q_in, k_in, v_in};
        void* const* const outs[3] = {q_out, k_out, v_out};
        world->w->fused_all_to_all(ins, outs, shape, elem_bytes, scatter_axis, gather_axis);
    });
}

spx_status spx_all_gather(spx_world* world, void* const* in, void* const* out,
                          const int64_t shape[4], int32_t elem_bytes, int32_t axis) {
    return guarded([&] {
        require_ptr(world, "world");
        require(in && out && shape, SPX_ERR_CONFIG, "null argument");
        world->w->all_gather(in, out, shape, elem_bytes, axis);
    });
}

spx_status spx_partition(int32_t world_size, int64_t heads, int64_t block_len, int64_t head_dim,
                         int64_t out[5]) {
    return guarded([&] {
        require_ptr(out, "out");
        require(heads >= 1 && head_dim >= 1, SPX_ERR_SHAPE, "bad head shape");
        const Partition p = Partition::make(world_size, heads, block_len, head_dim);
        out[0] = p.G;
        out[1] = p.S;
        out[2] = p.Lp;
        out[3] = p.Lq;
        out[4] = p.Hl;
    });
}

spx_status spx_exchange_plan(int32_t which, int32_t rank, int32_t world_size, int64_t heads,
                             int64_t block_len, int64_t head_dim, int64_t block_base_row,
                             int64_t* out, int64_t max_entries, int64_t* n_entries) {
    return guarded([&] {
        require(out && n_entries, SPX_ERR_CONFIG, "null argument");
        require(rank >= 0 && rank < world_size, SPX_ERR_COLLECTIVE, "rank out of range");
        const Partition p = Partition::make(world_size, heads, block_len, head_dim);
        const std::vector<Transfer> plan =
            which == 0 ? plan_qkv_exchange(p, rank, block_base_row) : plan_out_exchange(p, rank);
        require(static_cast<int64_t>(plan.size()) <= max_entries, SPX_ERR_RANGE,
                "plan has more entries than the output holds");
        for (size_t i = 0; i < plan.size(); ++i) {
            int64_t* r = out + 6 * i;
            r[0] = plan[i].peer;
            r[1] = plan[i].is_send;
            r[2] = plan[i].buf;
            r[3] = plan[i].offset;
            r[4] = plan[i].elems;
            r[5] = 0;
        }
        *n_entries = static_cast<int64_t>(plan.size());
    });
}

// ---- engine ---------------------------------------------------------------------------------
void spx_engine_config_defaults(spx_engine_config* c) {
    if (!c) return;
    std::memset(c, 0, sizeof(*c));
    c->frames = 3;
    c->grid_h = 4;
    c->grid_w = 4;
    c->num_blocks = 5;
    c->layers = 4;
    c->denoise_steps = 2;
    c->batch = 1;
    c->heads = 8;
    c->head_dim = 16;
    c->window_frames = -1;
    c->rope_base = 10000.0;
    c->band_split[0] = c->band_split[1] = c->band_split[2] = -1;
    c->seed = 0;
    c->force_start_frame_zero = 0;
    c->qk_norm = 0;
    c->norm_eps = 1e-6f;
    c->profile = 0;
    c->fuse_rope_epilogue = 1;
    c->ablation = SPX_ABLATION_ALL;
    c->adaln = 0;
    c->l2_prefetch = 0;  // opt-in: measured 0.4 % slower per chunk at the power cap (round 1)
    c->wan_block = 0;
    c->ffn_dim = 0;
    c->text_len = 512;
    c->text_dim = 4096;
    c->freq_dim = 256;
    c->sp_bit_exact = 0;
}

spx_status spx_engine_config_validate(const spx_engine_config* cfg, int32_t world_size) {
    return guarded([&] {
        require_ptr(cfg, "cfg");
        Engine::validate(*cfg, world_size);
    });
}

spx_status spx_engine_create(spx_world* world, const spx_engine_config* cfg, spx_engine** out) {
    return guarded([&] {
        require(world && cfg && out, SPX_ERR_CONFIG, "null argument");
        *out = nullptr;
        auto e = std::make_unique<spx_engine>();
        e->e = std::make_unique<Engine>(world->w.get(), *cfg);
        *out = e.release();
    });
}

void spx_engine_destroy(spx_engine* engine) { delete engine; }

spx_status spx_engine_info(const spx_engine* engine, int64_t out[8]) {
    return guarded([&] {
        require(engine && out, SPX_ERR_CONFIG, "null argument");
        engine->e->info(out);
    });
}

spx_status spx_engine_seed_weights(spx_engine* engine) {
    return guarded([&] {
        require_ptr(engine, "engine");
        engine->e->seed_weights();
    });
}

spx_status spx_engine_set_layer_weights(spx_engine* engine, int64_t layer, const uint16_t* wq,
                                        const uint16_t* wk, const uint16_t* wv,
                                        const uint16_t* wo) {
    return guarded([&] {
        require(engine && wq && wk && wv && wo, SPX_ERR_CONFIG, "null argument");
        engine->e->set_layer_weights(layer, wq, wk, wv, wo);
    });
}

spx_status spx_engine_set_norm_weights(spx_engine* engine, int64_t layer, const uint16_t* wq,
                                       const uint16_t* wk) {
    return guarded([&] {
        require(engine && wq && wk, SPX_ERR_CONFIG, "null argument");
        engine->e->set_norm_weights(layer, wq, wk);
    });
}

spx_status spx_engine_begin_block(spx_engine* engine, int64_t block_index) {
    return guarded([&] {
        require_ptr(engine, "engine");
        engine->e->begin_block(block_index);
    });
}

spx_status spx_engine_reset_cache(spx_engine* engine) {
    return guarded([&] {
        require_ptr(engine, "engine");
        engine->e->reset_cache();
    });
}

spx_status spx_engine_layer(spx_engine* engine, int64_t layer, int64_t block_index,
                            int64_t start_frame, void* const* x_local, void* const* y_local) {
    return guarded([&] {
        require(engine && x_local && y_local, SPX_ERR_CONFIG, "null argument");
        engine->e->layer_external(layer, block_index, start_frame, x_local, y_local);
    });
}

spx_status spx_engine_generate_block(spx_engine* engine, int64_t block,
                                     const uint16_t* noise_host, uint16_t* out_host) {
    return guarded([&] {
        require(engine && out_host, SPX_ERR_CONFIG, "null argument");
        engine->e->generate_block(block, noise_host, out_host);
    });
}

spx_status spx_engine_generate_block_device(spx_engine* engine, int64_t block,
                                            const void* const* noise_dev, void* const* out_dev) {
    return guarded([&] {
        require(engine && noise_dev && out_dev, SPX_ERR_CONFIG, "null argument");
        engine->e->generate_block_device(block, noise_dev, out_dev);
    });
}

spx_status spx_engine_generate_stream(spx_engine* engine, const int64_t* blocks, int64_t n,
                                     const uint16_t* const* noise_host, uint16_t* const* out_host) {
    return guarded([&] {
        require_ptr(engine, "engine");
        engine->e->generate_stream(blocks, n, noise_host, out_host);
    });
}

spx_status spx_engine_set_wan_layer(spx_engine* engine, int64_t layer,
                                    const spx_wan_layer_weights* w) {
    return guarded([&] {
        require(engine && w, SPX_ERR_CONFIG, "null argument");
        engine->e->set_wan_layer(layer, *w);
    });
}

spx_status spx_engine_set_wan_embeddings(spx_engine* engine, const spx_wan_embed_weights* w) {
    return guarded([&] {
        require(engine && w, SPX_ERR_CONFIG, "null argument");
        engine->e->set_wan_embeddings(*w);
    });
}

spx_status spx_engine_set_timesteps(spx_engine* engine, const float* t) {
    return guarded([&] {
        require_ptr(engine, "engine");
        engine->e->set_timesteps(t);
    });
}

spx_status spx_engine_set_context(spx_engine* engine, const uint16_t* text) {
    return guarded([&] {
        require_ptr(engine, "engine");
        engine->e->set_context(text);
    });
}

spx_status spx_engine_set_graphs(spx_engine* engine, int32_t on) {
    return guarded([&] {
        require_ptr(engine, "engine");
        engine->e->set_graphs(on != 0);
    });
}

spx_status spx_debug_engine_graphs(const spx_engine* engine, int64_t* count) {
    return guarded([&] {
        require(engine && count, SPX_ERR_CONFIG, "null argument");
        *count = engine->e->graph_count();
    });
}

spx_status spx_engine_denoise_step(spx_engine* engine, int64_t block, int64_t step,
                                   const void* const* x_local, void* const* y_local) {
    return guarded([&] {
        require(engine && x_local && y_local, SPX_ERR_CONFIG, "null argument");
        engine->e->denoise_step(block, step, x_local, y_local);
    });
}

spx_status spx_verify_stream(const spx_engine_config* cfg, int32_t world_size, const int* devices,
                             double tolerance, spx_verify_block* blocks, int64_t max_blocks,
                             int32_t* pass, spx_comm_stats* ledger) {
    return guarded([&] {
        require(cfg && blocks && pass, SPX_ERR_CONFIG, "null argument");
        require(max_blocks >= cfg->num_blocks, SPX_ERR_SHAPE,
                "blocks[] holds " + std::to_string(max_blocks) + " entries, the run has " +
                    std::to_string(cfg->num_blocks) + " blocks");
        // the variant: cfg on a LOCAL world of world_size ranks (devices may repeat)
        const int64_t L = cfg->frames * cfg->grid_h * cfg->grid_w;
        const size_t per_block = static_cast<size_t>(L * cfg->heads * cfg->head_dim);
        std::vector<uint16_t> got(per_block * static_cast<size_t>(cfg->num_blocks));
        std::vector<uint16_t> want(got.size());
        {
            World w(world_size, devices);
            Engine e(&w, *cfg);
            e.seed_weights();
            e.generate(got.data());
            if (ledger) *ledger = w.stats();
        }
        // the expected run: the P = 1 optimized path (= the reference pipeline at P = 1) with
        // the correct start frames (verify_stream, generator.cpp:149-177)
        {
            spx_engine_config rc = *cfg;
            rc.ablation = SPX_ABLATION_ALL;
            rc.force_start_frame_zero = 0;
            const int dev0 = devices ? devices[0] : current_device();
            World w(1, &dev0);
            Engine e(&w, rc);
            e.seed_weights();
            e.generate(want.data());
        }
        bool all = true;
        for (int64_t b = 0; b < cfg->num_blocks; ++b) {
            double mx = 0.0;
            for (size_t i = 0; i < per_block; ++i) {
                const size_t k = static_cast<size_t>(b) * per_block + i;
                const double d = std::fabs(bf16_to_f64(got[k]) - bf16_to_f64(want[k]));
                if (!(d <= mx)) mx = d;  // NaN propagates as a failure
            }
            blocks[b].block = b;
            blocks[b].max_abs_dev = mx;
            blocks[b].pass = mx <= tolerance ? 1 : 0;
            all = all && blocks[b].pass;
        }
        *pass = all ? 1 : 0;
    });
}

spx_status spx_engine_generate(spx_engine* engine, uint16_t* out_host) {
    return guarded([&] {
        require(engine && out_host, SPX_ERR_CONFIG, "null argument");
        engine->e->generate(out_host);
    });
}

spx_status spx_engine_synchronize(spx_engine* engine) {
    return guarded([&] {
        require_ptr(engine, "engine");
        engine->e->synchronize();
    });
}

spx_status spx_engine_stage_times(spx_engine* engine, double out_ms[6], int64_t* calls) {
    return guarded([&] {
        require(engine && out_ms, SPX_ERR_CONFIG, "null argument");
        engine->e->stage_times(out_ms, calls);
    });
}

spx_status spx_engine_reset_stage_times(spx_engine* engine) {
    return guarded([&] {
        require_ptr(engine, "engine");
        engine->e->reset_stage_times();
    });
}

spx_status spx_engine_set_profile(spx_engine* engine, int32_t on) {
    return guarded([&] {
        require_ptr(engine, "engine");
        require(on >= 0 && on <= 3, SPX_ERR_CONFIG, "profile level must be 0, 1, 2 or 3");
        engine->e->set_profile(on);
    });
}

spx_status spx_engine_stats(const spx_engine* engine, spx_comm_stats* out) {
    return guarded([&] {
        require(engine && out, SPX_ERR_CONFIG, "null argument");
        *out = engine->e->stats();
    });
}

spx_status spx_engine_set_modulation(spx_engine* engine, int64_t layer, const float* shift,
                                     const float* scale, const float* gate) {
    return guarded([&] {
        require(engine, SPX_ERR_CONFIG, "null engine");
        engine->e->set_modulation(layer, shift, scale, gate);
    });
}

spx_status spx_layernorm_modulate(const void* x, void* y, int64_t tokens, int64_t dim,
                                  const float* shift, const float* scale, float eps, void* stream) {
    return guarded([&] {
        require(x && y && shift && scale, SPX_ERR_CONFIG, "null buffer");
        ln_modulate_run(static_cast<const bf16*>(x), static_cast<bf16*>(y), tokens, dim, shift,
                        scale, eps, as_stream(stream));
    });
}

// tensor_checksum (proj/src/report.cpp:264-279): FNV-1a over the little-endian bytes of the
// fp64 values, as 16 hex digits (host utility for reference-compatible reports)
spx_status spx_checksum_f64(const double* p, int64_t n, char out[17]) {
    return guarded([&] {
        require(out && (p || n == 0) && n >= 0, SPX_ERR_CONFIG, "null argument");
        uint64_t h = 0xcbf29ce484222325ULL;
        for (int64_t i = 0; i < n; ++i) {
            uint64_t bits;
            std::memcpy(&bits, &p[i], 8);
            for (int b = 0; b < 8; ++b) {
                h ^= (bits >> (8 * b)) & 0xFFULL;
                h *= 0x100000001b3ULL;
            }
        }
        std::snprintf(out, 17, "%016llx", static_cast<unsigned long long>(h));
    });
}

spx_status spx_engine_ipc_export(spx_engine* engine, void* out, int64_t capacity, int64_t* bytes) {
    return guarded([&] {
        require(engine && bytes, SPX_ERR_CONFIG, "null argument");
        const std::vector<uint8_t> blob = engine->e->ipc_export();
        *bytes = static_cast<int64_t>(blob.size());
        if (out) {
            require(capacity >= *bytes, SPX_ERR_SHAPE, "ipc_export: buffer too small");
            std::memcpy(out, blob.data(), blob.size());
        }
    });
}

spx_status spx_engine_ipc_import(spx_engine* engine, const void* blobs, int64_t bytes_per_rank) {
    return guarded([&] {
        require(engine && blobs && bytes_per_rank > 0, SPX_ERR_CONFIG, "null argument");
        engine->e->ipc_import(static_cast<const uint8_t*>(blobs),
                              static_cast<size_t>(bytes_per_rank));
    });
}

// ---- debug ----------------------------------------------------------------------------------
spx_status spx_debug_naive_gemm(const void* a, const void* b, float* out, int64_t m, int64_t n,
                                int64_t k, void* stream) {
    return guarded([&] {
        require(a && b && out, SPX_ERR_CONFIG, "null buffer");
        naive_gemm_run(static_cast<const bf16*>(a), static_cast<const bf16*>(b), out,
                       static_cast<int>(m), static_cast<int>(n), static_cast<int>(k),
                       as_stream(stream));
    });
}

spx_status spx_debug_gemm_trace(int64_t* out, int64_t n) {
    return guarded([&] {
        require(out && n >= 0 && n <= 1024 * 16 * 4, SPX_ERR_CONFIG, "trace buffer");
        SPX_CUDA(cudaDeviceSynchronize());
        SPX_CUDA(cudaMemcpy(out, gemm_trace_buffer(), static_cast<size_t>(n) * 8,
                            cudaMemcpyDeviceToHost));
        // read-and-clear: the next traced launch starts from an empty buffer
        SPX_CUDA(cudaMemset(gemm_trace_buffer(), 0, 1024 * 16 * 4 * sizeof(int64_t)));
    });
}

spx_status spx_debug_spans(uint64_t* out, int64_t capacity, int64_t* count) {
    return guarded([&] {
        require(count, SPX_ERR_CONFIG, "null count");
        *count = span_count();
        if (out) span_dump(out, std::min(capacity / 2, *count));
    });
}

spx_status spx_debug_set_attn_v3(int32_t on) {
    return guarded([&] { attn_set_v3(on); });
}

spx_status spx_debug_set_attn_splits(int32_t splits) {
    return guarded([&] {
        require(splits >= 0 && splits <= 8, SPX_ERR_CONFIG, "attention splits must be 0..8");
        attn_force_splits(splits);
    });
}

spx_status spx_debug_set_gemm_variant(int32_t variant) {
    return guarded([&] {
        require(variant >= -1 && variant < gemm_num_variants(), SPX_ERR_CONFIG,
                "gemm variant out of range");
        gemm_force_variant(variant);
    });
}

spx_status spx_debug_naive_attention(const void* q, const void* k, const void* v, float* out,
                                     int64_t batch, int64_t sq, int64_t skv, int64_t heads,
                                     int64_t head_dim, void* stream) {
    return guarded([&] {
        require(q && k && v && out, SPX_ERR_CONFIG, "null buffer");
        naive_attention_run(static_cast<const bf16*>(q), static_cast<const bf16*>(k),
                            static_cast<const bf16*>(v), out, static_cast<int>(batch),
                            static_cast<int>(sq), static_cast<int>(skv), static_cast<int>(heads),
                            static_cast<int>(head_dim), as_stream(stream));
    });
}

}  // extern "C"
