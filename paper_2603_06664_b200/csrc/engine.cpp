// engine.cpp -- see engine.hpp.
#include "engine.hpp"

#include <cstdio>

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <string>
#include <functional>
#include <thread>

#include "common.hpp"
#include "host_rng.hpp"

namespace spx {

int64_t choose_head_groups(int64_t P, int64_t H) {
    for (int64_t g = P; g >= 1; --g)
        if (P % g == 0 && H % g == 0) return g;
    return 1;
}

namespace {

void fill_matrix_bf16(uint64_t seed, int64_t rows, int64_t cols, uint16_t* out) {
    HostRng rng(seed);
    const double scale = 1.0 / std::sqrt(static_cast<double>(cols));
    const int64_t n = rows * cols;
    for (int64_t i = 0; i < n; ++i) out[i] = f64_to_bf16(rng.next_normal() * scale);
}

template <class T>
T* dev_alloc(RankState& rs, size_t count) {
    void* p = nullptr;
    SPX_CUDA(cudaMalloc(&p, count * sizeof(T)));
    SPX_CUDA(cudaMemset(p, 0, count * sizeof(T)));
    rs.allocations.push_back(p);
    return static_cast<T*>(p);
}

}  // namespace

// GenerationConfig::validate (proj/src/generator.cpp:7-38) plus the device constraints.
void Engine::validate(const spx_engine_config& c, int world_size) {
    require(c.frames >= 1 && c.grid_h >= 1 && c.grid_w >= 1, SPX_ERR_SHAPE,
            "grid extents must be >= 1, got (" + std::to_string(c.frames) + ", " +
                std::to_string(c.grid_h) + ", " + std::to_string(c.grid_w) + ")");
    require(c.num_blocks >= 1 && c.layers >= 1 && c.denoise_steps >= 1, SPX_ERR_CONFIG,
            "num_blocks, layers and denoise_steps must be >= 1");
    require(c.batch >= 1 && c.heads >= 1 && c.head_dim >= 2 && c.head_dim % 2 == 0,
            SPX_ERR_CONFIG, "batch/heads must be >= 1 and head_dim even");
    require(world_size >= 1, SPX_ERR_CONFIG, "world_size must be >= 1");
    const int64_t L = c.frames * c.grid_h * c.grid_w;
    require(L % world_size == 0, SPX_ERR_PARTITION,
            "block length " + std::to_string(L) + " not divisible by world size " +
                std::to_string(world_size));
    BandSplit split = BandSplit::defaults_for(c.head_dim);
    if (c.band_split[0] >= 0 || c.band_split[1] >= 0 || c.band_split[2] >= 0)
        split = BandSplit{c.band_split[0], c.band_split[1], c.band_split[2]};
    require(split.total() == c.head_dim / 2, SPX_ERR_CONFIG, "band split must sum to head_dim/2");
    require(c.window_frames < 0 || c.window_frames >= c.frames, SPX_ERR_CONFIG,
            "window_frames smaller than one block is not supported");
    // device path constraints
    require(c.batch == 1, SPX_ERR_UNSUPPORTED, "device engine runs batch 1");
    require(c.head_dim == 16 || c.head_dim == 32 || c.head_dim == 64 || c.head_dim == 128,
            SPX_ERR_UNSUPPORTED,
            "device engine needs head_dim 16, 32, 64 or 128 (16 / 32: the reference's small "
            "configurations, attention on the SIMT path)");
    require(!c.wan_block || c.head_dim >= 64, SPX_ERR_UNSUPPORTED,
            "wan_block needs head_dim 64 or 128");
    const int64_t C = c.heads * c.head_dim;
    require(C % 64 == 0 && C <= 2048, SPX_ERR_UNSUPPORTED,
            "device engine needs a model dim that is a multiple of 64 and <= 2048");
    const int64_t G = choose_head_groups(world_size, c.heads);
    require(G <= 8 && world_size / G <= 8, SPX_ERR_PARTITION,
            "partition needs <= 8 head groups and <= 8 query splits");
    require(c.ablation >= 0 && c.ablation <= SPX_ABLATION_ALL, SPX_ERR_CONFIG,
            "ablation must be a combination of the three AblationFlags bits");
    require(c.adaln == 0 || c.adaln == 1, SPX_ERR_CONFIG, "adaln must be 0 or 1");
    require(c.qk_norm == 0 || c.qk_norm == 1, SPX_ERR_CONFIG, "qk_norm must be 0 or 1");
    require(c.wan_block == 0 || c.wan_block == 1, SPX_ERR_CONFIG, "wan_block must be 0 or 1");
    if (c.wan_block) {
        const int64_t F = wan_ffn_dim(c);
        require(F >= 64 && F % 64 == 0, SPX_ERR_UNSUPPORTED, "wan_block: ffn_dim must be a multiple of 64");
        require(c.text_len >= 1 && c.text_dim >= 64 && c.text_dim % 64 == 0, SPX_ERR_UNSUPPORTED,
                "wan_block: text_len >= 1 and text_dim a multiple of 64");
        require(c.freq_dim >= 16 && c.freq_dim % 16 == 0 && c.freq_dim <= 8192, SPX_ERR_UNSUPPORTED,
                "wan_block: freq_dim must be a multiple of 16, <= 8192");
        require(c.ablation == SPX_ABLATION_ALL, SPX_ERR_UNSUPPORTED,
                "wan_block runs the optimized schedule (ablation = ALL)");
    }
}

int64_t wan_ffn_dim(const spx_engine_config& c) {
    if (c.ffn_dim > 0) return c.ffn_dim;
    const int64_t C = c.heads * c.head_dim;
    return ceil_div(C * 35, 6 * 64) * 64;  // 8960 at the Wan2.1-1.3B dim 1536
}

Engine::Engine(World* world, const spx_engine_config& cfg) : world_(world), cfg_(cfg) {
    validate(cfg, world->size());
    if (cfg_.wan_block) {  // the full block carries the self-attention extensions
        cfg_.adaln = 1;
        cfg_.qk_norm = 1;
        FF_ = wan_ffn_dim(cfg_);
        TL_ = cfg_.text_len;
        TD_ = cfg_.text_dim;
        FD_ = cfg_.freq_dim;
    }
    if (world->transport() == SPX_TRANSPORT_PEER) {
        require(cfg.ablation == SPX_ABLATION_ALL, SPX_ERR_UNSUPPORTED,
                "the PEER transport runs the optimized schedule only (ablation = ALL)");
        require(world->size() <= kMaxPeers, SPX_ERR_UNSUPPORTED, "PEER transport: at most 8 ranks");
    }
    F_ = cfg.frames;
    Hg_ = cfg.grid_h;
    Wg_ = cfg.grid_w;
    HW_ = Hg_ * Wg_;
    L_ = F_ * HW_;
    H_ = cfg.heads;
    D_ = cfg.head_dim;
    C_ = H_ * D_;
    P_ = world->size();
    G_ = choose_head_groups(P_, H_);
    S_ = P_ / G_;
    Lp_ = L_ / P_;
    Lq_ = L_ / S_;
    Hl_ = H_ / G_;
    part_ = Partition::make(P_, H_, L_, D_);
    // the O-projection reads the head-group slabs through a 3-D TMA whose inner extent must be
    // a multiple of 64 elements; below that (small head_dim, many groups) the attention
    // epilogue stores o rows interleaved instead: (L/P, C) with group g at columns g H/G D
    o_interleaved_ = (Hl_ * D_) % 64 != 0;
    require(!o_interleaved_ || world->transport() != SPX_TRANSPORT_NCCL, SPX_ERR_UNSUPPORTED,
            "NCCL transport needs (heads / groups) x head_dim to be a multiple of 64");
    cap_frames_ = cfg.window_frames < 0 ? cfg.num_blocks * F_
                                        : ceil_div(cfg.window_frames, F_) * F_;
    frames_ = FrameRing(cap_frames_, cfg.window_frames);
    BandSplit split = BandSplit::defaults_for(D_);
    if (cfg.band_split[0] >= 0 || cfg.band_split[1] >= 0 || cfg.band_split[2] >= 0)
        split = BandSplit{cfg.band_split[0], cfg.band_split[1], cfg.band_split[2]};
    // temporal extent: every frame the run can address (generator.cpp:57-60)
    table_ = std::make_unique<RopeTable>(cfg.num_blocks * F_, Hg_, Wg_, D_, cfg.rope_base, split);
    allocate();
    build_plans();
}

Engine::~Engine() {
    drop_graphs();
    for (RankState& rs : ranks_) {
        cudaSetDevice(rs.device);
        cudaStreamSynchronize(rs.stream);
    }
    for (void* p : ipc_opened_) cudaIpcCloseMemHandle(p);
    for (RankState& rs : ranks_) {
        cudaSetDevice(rs.device);
        cudaStreamSynchronize(rs.stream);
        for (auto& ring : rs.rings) ring.release();
        for (void* p : rs.allocations) cudaFree(p);
        if (rs.ev_k3) cudaEventDestroy(rs.ev_k3);
        if (rs.ev_attn) cudaEventDestroy(rs.ev_attn);
        for (int b = 0; b < 2; ++b) {
            if (rs.ev_ready[b]) cudaEventDestroy(rs.ev_ready[b]);
            if (rs.ev_used[b]) cudaEventDestroy(rs.ev_used[b]);
        }
        if (rs.copy_stream) {
            cudaStreamSynchronize(rs.copy_stream);
            cudaStreamDestroy(rs.copy_stream);
        }
        if (rs.d2h_stream) {
            cudaStreamSynchronize(rs.d2h_stream);
            cudaStreamDestroy(rs.d2h_stream);
        }
        for (int b = 0; b < 2; ++b) {
            if (rs.ev_out_ready[b]) cudaEventDestroy(rs.ev_out_ready[b]);
            if (rs.ev_out_free[b]) cudaEventDestroy(rs.ev_out_free[b]);
        }
    }
    for (auto& kv : weights_) {
        cudaSetDevice(kv.first);
        for (void* p : kv.second.wan_allocs) cudaFree(p);
        cudaFree(kv.second.wqkv);
        cudaFree(kv.second.wo);
        cudaFree(kv.second.norm_q);
        cudaFree(kv.second.norm_k);
        cudaFree(kv.second.mod);
    }
    for (auto* set : {&pending_events_, &free_events_})
        for (StageEvents& se : *set)
            for (cudaEvent_t e : se.ev) cudaEventDestroy(e);
    if (noise_pinned_) cudaFreeHost(noise_pinned_);
    if (peer_error_host_) cudaFreeHost(peer_error_host_);
}

int Engine::local_of(int rank) const { return world_->local_index(rank); }

bf16* Engine::q_recv_of(int rank) const {
    if (world_->transport() == SPX_TRANSPORT_PEER) return peers_[static_cast<size_t>(rank)].q_recv;
    return ranks_[static_cast<size_t>(local_of(rank))].q_recv;
}

bf16* Engine::o_recv_of(int rank) const {
    if (world_->transport() == SPX_TRANSPORT_PEER) return peers_[static_cast<size_t>(rank)].o_recv;
    return ranks_[static_cast<size_t>(local_of(rank))].o_recv;
}

bf16* Engine::ring_k_of(int rank, int64_t layer) const {
    if (world_->transport() == SPX_TRANSPORT_PEER)
        return peers_[static_cast<size_t>(rank)].ring_k[static_cast<size_t>(layer)];
    return ranks_[static_cast<size_t>(local_of(rank))].rings[static_cast<size_t>(layer)].k;
}

bf16* Engine::ring_v_of(int rank, int64_t layer) const {
    if (world_->transport() == SPX_TRANSPORT_PEER)
        return peers_[static_cast<size_t>(rank)].ring_v[static_cast<size_t>(layer)];
    return ranks_[static_cast<size_t>(local_of(rank))].rings[static_cast<size_t>(layer)].v;
}

// ---- PEER transport: buffer handles and the device-side rank barrier ----
namespace {
constexpr uint32_t kIpcMagic = 0x53505849u;  // "SPXI"
struct IpcHeader {
    uint32_t magic;
    int32_t rank, world, layers;
    int64_t device_bytes;  // q_recv + o_recv + ring sizes, a shape cross-check
    int64_t handles;
};
}  // namespace

std::vector<uint8_t> Engine::ipc_export() const {
    require(world_->transport() == SPX_TRANSPORT_PEER, SPX_ERR_CONFIG,
            "ipc_export needs the PEER transport");
    const RankState& rs = ranks_[0];
    std::vector<const void*> ptrs = {rs.q_recv, rs.o_recv, rs.flags};
    for (const auto& ring : rs.rings) ptrs.push_back(ring.k);
    for (const auto& ring : rs.rings) ptrs.push_back(ring.v);
    IpcHeader h{kIpcMagic, rs.rank, static_cast<int32_t>(P_), static_cast<int32_t>(cfg_.layers),
                (Lq_ * Hl_ * D_ + G_ * Lp_ * Hl_ * D_ + 2 * cfg_.layers * rs.rings[0].rows() * Hl_ * D_),
                static_cast<int64_t>(ptrs.size())};
    std::vector<uint8_t> blob(sizeof(h) + ptrs.size() * sizeof(cudaIpcMemHandle_t));
    std::memcpy(blob.data(), &h, sizeof(h));
    SPX_CUDA(cudaSetDevice(rs.device));
    for (size_t i = 0; i < ptrs.size(); ++i) {
        cudaIpcMemHandle_t mh;
        SPX_CUDA(cudaIpcGetMemHandle(&mh, const_cast<void*>(ptrs[i])));
        std::memcpy(blob.data() + sizeof(h) + i * sizeof(mh), &mh, sizeof(mh));
    }
    return blob;
}

void Engine::ipc_import(const uint8_t* blobs, size_t per_rank) {
    require(world_->transport() == SPX_TRANSPORT_PEER, SPX_ERR_CONFIG,
            "ipc_import needs the PEER transport");
    require(!peers_ready_, SPX_ERR_CONFIG, "ipc_import: peers are already mapped");
    const RankState& rs = ranks_[0];
    const std::vector<uint8_t> mine = ipc_export();
    require(blobs && per_rank == mine.size(), SPX_ERR_SHAPE,
            "ipc_import: blob size " + std::to_string(per_rank) + ", expected " +
                std::to_string(mine.size()));
    SPX_CUDA(cudaSetDevice(rs.device));
    peers_.assign(static_cast<size_t>(P_), PeerView{});
    for (int r = 0; r < P_; ++r) {
        const uint8_t* b = blobs + static_cast<size_t>(r) * per_rank;
        IpcHeader h;
        std::memcpy(&h, b, sizeof(h));
        IpcHeader m;
        std::memcpy(&m, mine.data(), sizeof(m));
        require(h.magic == kIpcMagic && h.rank == r && h.world == P_ && h.layers == cfg_.layers &&
                    h.device_bytes == m.device_bytes && h.handles == m.handles,
                SPX_ERR_COLLECTIVE,
                "ipc_import: blob " + std::to_string(r) + " is not rank " + std::to_string(r) +
                    " of an engine with the same configuration");
        PeerView& v = peers_[static_cast<size_t>(r)];
        if (r == rs.rank) {
            v.q_recv = rs.q_recv;
            v.o_recv = rs.o_recv;
            v.flags = rs.flags;
            for (const auto& ring : rs.rings) {
                v.ring_k.push_back(ring.k);
                v.ring_v.push_back(ring.v);
            }
            continue;
        }
        auto open = [&](int64_t i) {
            cudaIpcMemHandle_t mh;
            std::memcpy(&mh, b + sizeof(h) + static_cast<size_t>(i) * sizeof(mh), sizeof(mh));
            void* p = nullptr;
            SPX_CUDA(cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess));
            ipc_opened_.push_back(p);
            return p;
        };
        v.q_recv = static_cast<bf16*>(open(0));
        v.o_recv = static_cast<bf16*>(open(1));
        v.flags = static_cast<uint64_t*>(open(2));
        for (int64_t l = 0; l < cfg_.layers; ++l) v.ring_k.push_back(static_cast<bf16*>(open(3 + l)));
        for (int64_t l = 0; l < cfg_.layers; ++l)
            v.ring_v.push_back(static_cast<bf16*>(open(3 + cfg_.layers + l)));
    }
    peers_ready_ = true;
}

void Engine::peer_barrier(RankState& rs, int slot) {
    PeerFlags f{};
    for (int r = 0; r < P_; ++r) f.rank_flags[r] = peers_[static_cast<size_t>(r)].flags;
    peer_barrier_run(f, rs.flags, static_cast<int>(P_), rs.rank, slot, peer_timeout_ns_,
                     peer_error_dev_, rs.stream);
}

void Engine::check_peer_error() {
    if (!peer_error_host_) return;
    const int e = *reinterpret_cast<volatile int*>(peer_error_host_);
    if (e == 0) return;
    *reinterpret_cast<volatile int*>(peer_error_host_) = 0;
    throw Error(SPX_ERR_COLLECTIVE,
                "PEER barrier timed out waiting for rank " + std::to_string(e - 1) + " (after " +
                    std::to_string(peer_timeout_ns_ / 1000000) +
                    " ms; a rank died or left the collective order, collectives.cpp:42-52)");
}

void Engine::allocate() {
    const bool nccl = world_->transport() == SPX_TRANSPORT_NCCL;
    const size_t slab = static_cast<size_t>(Lp_ * Hl_ * D_);
    for (int li = 0; li < world_->num_local(); ++li) {
        const LocalRank& lr = world_->local(li);
        SPX_CUDA(cudaSetDevice(lr.device));
        if (!weights_.count(lr.device)) {
            DeviceWeights w;
            w.device = lr.device;
            const size_t nqkv = static_cast<size_t>(cfg_.layers * 3 * C_ * C_);
            const size_t no = static_cast<size_t>(cfg_.layers * C_ * C_);
            const size_t nn = static_cast<size_t>(cfg_.layers * C_);
            SPX_CUDA(cudaMalloc(&w.wqkv, nqkv * sizeof(bf16)));
            SPX_CUDA(cudaMalloc(&w.wo, no * sizeof(bf16)));
            SPX_CUDA(cudaMalloc(&w.norm_q, nn * sizeof(bf16)));
            SPX_CUDA(cudaMalloc(&w.norm_k, nn * sizeof(bf16)));
            SPX_CUDA(cudaMalloc(&w.mod, 3 * nn * sizeof(float)));
            SPX_CUDA(cudaMemset(w.mod, 0, 3 * nn * sizeof(float)));
            SPX_CUDA(cudaMemset(w.wqkv, 0, nqkv * sizeof(bf16)));
            SPX_CUDA(cudaMemset(w.wo, 0, no * sizeof(bf16)));
            // norm weights default to 1.0 (bf16 0x3F80)
            std::vector<uint16_t> ones(nn, 0x3F80u);
            SPX_CUDA(cudaMemcpy(w.norm_q, ones.data(), nn * 2, cudaMemcpyHostToDevice));
            SPX_CUDA(cudaMemcpy(w.norm_k, ones.data(), nn * 2, cudaMemcpyHostToDevice));
            weights_[lr.device] = w;
        }
        RankState rs;
        rs.rank = lr.rank;
        rs.local = li;
        rs.device = lr.device;
        rs.stream = lr.stream;
        rs.g = static_cast<int>(lr.rank % G_);
        rs.p = static_cast<int>(lr.rank / G_);
        rs.x[0] = dev_alloc<bf16>(rs, static_cast<size_t>(Lp_ * C_));
        rs.x[1] = dev_alloc<bf16>(rs, static_cast<size_t>(Lp_ * C_));
        rs.qkv = dev_alloc<bf16>(rs, static_cast<size_t>(Lp_ * 3 * C_));
        if (cfg_.adaln) rs.xm = dev_alloc<bf16>(rs, static_cast<size_t>(Lp_ * C_));
        rs.q_recv = dev_alloc<bf16>(rs, static_cast<size_t>(Lq_ * Hl_ * D_));
        rs.o_recv = dev_alloc<bf16>(rs, static_cast<size_t>(G_) * slab);
        if (!(cfg_.ablation & SPX_ABLATION_FUSED_ALL_TO_ALL)) {  // all-gather targets (L, C)
            for (auto** g : {&rs.gq, &rs.gk, &rs.gv}) *g = dev_alloc<bf16>(rs, static_cast<size_t>(L_ * C_));
        }
        if (!(cfg_.ablation & SPX_ABLATION_PRECOMPUTED_FREQS)) {  // recomputed table slice
            const int64_t n = (cfg_.num_blocks * F_) * table_->pairs(0) + Hg_ * table_->pairs(1) +
                              Wg_ * table_->pairs(2);
            rs.tab_scratch = dev_alloc<float2>(rs, static_cast<size_t>(n));
        }
        if (world_->transport() == SPX_TRANSPORT_PEER) {
            // [kPeerSlots][P] shared flag words + [kPeerSlots] private epoch counters
            rs.flags = dev_alloc<uint64_t>(rs, static_cast<size_t>(kPeerSlots * P_ + kPeerSlots));
            SPX_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&peer_error_host_), sizeof(int),
                                   cudaHostAllocMapped));
            *peer_error_host_ = 0;
            SPX_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&peer_error_dev_),
                                              peer_error_host_, 0));
            const char* t = std::getenv("SPX_PEER_TIMEOUT_MS");
            const long long ms = t ? std::max(1LL, std::atoll(t)) : 60000LL;
            peer_timeout_ns_ = static_cast<uint64_t>(ms) * 1000000ull;
        }
        if (nccl) {
            rs.q_send = dev_alloc<bf16>(rs, static_cast<size_t>(G_) * slab);
            rs.k_send = dev_alloc<bf16>(rs, static_cast<size_t>(G_) * slab);
            rs.v_send = dev_alloc<bf16>(rs, static_cast<size_t>(G_) * slab);
            rs.o_send = dev_alloc<bf16>(rs, static_cast<size_t>(G_) * slab);
        }
        rs.rings.resize(static_cast<size_t>(cfg_.layers));
        for (auto& ring : rs.rings) {
            ring.device = lr.device;
            ring.tokens_per_frame = HW_;
            ring.capacity_frames = cap_frames_;
            ring.heads = Hl_;
            ring.head_dim = D_;
            ring.allocate();
        }
        SPX_CUDA(cudaEventCreateWithFlags(&rs.ev_k3, cudaEventDisableTiming));
        SPX_CUDA(cudaEventCreateWithFlags(&rs.ev_attn, cudaEventDisableTiming));
        ranks_.push_back(std::move(rs));
    }
    if (cfg_.wan_block) allocate_wan();
}

void Engine::build_plans() {
    for (RankState& rs : ranks_) {
        SPX_CUDA(cudaSetDevice(rs.device));
        table_->on_device(rs.device);  // the RoPE tables are resident before any capture
        const int sms = device_sm_count(rs.device);
        const DeviceWeights& w = weights_.at(rs.device);
        rs.qkv_plan.resize(static_cast<size_t>(cfg_.layers));
        rs.o_plan.resize(static_cast<size_t>(cfg_.layers));
        rs.attn_plan.resize(static_cast<size_t>(cfg_.layers));
        for (int64_t l = 0; l < cfg_.layers; ++l) {
            GemmOperands q{};
            q.a = cfg_.adaln ? rs.xm : rs.x[l % 2];
            q.a_row_stride = C_;
            q.a_group_stride = Lp_ * C_;
            q.groups = 1;
            q.k_inner = static_cast<int>(C_);
            q.b = w.wqkv + l * 3 * C_ * C_;
            q.b_row_stride = C_;
            q.out = rs.qkv;
            q.out_row_stride = 3 * C_;
            q.M = static_cast<int>(Lp_);
            q.N = static_cast<int>(3 * C_);
            q.K = static_cast<int>(C_);
            q.b_constant = true;  // weights: uploaded synchronously, never written by a kernel
            if (cfg_.wan_block) q.bias = w.wan.b_qkv + l * 3 * C_;
            q.allow_split_k = !cfg_.sp_bit_exact;  // split-K changes the k order
            gemm_plan(&rs.qkv_plan[l], q, sms);

            GemmOperands o{};
            o.a = rs.o_recv;
            if (o_interleaved_) {  // (L/P, C) rows, head group g at columns [g H/G D, ...)
                o.a_row_stride = C_;
                o.a_group_stride = Lp_ * C_;
                o.groups = 1;
                o.k_inner = static_cast<int>(C_);
            } else {               // [G][L/P][H/G D] slabs, un-interleaved by the 3-D TMA
                o.a_row_stride = Hl_ * D_;
                o.a_group_stride = Lp_ * Hl_ * D_;
                o.groups = static_cast<int>(G_);
                o.k_inner = static_cast<int>(Hl_ * D_);
            }
            o.b = w.wo + l * C_ * C_;
            o.b_row_stride = C_;
            o.out = rs.x[(l + 1) % 2];
            o.out_row_stride = C_;
            if (cfg_.adaln) {  // x + gate * (W_o o): the gated residual in the epilogue
                o.epi_mode = 1;
                o.residual = rs.x[l % 2];
                o.residual_row_stride = C_;
                o.gate = w.mod + (l * 3 + 2) * C_;
                if (cfg_.wan_block) {  // gate_msa of the step's modulation, + the o bias
                    o.gate = rs.mod_step + (l * 6 + 2) * C_;
                    o.bias = w.wan.b_o + l * C_;
                }
            }
            o.M = static_cast<int>(Lp_);
            o.N = static_cast<int>(C_);
            o.K = static_cast<int>(C_);
            o.b_constant = true;
            o.allow_split_k = !cfg_.sp_bit_exact;  // split-K changes the k order
            gemm_plan(&rs.o_plan[l], o, sms);
            // adaLN (not the full block): fuse the next layer's K1 into this projection
            rs.oln_plan.resize(static_cast<size_t>(cfg_.layers));
            static const bool fuse_ln = [] {  // SPX_FUSE_LN=0: K1 stays a separate launch (A/B)
                const char* e = std::getenv("SPX_FUSE_LN");
                return !(e && std::atoi(e) == 0);
            }();
            if (fuse_ln && cfg_.adaln && !cfg_.wan_block && l + 1 < cfg_.layers && gemm_ln_supported(o)) {
                const float* mn = w.mod + (l + 1) * 3 * C_;  // [shift | scale | gate] of layer l + 1
                gemm_ln_plan(&rs.oln_plan[static_cast<size_t>(l)], o, rs.xm, mn + C_, mn, false,
                             static_cast<float>(cfg_.norm_eps));
            }

            AttnOperands a{};
            a.q = rs.q_recv;
            a.q_rows = Lq_;
            a.k = rs.rings[l].k;
            a.v = rs.rings[l].v;
            a.kv_rows = rs.rings[l].rows();
            a.batch = 1;
            a.heads = static_cast<int>(Hl_);
            a.head_dim = static_cast<int>(D_);
            a.sq = static_cast<int>(Lq_);
            a.seg_start[0] = 0;
            a.seg_len[0] = static_cast<int>(HW_);  // placeholder until begin_block
            a.num_segs = 1;
            a.rows_per_chunk = static_cast<int>(Lp_);
            a.out_row_stride = o_interleaved_ ? C_ : Hl_ * D_;
            if (l == 0 && !cfg_.sp_bit_exact) {  // one split-KV workspace per rank (layers in stream order)
                const size_t ws = attn_workspace_bytes(a, attn_max_splits(a, sms));
                if (ws > 0) {
                    void* ptr = nullptr;
                    SPX_CUDA(cudaMalloc(&ptr, ws));
                    SPX_CUDA(cudaMemset(ptr, 0, ws));
                    rs.allocations.push_back(ptr);
                    rs.attn_ws = ptr;
                    rs.attn_ws_bytes = ws;
                }
            }
            a.workspace = rs.attn_ws;
            a.workspace_bytes = rs.attn_ws_bytes;
            a.prefer_v3 = cfg_.sp_bit_exact != 0;
            attn_plan(&rs.attn_plan[l], a, sms);
        }
    }
    if (cfg_.wan_block) build_wan_plans();
}

void Engine::info(int64_t out[8]) const {
    out[0] = G_;
    out[1] = S_;
    out[2] = L_;
    out[3] = Lp_;
    out[4] = Hl_;
    out[5] = Lq_;
    out[6] = cap_frames_;
    out[7] = C_;
}

void Engine::seed_weights() {
    const int64_t layers = cfg_.layers;
    const size_t mat = static_cast<size_t>(C_ * C_);
    const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    for (int64_t l0 = 0; l0 < layers; l0 += hw) {
        const int64_t l1 = std::min<int64_t>(layers, l0 + hw);
        std::vector<std::vector<uint16_t>> bufs(static_cast<size_t>(l1 - l0));
        std::vector<std::thread> threads;
        for (int64_t l = l0; l < l1; ++l) {
            threads.emplace_back([&, l] {
                std::vector<uint16_t>& b = bufs[static_cast<size_t>(l - l0)];
                b.resize(4 * mat);
                // AttentionLayerParams::seeded(H*D, derive_seed(seed, 0x20, layer))
                const uint64_t base = derive_seed(cfg_.seed, 0x20, static_cast<uint64_t>(l));
                for (int m = 0; m < 4; ++m)
                    fill_matrix_bf16(derive_seed(base, 11 + m), C_, C_, b.data() + m * mat);
            });
        }
        for (auto& t : threads) t.join();
        for (int64_t l = l0; l < l1; ++l) {
            const uint16_t* b = bufs[static_cast<size_t>(l - l0)].data();
            set_layer_weights(l, b, b + mat, b + 2 * mat, b + 3 * mat);
        }
    }
    // adaLN modulation (Wan init: N(0, 1) / sqrt(dim)), fp32
    for (int64_t l = 0; l < layers; ++l) {
        HostRng rng(derive_seed(cfg_.seed, 0x30, static_cast<uint64_t>(l)));
        std::vector<float> m(static_cast<size_t>(3 * C_));
        const double sc = 1.0 / std::sqrt(static_cast<double>(C_));
        for (float& e : m) e = static_cast<float>(rng.next_normal() * sc);
        set_modulation(l, m.data(), m.data() + C_, m.data() + 2 * C_);
    }
    if (cfg_.wan_block) seed_wan_weights();
}

// SPX_WAN_VPACK=0: K3 packs v too (A/B of the v-pack epilogue)
static bool vpack_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SPX_WAN_VPACK");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

void Engine::set_modulation(int64_t layer, const float* shift, const float* scale,
                            const float* gate) {
    require(layer >= 0 && layer < cfg_.layers, SPX_ERR_RANGE, "layer out of range");
    // kernels still in flight may read this layer's weights: drain the engine streams first
    synchronize();
    require(shift && scale && gate, SPX_ERR_CONFIG, "null modulation vector");
    for (auto& kv : weights_) {
        SPX_CUDA(cudaSetDevice(kv.first));
        float* m = kv.second.mod + layer * 3 * C_;
        SPX_CUDA(cudaMemcpy(m, shift, C_ * 4, cudaMemcpyHostToDevice));
        SPX_CUDA(cudaMemcpy(m + C_, scale, C_ * 4, cudaMemcpyHostToDevice));
        SPX_CUDA(cudaMemcpy(m + 2 * C_, gate, C_ * 4, cudaMemcpyHostToDevice));
    }
    sync_weight_devices();
}

void Engine::set_layer_weights(int64_t layer, const uint16_t* wq, const uint16_t* wk,
                               const uint16_t* wv, const uint16_t* wo) {
    require(layer >= 0 && layer < cfg_.layers, SPX_ERR_RANGE, "layer out of range");
    // kernels still in flight may read this layer's weights: drain the engine streams first
    synchronize();
    const size_t mat = static_cast<size_t>(C_ * C_);
    for (auto& kv : weights_) {
        SPX_CUDA(cudaSetDevice(kv.first));
        bf16* base = kv.second.wqkv + layer * 3 * mat;
        SPX_CUDA(cudaMemcpy(base, wq, mat * 2, cudaMemcpyHostToDevice));
        SPX_CUDA(cudaMemcpy(base + mat, wk, mat * 2, cudaMemcpyHostToDevice));
        SPX_CUDA(cudaMemcpy(base + 2 * mat, wv, mat * 2, cudaMemcpyHostToDevice));
        SPX_CUDA(cudaMemcpy(kv.second.wo + layer * mat, wo, mat * 2, cudaMemcpyHostToDevice));
    }
    sync_weight_devices();
}

void Engine::set_norm_weights(int64_t layer, const uint16_t* wq, const uint16_t* wk) {
    require(layer >= 0 && layer < cfg_.layers, SPX_ERR_RANGE, "layer out of range");
    // kernels still in flight may read this layer's weights: drain the engine streams first
    synchronize();
    for (auto& kv : weights_) {
        SPX_CUDA(cudaSetDevice(kv.first));
        SPX_CUDA(cudaMemcpy(kv.second.norm_q + layer * C_, wq, C_ * 2, cudaMemcpyHostToDevice));
        SPX_CUDA(cudaMemcpy(kv.second.norm_k + layer * C_, wk, C_ * 2, cudaMemcpyHostToDevice));
    }
    sync_weight_devices();
}

// the setters copy with cudaMemcpy on the legacy stream (a pageable H2D may return before its
// DMA lands, and the engine streams are non-blocking): finish the copies on every weight
// device before any later kernel can read them
void Engine::sync_weight_devices() {
    for (auto& kv : weights_) {
        SPX_CUDA(cudaSetDevice(kv.first));
        SPX_CUDA(cudaDeviceSynchronize());
    }
}

void Engine::reset_cache() {
    synchronize();
    frames_ = FrameRing(cap_frames_, cfg_.window_frames);
    have_block_ = false;
    current_block_ = -1;
}

void Engine::begin_block(int64_t block_index) {
    const int64_t first = frames_.update(block_index, F_);
    require(first + F_ <= cap_frames_, SPX_ERR_ALIGNMENT,
            "block frames straddle the ring end (capacity must be a multiple of the block)");
    block_base_row_ = first * HW_;
    auto segs = frames_.segments();
    require(!segs.empty() && segs.size() <= 2, SPX_ERR_RANGE, "kv ring segments");
    num_segs_ = static_cast<int>(segs.size());
    for (int s = 0; s < num_segs_; ++s) {
        seg_start_[s] = static_cast<int>(segs[static_cast<size_t>(s)].first * HW_);
        seg_len_[s] = static_cast<int>(segs[static_cast<size_t>(s)].second * HW_);
    }
    have_block_ = true;
    current_block_ = block_index;
}

RopeLaunch Engine::rope_launch(const RankState& rs, int64_t layer, int64_t start_frame) const {
    // LOCAL and PEER store straight into the destination rank's buffers
    const bool direct = world_->transport() != SPX_TRANSPORT_NCCL;
    RopeLaunch rl{};
    rl.in = rs.qkv;
    rl.in_row_stride = 3 * C_;
    rl.rows = Lp_;
    rl.rows_per_batch = Lp_;
    rl.heads = static_cast<int>(H_);
    rl.head_dim = static_cast<int>(D_);
    rl.groups = static_cast<int>(G_);
    rl.has_kv = 1;
    rl.row_offset = static_cast<int64_t>(rs.rank) * Lp_;  // i_g = r * L/P + i
    rl.hw = HW_;
    rl.grid_w = Wg_;
    rl.start_frame = start_frame;
    const DeviceRopeTable& t = table_->on_device(rs.device);
    for (int b = 0; b < 3; ++b) {
        rl.tab[b] = t.band[b];
        rl.pairs[b] = static_cast<int>(table_->pairs(b));
    }
    rl.tab_constant = 1;  // uploaded once at create time
    if (!(cfg_.ablation & SPX_ABLATION_PRECOMPUTED_FREQS)) {  // this call's recomputed slice
        rl.tab_constant = 0;
        rl.tab[0] = rs.tab_scratch;
        rl.tab[1] = rl.tab[0] + (start_frame + F_) * rl.pairs[0];
        rl.tab[2] = rl.tab[1] + Hg_ * rl.pairs[1];
    }
    if (cfg_.qk_norm) {
        const DeviceWeights& w = weights_.at(rs.device);
        rl.norm = 1;
        rl.norm_w_q = w.norm_q + layer * C_;
        rl.norm_w_k = w.norm_k + layer * C_;
        rl.norm_eps = cfg_.norm_eps;
    }
    const int64_t slab = Lp_ * Hl_ * D_;
    const int64_t row_elems = Hl_ * D_;
    for (int64_t g = 0; g < G_; ++g) {
        const int d = static_cast<int>(rs.p * G_ + g);
        if (direct) {
            rl.dst.q[g] = q_recv_of(d) + (rs.rank % G_) * slab;
        } else {
            rl.dst.q[g] = d == rs.rank ? rs.q_recv + (rs.rank % G_) * slab : rs.q_send + g * slab;
        }
        for (int64_t c = 0; c < S_; ++c) {
            const int dk = static_cast<int>(c * G_ + g);
            const int64_t row0 = block_base_row_ + static_cast<int64_t>(rs.rank) * Lp_;
            if (direct || dk == rs.rank) {
                rl.dst.k[g][c] = ring_k_of(dk, layer) + row0 * row_elems;
                rl.dst.v[g][c] = ring_v_of(dk, layer) + row0 * row_elems;
            } else {
                rl.dst.k[g][c] = rs.k_send + g * slab;
                rl.dst.v[g][c] = rs.v_send + g * slab;
            }
        }
    }
    rl.dst.copies = static_cast<int>(S_);
    rl.dst_row_stride = row_elems;
    return rl;
}

void Engine::run_layer(int64_t layer, int64_t start_frame,
                       const std::vector<const GemmPlan*>& qkv,
                       const std::vector<const GemmPlan*>& oproj,
                       const std::vector<const bf16*>& x_in) {
    require(have_block_, SPX_ERR_EMPTY_CACHE, "layer call before any block was registered");
    const bool local = world_->transport() == SPX_TRANSPORT_LOCAL;
    const bool peer = world_->transport() == SPX_TRANSPORT_PEER;
    const bool nccl = world_->transport() == SPX_TRANSPORT_NCCL;
    require(!peer || peers_ready_, SPX_ERR_COLLECTIVE,
            "PEER transport: exchange buffer handles first (spx_engine_ipc_import)");
    const int nl = static_cast<int>(ranks_.size());
    const int64_t slab = Lp_ * Hl_ * D_;

    StageEvents* prof = nullptr;
    // level 3: the attention bracket on every 8th call only (a live sample of the kernel's
    // duration that leaves the PDL chaining of the other calls intact)
    const bool sampled = cfg_.profile != 3 || (profile_seq_++ % 8) == 0;
    if (cfg_.profile && sampled) {
        SPX_CUDA(cudaSetDevice(ranks_[0].device));
        if (free_events_.empty()) {
            StageEvents se;
            for (auto& e : se.ev) SPX_CUDA(cudaEventCreate(&e));
            free_events_.push_back(se);
        }
        pending_events_.push_back(free_events_.back());
        free_events_.pop_back();
        prof = &pending_events_.back();
        prof->level = cfg_.profile == 1 ? 1 : 2;
    }
    auto mark = [&](int li, int k) {
        if (prof && li == 0 && (prof->level == 1 || k == 4 || k == 5))
            SPX_CUDA(cudaEventRecord(prof->ev[k], ranks_[0].stream));
    };

    // AblationFlags (sp_attention.cpp:229-292); the default is the optimized schedule
    const bool fused = cfg_.ablation & SPX_ABLATION_FUSED_ALL_TO_ALL;
    const bool local_rope = cfg_.ablation & SPX_ABLATION_LOCAL_ROPE;
    if (!(cfg_.ablation & SPX_ABLATION_PRECOMPUTED_FREQS)) {
        // recompute_slice (sp_attention.cpp:191-195): frames [0, s + F), all rows, all columns
        for (RankState& rs : ranks_) {
            SPX_CUDA(cudaSetDevice(rs.device));
            const int pairs[3] = {static_cast<int>(table_->pairs(0)), static_cast<int>(table_->pairs(1)),
                                  static_cast<int>(table_->pairs(2))};
            const int rows[3] = {static_cast<int>(start_frame + F_), static_cast<int>(Hg_),
                                 static_cast<int>(Wg_)};
            float2* band[3] = {rs.tab_scratch, rs.tab_scratch + rows[0] * pairs[0],
                               rs.tab_scratch + rows[0] * pairs[0] + rows[1] * pairs[1]};
            rope_table_run(band, rows, pairs, cfg_.rope_base, rs.stream);
        }
    }

    // K2 + K3 (the fused exchange is carried by K3's stores on the LOCAL transport)
    for (int li = 0; li < nl; ++li) {
        RankState& rs = ranks_[static_cast<size_t>(li)];
        SPX_CUDA(cudaSetDevice(rs.device));
        mark(li, 0);
        if (cfg_.wan_block) {  // K1 with shift_msa / scale_msa of this step's modulation
            const float* m = rs.mod_step + layer * 6 * C_;
            ln_modulate_run(x_in[static_cast<size_t>(li)], rs.xm, Lp_, C_, m, m + C_, cfg_.norm_eps,
                            rs.stream, false, true);
        } else if (cfg_.adaln && xm_ready_layer_ != layer) {
            // K1: x_in = LN(x)(1 + scale) + shift, the QKV GEMM's A operand (unless the previous
            // layer's fused O-projection already wrote it)
            const float* m = weights_.at(rs.device).mod + layer * 3 * C_;
            ln_modulate_run(x_in[static_cast<size_t>(li)], rs.xm, Lp_, C_, m, m + C_, cfg_.norm_eps,
                            rs.stream);
        }
        RopeLaunch rl = rope_launch(rs, layer, start_frame);
        if (!local_rope) rl.rotate = 0;  // exchange first, rotate after (apply_rope_global)
        if (!fused) {  // this rank's rows of the all-gathered q | k | v (all heads)
            rl.groups = 1;
            rl.dst = RopeDest{};
            const int64_t off = static_cast<int64_t>(rs.rank) * Lp_ * C_;
            rl.dst.q[0] = rs.gq + off;
            rl.dst.k[0][0] = rs.gk + off;
            rl.dst.v[0][0] = rs.gv + off;
            rl.dst.copies = 1;
            rl.dst_row_stride = C_;
        }
        const GemmPlan& qp = *qkv[static_cast<size_t>(li)];
        if (cfg_.fuse_rope_epilogue && gemm_rope_fusable(qp, rl)) {
            // K2+K3 in one kernel: RoPE + pack in the QKV GEMM epilogue (no qkv round trip)
            gemm_run(qp, rs.stream, &rl);
            mark(li, 1);
        } else if (rl.norm && fused && vpack_enabled() && gemm_vpack_fusable(qp, rl)) {
            // QK-norm: K3 needs whole q / k rows, but v only moves -- the QKV epilogue packs v
            // into the KV ring and K3 streams q | k (2/3 of the qkv round trip)
            rl.skip_v = 1;
            gemm_run(qp, rs.stream, &rl);
            mark(li, 1);
            rope_run(rl, rs.stream);
        } else {
            gemm_run(qp, rs.stream);
            mark(li, 1);
            rope_run(rl, rs.stream);
        }
        mark(li, 2);
        if (local) SPX_CUDA(cudaEventRecord(rs.ev_k3, rs.stream));
    }
    if (fused) {
        if (local) {
            for (int li = 0; li < nl; ++li) {
                RankState& rs = ranks_[static_cast<size_t>(li)];
                SPX_CUDA(cudaSetDevice(rs.device));
                for (int lj = 0; lj < nl; ++lj)
                    if (lj != li)
                        SPX_CUDA(cudaStreamWaitEvent(rs.stream, ranks_[static_cast<size_t>(lj)].ev_k3, 0));
            }
        } else if (peer && P_ > 1) {
            // K3 stored into the peers' buffers; every rank's stores land before attention
            peer_barrier(ranks_[0], 0);
        } else if (nccl && P_ > 1) {
            // one NCCL group == one round: the plan's sends and receives (exchange_plan.cpp)
            RankState& rs = ranks_[0];
            SPX_CUDA(cudaSetDevice(rs.device));
            run_plan(rs, layer, plan_qkv_exchange(part_, rs.rank, block_base_row_));
        }
        // ledger: one fused exchange (q: G-1 peers, k/v: P-1 peers per source) ...
        if (!capturing_) world_->add_stats(0, 0, 1, qkv_exchange_elements(part_), 1);
    } else {
        // three all-gathers along the sequence (collectives.cpp:180-201; ledger +1 each)
        const int64_t shape[4] = {1, Lp_, H_, D_};
        for (int t = 0; t < 3; ++t) {
            std::vector<void*> in, out;
            for (RankState& rs : ranks_) {
                bf16* g = t == 0 ? rs.gq : t == 1 ? rs.gk : rs.gv;
                in.push_back(g + static_cast<int64_t>(rs.rank) * Lp_ * C_);
                out.push_back(g);
            }
            world_->all_gather(in.data(), out.data(), shape, 2, 1);
        }
    }
    if (!local_rope) {
        // apply_rope_global after the exchange: in place on this rank's q and k rows
        for (RankState& rs : ranks_) {
            SPX_CUDA(cudaSetDevice(rs.device));
            const RopeLaunch base = rope_launch(rs, layer, start_frame);
            auto rotate_in_place = [&](bf16* x, int64_t rows, int64_t row_offset, int64_t heads) {
                RopeLaunch r = base;
                r.in = x;
                r.in_row_stride = heads * D_;
                r.rows = rows;
                r.rows_per_batch = rows;
                r.heads = static_cast<int>(heads);
                r.groups = 1;
                r.has_kv = 0;
                r.norm = 0;
                r.row_offset = row_offset;
                r.dst = RopeDest{};
                r.dst.q[0] = x;
                r.dst_row_stride = heads * D_;
                rope_run(r, rs.stream);
            };
            if (fused) {  // the head shard: q rows of this query split, k rows of the block
                rotate_in_place(rs.q_recv, Lq_, rs.p * Lq_, Hl_);
                rotate_in_place(rs.rings[static_cast<size_t>(layer)].k + block_base_row_ * Hl_ * D_,
                                L_, 0, Hl_);
            } else {      // the full sequence, every head (Alg. 1)
                rotate_in_place(rs.gq, L_, 0, H_);
                rotate_in_place(rs.gk, L_, 0, H_);
            }
        }
    }
    if (!fused) {
        // split_heads (collectives.cpp:298-312): this rank's head group (and query split)
        for (RankState& rs : ranks_) {
            SPX_CUDA(cudaSetDevice(rs.device));
            KvRingStorage& ring = rs.rings[static_cast<size_t>(layer)];
            Box4 bq{{1, Lq_, Hl_, D_}, {L_ * C_, C_, D_, 1}, {Lq_ * Hl_ * D_, Hl_ * D_, D_, 1}};
            copy_box_run(rs.q_recv, rs.gq + rs.p * Lq_ * C_ + rs.g * Hl_ * D_, bq, 2, rs.stream);
            Box4 bkv{{1, L_, Hl_, D_}, {L_ * C_, C_, D_, 1}, {L_ * Hl_ * D_, Hl_ * D_, D_, 1}};
            copy_box_run(ring.k + block_base_row_ * Hl_ * D_, rs.gk + rs.g * Hl_ * D_, bkv, 2, rs.stream);
            copy_box_run(ring.v + block_base_row_ * Hl_ * D_, rs.gv + rs.g * Hl_ * D_, bkv, 2, rs.stream);
        }
    }

    // K6 attention, output rows stored straight into their source's o_recv slab
    for (int li = 0; li < nl; ++li) {
        RankState& rs = ranks_[static_cast<size_t>(li)];
        SPX_CUDA(cudaSetDevice(rs.device));
        mark(li, 3);
        mark(li, 4);  // cache: bookkeeping only, the exchange already wrote the ring slots
        AttnPlan plan = rs.attn_plan[static_cast<size_t>(layer)];
        attn_set_segments(&plan, seg_start_, seg_len_, num_segs_);
        if (cfg_.l2_prefetch) {  // this layer's W_o and the next call's W_qkv into L2
            const DeviceWeights& w = weights_.at(rs.device);
            const int64_t next = (layer + 1) % cfg_.layers;
            plan.ops.l2_prefetch[0] = w.wo + layer * C_ * C_;
            plan.ops.l2_prefetch_bytes[0] = C_ * C_ * 2;
            plan.ops.l2_prefetch[1] = w.wqkv + next * 3 * C_ * C_;
            plan.ops.l2_prefetch_bytes[1] = 3 * C_ * C_ * 2;
        }
        for (int64_t c = 0; c < G_; ++c) {
            const int i = static_cast<int>(rs.p * G_ + c);
            if (local || peer) {
                plan.ops.out_base[c] = o_interleaved_ ? o_recv_of(i) + rs.g * Hl_ * D_
                                                      : o_recv_of(i) + rs.g * slab;
            } else {
                plan.ops.out_base[c] = i == rs.rank ? rs.o_recv + rs.g * slab : rs.o_send + c * slab;
            }
        }
        attn_run(plan, rs.stream);
        mark(li, 5);
        if (local) SPX_CUDA(cudaEventRecord(rs.ev_attn, rs.stream));
    }
    if (local) {
        for (int li = 0; li < nl; ++li) {
            RankState& rs = ranks_[static_cast<size_t>(li)];
            SPX_CUDA(cudaSetDevice(rs.device));
            for (int64_t g = 0; g < G_; ++g) {
                const int d = static_cast<int>(rs.p * G_ + g);
                const int ld = local_of(d);
                if (ld != li)
                    SPX_CUDA(cudaStreamWaitEvent(rs.stream, ranks_[static_cast<size_t>(ld)].ev_attn, 0));
            }
        }
    } else if (peer && P_ > 1) {
        // attention stored o rows into their sources' slabs (and every rank is past reading
        // this layer's q buffer, which the next call's K3 overwrites)
        peer_barrier(ranks_[0], 1);
    } else if (nccl && P_ > 1) {
        RankState& rs = ranks_[0];
        SPX_CUDA(cudaSetDevice(rs.device));
        run_plan(rs, layer, plan_out_exchange(part_, rs.rank));
    }
    // ... and one output all-to-all (G-1 peers per rank)
    if (!capturing_) world_->add_stats(0, 1, 0, out_exchange_elements(part_), 1);

    // K8 output projection
    bool fused_ln = true;  // every local rank ran the fused projection + next-layer K1
    for (int li = 0; li < nl; ++li) {
        RankState& rs = ranks_[static_cast<size_t>(li)];
        SPX_CUDA(cudaSetDevice(rs.device));
        // the step's own plan (not a caller's one-off layer call) with the next layer's K1 fused
        const GemmLnPlan* ln = (oproj[static_cast<size_t>(li)] == &rs.o_plan[static_cast<size_t>(layer)] &&
                                static_cast<size_t>(layer) < rs.oln_plan.size() &&
                                rs.oln_plan[static_cast<size_t>(layer)].ok)
                                   ? &rs.oln_plan[static_cast<size_t>(layer)]
                                   : nullptr;
        if (ln) {
            gemm_ln_run(*ln, rs.stream);
        } else {
            gemm_run(*oproj[static_cast<size_t>(li)], rs.stream);
        }
        fused_ln = fused_ln && ln != nullptr;
        mark(li, 6);
        if (cfg_.wan_block) run_wan_tail(rs, layer);  // cross-attention + FFN (token-local)
    }
    xm_ready_layer_ = fused_ln ? layer + 1 : -1;
}

void Engine::run_plan(RankState& rs, int64_t layer, const std::vector<Transfer>& plan) {
    KvRingStorage& ring = rs.rings[static_cast<size_t>(layer)];
    bf16* bases[8] = {rs.q_send, rs.k_send, rs.v_send, rs.o_send, rs.q_recv, ring.k, ring.v,
                      rs.o_recv};
    world_->group_start();
    for (const Transfer& t : plan) {
        bf16* p = bases[t.buf] + t.offset;
        const size_t bytes = static_cast<size_t>(t.elems) * sizeof(bf16);
        if (t.is_send) {
            world_->send(p, bytes, t.peer, rs.stream);
        } else {
            world_->recv(p, bytes, t.peer, rs.stream);
        }
    }
    world_->group_end();
}

void Engine::layer_external(int64_t layer, int64_t block, int64_t start_frame, void* const* x,
                            void* const* y) {
    require(layer >= 0 && layer < cfg_.layers, SPX_ERR_RANGE, "layer out of range");
    require(!cfg_.wan_block, SPX_ERR_UNSUPPORTED,
            "spx_engine_layer: the full Wan block runs through denoise_step / generate");
    require(start_frame >= 0 && start_frame + F_ <= cfg_.num_blocks * F_, SPX_ERR_RANGE,
            "block frames [" + std::to_string(start_frame) + ", " +
                std::to_string(start_frame + F_) + ") exceed table max_frames " +
                std::to_string(cfg_.num_blocks * F_));
    begin_block(block);  // KvCache::update of this call (idempotent within a block)
    std::vector<GemmPlan> qp(ranks_.size()), op(ranks_.size());
    std::vector<const GemmPlan*> qv, ov;
    std::vector<const bf16*> xv;
    for (size_t li = 0; li < ranks_.size(); ++li) {
        RankState& rs = ranks_[li];
        SPX_CUDA(cudaSetDevice(rs.device));
        GemmOperands q = rs.qkv_plan[static_cast<size_t>(layer)].ops;
        if (!cfg_.adaln) q.a = static_cast<const bf16*>(x[li]);  // adaLN: A is K1's output
        q.allow_split_k = !cfg_.sp_bit_exact;  // split-K changes the k order
        gemm_plan(&qp[li], q, device_sm_count(rs.device));
        GemmOperands o = rs.o_plan[static_cast<size_t>(layer)].ops;
        o.out = static_cast<bf16*>(y[li]);
        if (cfg_.adaln) o.residual = static_cast<const bf16*>(x[li]);
        o.allow_split_k = !cfg_.sp_bit_exact;  // split-K changes the k order
        gemm_plan(&op[li], o, device_sm_count(rs.device));
        qv.push_back(&qp[li]);
        ov.push_back(&op[li]);
        xv.push_back(static_cast<const bf16*>(x[li]));
    }
    xm_ready_layer_ = -1;  // a one-off layer call runs its own K1
    run_layer(layer, start_frame, qv, ov, xv);
}

void Engine::run_block(int64_t block, const std::function<void(int64_t)>& load_step) {
    require(block >= 0 && block < cfg_.num_blocks, SPX_ERR_RANGE, "block out of range");
    const int64_t start = cfg_.force_start_frame_zero ? 0 : block * F_;
    begin_block(block);
    for (int64_t step = 0; step < cfg_.denoise_steps; ++step) {
        load_step(step);  // fresh noise into x[0] of every local rank (steps do not chain)
        run_step(start, step);
    }
}

// the layers of one denoise step on x[0] of every local rank (output in x[layers % 2]):
// replayed from a CUDA graph per KV-ring state when graphs_allowed(), enqueued launch by
// launch otherwise
void Engine::run_step(int64_t start, int64_t step) {
    if (!graphs_allowed()) {
        run_step_eager(start, step);
        return;
    }
    RankState& rs = ranks_[0];
    SPX_CUDA(cudaSetDevice(rs.device));
    // everything a step's kernel parameters depend on besides the fixed buffers
    // (the Wan block's timestep embedding reads t[step]: the step is part of its state)
    const std::array<int64_t, 8> key{block_base_row_, num_segs_, seg_start_[0], seg_len_[0],
                                     seg_start_[1], seg_len_[1], start,
                                     cfg_.wan_block ? step : -1};
    auto it = graphs_.find(key);
    if (it == graphs_.end()) {
        // first sight of this state: run it launch by launch (lazy per-device set-up such as
        // table uploads and kernel attributes happens outside any capture) and capture on
        // the next occurrence
        if (seen_.insert(key).second) {
            run_step_eager(start, step);
            return;
        }
        if (graphs_.size() >= kMaxGraphs) {  // evict the least recently used
            auto lru = graphs_.begin();
            for (auto g = graphs_.begin(); g != graphs_.end(); ++g)
                if (g->second.last_use < lru->second.last_use) lru = g;
            SPX_CUDA(cudaStreamSynchronize(rs.stream));
            SPX_CUDA(cudaGraphExecDestroy(lru->second.exec));
            graphs_.erase(lru);
        }
        StepGraph sg;
        const int64_t l0 = launch_count();
        cudaGraph_t g = nullptr;
        SPX_CUDA(cudaStreamBeginCapture(rs.stream, cudaStreamCaptureModeThreadLocal));
        capturing_ = true;
        bool ok = true;
        try {
            run_step_eager(start, step);
        } catch (const Error&) {
            ok = false;
        }
        capturing_ = false;
        const cudaError_t ce = cudaStreamEndCapture(rs.stream, &g);
        cudaError_t ie = cudaErrorUnknown;
        if (ok && ce == cudaSuccess && g) ie = cudaGraphInstantiateWithFlags(&sg.exec, g, 0);
        static const bool graph_debug = std::getenv("SPX_GRAPH_DEBUG") != nullptr;
        if (graph_debug && g) {  // profiling: how many of the captured edges kept PDL
            size_t nn = 0, ne = 0;
            cudaGraphGetNodes(g, nullptr, &nn);
            cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &ne);
            std::vector<cudaGraphNode_t> from(ne), to(ne);
            std::vector<cudaGraphEdgeData> ed(ne);
            size_t ne2 = ne;
            cudaGraphGetEdges_v2(g, from.data(), to.data(), ed.data(), &ne2);
            size_t prog = 0;
            for (size_t i = 0; i < ne2; ++i) prog += ed[i].type == cudaGraphDependencyTypeProgrammatic;
            std::fprintf(stderr, "step graph: %zu nodes, %zu edges, %zu programmatic\n", nn, ne2, prog);
        }
        if (g) cudaGraphDestroy(g);
        sg.launches = launch_count() - l0;
        count_launch(static_cast<int>(-sg.launches));  // captured, not launched
        if (!ok || ce != cudaSuccess || ie != cudaSuccess) {
            // the step does not capture on this system: clear the capture error and stay on
            // the launch-by-launch path for this engine (nothing of the step ran)
            cudaGetLastError();
            graphs_enabled_ = false;
            run_step_eager(start, step);
            return;
        }
        it = graphs_.emplace(key, sg).first;
    }
    it->second.last_use = ++graph_clock_;
    SPX_CUDA(cudaGraphLaunch(it->second.exec, rs.stream));
    count_launch(static_cast<int>(it->second.launches));
    for (int64_t l = 0; l < cfg_.layers; ++l) {  // the ledger of the replayed layer calls
        world_->add_stats(0, 0, 1, qkv_exchange_elements(part_), 1);
        world_->add_stats(0, 1, 0, out_exchange_elements(part_), 1);
    }
}

bool Engine::graphs_allowed() const {
    static const bool env_on = [] {
        const char* e = std::getenv("SPX_GRAPHS");
        return !(e && std::atoi(e) == 0);
    }();
    // one local rank (multi-rank LOCAL worlds order their streams with host-side events),
    // no NCCL calls, the optimized schedule (its ledger is the fixed per-call pair above),
    // no per-stage profiling events and no span tracing
    return env_on && graphs_enabled_ && ranks_.size() == 1 &&
           world_->transport() != SPX_TRANSPORT_NCCL && cfg_.ablation == SPX_ABLATION_ALL &&
           cfg_.profile == 0 && !span_tracing() &&
           !(world_->transport() == SPX_TRANSPORT_PEER && !peers_ready_);
}

void Engine::drop_graphs() {
    if (graphs_.empty()) return;
    for (RankState& rs : ranks_) {
        cudaSetDevice(rs.device);
        cudaStreamSynchronize(rs.stream);
    }
    for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second.exec);
    graphs_.clear();
}

void Engine::run_step_eager(int64_t start, int64_t step) {
    xm_ready_layer_ = -1;  // layer 0 of every step runs its own K1
    if (cfg_.wan_block) {  // this step's timestep embedding -> every layer's modulation
        for (RankState& rs : ranks_) {
            SPX_CUDA(cudaSetDevice(rs.device));
            wan_time_embedding_run(rs.te, static_cast<int>(step), rs.stream);
        }
    }
    for (int64_t l = 0; l < cfg_.layers; ++l) {
        std::vector<const GemmPlan*> qv, ov;
        std::vector<const bf16*> xv;
        for (RankState& rs : ranks_) {
            qv.push_back(&rs.qkv_plan[static_cast<size_t>(l)]);
            ov.push_back(&rs.o_plan[static_cast<size_t>(l)]);
            xv.push_back(rs.x[l % 2]);
        }
        run_layer(l, start, qv, ov, xv);
    }
}

void Engine::denoise_step(int64_t block, int64_t step, const void* const* x, void* const* y) {
    require(block >= 0 && block < cfg_.num_blocks, SPX_ERR_RANGE, "block out of range");
    require(step >= 0 && step < cfg_.denoise_steps, SPX_ERR_RANGE,
            "denoise step " + std::to_string(step) + " out of range [0, " +
                std::to_string(cfg_.denoise_steps) + ")");
    const size_t slice_bytes = static_cast<size_t>(Lp_ * C_) * sizeof(bf16);
    begin_block(block);  // KvCache::update of this step (the block's slots are overwritten)
    for (RankState& rs : ranks_) {
        SPX_CUDA(cudaSetDevice(rs.device));
        SPX_CUDA(cudaMemcpyAsync(rs.x[0], x[rs.local], slice_bytes, cudaMemcpyDeviceToDevice,
                                 rs.stream));
    }
    run_step(cfg_.force_start_frame_zero ? 0 : block * F_, step);
    const int fin = static_cast<int>(cfg_.layers % 2);
    for (RankState& rs : ranks_) {
        SPX_CUDA(cudaSetDevice(rs.device));
        SPX_CUDA(cudaMemcpyAsync(y[rs.local], rs.x[fin], slice_bytes, cudaMemcpyDeviceToDevice,
                                 rs.stream));
    }
}

void Engine::generate_block(int64_t block, const uint16_t* noise_host, uint16_t* out_host) {
    const size_t block_elems = static_cast<size_t>(L_ * C_);
    const size_t slice_bytes = static_cast<size_t>(Lp_ * C_) * sizeof(bf16);
    if (noise_host) {
        // caller's noise: step s + 1 is uploaded (copy stream, into a staging buffer) while
        // step s computes; each step starts with a device copy staging -> x[0]
        for (RankState& rs : ranks_) {
            SPX_CUDA(cudaSetDevice(rs.device));
            if (!rs.copy_stream) {
                SPX_CUDA(cudaStreamCreateWithFlags(&rs.copy_stream, cudaStreamNonBlocking));
                for (int b = 0; b < 2; ++b) {
                    rs.nstage[b] = dev_alloc<bf16>(rs, static_cast<size_t>(Lp_ * C_));
                    SPX_CUDA(cudaEventCreateWithFlags(&rs.ev_ready[b], cudaEventDisableTiming));
                    SPX_CUDA(cudaEventCreateWithFlags(&rs.ev_used[b], cudaEventDisableTiming));
                }
            }
        }
        auto upload = [&](int64_t step) {
            for (RankState& rs : ranks_) {
                SPX_CUDA(cudaSetDevice(rs.device));
                const int b = static_cast<int>(step % 2);
                // the staging buffer's previous contents (step - 2) were consumed
                SPX_CUDA(cudaStreamWaitEvent(rs.copy_stream, rs.ev_used[b], 0));
                SPX_CUDA(cudaMemcpyAsync(rs.nstage[b],
                                         noise_host + static_cast<size_t>(step) * block_elems +
                                             static_cast<size_t>(rs.rank * Lp_ * C_),
                                         slice_bytes, cudaMemcpyHostToDevice, rs.copy_stream));
                SPX_CUDA(cudaEventRecord(rs.ev_ready[b], rs.copy_stream));
            }
        };
        // the previous call's last step may still read a staging buffer: order the first upload
        for (RankState& rs : ranks_) {
            SPX_CUDA(cudaSetDevice(rs.device));
            for (int b = 0; b < 2; ++b) SPX_CUDA(cudaEventRecord(rs.ev_used[b], rs.stream));
        }
        upload(0);
        run_block(block, [&](int64_t step) {
            for (RankState& rs : ranks_) {
                SPX_CUDA(cudaSetDevice(rs.device));
                const int b = static_cast<int>(step % 2);
                SPX_CUDA(cudaStreamWaitEvent(rs.stream, rs.ev_ready[b], 0));
                SPX_CUDA(cudaMemcpyAsync(rs.x[0], rs.nstage[b], slice_bytes, cudaMemcpyDeviceToDevice,
                                         rs.stream));
                SPX_CUDA(cudaEventRecord(rs.ev_used[b], rs.stream));
            }
            if (step + 1 < cfg_.denoise_steps) upload(step + 1);
        });
    } else {
        run_block(block, [&](int64_t step) {
            // block_noise (generator.cpp:42-46), drawn in full on every rank, then sliced
            if (!noise_pinned_) {
                SPX_CUDA(cudaMallocHost(reinterpret_cast<void**>(&noise_pinned_),
                                        block_elems * sizeof(uint16_t)));
            }
            world_->synchronize();  // the previous H2D from the staging buffer is done
            noise_f64_.resize(block_elems);
            fill_noise(derive_seed(cfg_.seed, 0x10, static_cast<uint64_t>(block),
                                   static_cast<uint64_t>(step)),
                       static_cast<int64_t>(block_elems), D_, noise_f64_.data());
            for (size_t i = 0; i < block_elems; ++i) noise_pinned_[i] = f64_to_bf16(noise_f64_[i]);
            for (RankState& rs : ranks_) {
                SPX_CUDA(cudaSetDevice(rs.device));
                SPX_CUDA(cudaMemcpyAsync(rs.x[0], noise_pinned_ + static_cast<size_t>(rs.rank * Lp_ * C_),
                                         slice_bytes, cudaMemcpyHostToDevice, rs.stream));
            }
        });
    }
    const int fin = static_cast<int>(cfg_.layers % 2);
    for (RankState& rs : ranks_) {
        SPX_CUDA(cudaSetDevice(rs.device));
        SPX_CUDA(cudaMemcpyAsync(out_host + static_cast<size_t>(rs.local) * Lp_ * C_, rs.x[fin],
                                 slice_bytes, cudaMemcpyDeviceToHost, rs.stream));
    }
    synchronize();
}

// Streaming generator (the paper's overlap theme): n blocks
// back to back with every host copy off the compute stream. The copy stream uploads step k + 1
// of the noise into one of two staging buffers while step k computes; at the end of a block
// the latent is copied (device to device) into one of two output staging buffers and a third
// stream downloads it to the host while the next block computes. The host thread only
// enqueues (graph launches + copies) and waits once at the end.
void Engine::generate_stream(const int64_t* blocks, int64_t n, const uint16_t* const* noise_host,
                             uint16_t* const* out_host) {
    require(n >= 0 && (n == 0 || (blocks && noise_host && out_host)), SPX_ERR_CONFIG,
            "null argument");
    for (int64_t i = 0; i < n; ++i)
        require(blocks[i] >= 0 && blocks[i] < cfg_.num_blocks && noise_host[i] && out_host[i],
                SPX_ERR_RANGE, "block " + std::to_string(i) + " out of range or null buffer");
    const size_t block_elems = static_cast<size_t>(L_ * C_);
    const size_t slice_bytes = static_cast<size_t>(Lp_ * C_) * sizeof(bf16);
    for (RankState& rs : ranks_) {
        SPX_CUDA(cudaSetDevice(rs.device));
        if (!rs.copy_stream) {
            SPX_CUDA(cudaStreamCreateWithFlags(&rs.copy_stream, cudaStreamNonBlocking));
            for (int b = 0; b < 2; ++b) {
                rs.nstage[b] = dev_alloc<bf16>(rs, static_cast<size_t>(Lp_ * C_));
                SPX_CUDA(cudaEventCreateWithFlags(&rs.ev_ready[b], cudaEventDisableTiming));
                SPX_CUDA(cudaEventCreateWithFlags(&rs.ev_used[b], cudaEventDisableTiming));
            }
        }
        if (!rs.d2h_stream) {
            SPX_CUDA(cudaStreamCreateWithFlags(&rs.d2h_stream, cudaStreamNonBlocking));
            for (int b = 0; b < 2; ++b) {
                rs.ostage[b] = dev_alloc<bf16>(rs, static_cast<size_t>(Lp_ * C_));
                SPX_CUDA(cudaEventCreateWithFlags(&rs.ev_out_ready[b], cudaEventDisableTiming));
                SPX_CUDA(cudaEventCreateWithFlags(&rs.ev_out_free[b], cudaEventDisableTiming));
            }
        }
        // earlier work (a previous call) may still read the staging buffers
        for (int b = 0; b < 2; ++b) {
            SPX_CUDA(cudaEventRecord(rs.ev_used[b], rs.stream));
            SPX_CUDA(cudaEventRecord(rs.ev_out_free[b], rs.d2h_stream));
        }
    }
    const int fin = static_cast<int>(cfg_.layers % 2);
    int64_t k = 0;  // global step counter (staging buffer k % 2)
    auto upload = [&](int64_t i, int64_t step, int64_t kk) {
        for (RankState& rs : ranks_) {
            SPX_CUDA(cudaSetDevice(rs.device));
            const int b = static_cast<int>(kk % 2);
            SPX_CUDA(cudaStreamWaitEvent(rs.copy_stream, rs.ev_used[b], 0));
            SPX_CUDA(cudaMemcpyAsync(rs.nstage[b],
                                     noise_host[i] + static_cast<size_t>(step) * block_elems +
                                         static_cast<size_t>(rs.rank * Lp_ * C_),
                                     slice_bytes, cudaMemcpyHostToDevice, rs.copy_stream));
            SPX_CUDA(cudaEventRecord(rs.ev_ready[b], rs.copy_stream));
        }
    };
    if (n > 0) upload(0, 0, 0);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t block = blocks[i];
        run_block(block, [&](int64_t step) {
            for (RankState& rs : ranks_) {
                SPX_CUDA(cudaSetDevice(rs.device));
                const int b = static_cast<int>(k % 2);
                SPX_CUDA(cudaStreamWaitEvent(rs.stream, rs.ev_ready[b], 0));
                SPX_CUDA(cudaMemcpyAsync(rs.x[0], rs.nstage[b], slice_bytes,
                                         cudaMemcpyDeviceToDevice, rs.stream));
                SPX_CUDA(cudaEventRecord(rs.ev_used[b], rs.stream));
            }
            // the next step's noise (this block's next step, or the next block's first)
            if (step + 1 < cfg_.denoise_steps)
                upload(i, step + 1, k + 1);
            else if (i + 1 < n)
                upload(i + 1, 0, k + 1);
            ++k;
        });
        for (RankState& rs : ranks_) {
            SPX_CUDA(cudaSetDevice(rs.device));
            const int b = static_cast<int>(i % 2);
            SPX_CUDA(cudaStreamWaitEvent(rs.stream, rs.ev_out_free[b], 0));
            SPX_CUDA(cudaMemcpyAsync(rs.ostage[b], rs.x[fin], slice_bytes, cudaMemcpyDeviceToDevice,
                                     rs.stream));
            SPX_CUDA(cudaEventRecord(rs.ev_out_ready[b], rs.stream));
            SPX_CUDA(cudaStreamWaitEvent(rs.d2h_stream, rs.ev_out_ready[b], 0));
            SPX_CUDA(cudaMemcpyAsync(out_host[i] + static_cast<size_t>(rs.local) * Lp_ * C_,
                                     rs.ostage[b], slice_bytes, cudaMemcpyDeviceToHost,
                                     rs.d2h_stream));
            SPX_CUDA(cudaEventRecord(rs.ev_out_free[b], rs.d2h_stream));
        }
    }
    for (RankState& rs : ranks_) {
        SPX_CUDA(cudaSetDevice(rs.device));
        SPX_CUDA(cudaStreamSynchronize(rs.d2h_stream));
        SPX_CUDA(cudaStreamSynchronize(rs.copy_stream));
    }
    synchronize();
}

void Engine::generate_block_device(int64_t block, const void* const* noise_dev,
                                   void* const* out_dev) {
    const size_t slice_bytes = static_cast<size_t>(Lp_ * C_) * sizeof(bf16);
    run_block(block, [&](int64_t step) {
        for (RankState& rs : ranks_) {
            SPX_CUDA(cudaSetDevice(rs.device));
            SPX_CUDA(cudaMemcpyAsync(rs.x[0],
                                     static_cast<const uint8_t*>(noise_dev[rs.local]) +
                                         static_cast<size_t>(step) * slice_bytes,
                                     slice_bytes, cudaMemcpyDeviceToDevice, rs.stream));
        }
    });
    const int fin = static_cast<int>(cfg_.layers % 2);
    for (RankState& rs : ranks_) {
        SPX_CUDA(cudaSetDevice(rs.device));
        SPX_CUDA(cudaMemcpyAsync(out_dev[rs.local], rs.x[fin], slice_bytes,
                                 cudaMemcpyDeviceToDevice, rs.stream));
    }
}

void Engine::generate(uint16_t* out_host) {
    const size_t per_block = static_cast<size_t>(ranks_.size()) * Lp_ * C_;
    for (int64_t b = 0; b < cfg_.num_blocks; ++b)
        generate_block(b, nullptr, out_host + static_cast<size_t>(b) * per_block);
}

void Engine::synchronize() {
    world_->synchronize();
    check_peer_error();
    harvest_events();
}

void Engine::harvest_events() {
    if (pending_events_.empty()) return;
    SPX_CUDA(cudaSetDevice(ranks_[0].device));
    for (StageEvents& se : pending_events_) {
        SPX_CUDA(cudaEventSynchronize(se.ev[se.level == 1 ? 6 : 5]));
        for (int k = 0; k < 6; ++k) {
            if (se.level != 1 && k != 4) continue;
            float ms = 0.0f;
            SPX_CUDA(cudaEventElapsedTime(&ms, se.ev[k], se.ev[k + 1]));
            stage_ms_[k] += ms;
        }
        ++profiled_calls_;
        free_events_.push_back(se);
    }
    pending_events_.clear();
}

void Engine::stage_times(double out_ms[6], int64_t* calls) {
    synchronize();
    for (int k = 0; k < 6; ++k) out_ms[k] = stage_ms_[k];
    if (calls) *calls = profiled_calls_;
}

void Engine::reset_stage_times() {
    synchronize();
    for (double& v : stage_ms_) v = 0.0;
    profiled_calls_ = 0;
}

}  // namespace spx
