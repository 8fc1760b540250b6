// engine.hpp -- the optimized Causal-RoPE SP schedule and the block-wise AR driver on device.
//
// Reference: sp_self_attention_engine with every ablation flag on
// (proj/src/sp_attention.cpp:197-313) driven by generate() (proj/src/generator.cpp:50-147).
//
// Partition: P = G * S ranks; rank r serves head group g = r mod G (H/G heads) and query
// split p = r / G (rows [p L/S, (p+1) L/S) of the block). Pure Ulysses is S = 1. Token rows
// stay sharded by rank (L/P each) for the projections.
//
// Per layer call and rank (one CUDA stream each):
//   K2  qkv[L/P][3C]      = x[L/P][C] W_qkv^T                       (tcgen05 GEMM)
//   K3  [RMSNorm] + Causal-RoPE(q, k), bf16, written straight into
//         q_recv of rank (p_src, g)   rows (src mod G) * L/P           (fused exchange,
//         KV ring of ranks (*, g)     rows base + src * L/P             one round)
//   K6  o = softmax(q K^T / sqrt D) V over the ring's <= 2 segments, rows scattered into
//         o_recv[g] of their source rank                              (output exchange)
//   K8  y[L/P][C]         = o_recv[G][L/P][H/G*D] W_o^T (3-D TMA un-interleave)
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <vector>

#include "../../include/spx.h"
#include "exchange_plan.hpp"
#include "kernels.hpp"
#include "kv_ring.hpp"
#include "rope_table.hpp"
#include "world.hpp"

namespace spx {

// the full Wan2.1 block's parameters beyond the self-attention projections (cfg.wan_block),
// one copy per device; [out][in] row-major bf16 matrices, fp32 vectors
struct WanWeights {
    float* b_qkv = nullptr;                  // [layers][3C] self-attention q | k | v biases
    float* b_o = nullptr;                    // [layers][C]
    float* n3_w = nullptr;                   // [layers][C] affine LayerNorm (norm3)
    float* n3_b = nullptr;
    bf16* cq = nullptr;                      // [layers][C][C] cross-attention projections
    bf16* ck = nullptr;
    bf16* cv = nullptr;
    bf16* co = nullptr;
    float* bcq = nullptr;                    // [layers][C]
    float* bck = nullptr;
    float* bcv = nullptr;
    float* bco = nullptr;
    bf16* cnq = nullptr;                     // [layers][C] cross-attention RMSNorm weights
    bf16* cnk = nullptr;
    bf16* w1 = nullptr;                      // [layers][F][C] FFN
    float* b1 = nullptr;                     // [layers][F]
    bf16* w2 = nullptr;                      // [layers][C][F]
    float* b2 = nullptr;                     // [layers][C]
    float* mod_param = nullptr;              // [layers][6][C]
    bf16* tw1 = nullptr;                     // [C][freq_dim] time embedding
    float* tb1 = nullptr;
    bf16* tw2 = nullptr;                     // [C][C]
    float* tb2 = nullptr;
    bf16* pw = nullptr;                      // [6C][C] time projection
    float* pb = nullptr;
    bf16* xw1 = nullptr;                     // [C][text_dim] text embedding
    float* xb1 = nullptr;
    bf16* xw2 = nullptr;                     // [C][C]
    float* xb2 = nullptr;
    float* tsteps = nullptr;                 // [denoise_steps]
    // per video: the text context and every layer's cross-attention K (RMSNorm'd) and V
    bf16* text = nullptr;                    // [text_len][text_dim]
    bf16* text_h = nullptr;                  // [text_len][C]
    bf16* ctx = nullptr;                     // [text_len][C]
    bf16* ktmp = nullptr;                    // [text_len][C]
    bf16* k_ctx = nullptr;                   // [layers][text_len][C]
    bf16* v_ctx = nullptr;
};

struct DeviceWeights {
    int device = 0;
    bf16* wqkv = nullptr;  // [layers][3C][C]
    bf16* wo = nullptr;    // [layers][C][C]
    bf16* norm_q = nullptr;  // [layers][C]
    bf16* norm_k = nullptr;
    float* mod = nullptr;  // [layers][3][C] adaLN shift | scale | gate (cfg.adaln)
    WanWeights wan;        // cfg.wan_block
    std::vector<void*> wan_allocs;
};

struct RankState {
    int rank = 0;
    int local = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
    int g = 0, p = 0;
    bf16* x[2] = {nullptr, nullptr};  // (L/P, C) ping-pong
    bf16* qkv = nullptr;              // (L/P, 3C)
    bf16* xm = nullptr;               // (L/P, C) adaLN-modulated layer input (cfg.adaln)
    bf16* q_recv = nullptr;           // (L/S, H/G, D)
    bf16* o_recv = nullptr;           // [G][L/P][H/G*D]
    bf16* q_send = nullptr;           // NCCL: [G][L/P][H/G][D]
    bf16* k_send = nullptr;
    bf16* v_send = nullptr;
    bf16* o_send = nullptr;           // NCCL: [G][L/P][H/G*D]
    bf16* gq = nullptr;               // ablation without the fused exchange: all-gathered
    bf16* gk = nullptr;               //   q, k, v of the whole block, (L, C)
    bf16* gv = nullptr;
    float2* tab_scratch = nullptr;    // ablation without precomputed freqs: per-call table
    uint64_t* flags = nullptr;        // PEER: [kPeerSlots][P] barrier epochs (IPC-shared)
    std::vector<KvRingStorage> rings; // per layer
    std::vector<GemmPlan> qkv_plan;   // per layer, A = x[layer % 2]
    std::vector<GemmPlan> o_plan;     // per layer, out = x[(layer + 1) % 2]
    // Wan mode (adaLN): layer l's O-projection fused with layer l + 1's LayerNorm + modulation
    // (gemm_ln.cu), writing x[(l + 1) % 2] and xm; ok = false where it does not apply
    std::vector<GemmLnPlan> oln_plan;
    std::vector<AttnPlan> attn_plan;  // per layer
    void* attn_ws = nullptr;          // split-KV workspace (shared by the layers)
    size_t attn_ws_bytes = 0;
    cudaEvent_t ev_k3 = nullptr;
    cudaEvent_t ev_attn = nullptr;
    // cfg.wan_block: the cross-attention and FFN tail of every layer, and the step's modulation
    bf16* ca_q = nullptr;             // (L/P, C) cross-attention q projection
    bf16* ca_qn = nullptr;            // (L/P, H, D) after its RMSNorm
    bf16* ca_o = nullptr;             // (L/P, C) cross-attention output
    bf16* ffn_h = nullptr;            // (L/P, F) GELU(x W1^T + b1)
    float* mod_step = nullptr;        // [layers][6][C] modulation of the current denoise step
    float* temb = nullptr;            // time-embedding scratch: sinus | h1 | e | e0
    WanTimeEmbed te;
    std::vector<GemmPlan> cq_plan, co_plan, f1_plan, f2_plan;  // per layer
    std::vector<AttnPlan> ca_plan;    // per layer: q over the cached context K/V
    // generate_block from host noise: the next denoise step's noise is uploaded on a copy
    // stream into a staging buffer while the current step computes
    bf16* nstage[2] = {nullptr, nullptr};
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_ready[2] = {nullptr, nullptr};
    cudaEvent_t ev_used[2] = {nullptr, nullptr};
    // generate_stream: block latents leave through two output staging buffers on a D2H stream
    bf16* ostage[2] = {nullptr, nullptr};
    cudaStream_t d2h_stream = nullptr;
    cudaEvent_t ev_out_ready[2] = {nullptr, nullptr};
    cudaEvent_t ev_out_free[2] = {nullptr, nullptr};
    std::vector<void*> allocations;
};

struct StageEvents {
    cudaEvent_t ev[7];
    int level = 1;  // 1: all seven stage marks; 2: the attention bracket (ev[4], ev[5]) only
};

class Engine {
  public:
    Engine(World* world, const spx_engine_config& cfg);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    static void validate(const spx_engine_config& cfg, int world_size);

    void info(int64_t out[8]) const;
    void seed_weights();
    void set_layer_weights(int64_t layer, const uint16_t* wq, const uint16_t* wk,
                           const uint16_t* wv, const uint16_t* wo);
    void set_norm_weights(int64_t layer, const uint16_t* wq, const uint16_t* wk);
    void set_modulation(int64_t layer, const float* shift, const float* scale, const float* gate);
    void set_wan_layer(int64_t layer, const spx_wan_layer_weights& w);
    void set_wan_embeddings(const spx_wan_embed_weights& w);
    void set_timesteps(const float* t);
    void set_context(const uint16_t* text);
    void begin_block(int64_t block_index);
    // a new video: every layer's KV cache empty again (generate() builds fresh caches,
    // generator.cpp:69-81); device ring memory is reused as is
    void reset_cache();
    void layer_external(int64_t layer, int64_t block, int64_t start_frame, void* const* x,
                        void* const* y);
    void generate_block(int64_t block, const uint16_t* noise_host, uint16_t* out_host);
    // device-resident variant (no host copies, no synchronisation): noise_dev[local] holds
    // (steps, L/P, C) bf16, out_dev[local] receives (L/P, C)
    void generate_block_device(int64_t block, const void* const* noise_dev, void* const* out_dev);
    void generate(uint16_t* out_host);
    // n blocks back to back (blocks[i] may repeat: a block re-denoised overwrites its slots),
    // noise_host[i]: (steps, L, C) bf16 of block i, out_host[i]: (rows of the local ranks, C);
    // host copies overlap the compute (upload of the next step, download of the last block)
    void generate_stream(const int64_t* blocks, int64_t n, const uint16_t* const* noise_host,
                         uint16_t* const* out_host);
    // one denoise step of a block (generator.cpp:94-110): x[local] (L/P, C) device bf16 in,
    // y[local] after every layer; asynchronous on the world's streams
    void denoise_step(int64_t block, int64_t step, const void* const* x, void* const* y);
    void synchronize();
    void stage_times(double out_ms[6], int64_t* calls);
    void reset_stage_times();
    // 0 off, 1 every stage (six CUDA-event intervals per call), 2 attention launch only,
    // 3 attention launch of every 8th call
    void set_profile(int level) { cfg_.profile = level; }
    // per-step CUDA graphs on (default) / off (every launch enqueued by the host)
    int64_t graph_count() const { return static_cast<int64_t>(graphs_.size()); }
    void set_graphs(bool on) {
        graphs_enabled_ = on;
        if (!on) drop_graphs();
    }
    spx_comm_stats stats() const { return world_->stats(); }
    // PEER transport: CUDA IPC handles of this rank's exchange buffers, and the mapping of
    // every peer's (blobs of all ranks in rank order)
    std::vector<uint8_t> ipc_export() const;
    void ipc_import(const uint8_t* blobs, size_t bytes_per_rank);

  private:
    void allocate();
    void run_block(int64_t block, const std::function<void(int64_t)>& load_step);
    void run_step(int64_t start_frame, int64_t step);
    void run_step_eager(int64_t start_frame, int64_t step);
    void run_wan_tail(RankState& rs, int64_t layer);
    void allocate_wan();
    void build_wan_plans();
    void seed_wan_weights();
    void compute_context();
    bool graphs_allowed() const;
    void drop_graphs();
    void build_plans();
    // x_in[local]: the layer input (the K1 source with cfg.adaln; otherwise the QKV plans'
    // A operand already points at it)
    void run_layer(int64_t layer, int64_t start_frame, const std::vector<const GemmPlan*>& qkv,
                   const std::vector<const GemmPlan*>& oproj, const std::vector<const bf16*>& x_in);
    void harvest_events();
    void run_plan(RankState& rs, int64_t layer, const std::vector<Transfer>& plan);
    RopeLaunch rope_launch(const RankState& rs, int64_t layer, int64_t start_frame) const;
    int local_of(int rank) const;
    // exchange destinations of a global rank: a local rank's buffers (LOCAL), or the IPC
    // mapping of a peer's (PEER; the own rank maps to its own buffers)
    bf16* q_recv_of(int rank) const;
    bf16* o_recv_of(int rank) const;
    bf16* ring_k_of(int rank, int64_t layer) const;
    bf16* ring_v_of(int rank, int64_t layer) const;
    void peer_barrier(RankState& rs, int slot);
    void check_peer_error();
    void sync_weight_devices();  // throws SPX_ERR_COLLECTIVE after a timed-out PEER barrier

    World* world_;
    spx_engine_config cfg_;
    // geometry
    int64_t F_, Hg_, Wg_, HW_, L_, H_, D_, C_, P_, G_, S_, Lp_, Lq_, Hl_;
    int64_t FF_ = 0, TL_ = 0, TD_ = 0, FD_ = 0;
    bool o_interleaved_ = false;  // attention output stored as (L/P, C) rows (see constructor)  // wan_block: ffn, text len / dim, freq dim
    int64_t cap_frames_ = 0;
    Partition part_{};
    std::unique_ptr<RopeTable> table_;
    std::map<int, DeviceWeights> weights_;
    std::vector<RankState> ranks_;  // local ranks
    FrameRing frames_;
    int64_t block_base_row_ = 0;
    int seg_start_[2] = {0, 0};
    int seg_len_[2] = {0, 0};
    int num_segs_ = 0;
    bool have_block_ = false;
    int64_t current_block_ = -1;
    // pinned staging for generated noise
    uint16_t* noise_pinned_ = nullptr;
    std::vector<double> noise_f64_;
    // PEER transport
    struct PeerView {
        bf16* q_recv = nullptr;
        bf16* o_recv = nullptr;
        uint64_t* flags = nullptr;
        std::vector<bf16*> ring_k, ring_v;
    };
    std::vector<PeerView> peers_;  // by global rank
    std::vector<void*> ipc_opened_;
    bool peers_ready_ = false;
    // per-step CUDA graphs, keyed by the KV-ring state and start frame (the only launch
    // parameters that change between steps); see run_step
    struct StepGraph {
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;
        uint64_t last_use = 0;
    };
    static constexpr size_t kMaxGraphs = 24;
    std::map<std::array<int64_t, 8>, StepGraph> graphs_;
    std::set<std::array<int64_t, 8>> seen_;  // states run once (captured on the next run)
    uint64_t graph_clock_ = 0;
    bool capturing_ = false;
    // the layer whose K1 output (xm) the previous fused O-projection already wrote (-1: none)
    int64_t xm_ready_layer_ = -1;
    bool graphs_enabled_ = true;
    int* peer_error_host_ = nullptr;  // host-mapped: 1 + the rank a PEER barrier timed out on
    int* peer_error_dev_ = nullptr;
    uint64_t peer_timeout_ns_ = 0;
    // profiling
    std::vector<StageEvents> pending_events_;
    std::vector<StageEvents> free_events_;
    double stage_ms_[6] = {0, 0, 0, 0, 0, 0};
    int64_t profiled_calls_ = 0;
    int64_t profile_seq_ = 0;
};

// G (head groups) for P ranks and H heads: the largest divisor of P that divides H
int64_t choose_head_groups(int64_t P, int64_t H);
// the Wan FFN hidden size of a config (cfg.ffn_dim, or the Wan2.1 ratio rounded to 64)
int64_t wan_ffn_dim(const spx_engine_config& c);

}  // namespace spx
