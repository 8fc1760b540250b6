// engine_wan.cpp -- the full Wan2.1 DiT block on the device engine (cfg.wan_block = 1).
//
// The reference model is attention-only; the Self-Forcing generator the paper
// accelerates runs Wan2.1-1.3B blocks, whose forward (wan/modules/model.py,
// WanAttentionBlock.forward) is, per layer l with e = modulation_param[l] + e0(t):
//
//   x = x + e[2] * self_attn(LN(x) (1 + e[1]) + e[0])          K1, K2+K3, K6, K8 (engine.cpp)
//   x = x + cross_attn(LN_affine(x), context)                  K1', Q GEMM, RMSNorm, K6, O GEMM
//   x = x + e[5] * ffn(LN(x) (1 + e[4]) + e[3])                K1, GEMM + GELU, GEMM
//
// with biases on every projection, QK-RMSNorm in both attentions and GELU(tanh) in the FFN.
// The cross-attention and the FFN are token-local: under sequence parallelism each rank runs
// them on its own L/P rows with every head and the full cached context, no exchange. The
// context K/V of every layer is computed once per video (set_context), the timestep
// embedding once per denoise step (wan.cu). Everything is bf16 storage, fp32 accumulation,
// on the same tcgen05 GEMM and attention kernels as the self-attention path.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.hpp"
#include "engine.hpp"
#include "host_rng.hpp"

namespace spx {

namespace {

template <class T>
T* wan_alloc(DeviceWeights& w, size_t count) {
    void* p = nullptr;
    SPX_CUDA(cudaMalloc(&p, count * sizeof(T)));
    SPX_CUDA(cudaMemset(p, 0, count * sizeof(T)));
    w.wan_allocs.push_back(p);
    return static_cast<T*>(p);
}

template <class T>
T* rank_alloc(RankState& rs, size_t count) {
    void* p = nullptr;
    SPX_CUDA(cudaMalloc(&p, count * sizeof(T)));
    SPX_CUDA(cudaMemset(p, 0, count * sizeof(T)));
    rs.allocations.push_back(p);
    return static_cast<T*>(p);
}

}  // namespace

void Engine::allocate_wan() {
    const size_t L = static_cast<size_t>(cfg_.layers), C = static_cast<size_t>(C_),
                 F = static_cast<size_t>(FF_), TL = static_cast<size_t>(TL_),
                 TD = static_cast<size_t>(TD_), FD = static_cast<size_t>(FD_);
    for (auto& kv : weights_) {
        SPX_CUDA(cudaSetDevice(kv.first));
        DeviceWeights& d = kv.second;
        WanWeights& w = d.wan;
        w.b_qkv = wan_alloc<float>(d, L * 3 * C);
        w.b_o = wan_alloc<float>(d, L * C);
        w.n3_w = wan_alloc<float>(d, L * C);
        w.n3_b = wan_alloc<float>(d, L * C);
        for (bf16** m : {&w.cq, &w.ck, &w.cv, &w.co}) *m = wan_alloc<bf16>(d, L * C * C);
        for (float** b : {&w.bcq, &w.bck, &w.bcv, &w.bco}) *b = wan_alloc<float>(d, L * C);
        w.cnq = wan_alloc<bf16>(d, L * C);
        w.cnk = wan_alloc<bf16>(d, L * C);
        w.w1 = wan_alloc<bf16>(d, L * F * C);
        w.b1 = wan_alloc<float>(d, L * F);
        w.w2 = wan_alloc<bf16>(d, L * C * F);
        w.b2 = wan_alloc<float>(d, L * C);
        w.mod_param = wan_alloc<float>(d, L * 6 * C);
        w.tw1 = wan_alloc<bf16>(d, C * FD);
        w.tb1 = wan_alloc<float>(d, C);
        w.tw2 = wan_alloc<bf16>(d, C * C);
        w.tb2 = wan_alloc<float>(d, C);
        w.pw = wan_alloc<bf16>(d, 6 * C * C);
        w.pb = wan_alloc<float>(d, 6 * C);
        w.xw1 = wan_alloc<bf16>(d, C * TD);
        w.xb1 = wan_alloc<float>(d, C);
        w.xw2 = wan_alloc<bf16>(d, C * C);
        w.xb2 = wan_alloc<float>(d, C);
        w.tsteps = wan_alloc<float>(d, static_cast<size_t>(cfg_.denoise_steps));
        w.text = wan_alloc<bf16>(d, TL * TD);
        w.text_h = wan_alloc<bf16>(d, TL * C);
        w.ctx = wan_alloc<bf16>(d, TL * C);
        w.ktmp = wan_alloc<bf16>(d, TL * C);
        w.k_ctx = wan_alloc<bf16>(d, L * TL * C);
        w.v_ctx = wan_alloc<bf16>(d, L * TL * C);
        // RMSNorm / affine-LayerNorm weights default to 1 (bf16 0x3F80, fp32 1.0f)
        std::vector<uint16_t> ones16(L * C, 0x3F80u);
        SPX_CUDA(cudaMemcpy(w.cnq, ones16.data(), L * C * 2, cudaMemcpyHostToDevice));
        SPX_CUDA(cudaMemcpy(w.cnk, ones16.data(), L * C * 2, cudaMemcpyHostToDevice));
        std::vector<float> ones32(L * C, 1.0f);
        SPX_CUDA(cudaMemcpy(w.n3_w, ones32.data(), L * C * 4, cudaMemcpyHostToDevice));
        // default schedule: t = 1000 -> 1000 / steps evenly (Self-Forcing's 4 steps:
        // 1000, 750, 500, 250)
        std::vector<float> ts(static_cast<size_t>(cfg_.denoise_steps));
        for (size_t i = 0; i < ts.size(); ++i)
            ts[i] = 1000.0f - 1000.0f * static_cast<float>(i) / static_cast<float>(ts.size());
        SPX_CUDA(cudaMemcpy(w.tsteps, ts.data(), ts.size() * 4, cudaMemcpyHostToDevice));
    }
    for (RankState& rs : ranks_) {
        SPX_CUDA(cudaSetDevice(rs.device));
        const size_t rows = static_cast<size_t>(Lp_);
        rs.ca_q = rank_alloc<bf16>(rs, rows * C);
        rs.ca_qn = rank_alloc<bf16>(rs, rows * C);
        rs.ca_o = rank_alloc<bf16>(rs, rows * C);
        rs.ffn_h = rank_alloc<bf16>(rs, rows * F);
        rs.mod_step = rank_alloc<float>(rs, L * 6 * C);
        rs.temb = rank_alloc<float>(rs, FD + C + C + 6 * C);
        const WanWeights& w = weights_.at(rs.device).wan;
        WanTimeEmbed& te = rs.te;
        te.tsteps = w.tsteps;
        te.freq_dim = static_cast<int>(FD_);
        te.dim = static_cast<int>(C_);
        te.layers = static_cast<int>(cfg_.layers);
        te.w1 = w.tw1;
        te.b1 = w.tb1;
        te.w2 = w.tw2;
        te.b2 = w.tb2;
        te.wp = w.pw;
        te.bp = w.pb;
        te.mod_param = w.mod_param;
        te.sinus = rs.temb;
        te.h1 = te.sinus + FD;
        te.e = te.h1 + C;
        te.e0 = te.e + C;
        te.mod = rs.mod_step;
    }
}

void Engine::build_wan_plans() {
    for (RankState& rs : ranks_) {
        SPX_CUDA(cudaSetDevice(rs.device));
        const int sms = device_sm_count(rs.device);
        const WanWeights& w = weights_.at(rs.device).wan;
        const size_t nl = static_cast<size_t>(cfg_.layers);
        rs.cq_plan.resize(nl);
        rs.co_plan.resize(nl);
        rs.f1_plan.resize(nl);
        rs.f2_plan.resize(nl);
        rs.ca_plan.resize(nl);
        for (int64_t l = 0; l < cfg_.layers; ++l) {
            bf16* xo = rs.x[(l + 1) % 2];  // the layer's output row block (after the self-attn)
            auto base = [&](const bf16* a, int64_t k, const bf16* b, bf16* out, int64_t n) {
                GemmOperands g{};
                g.a = a;
                g.a_row_stride = k;
                g.a_group_stride = Lp_ * k;
                g.groups = 1;
                g.k_inner = static_cast<int>(k);
                g.b = b;
                g.b_row_stride = k;
                g.out = out;
                g.out_row_stride = n;
                g.M = static_cast<int>(Lp_);
                g.N = static_cast<int>(n);
                g.K = static_cast<int>(k);
                g.b_constant = true;
                return g;
            };
            // cross-attention q = LN_affine(x) Wq^T + bq
            GemmOperands cq = base(rs.xm, C_, w.cq + l * C_ * C_, rs.ca_q, C_);
            cq.bias = w.bcq + l * C_;
            cq.allow_split_k = !cfg_.sp_bit_exact;  // split-K changes the k order
            gemm_plan(&rs.cq_plan[static_cast<size_t>(l)], cq, sms);
            // x += ca_o Wo^T + bo (in place, no gate)
            GemmOperands co = base(rs.ca_o, C_, w.co + l * C_ * C_, xo, C_);
            co.epi_mode = 1;
            co.residual = xo;
            co.residual_row_stride = C_;
            co.bias = w.bco + l * C_;
            co.allow_split_k = !cfg_.sp_bit_exact;  // split-K changes the k order
            gemm_plan(&rs.co_plan[static_cast<size_t>(l)], co, sms);
            // h = GELU(LN(x)(1 + scale_mlp) + shift_mlp) W1^T + b1)
            GemmOperands f1 = base(rs.xm, C_, w.w1 + l * FF_ * C_, rs.ffn_h, FF_);
            f1.epi_mode = 3;
            f1.bias = w.b1 + l * FF_;
            f1.allow_split_k = !cfg_.sp_bit_exact;  // split-K changes the k order
            gemm_plan(&rs.f1_plan[static_cast<size_t>(l)], f1, sms);
            // x += gate_mlp * (h W2^T + b2) (in place)
            GemmOperands f2 = base(rs.ffn_h, FF_, w.w2 + l * C_ * FF_, xo, C_);
            f2.epi_mode = 1;
            f2.residual = xo;
            f2.residual_row_stride = C_;
            f2.gate = rs.mod_step + (l * 6 + 5) * C_;
            f2.bias = w.b2 + l * C_;
            f2.allow_split_k = !cfg_.sp_bit_exact;  // split-K changes the k order
            gemm_plan(&rs.f2_plan[static_cast<size_t>(l)], f2, sms);
            // cross attention of this rank's rows (all heads) over the layer's context K/V;
            // no workspace: one CTA per (query tile, head), the same arithmetic at every P
            AttnOperands a{};
            a.q = rs.ca_qn;
            a.q_rows = Lp_;
            a.k = w.k_ctx + l * TL_ * C_;
            a.v = w.v_ctx + l * TL_ * C_;
            a.kv_rows = TL_;
            a.batch = 1;
            a.heads = static_cast<int>(H_);
            a.head_dim = static_cast<int>(D_);
            a.sq = static_cast<int>(Lp_);
            a.seg_start[0] = 0;
            a.seg_len[0] = static_cast<int>(TL_);
            a.num_segs = 1;
            a.out_base[0] = rs.ca_o;
            a.rows_per_chunk = static_cast<int>(Lp_);
            a.out_row_stride = C_;
            a.prefer_v3 = cfg_.sp_bit_exact != 0;
            attn_plan(&rs.ca_plan[static_cast<size_t>(l)], a, sms);
        }
    }
}

// RMSNorm over the C channels of `rows` rows of `in` (row stride in_stride) into dst (row
// stride C), weights w: K3 without rotation (the QK-RMSNorm of the cross-attention)
static RopeLaunch norm_only(const bf16* in, int64_t in_stride, int64_t rows, int64_t H, int64_t D,
                            int64_t hw, int64_t grid_w, const bf16* w, float eps, bf16* dst) {
    RopeLaunch r{};
    r.in = in;
    r.in_row_stride = in_stride;
    r.rows = rows;
    r.rows_per_batch = rows;
    r.heads = static_cast<int>(H);
    r.head_dim = static_cast<int>(D);
    r.groups = 1;
    r.has_kv = 0;
    r.hw = hw;
    r.grid_w = grid_w;
    r.norm = 1;
    r.norm_w_q = w;
    r.norm_eps = eps;
    r.rotate = 0;
    r.dst.q[0] = dst;
    r.dst.copies = 1;
    r.dst_row_stride = H * D;
    return r;
}

void Engine::run_wan_tail(RankState& rs, int64_t layer) {
    const size_t l = static_cast<size_t>(layer);
    const WanWeights& w = weights_.at(rs.device).wan;
    bf16* xo = rs.x[(layer + 1) % 2];
    // cross-attention: x += Wo attn(RMSNorm(Wq LN_affine(x) + bq), K_ctx, V_ctx) + bo
    ln_modulate_run(xo, rs.xm, Lp_, C_, w.n3_b + layer * C_, w.n3_w + layer * C_, cfg_.norm_eps,
                    rs.stream, true, false);
    gemm_run(rs.cq_plan[l], rs.stream);
    rope_run(norm_only(rs.ca_q, C_, Lp_, H_, D_, HW_, Wg_, w.cnq + layer * C_, cfg_.norm_eps, rs.ca_qn),
             rs.stream);
    attn_run(rs.ca_plan[l], rs.stream);
    gemm_run(rs.co_plan[l], rs.stream);
    // FFN: x += gate_mlp * (W2 GELU(W1 (LN(x)(1 + scale_mlp) + shift_mlp) + b1) + b2)
    const float* m = rs.mod_step + layer * 6 * C_;
    ln_modulate_run(xo, rs.xm, Lp_, C_, m + 3 * C_, m + 4 * C_, cfg_.norm_eps, rs.stream, false, true);
    gemm_run(rs.f1_plan[l], rs.stream);
    gemm_run(rs.f2_plan[l], rs.stream);
}

// the context K/V of every layer from the text already in w.text (set_context / seeding)
void Engine::compute_context() {
    for (auto& kv : weights_) {
        const int dev = kv.first;
        SPX_CUDA(cudaSetDevice(dev));
        WanWeights& w = kv.second.wan;
        cudaStream_t st = nullptr;
        for (RankState& rs : ranks_)
            if (rs.device == dev) {
                st = rs.stream;
                break;
            }
        const int sms = device_sm_count(dev);
        auto gemm = [&](const bf16* a, int64_t k, const bf16* b, bf16* out, const float* bias,
                        int epi) {
            GemmOperands g{};
            g.a = a;
            g.a_row_stride = k;
            g.a_group_stride = TL_ * k;
            g.groups = 1;
            g.k_inner = static_cast<int>(k);
            g.b = b;
            g.b_row_stride = k;
            g.out = out;
            g.out_row_stride = C_;
            g.M = static_cast<int>(TL_);
            g.N = static_cast<int>(C_);
            g.K = static_cast<int>(k);
            g.bias = bias;
            g.epi_mode = epi;
            GemmPlan plan;
            g.allow_split_k = !cfg_.sp_bit_exact;  // split-K changes the k order
            gemm_plan(&plan, g, sms);
            gemm_run(plan, st);
        };
        // text_embedding: Linear(text_dim, C), GELU(tanh), Linear(C, C)
        gemm(w.text, TD_, w.xw1, w.text_h, w.xb1, 3);
        gemm(w.text_h, C_, w.xw2, w.ctx, w.xb2, 0);
        for (int64_t l = 0; l < cfg_.layers; ++l) {
            gemm(w.ctx, C_, w.ck + l * C_ * C_, w.ktmp, w.bck + l * C_, 0);
            rope_run(norm_only(w.ktmp, C_, TL_, H_, D_, HW_, Wg_, w.cnk + l * C_, cfg_.norm_eps,
                               w.k_ctx + l * TL_ * C_),
                     st);
            gemm(w.ctx, C_, w.cv + l * C_ * C_, w.v_ctx + l * TL_ * C_, w.bcv + l * C_, 0);
        }
    }
    synchronize();
}

void Engine::set_context(const uint16_t* text) {
    require(cfg_.wan_block, SPX_ERR_CONFIG, "set_context needs cfg.wan_block = 1");
    require(text != nullptr, SPX_ERR_CONFIG, "null text");
    synchronize();
    for (auto& kv : weights_) {
        SPX_CUDA(cudaSetDevice(kv.first));
        SPX_CUDA(cudaMemcpy(kv.second.wan.text, text, static_cast<size_t>(TL_ * TD_) * 2,
                            cudaMemcpyHostToDevice));
    }
    sync_weight_devices();
    compute_context();
}

void Engine::set_timesteps(const float* t) {
    require(cfg_.wan_block, SPX_ERR_CONFIG, "set_timesteps needs cfg.wan_block = 1");
    require(t != nullptr, SPX_ERR_CONFIG, "null timesteps");
    synchronize();
    for (auto& kv : weights_) {
        SPX_CUDA(cudaSetDevice(kv.first));
        SPX_CUDA(cudaMemcpy(kv.second.wan.tsteps, t, static_cast<size_t>(cfg_.denoise_steps) * 4,
                            cudaMemcpyHostToDevice));
    }
    sync_weight_devices();
}

void Engine::set_wan_layer(int64_t layer, const spx_wan_layer_weights& in) {
    require(cfg_.wan_block, SPX_ERR_CONFIG, "set_wan_layer needs cfg.wan_block = 1");
    require(layer >= 0 && layer < cfg_.layers, SPX_ERR_RANGE, "layer out of range");
    synchronize();
    const size_t C = static_cast<size_t>(C_), F = static_cast<size_t>(FF_);
    for (auto& kv : weights_) {
        SPX_CUDA(cudaSetDevice(kv.first));
        WanWeights& w = kv.second.wan;
        auto put = [&](void* dst, const void* src, size_t bytes) {
            if (src) SPX_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
        };
        const int64_t l = layer;
        put(w.b_qkv + l * 3 * C, in.self_bq, C * 4);
        put(w.b_qkv + l * 3 * C + C, in.self_bk, C * 4);
        put(w.b_qkv + l * 3 * C + 2 * C, in.self_bv, C * 4);
        put(w.b_o + l * C, in.self_bo, C * 4);
        put(w.n3_w + l * C, in.norm3_w, C * 4);
        put(w.n3_b + l * C, in.norm3_b, C * 4);
        put(w.cq + l * C * C, in.cross_q, C * C * 2);
        put(w.ck + l * C * C, in.cross_k, C * C * 2);
        put(w.cv + l * C * C, in.cross_v, C * C * 2);
        put(w.co + l * C * C, in.cross_o, C * C * 2);
        put(w.bcq + l * C, in.cross_bq, C * 4);
        put(w.bck + l * C, in.cross_bk, C * 4);
        put(w.bcv + l * C, in.cross_bv, C * 4);
        put(w.bco + l * C, in.cross_bo, C * 4);
        put(w.cnq + l * C, in.cross_norm_q, C * 2);
        put(w.cnk + l * C, in.cross_norm_k, C * 2);
        put(w.w1 + l * F * C, in.ffn_w1, F * C * 2);
        put(w.b1 + l * F, in.ffn_b1, F * 4);
        put(w.w2 + l * C * F, in.ffn_w2, C * F * 2);
        put(w.b2 + l * C, in.ffn_b2, C * 4);
        put(w.mod_param + l * 6 * C, in.modulation, 6 * C * 4);
    }
    sync_weight_devices();
    // the cached context K/V depend on this layer's cross-attention K/V weights
    if (in.cross_k || in.cross_v || in.cross_bk || in.cross_bv || in.cross_norm_k) compute_context();
}

void Engine::set_wan_embeddings(const spx_wan_embed_weights& in) {
    require(cfg_.wan_block, SPX_ERR_CONFIG, "set_wan_embeddings needs cfg.wan_block = 1");
    synchronize();
    const size_t C = static_cast<size_t>(C_);
    for (auto& kv : weights_) {
        SPX_CUDA(cudaSetDevice(kv.first));
        WanWeights& w = kv.second.wan;
        auto put = [&](void* dst, const void* src, size_t bytes) {
            if (src) SPX_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
        };
        put(w.tw1, in.time_w1, C * static_cast<size_t>(FD_) * 2);
        put(w.tb1, in.time_b1, C * 4);
        put(w.tw2, in.time_w2, C * C * 2);
        put(w.tb2, in.time_b2, C * 4);
        put(w.pw, in.proj_w, 6 * C * C * 2);
        put(w.pb, in.proj_b, 6 * C * 4);
        put(w.xw1, in.text_w1, C * static_cast<size_t>(TD_) * 2);
        put(w.xb1, in.text_b1, C * 4);
        put(w.xw2, in.text_w2, C * C * 2);
        put(w.xb2, in.text_b2, C * 4);
    }
    sync_weight_devices();
    if (in.text_w1 || in.text_b1 || in.text_w2 || in.text_b2) compute_context();
}

// Synthetic Wan-block parameters (random init of the architecture; the reference has no Wan
// weights): N(0, 1/fan_in) matrices, N(0, 0.02^2) biases, norm weights 1 + N(0, 0.1^2),
// modulation parameters N(0, 1/C) (Wan's own init), a N(0, 1) text context. Drawn on the
// device by a counter-based generator seeded from derive_seed(seed, 0x40 + kind, layer).
void Engine::seed_wan_weights() {
    synchronize();
    const size_t C = static_cast<size_t>(C_), F = static_cast<size_t>(FF_);
    for (auto& kv : weights_) {
        SPX_CUDA(cudaSetDevice(kv.first));
        WanWeights& w = kv.second.wan;
        cudaStream_t st = nullptr;  // legacy stream, drained by sync_weight_devices below
        auto mat = [&](bf16* p, size_t n, size_t fan_in, uint64_t kind, int64_t l) {
            fill_normal_bf16_run(p, static_cast<int64_t>(n),
                                 derive_seed(cfg_.seed, 0x40 + kind, static_cast<uint64_t>(l + 1)),
                                 1.0f / std::sqrt(static_cast<float>(fan_in)), 0.0f, st);
        };
        auto vec = [&](float* p, size_t n, float scale, float offset, uint64_t kind, int64_t l) {
            fill_normal_f32_run(p, static_cast<int64_t>(n),
                                derive_seed(cfg_.seed, 0x40 + kind, static_cast<uint64_t>(l + 1)),
                                scale, offset, st);
        };
        for (int64_t l = 0; l < cfg_.layers; ++l) {
            vec(w.b_qkv + l * 3 * C, 3 * C, 0.02f, 0.0f, 1, l);
            vec(w.b_o + l * C, C, 0.02f, 0.0f, 2, l);
            vec(w.n3_w + l * C, C, 0.1f, 1.0f, 3, l);
            vec(w.n3_b + l * C, C, 0.02f, 0.0f, 4, l);
            mat(w.cq + l * C * C, C * C, C, 5, l);
            mat(w.ck + l * C * C, C * C, C, 6, l);
            mat(w.cv + l * C * C, C * C, C, 7, l);
            mat(w.co + l * C * C, C * C, C, 8, l);
            vec(w.bcq + l * C, C, 0.02f, 0.0f, 9, l);
            vec(w.bck + l * C, C, 0.02f, 0.0f, 10, l);
            vec(w.bcv + l * C, C, 0.02f, 0.0f, 11, l);
            vec(w.bco + l * C, C, 0.02f, 0.0f, 12, l);
            fill_normal_bf16_run(w.cnq + l * C, static_cast<int64_t>(C),
                                 derive_seed(cfg_.seed, 0x40 + 13, static_cast<uint64_t>(l + 1)), 0.1f,
                                 1.0f, st);
            fill_normal_bf16_run(w.cnk + l * C, static_cast<int64_t>(C),
                                 derive_seed(cfg_.seed, 0x40 + 14, static_cast<uint64_t>(l + 1)), 0.1f,
                                 1.0f, st);
            mat(w.w1 + l * F * C, F * C, C, 15, l);
            vec(w.b1 + l * F, F, 0.02f, 0.0f, 16, l);
            mat(w.w2 + l * C * F, C * F, F, 17, l);
            vec(w.b2 + l * C, C, 0.02f, 0.0f, 18, l);
            vec(w.mod_param + l * 6 * C, 6 * C, 1.0f / std::sqrt(static_cast<float>(C)), 0.0f, 19, l);
        }
        mat(w.tw1, C * static_cast<size_t>(FD_), static_cast<size_t>(FD_), 20, 0);
        vec(w.tb1, C, 0.02f, 0.0f, 21, 0);
        mat(w.tw2, C * C, C, 22, 0);
        vec(w.tb2, C, 0.02f, 0.0f, 23, 0);
        mat(w.pw, 6 * C * C, C, 24, 0);
        vec(w.pb, 6 * C, 0.02f, 0.0f, 25, 0);
        mat(w.xw1, C * static_cast<size_t>(TD_), static_cast<size_t>(TD_), 26, 0);
        vec(w.xb1, C, 0.02f, 0.0f, 27, 0);
        mat(w.xw2, C * C, C, 28, 0);
        vec(w.xb2, C, 0.02f, 0.0f, 29, 0);
        fill_normal_bf16_run(w.text, TL_ * TD_, derive_seed(cfg_.seed, 0x40 + 30, 0), 1.0f, 0.0f, st);
    }
    sync_weight_devices();
    compute_context();
}

}  // namespace spx
