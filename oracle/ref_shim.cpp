// ref_shim.cpp -- C entry points over the UNMODIFIED reference sources (test/bench
// infrastructure only). Compiled together with /root/reference/proj/src/{tensor,rope,
// collectives,kv_cache,sp_attention,generator}.cpp into oracle/_ref/libspattn_ref.so by
// oracle/Makefile; nothing here re-implements reference logic, it only marshals arguments.
//
//   ref_generate ....... spattn::generate (proj/src/generator.cpp:50-147), any variant/P
//   ref_sample_call .... times the reference's own per-call operators (project_tokens,
//                        apply_rope_global, KvCache, scaled_dot_product_attention) on a
//                        bounded sample of one layer call, spread over host threads, and
//                        extrapolates the full call (bench.py cpu_baseline / --impl reference)
#include <chrono>
#include <cstdint>
#include <cstring>
#include <optional>
#include <thread>
#include <vector>

#include "spattn/generator.hpp"
#include "spattn/kv_cache.hpp"
#include "spattn/rope.hpp"
#include "spattn/sp_attention.hpp"
#include "spattn/tensor.hpp"

using namespace spattn;

extern "C" {

// cfg: frames, Hg, Wg, blocks, layers, steps, heads, head_dim, world, window(<0 none),
//      variant (0 reference, 1 baseline, 2 optimized), ablation mask (bit0 fused, bit1 local
//      rope, bit2 precomputed), force_start_frame_zero
// out: blocks x L x H x D; ledger (5 int64) optional. Returns 0, or 1 + error kind on throw.
int ref_generate(const int64_t* cfg, uint64_t seed, double* out, int64_t* ledger) {
    try {
        GenerationConfig c;
        c.grid_per_block = GridSpec{cfg[0], cfg[1], cfg[2]};
        c.num_blocks = cfg[3];
        c.layers = cfg[4];
        c.denoise_steps = cfg[5];
        c.heads = cfg[6];
        c.head_dim = cfg[7];
        c.world_size = static_cast<int>(cfg[8]);
        if (cfg[9] >= 0) c.window_frames = cfg[9];
        const int64_t mask = cfg[11];
        AblationFlags f{(mask & 1) != 0, (mask & 2) != 0, (mask & 4) != 0};
        if (cfg[10] == 0) c.variant = PipelineVariant::reference();
        if (cfg[10] == 1) c.variant = PipelineVariant::baseline();
        if (cfg[10] == 2) c.variant = PipelineVariant::optimized(f);
        c.force_start_frame_zero = cfg[12] != 0;
        c.seed = seed;
        GenerationResult r = generate(c);
        size_t off = 0;
        for (const Tensor4& t : r.block_outputs) {
            std::memcpy(out + off, t.data(), static_cast<size_t>(t.numel()) * sizeof(double));
            off += static_cast<size_t>(t.numel());
        }
        if (ledger) {
            ledger[0] = r.profile.ledger.all_gather;
            ledger[1] = r.profile.ledger.all_to_all;
            ledger[2] = r.profile.ledger.fused_all_to_all;
            ledger[3] = r.profile.ledger.elements_sent;
            ledger[4] = r.profile.ledger.rounds;
        }
        return 0;
    } catch (const ShapeError&) {
        return 2;
    } catch (const PartitionError&) {
        return 3;
    } catch (const ConfigError&) {
        return 4;
    } catch (const RangeError&) {
        return 5;
    } catch (...) {
        return 1;
    }
}

// One reference layer call (reference_self_attention at P = 1, sp_attention.cpp:317-348) on
// the shape (F, Hg, Wg, H, D) with a cache of kv_frames frames, timed on a bounded sample:
// `tokens` projected tokens and `rows` attention query rows per thread, `threads` threads.
// out[0] = extrapolated seconds for the full call; out[1..5] = per-stage seconds (qkv, rope,
// cache, attention, output) extrapolated; out[6] = sample wall seconds.
int ref_sample_call(const int64_t* shape, int64_t kv_frames, int64_t tokens, int64_t rows,
                    int64_t threads, double* out) {
    try {
        const int64_t F = shape[0], Hg = shape[1], Wg = shape[2], H = shape[3], D = shape[4];
        const int64_t L = F * Hg * Wg, dim = H * D;
        using clk = std::chrono::steady_clock;
        const auto wall0 = clk::now();
        Rng rng(derive_seed(0, 0x77));
        const AttentionLayerParams params = AttentionLayerParams::seeded(dim, derive_seed(0, 0x20, 0));
        const RopeFrequencyTable table = precompute_frequencies(kv_frames + F, Hg, Wg, D);
        const Tensor4 x_tok = random_tensor(Shape4{1, tokens, H, D}, rng);
        const Tensor4 q_full = random_tensor(Shape4{1, L, H, D}, rng);
        const Tensor4 kv_block = random_tensor(Shape4{1, L, H, D}, rng);

        // projections: 3 (qkv) + 1 (o) project_tokens over `tokens` tokens per thread
        auto t0 = clk::now();
        {
            std::vector<std::thread> ts;
            for (int64_t t = 0; t < threads; ++t)
                ts.emplace_back([&] {
                    Tensor4 a = project_tokens(x_tok, params.w_q);
                    Tensor4 b = project_tokens(x_tok, params.w_k);
                    Tensor4 c = project_tokens(x_tok, params.w_v);
                    Tensor4 d = project_tokens(a, params.w_o);
                    (void)b;
                    (void)c;
                    (void)d;
                });
            for (auto& th : ts) th.join();
        }
        const double proj_s = std::chrono::duration<double>(clk::now() - t0).count();
        const double proj_call = proj_s * static_cast<double>(L) / static_cast<double>(tokens * threads);

        // rope on the full q and k (cheap, measured in full)
        t0 = clk::now();
        Tensor4 qr = apply_rope_global(q_full, GridSpec{F, Hg, Wg}, table, kv_frames);
        Tensor4 kr = apply_rope_global(kv_block, GridSpec{F, Hg, Wg}, table, kv_frames);
        const double rope_s = std::chrono::duration<double>(clk::now() - t0).count();

        // cache: kv_frames history + this block, then read (measured in full)
        t0 = clk::now();
        KvCache cache(Hg * Wg);
        for (int64_t b = 0; b * F < kv_frames; ++b) cache.update(b, kv_block, kv_block);
        cache.update(1000000, kr, kv_block);
        auto kv = cache.read();
        const double cache_s = std::chrono::duration<double>(clk::now() - t0).count();

        // attention: `rows` query rows per thread against the full cache
        t0 = clk::now();
        {
            std::vector<std::thread> ts;
            for (int64_t t = 0; t < threads; ++t)
                ts.emplace_back([&, t] {
                    Tensor4 qs = qr.slice(Axis::Seq, (t * rows) % (L - rows + 1), rows);
                    Tensor4 o = scaled_dot_product_attention(qs, kv.first, kv.second);
                    (void)o;
                });
            for (auto& th : ts) th.join();
        }
        const double attn_s = std::chrono::duration<double>(clk::now() - t0).count();
        const double attn_call = attn_s * static_cast<double>(L) / static_cast<double>(rows * threads);

        out[1] = proj_call * 0.75;
        out[2] = rope_s;
        out[3] = cache_s;
        out[4] = attn_call;
        out[5] = proj_call * 0.25;
        out[0] = out[1] + out[2] + out[3] + out[4] + out[5];
        out[6] = std::chrono::duration<double>(clk::now() - wall0).count();
        return 0;
    } catch (...) {
        return 1;
    }
}

}  // extern "C"
