// attention.cu -- K6: chunk-causal flash attention over the rolling KV ring.
//
// Reference semantics: scaled_dot_product_attention (proj/src/tensor.cpp:161-209): per
// (b, h, i) logits q.k/sqrt(D), max-subtracted softmax, o = sum w v / sum w, NO mask -- the
// block causality is structural (the cache only exposes past + current frames). Softmax is
// order-invariant, so the ring's two chronological segments are visited in storage order.
//
// Two kernels, one CTA per 128-row query tile of one head (or a piece of its kv range), the kv
// range split between two softmax warpgroups that ping-pong against one MMA thread; host
// selection in attn_run:
//   attn_fwd_v3_kernel  one O accumulator shared by both warpgroups, separate P buffers;
//                       persistent over the tiles when every tile is whole, or (kPair) a 2-CTA
//                       cluster per tile, each CTA half of the kv range, merged through DSMEM
//   attn_fwd_v2_kernel  per-warpgroup O; mixed layouts (unsplit tiles first, then split-KV tiles
//                       merged through a workspace) and the single-wave unsplit layouts
// (Measured slower and removed: CTA-pair MMAs, K/V multicast across a CTA pair, v2's own
// DSMEM pair merge, stream-K pieces, a slot-1 epilogue -- DESIGN.md section 5 has the numbers.)
#include <algorithm>

#include <atomic>
#include <cstdio>
#include <vector>
#include <tuple>
#include <mutex>
#include <map>
#include <functional>
#include <cstdlib>

#include "common.hpp"
#include "kernels.hpp"
#include "sm100.cuh"
#include "tma.hpp"

namespace spx {

using namespace sm100;

namespace {

constexpr int kBQ = 128;     // query rows per CTA
constexpr int kBKV = 128;    // kv rows per tile
// exponentials computed by the FMA-pipe polynomial, out of every 8 (the rest on MUFU.EX2).
// Re-measured once the profiling branch was compiled out of the exp loop (it had been
// predicated into every element): 3 of 8 0.1080-0.1100 vs 0 of 8 0.1097-0.1111 ms at the
// Wan chunk (4 of 8 is slower again, 0.1146) -- the MUFU pipe is close to its limit.
#ifndef SPX_POLY_OF_8
#define SPX_POLY_OF_8 3  // 3 of every 8 exponentials on the FMA pipe (A/B after the loop cleanup: ~1-1.5 %)
#endif
// P_i hand-off to the MMA thread: one arrival per softmax warp (after __syncwarp) instead of
// one per thread
// profiling-only variants of the hot loop (SPX_ATTN_EXPERIMENT=2: exponentials on the FMA
// pipe) are compiled in only with -DSPX_ATTN_PROFILING=1: a runtime branch inside the
// unrolled exp loop is predicated, i.e. it costs issue slots on every element
// the same share for v3 (separate tuning: A/B on one box, kbench attn, 2 reps: of 1 / 2 / 3 /
// 4 / 5 -> 0.1043 / 0.1048 / 0.1054 / 0.1060 / 0.1094 ms at the Wan chunk and 0.670 / 0.680 /
// 0.686 / 0.688 / 0.716 ms at 32760 keys). The persistent v3 re-tuned (profiles/r02aq, 2 reps):
// 0 / 1 / 2 -> 0.1014 / 0.1016 / 0.1037 ms at the chunk, 0.669 / 0.677 / 0.690 ms at 32760 keys:
// every exponential on the MUFU
#ifndef SPX_V3_POLY_OF_8
#define SPX_V3_POLY_OF_8 0
#endif
#ifndef SPX_ATTN_PROFILING
#define SPX_ATTN_PROFILING 0
#endif
#ifndef SPX_PFULL_PER_WARP
#define SPX_PFULL_PER_WARP 0
#endif

struct AttnParams {
    int sq;
    int seg_start[2];
    int seg_len[2];
    int seg_tiles0;   // kv tiles in segment 0
    int total_tiles;
    float scale_log2;
    bf16* out_base[8];
    int rows_per_chunk;
    int64_t out_row_stride;
    int64_t out_batch_stride;
    // split-KV (v2 kernel). Cluster modes: gridDim.z CTAs per (query tile, head). Mode 0: a
    // 1-D grid; tiles (t = head * qt + q_tile) below n_full run unsplit, the rest in `splits`
    int splits;
    int n_full;
    int qt;           // query tiles per head (unpadded)
    int heads;
    int q_tiles;
    int* counters;   // [q_tiles][heads], zero between launches
    float* ws_lse;   // [splits][q_tiles * 128][heads]
    float* ws_o;     // [splits][q_tiles * 128][heads][D]
    int experiment;  // profiling only (SPX_ATTN_EXPERIMENT): 1 skip softmax math, 2 no MUFU
    const uint8_t* pf[2];  // L2 prefetch ranges (see AttnOperands::l2_prefetch)
    int64_t pf_bytes[2];
    long long* trace;      // SPX_ATTN_EXPERIMENT=5: per-CTA clock64 marks [cta][16][4]
    unsigned long long* span;  // SPX_SPAN_TRACE
    // raw operand pointers (v3's exact fallback path and the small-D kernel)
    const bf16* q_ptr;
    const bf16* k_ptr;
    const bf16* v_ptr;
    int64_t q_row_stride;   // elements between query rows (heads * D)
    int64_t kv_row_stride;  // elements between kv rows
};

__device__ __forceinline__ void attn_mark(const AttnParams& p, int k) {
    if (p.experiment != 5) return;
    const int64_t me = (static_cast<int64_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    if (me < 1024) p.trace[me * 64 + k] = clock64();
}
// profiling (SPX_ATTN_EXPERIMENT=5): global start (slot 7) / end (slot 8) in globaltimer ns and
// the SM id (slot 9) of this CTA, for a per-SM timeline across CTAs
__device__ __forceinline__ void attn_mark_global(const AttnParams& p, int k) {
    if (p.experiment != 5) return;
    const int64_t me = (static_cast<int64_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    if (me >= 1024) return;
    p.trace[me * 64 + k] = static_cast<long long>(globaltimer_ns());
    if (k == 7) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.trace[me * 64 + 9] = smid;
    }
}

// this CTA's share of the L2 prefetch ranges, 16 KB bulk prefetches (no smem, no barrier)
__device__ __forceinline__ void l2_prefetch_share(const AttnParams& p) {
    const int64_t ctas = static_cast<int64_t>(gridDim.x) * gridDim.y * gridDim.z;
    const int64_t me = (static_cast<int64_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    for (int r = 0; r < 2; ++r) {
        const int64_t n = p.pf_bytes[r];
        if (n <= 0) continue;
        constexpr int64_t kPiece = 16384;
        const int64_t pieces = (n + kPiece - 1) / kPiece;
        for (int64_t i = me; i < pieces; i += ctas) {
            const int64_t off = i * kPiece;
            const uint32_t bytes = static_cast<uint32_t>(min(kPiece, n - off)) & ~15u;
            if (bytes)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.pf[r] + off), "r"(bytes)
                             : "memory");
        }
    }
}

__device__ __forceinline__ void kv_tile_coords(const AttnParams& p, int j, int& row, int& valid) {
    if (j < p.seg_tiles0) {
        row = p.seg_start[0] + j * kBKV;
        valid = min(kBKV, p.seg_len[0] - j * kBKV);
    } else {
        const int t = j - p.seg_tiles0;
        row = p.seg_start[1] + t * kBKV;
        valid = min(kBKV, p.seg_len[1] - t * kBKV);
    }
}

// =========================================================================================
// v2: one 128-row query tile per CTA, its KV range split between two softmax warpgroups
// (slot 0: first half of the kv tiles, slot 1: second half) that ping-pong against the
// single MMA thread, P written back into TMEM over its S (TS-MMA: A operand from TMEM),
// K/V tiles streamed through one 6-deep smem ring in exact MMA consumption order, and the
// two partial (O, m, l) merged in-CTA at the end (TMEM is CTA-wide: each warpgroup reads
// both O accumulators for its half of the head dim).
//
//   warp 0      TMA producer            warp 1   MMA issuer (one thread)
//   warp 2      TMEM allocator          warp 3   idle
//   warps 4-7   softmax slot 0          warps 8-11 softmax slot 1
//   TMEM: S0 | S1 | O0 | O1 (128 columns each); P_i (bf16 pairs) over S_i columns 0..63
// =========================================================================================
constexpr int kThreadsV2 = 384;
#ifndef SPX_ATTN_SLOTS
#define SPX_ATTN_SLOTS 4  // K/V ring depth: 4 measured ~1 % faster than 5 at the Wan chunk (A/B, same box)
#endif
constexpr int kSlotsV2 = SPX_ATTN_SLOTS;

template <int D, int kMode = 0>
struct SmemV2 {
    static constexpr uint32_t kChunks = D / 64;
    static constexpr uint32_t kTileBytes = kBKV * D * 2;
    static constexpr uint32_t kSlots = D == 128 ? kSlotsV2 : 2 * kSlotsV2;
    static constexpr uint32_t kQBytes = kBQ * D * 2;
    static constexpr uint32_t kOffQ = 0;
    static constexpr uint32_t kOffRing = kOffQ + kQBytes;
    static constexpr uint32_t kOffBar = kOffRing + kSlots * kTileBytes;
    // q_full, slot_full/empty[kSlots], s_full/p_full/pv_done[2], merge, xfer_free
    static constexpr uint32_t kNumBars = 1 + 2 * kSlots + 6 + 1 + 1;
    static constexpr uint32_t kOffStats = kOffBar + ((kNumBars * 8 + 8 + 15) / 16) * 16;
    static constexpr uint32_t kBytes = kOffStats + 4 * 128 * 4 + 1024;
};

__device__ __forceinline__ void setmaxnreg_dec56() {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
}
__device__ __forceinline__ void setmaxnreg_inc224() {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;" ::: "memory");
}
__device__ __forceinline__ int opaque_i32(int x) {
    asm volatile("" : "+r"(x));
    return x;
}
__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
    asm volatile("" : "+r"(x));
    return x;
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
        : "memory");
}

// ---- packed f32x2 arithmetic (FFMA2 / FADD2: two lanes per issue slot on sm_100) ----
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3}; mov.b64 rb, {%4, %5}; mov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3}; mov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3}; mov.b64 rb, {%4, %5};\n\t"
        "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float fmax3f(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
// ex2_poly on a pair with packed arithmetic: 2 clamps + 3 FADD2 + 3 FFMA2 + 2 IMAD per pair.
// bits(t) = 0x4B400000 + round(x); the constant's low 9 bits are zero, so
// bits(t) << 23 == round(x) << 23 (mod 2^32) and the exponent add is one IMAD.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
    constexpr float kC = 12582912.0f;  // 1.5 * 2^23
    x.x = fmaxf(x.x, -126.0f);
    x.y = fmaxf(x.y, -126.0f);
    const float2 t = fadd2(x, make_float2(kC, kC));
    const float2 f = fsub2(x, fsub2(t, make_float2(kC, kC)));
    float2 p = ffma2(make_float2(0.0553458875f, 0.0553458875f), f,
                     make_float2(0.24260599f, 0.24260599f));
    p = ffma2(p, f, make_float2(0.69322751f, 0.69322751f));
    p = ffma2(p, f, make_float2(0.999927776f, 0.999927776f));
    return make_float2(
        __int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
        __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// kMode 5: every (query tile, head) in exactly 2 kv splits, the two CTAs of a 2-CTA cluster.
// Split 1 bulk-copies its normalised fp32 partial and log-sum-exp straight into split 0's
// shared memory (DSMEM) and split 0 merges: no workspace round trip through L2, no completion
// wait + atomic on the critical path.
template <int D, int kMode>
__global__ void __launch_bounds__(kThreadsV2, 1)
    attn_fwd_v2_kernel(const __grid_constant__ CUtensorMap map_q,
                       const __grid_constant__ CUtensorMap map_k,
                       const __grid_constant__ CUtensorMap map_v, const AttnParams p) {
    using L = SmemV2<D, kMode>;
    constexpr uint32_t kSlots = L::kSlots;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* sQ = smem + L::kOffQ;
    uint8_t* ring = smem + L::kOffRing;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
    uint64_t* q_full = bars;
    uint64_t* slot_full = bars + 1;
    uint64_t* slot_empty = slot_full + kSlots;
    uint64_t* s_full = slot_empty + kSlots;  // [2]
    uint64_t* p_full = s_full + 2;           // [2]
    uint64_t* pv_done = p_full + 2;          // [2]
    uint64_t* merge_bar = pv_done + 2;       // split-KV: other splits' partials landed
    uint64_t* xfer_free = merge_bar + 1;     // (unused since the DSMEM pair merge moved to v3)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xfer_free + 1);
    float* st_m = reinterpret_cast<float*>(smem + L::kOffStats);  // [2][128]
    float* st_l = st_m + 256;                                     // [2][128]

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    pdl_trigger();
    span_begin(p.span);
    if (threadIdx.x == 0) {
        attn_mark(p, 4);  // CTA entry
        attn_mark_global(p, 7);
    }
    int q_tile, head, split, ns;
    {  // full tiles first (block order ~ issue order), then the split ones
        const int b = static_cast<int>(blockIdx.x);
        int t;
        if (b < p.n_full) {
            t = b;
            split = 0;
            ns = 1;
        } else {  // split index outermost: concurrent CTAs share a kv range (L2 reuse)
            const int k = b - p.n_full;
            const int nsplit_tiles = p.qt * p.heads - p.n_full;
            t = p.n_full + k % nsplit_tiles;
            split = k / nsplit_tiles;
            ns = p.splits;
        }
        q_tile = t % p.qt;
        head = t / p.qt;
    }
    // this CTA's share [tb, tb + n_total) of the kv tiles, halved between the warpgroups
    const int tb = static_cast<int>((static_cast<int64_t>(split) * p.total_tiles) / ns);
    const int n_total = static_cast<int>((static_cast<int64_t>(split + 1) * p.total_tiles) / ns) - tb;
    const int n0 = (n_total + 1) / 2;
    const int n1 = n_total - n0;
    __shared__ int s_last;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&map_q);
        tma_prefetch_desc(&map_k);
        tma_prefetch_desc(&map_v);
        mbar_init(q_full, 1);
        for (uint32_t s = 0; s < kSlots; ++s) {
            mbar_init(&slot_full[s], 1);
            mbar_init(&slot_empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], SPX_PFULL_PER_WARP ? 4 : 128);
            mbar_init(&pv_done[i], 1);
        }
        mbar_init(merge_bar, 1);
        mbar_init(xfer_free, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (warp == 3 && lane == 0) l2_prefetch_share(p);  // constant data: before the PDL wait
    pdl_wait();  // q and the KV ring slots were written by the previous kernel(s)
    if (threadIdx.x == 0) attn_mark(p, 0);

    if (warp < 4) {
        setmaxnreg_dec56();
        if (warp == 0 && lane == 0) {
            // ---------------- TMA producer: the MMA consumption order ----------------
            uint32_t t = 0;
            mbar_arrive_expect_tx(q_full, kBQ * D * 2);
#pragma unroll
            for (int c = 0; c < (int)L::kChunks; ++c)
                tma_load_3d(sQ + c * (kBQ * 128), &map_q, q_full, c * 64, head, q_tile * kBQ);
            auto load = [&](bool is_v, int g) {
                const uint32_t slot = t % kSlots;
                const uint32_t ph = (t / kSlots) & 1;
                mbar_wait(&slot_empty[slot], ph ^ 1);
                mbar_arrive_expect_tx(&slot_full[slot], L::kTileBytes);
                int row, valid;
                kv_tile_coords(p, tb + g, row, valid);
                uint8_t* dst = ring + slot * L::kTileBytes;
#pragma unroll
                for (int c = 0; c < (int)L::kChunks; ++c)
                    tma_load_3d(dst + c * (kBKV * 128), is_v ? &map_v : &map_k, &slot_full[slot],
                                c * 64, head, row);
                ++t;
            };
            load(false, 0);
            if (n1 > 0) load(false, n0);
            for (int j = 0; j < n0; ++j) {
                load(true, j);
                if (j + 1 < n0) load(false, j + 1);
                if (j < n1) {
                    load(true, n0 + j);
                    if (j + 1 < n1) load(false, n0 + j + 1);
                }
            }
        } else if (warp == 1) {
            // ---------------- MMA issuer ----------------
            // The whole warp runs the control flow (waits, slot and descriptor arithmetic stay
            // warp-uniform, in uniform registers); one elected lane issues the tcgen05 ops.
            const bool issuer = elect_one();
            constexpr uint32_t idesc_s = make_idesc_bf16(kBQ, kBKV, false, false);
            constexpr uint32_t idesc_o = make_idesc_bf16(kBQ, D, false, true);
            const uint32_t q_addr = smem_u32(sQ);
            const uint32_t ring_addr = smem_u32(ring);
            uint32_t t = 0;
            auto take = [&]() {
                const uint32_t slot = t % kSlots;
                mbar_wait(&slot_full[slot], (t / kSlots) & 1);
                tc_fence_after();
                ++t;
                return slot;
            };
            auto issue_s = [&](int i) {
                const uint32_t slot = take();
                const uint32_t k_addr = ring_addr + slot * L::kTileBytes;
                if (issuer) {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
                        umma_bf16_ss(tmem_base + i * 128, make_desc_sw128(q_addr + off, 16, 1024),
                                     make_desc_sw128(k_addr + off, 16, 1024), idesc_s, kk > 0);
                    }
                    umma_commit(&s_full[i]);
                    umma_commit(&slot_empty[slot]);
                }
                __syncwarp();
            };
            auto issue_pv = [&](int i, int j) {
                const uint32_t slot = take();
                if (p.experiment != 3)  // 3: profiling, MMA stream without softmax
                    mbar_wait(&p_full[i], j & 1);
                tc_fence_after();
                const uint32_t v_addr = ring_addr + slot * L::kTileBytes;
                if (issuer) {
#pragma unroll
                    for (int kk = 0; kk < kBKV / 16; ++kk)
                        umma_bf16_ts(tmem_base + 256 + i * 128, tmem_base + i * 128 + kk * 8,
                                     make_desc_sw128(v_addr + kk * 16 * 128, kBKV * 128, 1024),
                                     idesc_o, (j | kk) != 0);
                    umma_commit(&pv_done[i]);
                    umma_commit(&slot_empty[slot]);
                }
                __syncwarp();
            };
            mbar_wait(q_full, 0);
            tc_fence_after();
            issue_s(0);
            if (n1 > 0) issue_s(1);
            for (int j = 0; j < n0; ++j) {
                issue_pv(0, j);
                if (j + 1 < n0) issue_s(0);
                if (j < n1) {
                    issue_pv(1, j);
                    if (j + 1 < n1) issue_s(1);
                }
            }
        }
    } else {
        setmaxnreg_inc224();
        // ---------------- softmax warpgroups ----------------
        const int i = (warp - 4) / 4;           // slot
        const int q = warp % 4;                 // TMEM lane quarter
        const int r = q * 32 + lane;            // query row in the tile == TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        const uint32_t t_s = tmem_base + i * 128 + lane_off;
        const uint32_t t_o = tmem_base + 256 + i * 128 + lane_off;
        const int n = i == 0 ? n0 : n1;
        const int g0 = tb + (i == 0 ? 0 : n0);
        const float scale = p.scale_log2;
        float m_run = -INFINITY;
        float l_run = 0.0f;
        for (int j = 0; j < (p.experiment == 3 ? 0 : n); ++j) {
            int row, valid;
            kv_tile_coords(p, g0 + j, row, valid);
            mbar_wait(&s_full[i], j & 1);
            // PV_i(j - 1) precedes QK_i(j) in the MMA pipe, so this phase is complete already;
            // observing every phase keeps the barrier protocol explicit (compute-sanitizer
            // synccheck flags committed phases nobody waits on)
            if (j > 0) mbar_wait(&pv_done[i], (j - 1) & 1);
            tc_fence_after();
            if (p.experiment == 1) {  // profiling: MMA/TMA/barrier skeleton only
                tc_fence_before();
                if (SPX_PFULL_PER_WARP) __syncwarp();
                if (!SPX_PFULL_PER_WARP || lane == 0) mbar_arrive(&p_full[i]);
                continue;
            }
            // Exponent offset: the row max of the WG's FIRST tile only. Softmax is invariant to
            // the offset and P (bf16) / O, l (fp32) have the range for values far above 1, so
            // later tiles skip the per-tile max (43 3-input max ops per row); the tile's row sum
            // guards against overflow: if any exp exceeded 2^64 (a logit > offset + 64, in log2
            // units; rare), the tile is redone with its true max and O, l rescaled.
            uint32_t u[kBKV];
            auto load_s = [&]() {
#pragma unroll
                for (int c = 0; c < kBKV / 32; ++c)
                    tmem_ld32(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&u[c * 32]));
                tmem_ld_wait();
                if (valid < kBKV) {  // ragged tail tile only: masked logits -> -inf (exp -> 0)
#pragma unroll
                    for (int c = 0; c < kBKV; ++c)
                        if (c >= valid) u[c] = 0xff800000u;
                }
            };
            auto row_max = [&]() {  // four independent 3-input max chains
                float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int c = 0; c < kBKV; c += 8) {
#pragma unroll
                    for (int k4 = 0; k4 < 4; ++k4)
                        mq[k4] = fmax3f(mq[k4], __uint_as_float(u[c + 2 * k4]),
                                        __uint_as_float(u[c + 2 * k4 + 1]));
                }
                return fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
            };
            uint32_t pk[kBKV / 2];
            auto exp_tile = [&]() {  // P = exp2(s scale - m_run), bf16 pairs; returns the sum
                const float2 sc2 = make_float2(scale, scale);
                const float2 nm2 = make_float2(-m_run, -m_run);
                float2 ls[4];
#pragma unroll
                for (int e = 0; e < kBKV / 2; ++e) {
                    const float2 x = ffma2(
                        make_float2(__uint_as_float(u[2 * e]), __uint_as_float(u[2 * e + 1])), sc2,
                        nm2);
                    float2 pr;
                    if ((e & 7) >= 8 - SPX_POLY_OF_8) {  // part of the exponentials on the FMA pipe
                        pr = ex2_poly2(x);
                    } else {
#if SPX_ATTN_PROFILING
                        if (p.experiment == 2) {  // profiling: no MUFU
                            pr.x = fmaf(x.x, 0.03125f, 1.0f);
                            pr.y = fmaf(x.y, 0.03125f, 1.0f);
                        } else
#endif
                        {
                            pr.x = ex2_approx(x.x);
                            pr.y = ex2_approx(x.y);
                        }
                    }
                    ls[e & 3] = e < 4 ? pr : fadd2(ls[e & 3], pr);  // (unrolled: no add of 0)
                    pk[e] = pack_bf16x2(pr.x, pr.y);
                }
                const float2 s01 = fadd2(fadd2(ls[0], ls[1]), fadd2(ls[2], ls[3]));
                return s01.x + s01.y;
            };
            load_s();
            if (j == 0) m_run = row_max() * scale;
            float lt = exp_tile();
            if (j > 0 && __any_sync(0xffffffffu, !(lt < 1.8446744e19f))) {  // 2^64, or inf / NaN
                load_s();  // S is still in TMEM (P not written yet)
                const float m_new = fmaxf(m_run, row_max() * scale);  // (PV_i(j - 1) done: above)
                const float alpha = ex2_approx(m_run - m_new);
#pragma unroll 1
                for (int c = 0; c < D / 32; ++c) {
                    uint32_t o[32];
                    tmem_ld32(t_o + c * 32, o);
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
                    tmem_st32(t_o + c * 32, o);
                }
                tmem_st_wait();
                l_run *= alpha;
                m_run = m_new;
                lt = exp_tile();
            }
            l_run += lt;
#pragma unroll
            for (int c = 0; c < kBKV / 32; ++c) tmem_st16(t_s + c * 16, &pk[c * 16]);
            tmem_st_wait();
            tc_fence_before();
            if (SPX_PFULL_PER_WARP) __syncwarp();
            if (!SPX_PFULL_PER_WARP || lane == 0) mbar_arrive(&p_full[i]);
        }
        if (n > 0) {
            mbar_wait(&pv_done[i], (n - 1) & 1);
            tc_fence_after();
        }
        // ---------------- epilogue ----------------
        if (threadIdx.x == 128) attn_mark(p, 1);
        st_m[i * 128 + r] = m_run;
        st_l[i * 128 + r] = l_run;
        tc_fence_before();
        named_bar_sync(1, 256);
        tc_fence_after();
        // merge the two partial softmaxes; warpgroup i stores head-dim columns [i D/2, (i+1) D/2)
        const int qi = q_tile * kBQ + r;
        const float m0 = st_m[r], l0 = st_l[r];
        const float m1 = n1 > 0 ? st_m[128 + r] : -INFINITY;
        const float l1 = n1 > 0 ? st_l[128 + r] : 0.0f;
        const float mm = fmaxf(m0, m1);
        const float a0 = ex2_approx(m0 - mm);
        const float a1 = n1 > 0 ? ex2_approx(m1 - mm) : 0.0f;
        const float inv = 1.0f / (l0 * a0 + l1 * a1);
        const float w0 = a0 * inv, w1 = a1 * inv;
        bf16* dst = nullptr;
        if (qi < p.sq) {
            const int chunk = qi / p.rows_per_chunk;
            dst = p.out_base[chunk] +
                  static_cast<int64_t>(qi - chunk * p.rows_per_chunk) * p.out_row_stride +
                  static_cast<int64_t>(head) * D;
        }
        const uint32_t t_o0 = tmem_base + 256 + lane_off;
        const uint32_t t_o1 = tmem_base + 384 + lane_off;
        if (ns == 1) {
            // rows staged as bf16 in the idle Q smem (16-byte units XOR-swizzled by row), then
            // copied out by all 256 softmax threads so that each store instruction writes whole
            // 128/256-byte row segments (the per-row 16-byte stores of a warp hit 32 rows)
            constexpr uint32_t kRowBytes = D * 2;
            constexpr uint32_t kU = kRowBytes / 16;
            const uint32_t s_base = smem_u32(smem);
#pragma unroll 1
            for (int c = i * (D / 64); c < (i + 1) * (D / 64); ++c) {
                uint32_t o0[32], o1[32];
                tmem_ld32(t_o0 + c * 32, o0);
                if (n1 > 0) tmem_ld32(t_o1 + c * 32, o1);
                tmem_ld_wait();
                float f[32];
#pragma unroll
                for (int e = 0; e < 32; ++e)
                    f[e] = __uint_as_float(o0[e]) * w0 + (n1 > 0 ? __uint_as_float(o1[e]) * w1 : 0.0f);
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const uint32_t unit = static_cast<uint32_t>(c * 4 + v);
                    const uint32_t a = s_base + static_cast<uint32_t>(r) * kRowBytes +
                                       ((unit ^ (static_cast<uint32_t>(r) & (kU - 1))) << 4);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a),
                                 "r"(pack_bf16x2(f[8 * v + 0], f[8 * v + 1])),
                                 "r"(pack_bf16x2(f[8 * v + 2], f[8 * v + 3])),
                                 "r"(pack_bf16x2(f[8 * v + 4], f[8 * v + 5])),
                                 "r"(pack_bf16x2(f[8 * v + 6], f[8 * v + 7]))
                                 : "memory");
                }
            }
            named_bar_sync(1, 256);
            const int tid = static_cast<int>(threadIdx.x) - 128;
#pragma unroll 1
            for (int idx = tid; idx < kBQ * static_cast<int>(kU); idx += 256) {
                const int row = idx / static_cast<int>(kU);
                const uint32_t u = static_cast<uint32_t>(idx) % kU;
                const int q_row = q_tile * kBQ + row;
                if (q_row >= p.sq) continue;
                uint4 w;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                             : "r"(s_base + static_cast<uint32_t>(row) * kRowBytes +
                                   ((u ^ (static_cast<uint32_t>(row) & (kU - 1))) << 4))
                             : "memory");
                const int chunk = q_row / p.rows_per_chunk;
                bf16* drow = p.out_base[chunk] +
                             static_cast<int64_t>(q_row - chunk * p.rows_per_chunk) * p.out_row_stride +
                             static_cast<int64_t>(head) * D;
                *reinterpret_cast<uint4*>(drow + u * 8) = w;
            }
        } else {
            // ---- split-KV ----
            // Each split CTA stages its normalised fp32 partial (128 rows x D) in the now idle
            // Q/ring smem (16-byte units XOR-swizzled by row: conflict-free, the swizzle travels
            // with the bytes) and writes it to its own contiguous workspace block with ONE
            // bulk copy; the last split of the tile bulk-loads the others back into smem and
            // merges them lse-weighted. Workspace: [tile][split][128][D] fp32, [tile][split][128]
            // lse, tile = head * q_tiles + q_tile.
            constexpr uint32_t kUnits = D / 4;                  // 16-byte units per fp32 row
            constexpr uint32_t kPartBytes = kBQ * D * 4;        // one partial
            constexpr int kMaxOthers = static_cast<int>(L::kOffBar / kPartBytes) - 1;
            const uint32_t s_base = smem_u32(smem);
            auto unit_addr = [&](uint32_t buf, int row, uint32_t u) {
                return s_base + buf * kPartBytes + static_cast<uint32_t>(row) * (kUnits * 16) +
                       ((u ^ (static_cast<uint32_t>(row) & (kUnits - 1))) << 4);
            };
            const int64_t tile = static_cast<int64_t>(head) * p.q_tiles + q_tile;
            float* ws_tile = p.ws_o + tile * p.splits * (kBQ * D);
            float* lse_tile = p.ws_lse + tile * p.splits * kBQ;
#pragma unroll 1
            for (int c = i * (D / 64); c < (i + 1) * (D / 64); ++c) {
                uint32_t o0[32], o1[32];
                tmem_ld32(t_o0 + c * 32, o0);
                if (n1 > 0) tmem_ld32(t_o1 + c * 32, o1);
                tmem_ld_wait();
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                    float f[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        f[e] = __uint_as_float(o0[4 * v + e]) * w0 +
                               (n1 > 0 ? __uint_as_float(o1[4 * v + e]) * w1 : 0.0f);
                    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                                     unit_addr(0, r, static_cast<uint32_t>(c * 8 + v))),
                                 "f"(f[0]), "f"(f[1]), "f"(f[2]), "f"(f[3])
                                 : "memory");
                }
            }
            if (i == 0) __stcg(lse_tile + split * kBQ + r, mm + __log2f(l0 * a0 + l1 * a1));
            fence_proxy_async_smem();  // generic-proxy smem writes -> the bulk copy's reads
            named_bar_sync(1, 256);
            if (threadIdx.x == 128) {
                attn_mark(p, 2);
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                 ws_tile + static_cast<int64_t>(split) * (kBQ * D)),
                             "r"(s_base), "r"(kPartBytes)
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                asm volatile("fence.proxy.async.global;" ::: "memory");
                __threadfence();
                int* ctr = p.counters + tile;
                const int prev = atomicAdd(ctr, 1);
                s_last = prev == ns - 1;
                if (s_last) *ctr = 0;  // every split has arrived: re-arm for the next launch
            }
            named_bar_sync(1, 256);
            if (threadIdx.x == 128) attn_mark(p, 5);  // split arrival counted
            if (s_last) {
                __threadfence();
                float lse_max = -INFINITY;
                for (int z = 0; z < ns; ++z) lse_max = fmaxf(lse_max, __ldcg(lse_tile + z * kBQ + r));
                float acc[D / 2];
                float wsum;
                {  // own partial (staging buffer 0)
                    const float wz = ex2_approx(__ldcg(lse_tile + split * kBQ + r) - lse_max);
                    wsum = wz;
#pragma unroll
                    for (int v = 0; v < D / 8; ++v) {
                        float4 t;
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w)
                                     : "r"(unit_addr(0, r, static_cast<uint32_t>(i * (D / 8) + v))));
                        acc[4 * v + 0] = wz * t.x;
                        acc[4 * v + 1] = wz * t.y;
                        acc[4 * v + 2] = wz * t.z;
                        acc[4 * v + 3] = wz * t.w;
                    }
                }
                // the other splits in batches of kMaxOthers (other index o -> split z)
                uint32_t phase = 0;
                const int others = ns - 1;
                for (int o0 = 0; o0 < others; o0 += kMaxOthers) {
                    const int cnt = min(kMaxOthers, others - o0);
                    named_bar_sync(1, 256);  // buffers 1.. are free (previous batch read)
                    if (threadIdx.x == 128) {
                        mbar_arrive_expect_tx(merge_bar, static_cast<uint32_t>(cnt) * kPartBytes);
                        for (int b = 0; b < cnt; ++b) {
                            const int z = o0 + b < split ? o0 + b : o0 + b + 1;
                            asm volatile(
                                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
                                " [%0], [%1], %2, [%3];" ::"r"(s_base + (b + 1) * kPartBytes),
                                "l"(ws_tile + static_cast<int64_t>(z) * (kBQ * D)), "r"(kPartBytes),
                                "r"(smem_u32(merge_bar))
                                : "memory");
                        }
                    }
                    mbar_wait(merge_bar, phase);
                    if (threadIdx.x == 128) attn_mark(p, 6);  // other partials landed
                    phase ^= 1;
                    for (int b = 0; b < cnt; ++b) {
                        const int z = o0 + b < split ? o0 + b : o0 + b + 1;
                        const float wz = ex2_approx(__ldcg(lse_tile + z * kBQ + r) - lse_max);
                        wsum += wz;
#pragma unroll
                        for (int v = 0; v < D / 8; ++v) {
                            float4 t;
                            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                         : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w)
                                         : "r"(unit_addr(static_cast<uint32_t>(b + 1), r,
                                                         static_cast<uint32_t>(i * (D / 8) + v))));
                            acc[4 * v + 0] = fmaf(wz, t.x, acc[4 * v + 0]);
                            acc[4 * v + 1] = fmaf(wz, t.y, acc[4 * v + 1]);
                            acc[4 * v + 2] = fmaf(wz, t.z, acc[4 * v + 2]);
                            acc[4 * v + 3] = fmaf(wz, t.w, acc[4 * v + 3]);
                        }
                    }
                }
                if (dst) {
                    const float inv_w = 1.0f / wsum;
                    uint4* d4 = reinterpret_cast<uint4*>(dst + i * (D / 2));
#pragma unroll
                    for (int v = 0; v < D / 16; ++v)
                        d4[v] = make_uint4(pack_bf16x2(acc[8 * v + 0] * inv_w, acc[8 * v + 1] * inv_w),
                                           pack_bf16x2(acc[8 * v + 2] * inv_w, acc[8 * v + 3] * inv_w),
                                           pack_bf16x2(acc[8 * v + 4] * inv_w, acc[8 * v + 5] * inv_w),
                                           pack_bf16x2(acc[8 * v + 6] * inv_w, acc[8 * v + 7] * inv_w));
                }
            }
        }
    }
    if (threadIdx.x == 128) {
        attn_mark(p, 3);
        attn_mark_global(p, 8);
    }
    tc_fence_before();
    __syncthreads();
    span_end(p.span);
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

template <int D, int kMode>
void attn_v2_launch(dim3 grid, const AttnPlan& plan, const AttnParams& p, cudaStream_t stream) {
    static bool done[64] = {};
    int dev = 0;
    SPX_CUDA(cudaGetDevice(&dev));
    if (!done[dev & 63]) {
        SPX_CUDA(cudaFuncSetAttribute(attn_fwd_v2_kernel<D, kMode>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(SmemV2<D, kMode>::kBytes)));
        done[dev & 63] = true;
    }
    launch_pdl(attn_fwd_v2_kernel<D, kMode>, grid, dim3(kThreadsV2), SmemV2<D, kMode>::kBytes,
               stream, plan.map_q, plan.map_k, plan.map_v, p);
}


// the v3 slots' exponent-offset exchange: one barrier instruction for both call sites (a slot
// with no kv tiles joins from outside its loop), so the barrier is not seen as divergent
__device__ __noinline__ void v3_offset_exchange_barrier() { named_bar_sync(1, 256); }

// =========================================================================================
// v3: the kv range of a 128-row query tile is split between two softmax warpgroups as in v2,
// but the two slots accumulate into ONE O (TMEM) with a common exponent offset (the max over
// both slots' first tiles, exchanged once), which frees the TMEM for separate P buffers:
//   S0 | S1 | O | P0 | P1  = 128 + 128 + 128 + 64 + 64 columns.
// With P no longer written over S, the MMA issues S_i(j+1) as soon as the softmax has loaded
// S_i(j) into registers (s_free), so a slot's dependency chain per tile is softmax + PV
// instead of softmax + PV + QK^T. MMA issue order (= the producer's ring order):
//   QK0(0) QK1(0) | QK0(j+1) PV0(j) QK1(j+1) PV1(j) | ...
// Persistent: a CTA walks query tiles blockIdx.x, blockIdx.x + gridDim.x, ... (grid = min(tiles,
// SMs)). Q is double-buffered in shared memory and the barrier phases run on across tiles, so
// the producer loads Q and the first K/V tiles of tile k+1, and the MMA issues its first
// QK^T, while the softmax warps run the epilogue of tile k; O is handed over as soon as the
// epilogue has it in registers (o_free). The CTA prologue (barriers, TMEM, descriptors) and
// the launch gap between CTAs are paid once per SM instead of once per tile.
// Overflow: the fixed offset covers logits up to offset + 64 (log2 units) exactly; if a later
// tile's exponentials exceed 2^64 (or are not finite), the shared O cannot be rescaled
// without stopping both slots, so the CTA flags it and recomputes that tile's rows exactly on
// the CUDA cores after its main loop (never taken for sane inputs; tested).
// =========================================================================================
template <int D>
struct SmemV3 {
    static constexpr uint32_t kChunks = D / 64;
    static constexpr uint32_t kTileBytes = kBKV * D * 2;
    static constexpr uint32_t kSlots = D == 128 ? kSlotsV2 : 2 * kSlotsV2;
    static constexpr uint32_t kQBytes = kBQ * D * 2;
    static constexpr uint32_t kOffQ = 0;  // [2] query tiles (also the epilogue's row staging)
    static constexpr uint32_t kOffRing = kOffQ + 2 * kQBytes;
    static constexpr uint32_t kOffBar = kOffRing + kSlots * kTileBytes;
    // q_full[2], slot_full/empty[kSlots], s_full/p_full/pv_done/s_free[2], o_free, q_free[2],
    // merge, xfer_free (pair-split mode)
    static constexpr uint32_t kNumBars = 2 + 2 * kSlots + 8 + 1 + 2 + 2;
    static constexpr uint32_t kOffStats = kOffBar + ((kNumBars * 8 + 8 + 15) / 16) * 16;
    static constexpr uint32_t kBytes = kOffStats + 4 * 128 * 4 + 1024;
};

// kMode (the CTA's list of pieces = (tile, kv range)):
//   0  persistent: tiles blockIdx.x, + gridDim.x, ..., each over its whole kv range
//   1  pair split: a 2-CTA cluster per tile, CTA r takes half r of the kv range (the per-rank
//      shapes of P = 8); the halves' normalised fp32 partials merge lse-weighted through DSMEM
//      in CTA 0
//   2  triple: cluster c owns tiles 3c, 3c + 1, 3c + 2; CTA r takes tile 3c + r whole, then
//      half r of tile 3c + 2, merged as in mode 1 (1.5 tiles per SM: the P = 2 per-rank shape's
//      222 tiles on 148 SMs)
// Modes 1 and 2 launch as 2-CTA clusters.
template <int D, int kMode>
__global__ void __launch_bounds__(kThreadsV2, 1)
    attn_fwd_v3_kernel(const __grid_constant__ CUtensorMap map_q,
                       const __grid_constant__ CUtensorMap map_k,
                       const __grid_constant__ CUtensorMap map_v, const AttnParams p) {
    using L = SmemV3<D>;
    constexpr uint32_t kSlots = L::kSlots;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* sQ = smem + L::kOffQ;
    uint8_t* ring = smem + L::kOffRing;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
    uint64_t* q_full = bars;                 // [2]
    uint64_t* slot_full = bars + 2;
    uint64_t* slot_empty = slot_full + kSlots;
    uint64_t* s_full = slot_empty + kSlots;  // [2]
    uint64_t* p_full = s_full + 2;           // [2]
    uint64_t* pv_done = p_full + 2;          // [2]
    uint64_t* s_free = pv_done + 2;          // [2]
    uint64_t* o_free = s_free + 2;           // the epilogue holds O in registers
    uint64_t* q_free = o_free + 1;           // [2] the epilogue's row staging in Q buffer b is done
    uint64_t* merge_bar = q_free + 2;        // pair: split 1's partial landed in CTA 0
    uint64_t* xfer_free = merge_bar + 1;     // pair, split 1: CTA 0's ring is free for the partial
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xfer_free + 1);
    float* st_m = reinterpret_cast<float*>(smem + L::kOffStats);  // [2][128]
    float* st_l = st_m + 256;                                     // [2][128]
    __shared__ int s_ovf;

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    pdl_trigger();
    span_begin(p.span);
    if (threadIdx.x == 0) {
        attn_mark(p, 4);  // CTA entry
        attn_mark_global(p, 7);
    }
    constexpr bool kPair = kMode != 0;  // a 2-CTA cluster: the last piece merges through DSMEM
    const int num_tiles = p.qt * p.heads;
    const int split = kPair ? static_cast<int>(cluster_ctarank()) : 0;
    const int NT = p.total_tiles;
    const int half_b = (NT + 1) / 2;
    // piece `it` of this CTA: tile, kv tiles [kb, ke); false past the last piece
    auto piece = [&](int it, int& tile, int& kb, int& ke) -> bool {
        if constexpr (kMode == 0) {
            tile = static_cast<int>(blockIdx.x) + it * static_cast<int>(gridDim.x);
            kb = 0;
            ke = NT;
            return tile < num_tiles;
        } else {
            const int c = static_cast<int>(blockIdx.x >> 1);
            const int last = kMode == 1 ? 0 : 1;
            if (it > last) return false;
            tile = kMode == 1 ? c : (it == 0 ? 3 * c + split : 3 * c + 2);
            const bool halved = it == last;
            kb = halved && split ? half_b : 0;
            ke = halved && !split ? half_b : NT;
            return tile < num_tiles;
        }
    };
    // the CTA's last piece is the merged half in modes 1 / 2
    auto merged = [&](int it) { return kPair && it == (kMode == 1 ? 0 : 1); };

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&map_q);
        tma_prefetch_desc(&map_k);
        tma_prefetch_desc(&map_v);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&q_full[b], 1);
            mbar_init(&q_free[b], 256);  // every softmax thread, after its last staging read
        }
        for (uint32_t s = 0; s < kSlots; ++s) {
            mbar_init(&slot_full[s], 1);
            mbar_init(&slot_empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 4);   // one arrival per softmax warp
            mbar_init(&pv_done[i], 1);
            mbar_init(&s_free[i], 4);   // one arrival per softmax warp
        }
        mbar_init(o_free, 8);  // one arrival per softmax warp
        mbar_init(merge_bar, 1);
        mbar_init(xfer_free, 1);
        s_ovf = 0;
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    if constexpr (kPair)
        cluster_sync_all();  // the partner's barriers exist before any remote arrival
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t t_O = tmem_base + 256;
    if (warp == 3 && lane == 0) l2_prefetch_share(p);  // constant data (weights): before the PDL wait
    pdl_wait();  // q and the KV ring slots were written by the previous kernel(s)
    if (threadIdx.x == 0) attn_mark(p, 0);

    if (warp < 4) {
        setmaxnreg_dec56();
        if (warp == 0 && lane == 0) {
            // ---------------- TMA producer: the MMA consumption order ----------------
            uint32_t t = 0;
            int it = 0;
            for (int tile, kb, ke; piece(it, tile, kb, ke); ++it) {
                const int n0 = (ke - kb + 1) / 2;
                const int n1 = ke - kb - n0;
                const int q_tile = tile % p.qt;
                const int head = tile / p.qt;
                const int b = it & 1;
                if (it >= 2) mbar_wait(&q_free[b], ((it - 2) >> 1) & 1);  // tile it-2's staging done
                mbar_arrive_expect_tx(&q_full[b], L::kQBytes);
#pragma unroll
                for (int c = 0; c < (int)L::kChunks; ++c)
                    tma_load_3d(sQ + b * L::kQBytes + c * (kBQ * 128), &map_q, &q_full[b], c * 64, head,
                                q_tile * kBQ);
                auto load = [&](bool is_v, int g) {
                    const uint32_t slot = t % kSlots;
                    const uint32_t ph = (t / kSlots) & 1;
                    mbar_wait(&slot_empty[slot], ph ^ 1);
                    mbar_arrive_expect_tx(&slot_full[slot], L::kTileBytes);
                    int row, valid;
                    kv_tile_coords(p, g, row, valid);
                    uint8_t* dst = ring + slot * L::kTileBytes;
#pragma unroll
                    for (int c = 0; c < (int)L::kChunks; ++c)
                        tma_load_3d(dst + c * (kBKV * 128), is_v ? &map_v : &map_k, &slot_full[slot],
                                    c * 64, head, row);
                    ++t;
                };
                load(false, kb);
                if (n1 > 0) load(false, kb + n0);
                for (int j = 0; j < n0; ++j) {
                    if (j + 1 < n0) load(false, kb + j + 1);
                    load(true, kb + j);
                    if (j < n1) {
                        if (j + 1 < n1) load(false, kb + n0 + j + 1);
                        load(true, kb + n0 + j);
                    }
                }
            }
        } else if (warp == 1) {
            // ---------------- MMA issuer ----------------
            const bool issuer = elect_one();
            constexpr uint32_t idesc_s = make_idesc_bf16(kBQ, kBKV, false, false);
            constexpr uint32_t idesc_o = make_idesc_bf16(kBQ, D, false, true);
            const uint32_t ring_addr = smem_u32(ring);
            uint32_t t = 0;
            uint32_t gs0 = 0, gs1 = 0;  // S tiles issued per slot (all tiles of this CTA)
            uint32_t gp0 = 0, gp1 = 0;  // PV tiles issued per slot
            auto take = [&]() {
                const uint32_t slot = t % kSlots;
                mbar_wait(&slot_full[slot], (t / kSlots) & 1);
                tc_fence_after();
                ++t;
                return slot;
            };
            int it = 0;
            for (int tile, kb, ke; piece(it, tile, kb, ke); ++it) {
                const int n0 = (ke - kb + 1) / 2;
                const int n1 = ke - kb - n0;
                const int b = it & 1;
                const uint32_t q_addr = smem_u32(sQ + b * L::kQBytes);
                bool first_pv = true;
                auto issue_s = [&](int i) {
                    const uint32_t g = i == 0 ? gs0 : gs1;
                    if (g > 0) {  // the softmax holds S_i(previous) in registers
                        mbar_wait(&s_free[i], (g - 1) & 1);
                        tc_fence_after();
                    }
                    const uint32_t slot = take();
                    const uint32_t k_addr = ring_addr + slot * L::kTileBytes;
                    if (issuer) {
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {
                            const uint32_t off = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
                            umma_bf16_ss(tmem_base + i * 128, make_desc_sw128(q_addr + off, 16, 1024),
                                         make_desc_sw128(k_addr + off, 16, 1024), idesc_s, kk > 0);
                        }
                        umma_commit(&s_full[i]);
                        umma_commit(&slot_empty[slot]);
                    }
                    if (i == 0)
                        ++gs0;
                    else
                        ++gs1;
                    __syncwarp();
                };
                auto issue_pv = [&](int i) {
                    const uint32_t slot = take();
                    mbar_wait(&p_full[i], (i == 0 ? gp0 : gp1) & 1);
                    if (first_pv && it > 0) mbar_wait(o_free, (it - 1) & 1);  // tile it-1's O is read
                    tc_fence_after();
                    const uint32_t v_addr = ring_addr + slot * L::kTileBytes;
                    const uint32_t t_p = tmem_base + 384 + i * 64;
                    if (issuer) {
#pragma unroll
                        for (int kk = 0; kk < kBKV / 16; ++kk)
                            umma_bf16_ts(t_O, t_p + kk * 8,
                                         make_desc_sw128(v_addr + kk * 16 * 128, kBKV * 128, 1024),
                                         idesc_o, (first_pv && kk == 0) ? 0u : 1u);
                        umma_commit(&pv_done[i]);
                        umma_commit(&slot_empty[slot]);
                    }
                    if (i == 0)
                        ++gp0;
                    else
                        ++gp1;
                    first_pv = false;
                    __syncwarp();
                };
                mbar_wait(&q_full[b], (it >> 1) & 1);
                tc_fence_after();
                issue_s(0);
                if (n1 > 0) issue_s(1);
                for (int j = 0; j < n0; ++j) {
                    if (j + 1 < n0) issue_s(0);
                    issue_pv(0);
                    if (j < n1) {
                        if (j + 1 < n1) issue_s(1);
                        issue_pv(1);
                    }
                }
            }
        }
    } else {
        setmaxnreg_inc224();
        // ---------------- softmax warpgroups ----------------
        const int i = (warp - 4) / 4;           // slot
        const int q = warp % 4;                 // TMEM lane quarter
        const int r = q * 32 + lane;            // query row in the tile == TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        const uint32_t t_s = tmem_base + i * 128 + lane_off;
        const uint32_t t_p = tmem_base + 384 + i * 64 + lane_off;
        const float scale = p.scale_log2;
        constexpr uint32_t kRowBytes = D * 2;
        constexpr uint32_t kU = kRowBytes / 16;
        int it = 0;
        uint32_t gbase = 0;  // this slot's kv tiles in the CTA's earlier pieces
        for (int tile, kb, ke; piece(it, tile, kb, ke); ++it) {
        const int n0 = (ke - kb + 1) / 2;
        const int n = i == 0 ? n0 : ke - kb - n0;
        const int g0 = kb + (i == 0 ? 0 : n0);
        const int q_tile = tile % p.qt;
        const int head = tile / p.qt;
        const int b = it & 1;
        float m_run = -INFINITY;
        float l_run = 0.0f;
        bool ovf = false;
        if (n == 0) {  // (a one-tile kv range: slot 1 idle) still joins the offset exchange
            st_m[i * 128 + r] = -INFINITY;
            v3_offset_exchange_barrier();
        }
        for (int j = 0; j < n; ++j) {
            const uint32_t G = gbase + static_cast<uint32_t>(j);
            int row, valid;
            kv_tile_coords(p, g0 + j, row, valid);
            mbar_wait(&s_full[i], G & 1);
            tc_fence_after();
            uint32_t u[kBKV];
#pragma unroll
            for (int c = 0; c < kBKV / 32; ++c)
                tmem_ld32(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&u[c * 32]));
            tmem_ld_wait();
            // S_i is in registers: the MMA may overwrite it with S_i(j + 1)
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_free[i]);
            if (valid < kBKV) {  // ragged tail tile only: masked logits -> -inf (exp -> 0)
#pragma unroll
                for (int c = 0; c < kBKV; ++c)
                    if (c >= valid) u[c] = 0xff800000u;
            }
            if (j == 0) {  // common exponent offset: max over both slots' first tiles
                float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int c = 0; c < kBKV; c += 8) {
#pragma unroll
                    for (int k4 = 0; k4 < 4; ++k4)
                        mq[k4] = fmax3f(mq[k4], __uint_as_float(u[c + 2 * k4]),
                                        __uint_as_float(u[c + 2 * k4 + 1]));
                }
                st_m[i * 128 + r] = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])) * scale;
                v3_offset_exchange_barrier();
                m_run = fmaxf(st_m[r], st_m[128 + r]);
            }
            uint32_t pk[kBKV / 2];
            float lt;
            {  // P = exp2(s scale - m), bf16 pairs; lt = the row sum
                const float2 sc2 = make_float2(scale, scale);
                const float2 nm2 = make_float2(-m_run, -m_run);
                float2 ls[4];
#pragma unroll
                for (int e = 0; e < kBKV / 2; ++e) {
                    const float2 x = ffma2(
                        make_float2(__uint_as_float(u[2 * e]), __uint_as_float(u[2 * e + 1])), sc2, nm2);
                    float2 pr;
                    if ((e & 7) >= 8 - SPX_V3_POLY_OF_8) {
                        pr = ex2_poly2(x);
                    } else {
                        pr.x = ex2_approx(x.x);
                        pr.y = ex2_approx(x.y);
                    }
                    ls[e & 3] = e < 4 ? pr : fadd2(ls[e & 3], pr);
                    pk[e] = pack_bf16x2(pr.x, pr.y);
                }
                const float2 s01 = fadd2(fadd2(ls[0], ls[1]), fadd2(ls[2], ls[3]));
                lt = s01.x + s01.y;
            }
            ovf = ovf || !(lt < 1.8446744e19f);  // 2^64, or inf / NaN
            l_run += lt;
            // P_i(j - 1) has been read by its PV before P_i(j) overwrites the buffer (at j = 0
            // the previous tile's epilogue waited for its last PV)
            if (j > 0) {
                mbar_wait(&pv_done[i], (G - 1) & 1);
                tc_fence_after();
            }
#pragma unroll
            for (int c = 0; c < kBKV / 32; ++c) tmem_st16(t_p + c * 16, &pk[c * 16]);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[i]);
        }
        if (n > 0) {
            mbar_wait(&pv_done[i], (gbase + static_cast<uint32_t>(n) - 1) & 1);
            tc_fence_after();
        }
        if (ovf) s_ovf = 1;
        if (threadIdx.x == 128) {
            attn_mark(p, 1);  // softmax loop done (last tile's)
            if (it < 4) attn_mark(p, 10 + it);  // per piece: loop end
        }
        // ---------------- epilogue: O / (l0 + l1), rows staged in this tile's Q buffer ----------------
        st_l[i * 128 + r] = l_run;
        tc_fence_before();
        named_bar_sync(1, 256);  // both slots' last PVs are done; l and the flag are visible
        tc_fence_after();
        const float inv = 1.0f / (st_l[r] + st_l[128 + r]);
        const bool fallback = s_ovf != 0;
        gbase += static_cast<uint32_t>(n);
        if (merged(it)) {
        // ---------------- pair split: merge the two kv halves through DSMEM ----------------
        // normalised fp32 partials, 16-byte units XOR-swizzled by row (conflict-free both ways);
        // split 1 stages its partial + lse at offset 0 of its shared memory and bulk-copies
        // them into CTA 0's idle ring once CTA 0's MMAs are done; CTA 0 merges from TMEM +
        // shared memory, stages bf16 rows at offset 0 and stores them. lse = +inf marks a half
        // that overflowed: CTA 0 then recomputes the row exactly.
        constexpr uint32_t kPartBytes = kBQ * D * 4;
        constexpr uint32_t kPU = D / 4;  // 16-byte units per fp32 row
        static_assert(2 * kPartBytes + kBQ * 4 <= L::kOffBar, "pair merge buffers in the Q + ring smem");
        const uint32_t s0 = smem_u32(smem);
        auto punit = [&](uint32_t base, uint32_t u) {
            return base + static_cast<uint32_t>(r) * (kPU * 16) + ((u ^ (static_cast<uint32_t>(r) & (kPU - 1))) << 4);
        };
        const float l_sum = st_l[r] + st_l[128 + r];
        const float lse_own = fallback ? INFINITY : m_run + __log2f(l_sum);
        if (split == 1) {
            if (!fallback) {
#pragma unroll 1
                for (int c = 0; c < D / 64; ++c) {
                    const int cc = i * (D / 64) + c;
                    uint32_t o[32];
                    tmem_ld32(t_O + lane_off + cc * 32, o);
                    tmem_ld_wait();
#pragma unroll
                    for (int v = 0; v < 8; ++v)
                        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(punit(s0, cc * 8 + v)),
                                     "f"(__uint_as_float(o[4 * v]) * inv), "f"(__uint_as_float(o[4 * v + 1]) * inv),
                                     "f"(__uint_as_float(o[4 * v + 2]) * inv), "f"(__uint_as_float(o[4 * v + 3]) * inv)
                                     : "memory");
                }
            }
            if (i == 0)
                asm volatile("st.shared.f32 [%0], %1;" ::"r"(s0 + kPartBytes + r * 4), "f"(lse_own) : "memory");
            fence_proxy_async_smem();  // generic-proxy smem writes -> the bulk copies' reads
            named_bar_sync(1, 256);
            if (threadIdx.x == 128) {
                mbar_wait_cluster(xfer_free, 0);
                const uint32_t mb = peer_smem_addr(merge_bar, 0);
                bulk_copy_to_peer(peer_smem_addr(smem + kPartBytes, 0), s0, kPartBytes, mb);
                bulk_copy_to_peer(peer_smem_addr(smem + 2 * kPartBytes, 0), s0 + kPartBytes, kBQ * 4, mb);
            }
        } else {
            if (threadIdx.x == 128) {  // our MMAs are done: the partner may fill our ring
                mbar_arrive_expect_tx(merge_bar, kPartBytes + kBQ * 4);
                mbar_arrive_remote(peer_smem_addr(xfer_free, 1));
            }
            mbar_wait(merge_bar, 0);
            float lse1;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(lse1) : "r"(s0 + 2 * kPartBytes + r * 4) : "memory");
            const bool exact = fallback || !(lse1 < INFINITY);
            auto stage = [&](int cc, const float* f) {  // bf16 row r, columns [32 cc, 32 cc + 32)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const uint32_t unit = static_cast<uint32_t>(cc * 4 + v);
                    const uint32_t a = s0 + static_cast<uint32_t>(r) * kRowBytes +
                                       ((unit ^ (static_cast<uint32_t>(r) & (kU - 1))) << 4);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a),
                                 "r"(pack_bf16x2(f[8 * v + 0], f[8 * v + 1])), "r"(pack_bf16x2(f[8 * v + 2], f[8 * v + 3])),
                                 "r"(pack_bf16x2(f[8 * v + 4], f[8 * v + 5])), "r"(pack_bf16x2(f[8 * v + 6], f[8 * v + 7]))
                                 : "memory");
                }
            };
            if (!exact) {
                const float lm = fmaxf(lse_own, lse1);
                const float wa = ex2_approx(lse_own - lm), wb = ex2_approx(lse1 - lm);
                const float iw = 1.0f / (wa + wb);
                const float ca = wa * iw * inv, cb = wb * iw;
#pragma unroll 1
                for (int c = 0; c < D / 64; ++c) {
                    const int cc = i * (D / 64) + c;
                    uint32_t o[32];
                    tmem_ld32(t_O + lane_off + cc * 32, o);
                    tmem_ld_wait();
                    float f[32];
#pragma unroll
                    for (int v = 0; v < 8; ++v) {
                        float4 y;
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(y.x), "=f"(y.y), "=f"(y.z), "=f"(y.w)
                                     : "r"(punit(s0 + kPartBytes, cc * 8 + v)));
                        f[4 * v] = fmaf(__uint_as_float(o[4 * v]), ca, cb * y.x);
                        f[4 * v + 1] = fmaf(__uint_as_float(o[4 * v + 1]), ca, cb * y.y);
                        f[4 * v + 2] = fmaf(__uint_as_float(o[4 * v + 2]), ca, cb * y.z);
                        f[4 * v + 3] = fmaf(__uint_as_float(o[4 * v + 3]), ca, cb * y.w);
                    }
                    stage(cc, f);
                }
            } else {
                // exact recompute of row r over the whole kv range, columns [i D/2, (i+1) D/2)
                const int qi = q_tile * kBQ + r;
                float acc[D / 2];
#pragma unroll
                for (int d = 0; d < D / 2; ++d) acc[d] = 0.0f;
                float m = -INFINITY, l = 0.0f;
                if (qi < p.sq) {
                    const bf16* qr = p.q_ptr + static_cast<int64_t>(qi) * p.q_row_stride + head * D;
                    const int total = p.seg_len[0] + p.seg_len[1];
                    for (int jj = 0; jj < total; ++jj) {
                        const int kr = jj < p.seg_len[0] ? p.seg_start[0] + jj : p.seg_start[1] + (jj - p.seg_len[0]);
                        const bf16* krow = p.k_ptr + static_cast<int64_t>(kr) * p.kv_row_stride + head * D;
                        const bf16* vrow = p.v_ptr + static_cast<int64_t>(kr) * p.kv_row_stride + head * D + i * (D / 2);
                        float sdot = 0.0f;
                        for (int d = 0; d < D; ++d) sdot = fmaf(__bfloat162float(qr[d]), __bfloat162float(krow[d]), sdot);
                        sdot *= scale;
                        const float mn = fmaxf(m, sdot);
                        const float a = exp2f(m - mn), e = exp2f(sdot - mn);
                        l = l * a + e;
#pragma unroll
                        for (int d = 0; d < D / 2; ++d) acc[d] = acc[d] * a + e * __bfloat162float(vrow[d]);
                        m = mn;
                    }
                }
                const float il = 1.0f / l;
#pragma unroll
                for (int d = 0; d < D / 2; ++d) acc[d] *= il;
#pragma unroll
                for (int c = 0; c < D / 64; ++c) stage(i * (D / 64) + c, &acc[c * 32]);
            }
            named_bar_sync(1, 256);  // staged rows visible
            const int tid = static_cast<int>(threadIdx.x) - 128;
            const int r0 = q_tile * kBQ;
#pragma unroll 1
            for (int idx = tid; idx < kBQ * static_cast<int>(kU); idx += 256) {
                const int row = idx / static_cast<int>(kU);
                const uint32_t uu = static_cast<uint32_t>(idx) % kU;
                const int q_row = r0 + row;
                if (q_row >= p.sq) continue;
                uint4 w;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                             : "r"(s0 + static_cast<uint32_t>(row) * kRowBytes +
                                   ((uu ^ (static_cast<uint32_t>(row) & (kU - 1))) << 4))
                             : "memory");
                const int chunk = q_row / p.rows_per_chunk;
                bf16* drow = p.out_base[chunk] + static_cast<int64_t>(q_row - chunk * p.rows_per_chunk) * p.out_row_stride +
                             static_cast<int64_t>(head) * D;
                *reinterpret_cast<uint4*>(drow + uu * 8) = w;
            }
        }
        } else {
        // this slot's half of the O columns, 32 at a time: normalise, stage in this tile's Q
        // buffer (every QK^T of the tile is done); O is handed to the next tile's PV as soon as
        // the last chunk is in registers
        const uint32_t s_base = smem_u32(sQ + b * L::kQBytes);
        if (!fallback) {
#pragma unroll 1
            for (int c = 0; c < D / 64; ++c) {
                const int cc = i * (D / 64) + c;
                uint32_t o[32];
                tmem_ld32(t_O + lane_off + cc * 32, o);
                tmem_ld_wait();
                if (c == D / 64 - 1) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(o_free);
                }
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const uint32_t unit = static_cast<uint32_t>(cc * 4 + v);
                    const uint32_t a = s_base + static_cast<uint32_t>(r) * kRowBytes +
                                       ((unit ^ (static_cast<uint32_t>(r) & (kU - 1))) << 4);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a),
                                 "r"(pack_bf16x2(__uint_as_float(o[8 * v + 0]) * inv, __uint_as_float(o[8 * v + 1]) * inv)),
                                 "r"(pack_bf16x2(__uint_as_float(o[8 * v + 2]) * inv, __uint_as_float(o[8 * v + 3]) * inv)),
                                 "r"(pack_bf16x2(__uint_as_float(o[8 * v + 4]) * inv, __uint_as_float(o[8 * v + 5]) * inv)),
                                 "r"(pack_bf16x2(__uint_as_float(o[8 * v + 6]) * inv, __uint_as_float(o[8 * v + 7]) * inv))
                                 : "memory");
                }
            }
        } else {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(o_free);  // O is not read on this path
            // exact recompute of this thread's row, columns [i D/2, (i + 1) D/2), from global
            // memory with a running max (rare path; see the kernel comment)
            const int qi = q_tile * kBQ + r;
            float acc[D / 2];
#pragma unroll
            for (int d = 0; d < D / 2; ++d) acc[d] = 0.0f;
            float m = -INFINITY, l = 0.0f;
            if (qi < p.sq) {
                const bf16* qr = p.q_ptr + static_cast<int64_t>(qi) * p.q_row_stride + head * D;
                const int total = p.seg_len[0] + p.seg_len[1];
                for (int jj = 0; jj < total; ++jj) {
                    const int kr = jj < p.seg_len[0] ? p.seg_start[0] + jj : p.seg_start[1] + (jj - p.seg_len[0]);
                    const bf16* krow = p.k_ptr + static_cast<int64_t>(kr) * p.kv_row_stride + head * D;
                    const bf16* vrow = p.v_ptr + static_cast<int64_t>(kr) * p.kv_row_stride + head * D + i * (D / 2);
                    float sdot = 0.0f;
                    for (int d = 0; d < D; ++d) sdot = fmaf(__bfloat162float(qr[d]), __bfloat162float(krow[d]), sdot);
                    sdot *= scale;
                    const float mn = fmaxf(m, sdot);
                    const float a = exp2f(m - mn), e = exp2f(sdot - mn);
                    l = l * a + e;
#pragma unroll
                    for (int d = 0; d < D / 2; ++d) acc[d] = acc[d] * a + e * __bfloat162float(vrow[d]);
                    m = mn;
                }
            }
            const float il = 1.0f / l;
#pragma unroll
            for (int v = 0; v < D / 16; ++v) {
                const uint32_t unit = static_cast<uint32_t>(i * (D / 16) + v);
                const uint32_t a = s_base + static_cast<uint32_t>(r) * kRowBytes +
                                   ((unit ^ (static_cast<uint32_t>(r) & (kU - 1))) << 4);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a),
                             "r"(pack_bf16x2(acc[8 * v + 0] * il, acc[8 * v + 1] * il)),
                             "r"(pack_bf16x2(acc[8 * v + 2] * il, acc[8 * v + 3] * il)),
                             "r"(pack_bf16x2(acc[8 * v + 4] * il, acc[8 * v + 5] * il)),
                             "r"(pack_bf16x2(acc[8 * v + 6] * il, acc[8 * v + 7] * il))
                             : "memory");
            }
        }
        named_bar_sync(1, 256);  // staged rows visible; every thread has read s_ovf and st_l
        if (threadIdx.x == 128) s_ovf = 0;  // re-armed for the next tile
        const int tid = static_cast<int>(threadIdx.x) - 128;
        // output chunks of this tile's rows: with chunks of >= 128 rows a tile spans at most two,
        // split at row `split` (no division per store); smaller chunks divide per row
        const int r0 = q_tile * kBQ;
        const int rpc = p.rows_per_chunk;
        const int c0 = r0 / rpc;
        const int split = (c0 + 1) * rpc - r0;
        const int64_t ostride = p.out_row_stride;
        bf16* base0 = p.out_base[c0] + static_cast<int64_t>(r0 - c0 * rpc) * ostride + static_cast<int64_t>(head) * D;
        bf16* base1 = split < kBQ && c0 + 1 < 8
                          ? p.out_base[c0 + 1] - static_cast<int64_t>(split) * ostride + static_cast<int64_t>(head) * D
                          : base0;
#pragma unroll 1
        for (int idx = tid; idx < kBQ * static_cast<int>(kU); idx += 256) {
            const int row = idx / static_cast<int>(kU);
            const uint32_t uu = static_cast<uint32_t>(idx) % kU;
            const int q_row = r0 + row;
            if (q_row >= p.sq) continue;
            uint4 w;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                         : "r"(s_base + static_cast<uint32_t>(row) * kRowBytes +
                               ((uu ^ (static_cast<uint32_t>(row) & (kU - 1))) << 4))
                         : "memory");
            bf16* drow;
            if (rpc >= kBQ) {
                drow = (row < split ? base0 : base1) + static_cast<int64_t>(row) * ostride;
            } else {
                const int chunk = q_row / rpc;
                drow = p.out_base[chunk] + static_cast<int64_t>(q_row - chunk * rpc) * ostride +
                       static_cast<int64_t>(head) * D;
            }
            *reinterpret_cast<uint4*>(drow + uu * 8) = w;
        }
        // this thread's staging reads are done: the producer may load tile it + 2's Q here
        // (generic-proxy reads before an async-proxy write: the mbarrier orders them)
        mbar_arrive(&q_free[b]);
        }  // merged piece
        if (threadIdx.x == 128 && it < 4) attn_mark(p, 20 + it);  // per piece: epilogue end
        }  // tiles
    }
    tc_fence_before();
    // pair: split 1's shared memory is read by its bulk copies until CTA 0 has the partial
    if constexpr (kPair) cluster_sync_all();
    __syncthreads();
    span_end(p.span);
    if (threadIdx.x == 128) {
        attn_mark(p, 3);
        attn_mark_global(p, 8);
    }
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

template <int D, int kMode = 0>
void attn_v3_launch(dim3 grid, const AttnPlan& plan, const AttnParams& p, cudaStream_t stream) {
    static bool done[64] = {};
    int dev = 0;
    SPX_CUDA(cudaGetDevice(&dev));
    if (!done[dev & 63]) {
        SPX_CUDA(cudaFuncSetAttribute(attn_fwd_v3_kernel<D, kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(SmemV3<D>::kBytes)));
        done[dev & 63] = true;
    }
    if constexpr (kMode != 0)
        launch_pdl_cluster(attn_fwd_v3_kernel<D, kMode>, grid, dim3(kThreadsV2), SmemV3<D>::kBytes, stream, 2,
                           plan.map_q, plan.map_k, plan.map_v, p);
    else
        launch_pdl(attn_fwd_v3_kernel<D, kMode>, grid, dim3(kThreadsV2), SmemV3<D>::kBytes, stream, plan.map_q,
                   plan.map_k, plan.map_v, p);
}

// head_dim 16 / 32 (the reference's default and desk configurations, GenerationConfig
// defaults D = 16: generator.hpp:14-42): below the 64-element rows the tcgen05 / TMA tile
// layout is built for; these shapes are tiny (48-token blocks), so a SIMT kernel serves them.
// One warp per (query row, head); lanes stride over the keys of both ring segments with a
// per-lane online softmax, merged across the warp at the end. Same output addressing as K6.
template <int D>
__global__ void __launch_bounds__(128) attn_small_kernel(const bf16* __restrict__ q,
                                                        const bf16* __restrict__ k,
                                                        const bf16* __restrict__ v,
                                                        const AttnParams p, int64_t q_stride,
                                                        int64_t kv_stride) {
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x % 32;
    const int64_t pair = static_cast<int64_t>(blockIdx.x) * 4 + threadIdx.x / 32;
    if (pair >= static_cast<int64_t>(p.sq) * p.heads) return;
    const int row = static_cast<int>(pair / p.heads);
    const int head = static_cast<int>(pair % p.heads);
    float qf[D];
#pragma unroll
    for (int d = 0; d < D; ++d) qf[d] = __bfloat162float(q[row * q_stride + head * D + d]) * p.scale_log2;
    const int total = p.seg_len[0] + p.seg_len[1];
    float m = -INFINITY, l = 0.0f, acc[D];
#pragma unroll
    for (int d = 0; d < D; ++d) acc[d] = 0.0f;
    for (int j = lane; j < total; j += 32) {
        const int r = j < p.seg_len[0] ? p.seg_start[0] + j : p.seg_start[1] + (j - p.seg_len[0]);
        const bf16* kr = k + static_cast<int64_t>(r) * kv_stride + head * D;
        const bf16* vr = v + static_cast<int64_t>(r) * kv_stride + head * D;
        float s = 0.0f;
#pragma unroll
        for (int d = 0; d < D; ++d) s = fmaf(qf[d], __bfloat162float(kr[d]), s);
        const float mn = fmaxf(m, s);
        const float a = exp2f(m - mn), e = exp2f(s - mn);
        l = l * a + e;
#pragma unroll
        for (int d = 0; d < D; ++d) acc[d] = acc[d] * a + e * __bfloat162float(vr[d]);
        m = mn;
    }
    float mw = m;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, o));
    const float a = m == -INFINITY ? 0.0f : exp2f(m - mw);
    l *= a;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    const float inv = 1.0f / l;
    const int chunk = row / p.rows_per_chunk;
    bf16* dst = p.out_base[chunk] + static_cast<int64_t>(row - chunk * p.rows_per_chunk) * p.out_row_stride +
                static_cast<int64_t>(head) * D;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        float x = acc[d] * a;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == d % 32) dst[d] = __float2bfloat16_rn(x * inv);
    }
}

}  // namespace

namespace {
// kv splits for n (query tile x head) CTAs over `tiles` kv tiles: the modelled time
//   waves(n s) x (c + tiles / s)          [kv-tile units]
// with the fixed per-CTA cost c = 3.3 tiles unsplit, 9 tiles split (fp32 partial staging, the
// bulk copy out, the last CTA's bulk loads + merge), fitted to B200 sweeps (tools/kbench.py,
// SPX_ATTN_SPLITS=1..8: e.g. 2340x4680x3 s=2 29.5 vs s=1 40.1 us; 2340x32760x3 s=5 113.7 vs
// s=1 234.8; 4680x4680x6 s=1 80.8 vs s=2 82.3). Every CTA keeps >= 2 kv tiles (one per
// softmax warpgroup).
int choose_splits(int64_t n, int64_t tiles, int sm_count, int cap) {
    int best = 1;
    double best_t = 1e30;
    for (int sp = 1; sp <= cap; ++sp) {
        if (sp > 1 && tiles / sp < 2) break;
        const double waves = static_cast<double>(ceil_div(n * sp, sm_count));
        const double t = waves * ((sp == 1 ? 3.3 : 9.0) + static_cast<double>(tiles) / sp);
        if (t < best_t * 0.97) {  // a split must win clearly (the model is coarse)
            best_t = t;
            best = sp;
        }
    }
    return best;
}
}  // namespace

// the shared-O / early-S kernel (v3) for unsplit and 2-split layouts: SPX_ATTN_V3 = 0 never
// (v2 everywhere), otherwise always (the persistent v3 measured 3-5 % faster than v2 on the
// single-wave layouts too: 4680 x 4680 x 3 0.0359 vs 0.0375 ms, profiles/r02au)
std::atomic<int> g_attn_v3{[] {
    const char* e = std::getenv("SPX_ATTN_V3");
    return e ? std::atoi(e) : 1;
}()};
bool attn_v3_enabled() { return g_attn_v3.load(std::memory_order_relaxed) != 0; }
void attn_set_v3(int on) { g_attn_v3.store(on, std::memory_order_relaxed); }

// SPX_ATTN_V3_PERSISTENT=0: one CTA per query tile (the pre-persistent launch shape; A/B)
bool v3_persistent() {
    static const bool on = [] {
        const char* e = std::getenv("SPX_ATTN_V3_PERSISTENT");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

std::atomic<int> g_forced_splits{[] {  // tuning override: SPX_ATTN_SPLITS=<1..8>
    const char* e = std::getenv("SPX_ATTN_SPLITS");
    return e ? std::max(1, std::min(8, std::atoi(e))) : 0;
}()};

void attn_force_splits(int s) { g_forced_splits.store(s, std::memory_order_relaxed); }

namespace {
// Mixed layout for mode 0: the first n_full (query tile, head) tiles unsplit, the remaining
// ones in s2 splits, scored by a greedy list-scheduling simulation of the CTAs in block order
// on sm_count SMs with the same per-CTA costs as choose_splits (full: 3.3 + tiles, split:
// 9 + tiles / s2, in kv-tile units). E.g. 222 tiles x 37 kv tiles on 148 SMs: 148 full + 74
// tiles in halves (one full and one half CTA per SM) instead of 1.5 waves of full CTAs.
struct Layout {
    int n_full, s2;
};
double simulate(int64_t full, int64_t split_ctas, double t_full, double t_split, int sms) {
    // full CTAs land round-robin (identical durations); split CTAs greedily on the earliest
    // free SM (min-heap)
    std::vector<double> busy(static_cast<size_t>(sms));
    for (int i = 0; i < sms; ++i)
        busy[static_cast<size_t>(i)] = t_full * static_cast<double>(full / sms + (i < full % sms ? 1 : 0));
    std::make_heap(busy.begin(), busy.end(), std::greater<double>());
    for (int64_t i = 0; i < split_ctas; ++i) {
        std::pop_heap(busy.begin(), busy.end(), std::greater<double>());
        busy.back() += t_split;
        std::push_heap(busy.begin(), busy.end(), std::greater<double>());
    }
    return *std::max_element(busy.begin(), busy.end());
}
Layout choose_layout(int64_t T, int64_t tiles, int sms, int cap) {
    static std::mutex mu;
    static std::map<std::tuple<int64_t, int64_t, int, int>, Layout> cache;
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_tuple(T, tiles, sms, cap);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    Layout best{static_cast<int>(T), 1};
    double best_t = simulate(T, 0, 3.3 + static_cast<double>(tiles), 0.0, sms);
    for (int s2 = 2; s2 <= cap; ++s2) {
        if (tiles / s2 < 2) break;
        const double ts = 9.0 + static_cast<double>(ceil_div(tiles, s2));
        // the split part beyond ~2 waves of CTAs never beats fewer, longer splits
        for (int64_t F = T - 1; F >= std::max<int64_t>(0, T - 2 * sms); --F) {
            const double t = simulate(F, (T - F) * s2, 3.3 + static_cast<double>(tiles), ts, sms);
            if (t < best_t * 0.97) {  // a split must win clearly (the model is coarse)
                best_t = t;
                best = {static_cast<int>(F), s2};
            }
        }
    }
    cache[key] = best;
    return best;
}
}  // namespace

int attn_max_splits(const AttnOperands& ops, int sm_count) {
    const int forced = g_forced_splits.load(std::memory_order_relaxed);
    if (forced) return forced;
    // the workspace is sized for the longest kv range the buffers can hold (splits grow
    // with the kv length)
    const int64_t n = ceil_div(static_cast<int64_t>(ops.sq), kBQ) * ops.heads * ops.batch;
    const int64_t tiles = ceil_div(ops.kv_rows, kBKV);
    return std::max(choose_splits(n, tiles, sm_count, 8), choose_layout(n, tiles, sm_count, 8).s2);
}

size_t attn_workspace_bytes(const AttnOperands& ops, int max_splits) {
    if (max_splits <= 1) return 0;
    const size_t tiles = static_cast<size_t>((ceil_div(static_cast<int64_t>(ops.sq), kBQ) + 1) & ~1);
    const size_t rows = tiles * kBQ;  // query tiles padded to whole CTA pairs
    const size_t ctr = (rows / kBQ * ops.heads * sizeof(int) + 255) / 256 * 256;
    const size_t lse = (max_splits * rows * ops.heads * sizeof(float) + 255) / 256 * 256;
    return ctr + lse + max_splits * rows * ops.heads * ops.head_dim * sizeof(float);
}

void attn_plan(AttnPlan* plan, const AttnOperands& ops, int sm_count) {
    require(ops.head_dim == 16 || ops.head_dim == 32 || ops.head_dim == 64 || ops.head_dim == 128,
            SPX_ERR_UNSUPPORTED,
            "attention: head_dim must be 16, 32, 64 or 128 (got " + std::to_string(ops.head_dim) + ")");
    require(ops.batch == 1, SPX_ERR_UNSUPPORTED, "attention kernel: batch must be 1");
    require(ops.sq > 0 && ops.heads > 0, SPX_ERR_SHAPE, "attention: empty problem");
    require(ops.rows_per_chunk > 0 && ceil_div(ops.sq, ops.rows_per_chunk) <= 8, SPX_ERR_SHAPE,
            "attention: at most 8 output chunks");
    plan->ops = ops;
    if (ops.head_dim < 64) {  // SIMT path (attn_small_kernel): no tensor maps, no splits
        attn_set_segments(plan, ops.seg_start, ops.seg_len, ops.num_segs);
        plan->max_splits = 1;
        return;
    }
    char err[256];
    const uint32_t box[3] = {64, 1, 128};
    {
        const uint64_t dims[3] = {static_cast<uint64_t>(ops.head_dim),
                                  static_cast<uint64_t>(ops.heads),
                                  static_cast<uint64_t>(ops.q_rows)};
        const uint64_t strides[2] = {static_cast<uint64_t>(ops.head_dim) * 2,
                                     static_cast<uint64_t>(ops.heads) * ops.head_dim * 2};
        require(make_tma_map_bf16(&plan->map_q, ops.q, 3, dims, strides, box, err, sizeof(err)),
                SPX_ERR_ALIGNMENT, err);
    }
    {
        const uint64_t dims[3] = {static_cast<uint64_t>(ops.head_dim),
                                  static_cast<uint64_t>(ops.heads),
                                  static_cast<uint64_t>(ops.kv_rows)};
        const uint64_t strides[2] = {static_cast<uint64_t>(ops.head_dim) * 2,
                                     static_cast<uint64_t>(ops.heads) * ops.head_dim * 2};
        require(make_tma_map_bf16(&plan->map_k, ops.k, 3, dims, strides, box, err, sizeof(err)),
                SPX_ERR_ALIGNMENT, err);
        require(make_tma_map_bf16(&plan->map_v, ops.v, 3, dims, strides, box, err, sizeof(err)),
                SPX_ERR_ALIGNMENT, err);
    }
    attn_set_segments(plan, ops.seg_start, ops.seg_len, ops.num_segs);
    plan->max_splits = ops.batch == 1 ? attn_max_splits(ops, sm_count) : 1;
    if (plan->max_splits > 1 &&
        (ops.workspace == nullptr || ops.workspace_bytes < attn_workspace_bytes(ops, plan->max_splits)))
        plan->max_splits = 1;  // no (or too small a) workspace: one CTA per tile
}

void attn_set_segments(AttnPlan* plan, const int* seg_start, const int* seg_len, int num_segs) {
    require(num_segs >= 1 && num_segs <= 2, SPX_ERR_SHAPE, "attention: 1 or 2 kv segments");
    int total = 0;
    for (int s = 0; s < 2; ++s) {
        plan->ops.seg_start[s] = s < num_segs ? seg_start[s] : 0;
        plan->ops.seg_len[s] = s < num_segs ? seg_len[s] : 0;
        require(plan->ops.seg_len[s] >= 0 &&
                    plan->ops.seg_start[s] + plan->ops.seg_len[s] <= plan->ops.kv_rows,
                SPX_ERR_RANGE, "attention: kv segment out of range");
        total += plan->ops.seg_len[s];
    }
    plan->ops.num_segs = num_segs;
    require(total > 0, SPX_ERR_EMPTY_CACHE, "attention over an empty key/value set");
}

void attn_run(const AttnPlan& plan, cudaStream_t stream) {
    const AttnOperands& o = plan.ops;
    AttnParams p{};
    p.sq = o.sq;
    for (int s = 0; s < 2; ++s) {
        p.seg_start[s] = o.seg_start[s];
        p.seg_len[s] = o.seg_len[s];
    }
    if (o.head_dim < 64) {
        p.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(o.head_dim));
        for (int i = 0; i < 8; ++i) p.out_base[i] = o.out_base[i];
        p.rows_per_chunk = o.rows_per_chunk;
        p.out_row_stride = o.out_row_stride;
        p.heads = o.heads;
        const int64_t pairs = static_cast<int64_t>(o.sq) * o.heads;
        const dim3 grid(static_cast<unsigned>(ceil_div(pairs, 4)));
        const int64_t qs = static_cast<int64_t>(o.heads) * o.head_dim;
        if (o.head_dim == 16)
            launch_pdl(attn_small_kernel<16>, grid, dim3(128), 0, stream, o.q, o.k, o.v, p, qs, qs);
        else
            launch_pdl(attn_small_kernel<32>, grid, dim3(128), 0, stream, o.q, o.k, o.v, p, qs, qs);
        SPX_CUDA_LAUNCH();
        count_launch();
        return;
    }
    p.seg_tiles0 = static_cast<int>(ceil_div(o.seg_len[0], kBKV));
    p.total_tiles = p.seg_tiles0 + static_cast<int>(ceil_div(o.seg_len[1], kBKV));
    p.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(o.head_dim));
    static const int experiment = [] {
        const char* e = std::getenv("SPX_ATTN_EXPERIMENT");
        return e ? std::atoi(e) : 0;
    }();
    p.experiment = experiment;
    if (experiment == 5) p.trace = gemm_trace_buffer();
    p.span = span_slot();
    for (int i = 0; i < 8; ++i) p.out_base[i] = o.out_base[i];
    p.rows_per_chunk = o.rows_per_chunk;
    for (int r = 0; r < 2; ++r) {
        p.pf[r] = static_cast<const uint8_t*>(o.l2_prefetch[r]);
        p.pf_bytes[r] = o.l2_prefetch[r] ? o.l2_prefetch_bytes[r] : 0;
    }
    p.out_row_stride = o.out_row_stride;
    p.out_batch_stride = o.out_batch_stride;
    p.q_ptr = o.q;
    p.k_ptr = o.k;
    p.v_ptr = o.v;
    p.q_row_stride = static_cast<int64_t>(o.heads) * o.head_dim;
    p.kv_row_stride = static_cast<int64_t>(o.heads) * o.head_dim;
    // kv splits for this call's kv length, within the planned workspace
    {
        int dev = 0;
        SPX_CUDA(cudaGetDevice(&dev));
        const int64_t n = ceil_div(static_cast<int64_t>(o.sq), kBQ) * o.heads * o.batch;
        const bool forced = g_forced_splits.load(std::memory_order_relaxed) != 0;
        p.qt = static_cast<int>(ceil_div(o.sq, kBQ));
        if (forced || o.head_dim != 128) {  // uniform splits
            const int want = forced ? plan.max_splits
                                    : choose_splits(n, p.total_tiles, device_sm_count(dev), plan.max_splits);
            p.splits = std::max(1, std::min(want, p.total_tiles / 2));
            p.n_full = p.splits == 1 ? static_cast<int>(n) : 0;
        } else {
            Layout lay = choose_layout(n, p.total_tiles, device_sm_count(dev), plan.max_splits);
            static const char* forced_layout = std::getenv("SPX_ATTN_LAYOUT");  // "F,s2" (tuning)
            if (forced_layout) {
                int f = 0, s2 = 1;
                if (std::sscanf(forced_layout, "%d,%d", &f, &s2) == 2)
                    lay = {f, std::min(s2, plan.max_splits)};
            }
            static const bool verbose = std::getenv("SPX_ATTN_VERBOSE") != nullptr;
            if (verbose)
                std::fprintf(stderr, "attention layout: T=%lld tiles=%d -> n_full=%d s2=%d (cap %d)\n",
                             static_cast<long long>(n), p.total_tiles, lay.n_full, lay.s2, plan.max_splits);
            p.splits = std::max(1, std::min(lay.s2, p.total_tiles / 2));
            p.n_full = p.splits == 1 ? static_cast<int>(n) : lay.n_full;
        }
    }
    p.heads = o.heads;
    p.q_tiles = static_cast<int>((ceil_div(o.sq, kBQ) + 1) & ~1);  // workspace stride (pairs)
    if (p.splits > 1 && p.n_full < p.qt * o.heads) {
        const size_t rows = static_cast<size_t>(p.q_tiles) * kBQ;
        uint8_t* ws = static_cast<uint8_t*>(o.workspace);
        const size_t ctr = (rows / kBQ * o.heads * sizeof(int) + 255) / 256 * 256;
        const size_t lse = (plan.max_splits * rows * o.heads * sizeof(float) + 255) / 256 * 256;
        p.counters = reinterpret_cast<int*>(ws);
        p.ws_lse = reinterpret_cast<float*>(ws + ctr);
        p.ws_o = reinterpret_cast<float*>(ws + ctr + lse);
    }
    {
        const int64_t T = static_cast<int64_t>(p.qt) * o.heads;
        int dev = 0;
        SPX_CUDA(cudaGetDevice(&dev));
        const int sms = device_sm_count(dev);
        static const bool pair_merge = [] {  // SPX_ATTN_SPLIT_PAIR=0: the workspace merge
            const char* e = std::getenv("SPX_ATTN_SPLIT_PAIR");
            return !(e && std::atoi(e) == 0);
        }();
        static const bool triple_on = [] {  // SPX_ATTN_TRIPLE=0: no triple layout (A/B)
            const char* e = std::getenv("SPX_ATTN_TRIPLE");
            return !(e && std::atoi(e) == 0);
        }();
        // triple layout: 1.5 tiles per SM (one whole tile per CTA plus half of a third per
        // 2-CTA cluster) when the tiles are 3 per cluster and fill the SMs in 1-2 waves (the
        // P = 2 per-rank shape: 222 tiles on 148 SMs). Measured (profiles/r02bh): 0.0662 ->
        // 0.0638 ms at 4680 x 4680 x 6 (37 kv tiles), but 0.355 -> 0.360 ms at 256 kv tiles (the
        // half pieces and the merge cost more than the balance gains there): short kv ranges only
        const int64_t clusters3 = T / 3;
        const bool triple = triple_on && !o.prefer_v3 && T % 3 == 0 && T > sms && clusters3 <= sms / 2 &&
                            5 * clusters3 >= 4 * (sms / 2) && p.total_tiles >= 8 && p.total_tiles <= 48 &&
                            (p.experiment == 0 || p.experiment == 5) && g_attn_v3.load(std::memory_order_relaxed) != 0 &&
                            !g_forced_splits.load(std::memory_order_relaxed);
        if (triple) {
            const dim3 g3(static_cast<unsigned>(2 * clusters3));
            if (o.head_dim == 128)
                attn_v3_launch<128, 2>(g3, plan, p, stream);
            else
                attn_v3_launch<64, 2>(g3, plan, p, stream);
        } else if (pair_merge && p.n_full == 0 && p.splits == 2 && g_attn_v3.load(std::memory_order_relaxed) != 0 &&
            (p.experiment == 0 || p.experiment == 5)) {
            // every tile in 2 kv halves: the shared-O kernel as 2-CTA clusters merging via DSMEM
            const dim3 g2(static_cast<unsigned>(2 * T));
            if (o.head_dim == 128)
                attn_v3_launch<128, 1>(g2, plan, p, stream);
            else
                attn_v3_launch<64, 1>(g2, plan, p, stream);
        } else if (p.n_full == T && (p.experiment == 0 || p.experiment == 5) &&
                   g_attn_v3.load(std::memory_order_relaxed) != 0) {
            // every tile unsplit: the shared-O / early-S kernel, persistent over the tiles
            const dim3 gv3(static_cast<unsigned>(std::min<int64_t>(T, v3_persistent() ? sms : T)));
            if (o.head_dim == 128)
                attn_v3_launch<128>(gv3, plan, p, stream);
            else
                attn_v3_launch<64>(gv3, plan, p, stream);
        } else {  // mode 0: 1-D grid, n_full unsplit tiles then the split ones
            const dim3 g1(static_cast<unsigned>(p.n_full + (T - p.n_full) * p.splits));
            if (o.head_dim == 128)
                attn_v2_launch<128, 0>(g1, plan, p, stream);
            else
                attn_v2_launch<64, 0>(g1, plan, p, stream);
        }
    }
    SPX_CUDA_LAUNCH();
    count_launch();
}

}  // namespace spx
