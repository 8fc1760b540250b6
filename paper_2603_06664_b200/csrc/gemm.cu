// gemm.cu -- K2/K8: the QKV and output projections (reference: project_tokens,
// proj/src/sp_attention.cpp:51-75, y[t,:] = W x[t,:] with W [out][in] row-major) as one
// persistent, warp-specialised tcgen05 GEMM:
//
//   out[M][N] = A[M][K] * B[N][K]^T        A = tokens (bf16), B = W (bf16, K-major)
//
//   warp 0      : TMA producer (A box 64x128 from a 3-D [G][M][k_inner] map, B box 64xBN)
//   warp 1      : single-thread tcgen05.mma issuer, M=128 x N=BN x K=16 per instruction,
//                 fp32 accumulator double-buffered in TMEM (2 x BN columns)
//   warp 2      : TMEM allocator
//   warps 4..11 : epilogue (two warps per TMEM lane quarter, half the columns each),
//                 tcgen05.ld -> (gate, residual | RoPE + pack) -> bf16 -> global
//
// The smem ring is 4 stages of (A 16 KB + B BN*128 B), SWIZZLE_128B everywhere.
#include <atomic>
#include <cstdlib>

#include "common.hpp"
#include "kernels.hpp"
#include "rope_device.cuh"
#include "sm100.cuh"
#include "tma.hpp"

namespace spx {

using namespace sm100;

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kStages = 4;
constexpr int kThreads = 384;
constexpr int kEpiWarps = 8;  // warps 4..11: two per TMEM lane quarter, splitting the columns
// epi_mode 2 stages the rank's slice of the RoPE band tables in smem: T rows of the frames
// its tokens span, all H rows, all W rows (the scattered per-row table reads from L1/L2 cost
// more than the whole mainloop: 0.111 vs 0.054 ms for the Wan QKV GEMM)
constexpr int kRopeSmemPairs = 2048;
// per epilogue warp: 32 rows x 32 bf16 columns staged for the coalescing transpose
constexpr int kEpiStageBytes = 32 * 64;

struct GemmParams {
    int M, N, K, k_inner;
    int num_m_tiles, num_n_tiles;
    bf16* out;
    int64_t ldo;
    int epi_mode;
    const bf16* residual;
    int64_t ldr;
    const float* gate;
    const float* bias;
    RopeLaunch rope;  // epi_mode 2
    // epi_mode 2 lookups (host-computed: no integer division in the epilogue)
    int head_shift;         // log2(head_dim)
    int8_t head_group[16];  // head -> its head group g
    int8_t head_slot[16];   // head -> index within the group
    int n_fastest;    // tile raster: 1 = n index fastest (concurrent CTAs share A row blocks:
                      // A larger than B), 0 = m fastest (concurrent CTAs share B = weights)
    int b_early;      // stages whose B tile the producer loaded before griddepcontrol.wait
    int experiment;   // profiling (SPX_GEMM_EXPERIMENT): 1 = rope epilogue without rotation,
                      // 5 = per-tile clock64 timeline of the pair kernel into `trace`
    long long* trace;  // [cta][16 tiles][4]: mma start, mma issued, epilogue start, end
    unsigned long long* span;  // SPX_SPAN_TRACE
};

__device__ __forceinline__ int tile_m(const GemmParams& p, int tile) {
    return p.n_fastest ? tile / p.num_n_tiles : tile % p.num_m_tiles;
}
__device__ __forceinline__ int tile_n(const GemmParams& p, int tile) {
    return p.n_fastest ? tile % p.num_n_tiles : tile / p.num_m_tiles;
}

__device__ __forceinline__ void trace_mark(const GemmParams& p, int it, int kind) {
    if (p.experiment == 5 && it < 14) p.trace[(blockIdx.x * 16 + it) * 4 + kind] = clock64();
}

// kRopeSmem = false (single-CTA kernel, epilogues without RoPE): the table area is traded for
// a fifth pipeline stage where it fits (128 x 192: the O-projection's exact 2-wave tile;
// 18.6 -> 18.3 us standalone, -0.8 us per layer call in the engine)
template <int BN, bool kRopeSmem>
__host__ __device__ constexpr int gemm_stages() { return (!kRopeSmem && BN == 192) ? 5 : kStages; }
template <int BN, bool kRopeSmem = true, int kSplit = 1>
constexpr size_t gemm_smem_bytes() {
    return 1024 + static_cast<size_t>(gemm_stages<BN, kRopeSmem>()) * (kBM * kBK * 2 + BN * kBK * 2) +
           256 + (kRopeSmem ? kRopeSmemPairs * 8 : 0) + kEpiWarps * kEpiStageBytes +
           (kSplit > 1 ? static_cast<size_t>(kBM) * BN * 4 : 0);
}


// ---- RoPE band tables staged in smem (epi_mode 2; layout in rope_device.cuh) ----
// every thread of the CTA: copy the slice (before the CTA-wide barrier that follows setup)
__device__ __forceinline__ void rope_stage_tables(const RopeLaunch& l, uint32_t st) {
    rope_stage_tables(l, st, static_cast<int>(threadIdx.x), static_cast<int>(blockDim.x));
}

// a token row's three band rows in the staged tables (shared-memory byte addresses, computed
// once per row per tile; explicit ld.shared keeps the reads off the generic/long-scoreboard path)
struct RopeRow {
    uint32_t t;  // T band row of its frame
    uint32_t h;  // H band row
    uint32_t w;  // W band row
    bool valid;
};

__device__ __forceinline__ RopeRow rope_row(const RopeLaunch& l, const RopeSmem& r, uint32_t st,
                                            int row) {
    int t, h, w;
    rope_thw(l, row, t, h, w);
    return {st + 8u * static_cast<uint32_t>((t - r.t_lo) * l.pairs[0]),
            st + 8u * static_cast<uint32_t>(r.off_h + h * l.pairs[1]),
            st + 8u * static_cast<uint32_t>(r.off_w + w * l.pairs[2]), true};
}

// epi_mode 2: RoPE of a 32-column slice of one head of q or k for token `row` at (t, h, w):
// pairs (2j, 2j+1) rotate in fp32 (rope.cpp:106-126) before the single bf16 rounding. All 16
// (cos, sin) pairs are loaded before any math (branch-free band selection), so the shared-
// memory latency is paid once per slice, not once per pair.
__device__ __forceinline__ void rope_rotate_chunk(const RopeLaunch& l, const RopeRow& rr, int d0,
                                                  float (&f)[32]) {
    // pair j = j0 + e lies in band T below k0, H below k1, W above (warp-uniform breakpoints);
    // each band's row base is offset so that base + 8 e addresses pair j
    const int j0 = d0 / 2;
    const int k0 = l.pairs[0] - j0, k1 = l.pairs[0] + l.pairs[1] - j0;
    const uint32_t tb = rr.t + 8u * j0, hb = rr.h - 8u * k0, wb = rr.w - 8u * k1;
    float2 cs[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        const uint32_t base = e < k0 ? tb : (e < k1 ? hb : wb);
        cs[e] = lds_f2(base + 8u * e);
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        const float x0 = f[2 * e], x1 = f[2 * e + 1];
        f[2 * e] = x0 * cs[e].x - x1 * cs[e].y;
        f[2 * e + 1] = x0 * cs[e].y + x1 * cs[e].x;
    }
}

// Destinations of a 32-column slice (warp-uniform): column `col0` of row 0. epi_mode 2 is the
// pack of the fused all-to-all, as K3 does: q slices go to their head group's q slab, k / v
// slices to every KV-ring copy of the group.
struct ChunkDst {
    int which, g, n;  // which: 0 q, 1 k, 2 v (epi_mode 2); -1 the plain output
    int d0;           // first head-dim element of the slice (epi_mode 2)
    int64_t off, stride;
};

__device__ __forceinline__ ChunkDst chunk_dst(const GemmParams& p, int col0) {
    if (p.epi_mode != 2 && p.epi_mode != 4) return {-1, 0, 1, 0, col0, p.ldo};
    const RopeLaunch& l = p.rope;
    const int C = l.heads << p.head_shift;
    const int which = (col0 >= C) + (col0 >= 2 * C);
    if (p.epi_mode == 4 && which < 2) return {-1, 0, 1, 0, col0, p.ldo};  // q | k: plain output
    const int c = col0 - which * C;
    const int head = c >> p.head_shift;
    const int d0 = c & ((1 << p.head_shift) - 1);
    return {which, p.head_group[head], which == 0 ? 1 : l.dst.copies, d0,
            (static_cast<int64_t>(p.head_slot[head]) << p.head_shift) + d0, l.dst_row_stride};
}

__device__ __forceinline__ bf16* chunk_base(const GemmParams& p, const ChunkDst& d, int cp) {
    bf16* b = d.which < 0 ? p.out
              : d.which == 0 ? p.rope.dst.q[d.g]
              : d.which == 1 ? p.rope.dst.k[d.g][cp] : p.rope.dst.v[d.g][cp];
    return b + d.off;
}

// One 32-column slice of the warp's 32 accumulator rows (lane = row) -> (gate, residual |
// RoPE) -> bf16 -> global. The slice is transposed through the warp's 2 KB of shared memory
// (16-byte units XOR-swizzled, conflict-free both ways) so each store instruction writes
// 8 rows x 64 contiguous bytes (full sectors) instead of 32 rows x 16 bytes.
__device__ __forceinline__ void epilogue_chunk(const GemmParams& p, int row0, int lane, int col0,
                                               const uint32_t (&r)[32], uint32_t stage,
                                               const RopeRow& rr = RopeRow{},
                                               const uint4* res_pre = nullptr) {
    if (col0 >= p.N) return;  // warp-uniform
    const int row = row0 + lane;
    float f[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(r[j]);
    const ChunkDst d = chunk_dst(p, col0);
    if (p.epi_mode != 2 && p.bias) {  // warp-uniform; the 32 bias values are a broadcast load
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias + col0 + j));
            f[j] += b.x;
            f[j + 1] += b.y;
            f[j + 2] += b.z;
            f[j + 3] += b.w;
        }
    }
    if (p.epi_mode == 2) {
        if (d.which < 2 && rr.valid) rope_rotate_chunk(p.rope, rr, d.d0, f);
    } else if (p.epi_mode == 1 && row < p.M) {
        const uint4* res = reinterpret_cast<const uint4*>(p.residual + row * p.ldr + col0);
        float g[32];
#pragma unroll
        for (int j = 0; j < 32; j += 4) {  // the gate: broadcast float4 loads
            const float4 gv = p.gate ? __ldg(reinterpret_cast<const float4*>(p.gate + col0 + j))
                                     : make_float4(1.0f, 1.0f, 1.0f, 1.0f);
            g[j] = gv.x;
            g[j + 1] = gv.y;
            g[j + 2] = gv.z;
            g[j + 3] = gv.w;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 rv = res_pre ? res_pre[q] : res[q];
            const uint32_t rw[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float2 rs = unpack_bf16x2(rw[e]);
                const int j = q * 8 + e * 2;
                f[j] = rs.x + g[j] * f[j];
                f[j + 1] = rs.y + g[j + 1] * f[j + 1];
            }
        }
    } else if (p.epi_mode == 3) {
        // GELU, tanh approximation (torch.nn.GELU(approximate="tanh"), the Wan FFN):
        // 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))
        // tanh on the SFU (tanh.approx.f32: ~2^-11 relative, below the bf16 output rounding);
        // tanhf's software sequence made this epilogue cost 20 us on the 1536 -> 8960 FFN
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const float x = f[j];
            const float u = 0.7978845608028654f * fmaf(0.044715f * x, x * x, x);
            float t;
            asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
            f[j] = 0.5f * x * (1.0f + t);
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t a = stage + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a),
                     "r"(pack_bf16x2(f[q * 8 + 0], f[q * 8 + 1])), "r"(pack_bf16x2(f[q * 8 + 2], f[q * 8 + 3])),
                     "r"(pack_bf16x2(f[q * 8 + 4], f[q * 8 + 5])), "r"(pack_bf16x2(f[q * 8 + 6], f[q * 8 + 7]))
                     : "memory");
    }
    __syncwarp();
    const int u = lane & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int rr_ = (lane >> 2) + 8 * i;
        uint4 w;
        const uint32_t a = stage + rr_ * 64 + ((u ^ ((rr_ >> 1) & 3)) << 4);
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                     : "r"(a)
                     : "memory");
        const int grow = row0 + rr_;
        if (grow < p.M) {
            for (int cp = 0; cp < d.n; ++cp)
                *reinterpret_cast<uint4*>(chunk_base(p, d, cp) + static_cast<int64_t>(grow) * d.stride +
                                          u * 8) = w;
        }
    }
    __syncwarp();  // the slice's shared memory is read before the next slice overwrites it
}

// kSplit = 2 (split-K, launched as 2-CTA clusters, BN = 128): both CTAs of a cluster own the
// same output tile; CTA r accumulates k-blocks [r K/2, (r+1) K/2) in its own TMEM. CTA 1's
// epilogue warps store their fp32 partial into CTA 0's shared memory (DSMEM, a [chunk][4-column
// group][row] float4 layout: conflict-free on both sides) and arrive on CTA 0's pfull; CTA 0 adds
// it to its accumulator and runs the epilogue, then hands the buffer back (pempty in CTA 1). For
// the short-M per-rank shapes (585-1170 rows at P = 4 / 8), whose tiles cannot fill the SMs: each
// SM streams half the operand bytes of the tile (the L2 -> SM inflow is what bounds them).
template <int BN, bool kRopeSmem = true, int kSplit = 1>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_b, const GemmParams p) {
    static_assert(kSplit == 1 || (kSplit == 2 && BN == 128), "split-K: 2-CTA clusters, BN = 128");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    constexpr uint32_t kABytes = kBM * kBK * 2;
    constexpr uint32_t kBBytes = BN * kBK * 2;
    constexpr uint32_t kTmemCols = 2 * BN <= 256 ? 256 : 512;  // power of two >= 2 x BN
    constexpr int kStages = gemm_stages<BN, kRopeSmem>();
    uint8_t* sA = smem;
    uint8_t* sB = smem + kStages * kABytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint64_t* pfull = tempty + 2;   // split-K (CTA 0): CTA 1's partial landed
    uint64_t* pempty = pfull + 1;   // split-K (CTA 1): CTA 0 has consumed the partial buffer
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pempty + 1);
    const uint32_t s_rope = smem_u32(reinterpret_cast<uint8_t*>(full) + 256);
    const uint32_t s_stage =
        s_rope + (kRopeSmem ? kRopeSmemPairs * 8 : 0) + (threadIdx.x / 32 - 4) * kEpiStageBytes;
    const uint32_t s_part = s_rope + (kRopeSmem ? kRopeSmemPairs * 8 : 0) + kEpiWarps * kEpiStageBytes;
    const RopeSmem rope_l = p.epi_mode == 2 ? rope_smem_layout(p.rope) : RopeSmem{};

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int split = kSplit > 1 ? static_cast<int>(cluster_ctarank()) : 0;
    const int tile0 = static_cast<int>(blockIdx.x) / kSplit;   // this CTA's first tile
    const int tile_step = static_cast<int>(gridDim.x) / kSplit;
    pdl_trigger();  // the next kernel may launch; it waits for this grid before its main loop
    span_begin(p.span);
    if (threadIdx.x == 0 && p.experiment == 5) {
        p.trace[(blockIdx.x * 16 + 15) * 4 + 0] = clock64();
        p.trace[(blockIdx.x * 16 + 14) * 4 + 0] = static_cast<long long>(globaltimer_ns());
    }
    const int num_tiles = p.num_m_tiles * p.num_n_tiles;
    const int num_kt_all = p.K / kBK;
    const int kt_begin = split * num_kt_all / kSplit;  // this CTA's k-blocks
    const int num_kt = (split + 1) * num_kt_all / kSplit - kt_begin;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&map_a);
        tma_prefetch_desc(&map_b);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kEpiWarps);  // one arrival per epilogue warp
        }
        mbar_init(pfull, kEpiWarps * 32);   // every epilogue thread of CTA 1
        mbar_init(pempty, kEpiWarps * 32);  // every epilogue thread of CTA 0
        fence_mbar_init();
        // B (weights) of this CTA's first tile: not produced by the previous kernel, so it
        // streams in while that kernel drains; A follows after the PDL wait
        if (tile0 < num_tiles) {
            const int n0 = tile_n(p, tile0) * BN;
            for (int kt = 0; kt < p.b_early; ++kt) {
                mbar_arrive_expect_tx(&full[kt], kABytes + kBBytes);
                tma_load_2d(sB + kt * kBBytes, &map_b, &full[kt], (kt_begin + kt) * kBK, n0);
            }
        }
    }
    if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
    // a constant (uploaded) RoPE table is staged while the previous kernel drains
    if constexpr (kRopeSmem)
        if (p.epi_mode == 2 && p.rope.tab_constant) rope_stage_tables(p.rope, s_rope);
    // the previous kernel's outputs (A operand, destinations, a per-call RoPE table) are
    // complete past this point; everything above overlapped its tail
    pdl_wait();
    if constexpr (kRopeSmem)
        if (p.epi_mode == 2 && !p.rope.tab_constant) rope_stage_tables(p.rope, s_rope);
    tc_fence_before();
    if constexpr (kSplit > 1)
        cluster_sync_all();  // the peer's pfull / pempty exist before any remote arrival
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0 && p.experiment == 5) p.trace[(blockIdx.x * 16 + 15) * 4 + 1] = clock64();

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = tile0; tile < num_tiles; tile += tile_step) {
                const int m0 = tile_m(p, tile) * kBM;
                const int n0 = tile_n(p, tile) * BN;
                for (int kt = 0; kt < num_kt; ++kt) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    const bool early = tile == tile0 && kt < p.b_early;
                    if (!early) mbar_arrive_expect_tx(&full[stage], kABytes + kBBytes);
                    const int k0 = (kt_begin + kt) * kBK;
                    tma_load_3d(sA + stage * kABytes, &map_a, &full[stage], k0 % p.k_inner, m0,
                                k0 / p.k_inner);
                    if (!early) tma_load_2d(sB + stage * kBBytes, &map_b, &full[stage], k0, n0);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // whole warp: uniform control flow and descriptors; one elected lane issues
        const bool issuer = elect_one();
        {
            constexpr uint32_t idesc = make_idesc_bf16(kBM, BN, false, false);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int tile = tile0; tile < num_tiles; tile += tile_step, ++it) {
                const int acc = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                mbar_wait(&tempty[acc], aphase ^ 1);
                tc_fence_after();
                if (issuer) trace_mark(p, it, 0);
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kt = 0; kt < num_kt; ++kt) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_addr = smem_u32(sA + stage * kABytes);
                    const uint32_t b_addr = smem_u32(sB + stage * kBBytes);
                    if (issuer) {
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k) {
                            umma_bf16_ss(d_tmem, make_desc_sw128(a_addr + k * 32, 16, 1024),
                                         make_desc_sw128(b_addr + k * 32, 16, 1024), idesc,
                                         (kt | k) != 0);
                        }
                        umma_commit(&empty[stage]);
                    }
                    __syncwarp();
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (issuer) umma_commit(&tfull[acc]);
                if (issuer) trace_mark(p, it, 1);
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        const int ew = warp % 4;         // TMEM lane quarter this warp may access
        const int half = (warp - 4) / 4;  // which half of the tile's columns
        // split-K partial buffer: [chunk][4-column group][row] float4, this thread's row
        const uint32_t part_row = s_part + static_cast<uint32_t>(ew * 32 + lane) * 16u;
        // the accumulator chunk c of this thread's row (+ CTA 1's partial on CTA 0)
        auto load_acc = [&](uint32_t t_row, int c, uint32_t (&r)[32]) {
            tmem_ld32(t_row + c * 32, r);
            tmem_ld_wait();
            if constexpr (kSplit > 1) {
#pragma unroll
                for (int j4 = 0; j4 < 8; ++j4) {
                    float4 v;
                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                                 : "r"(part_row + static_cast<uint32_t>(c * 8 + j4) * (kBM * 16u)));
                    r[4 * j4 + 0] = __float_as_uint(__uint_as_float(r[4 * j4 + 0]) + v.x);
                    r[4 * j4 + 1] = __float_as_uint(__uint_as_float(r[4 * j4 + 1]) + v.y);
                    r[4 * j4 + 2] = __float_as_uint(__uint_as_float(r[4 * j4 + 2]) + v.z);
                    r[4 * j4 + 3] = __float_as_uint(__uint_as_float(r[4 * j4 + 3]) + v.w);
                }
            }
        };
        int it = 0;
        for (int tile = tile0; tile < num_tiles; tile += tile_step, ++it) {
            const int acc = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            const int m0 = tile_m(p, tile) * kBM;
            const int n0 = tile_n(p, tile) * BN;
            const int row = m0 + ew * 32 + lane;
            if constexpr (kSplit > 1) {
                if (split == 1) {
                    // ship the partial into CTA 0's buffer once CTA 0 has consumed the last one
                    mbar_wait(&tfull[acc], aphase);
                    tc_fence_after();
                    mbar_wait_cluster(pempty, (it & 1) ^ 1);
                    uint32_t peer_row;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(peer_row) : "r"(part_row));
                    const uint32_t t_row = tmem_base + acc * BN + (static_cast<uint32_t>(ew * 32) << 16);
#pragma unroll
                    for (int c = half * (BN / 64); c < (half + 1) * (BN / 64); ++c) {
                        uint32_t r[32];
                        tmem_ld32(t_row + c * 32, r);
                        tmem_ld_wait();
#pragma unroll
                        for (int j4 = 0; j4 < 8; ++j4)
                            asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                                             peer_row + static_cast<uint32_t>(c * 8 + j4) * (kBM * 16u)),
                                         "r"(r[4 * j4]), "r"(r[4 * j4 + 1]), "r"(r[4 * j4 + 2]), "r"(r[4 * j4 + 3])
                                         : "memory");
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                    uint32_t peer_full;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(peer_full) : "r"(smem_u32(pfull)));
                    mbar_arrive_remote(peer_full);  // release.cluster: the stores above are visible
                    continue;
                }
            }
            if (p.epi_mode == 1) {
                // residual epilogue: this lane's residual row segments are loaded before the
                // accumulator is waited for (one L2 round trip per tile, overlapping the MMA,
                // instead of one per 32-column slice on the epilogue's critical path)
                constexpr int kS = BN / 64;
                uint4 res_pre[kS][4];
#pragma unroll
                for (int ci = 0; ci < kS; ++ci) {
                    const int col = n0 + (half * kS + ci) * 32;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        res_pre[ci][q] = (row < p.M && col < p.N)
                                             ? reinterpret_cast<const uint4*>(p.residual + row * p.ldr + col)[q]
                                             : make_uint4(0, 0, 0, 0);
                }
                mbar_wait(&tfull[acc], aphase);
                tc_fence_after();
                if constexpr (kSplit > 1) mbar_wait_cluster(pfull, it & 1);
                if (warp == 4 && lane == 0) trace_mark(p, it, 2);
                const uint32_t t_row = tmem_base + acc * BN + (static_cast<uint32_t>(ew * 32) << 16);
#pragma unroll
                for (int ci = 0; ci < kS; ++ci) {
                    const int c = half * kS + ci;
                    uint32_t r[32];
                    load_acc(t_row, c, r);
                    epilogue_chunk(p, m0 + ew * 32, lane, n0 + c * 32, r, s_stage, RopeRow{}, res_pre[ci]);
                }
            } else {
            mbar_wait(&tfull[acc], aphase);
            tc_fence_after();
            if constexpr (kSplit > 1) mbar_wait_cluster(pfull, it & 1);
            if (warp == 4 && lane == 0) trace_mark(p, it, 2);
            const uint32_t t_row = tmem_base + acc * BN + (static_cast<uint32_t>(ew * 32) << 16);
            RopeRow rr{};
            if (p.epi_mode == 2 && row < p.M) rr = rope_row(p.rope, rope_l, s_rope, row);
            if (p.experiment == 1 || !p.rope.rotate) rr.valid = false;
#pragma unroll 1
            for (int c = half * (BN / 64); c < (half + 1) * (BN / 64); ++c) {
                uint32_t r[32];
                load_acc(t_row, c, r);
                epilogue_chunk(p, m0 + ew * 32, lane, n0 + c * 32, r, s_stage, rr);
            }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if constexpr (kSplit > 1) {  // the partial buffer is free for CTA 1's next tile
                uint32_t peer_empty;
                asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(peer_empty) : "r"(smem_u32(pempty)));
                mbar_arrive_remote(peer_empty);
            }
            if (warp == 4 && lane == 0) trace_mark(p, it, 3);
        }
    }
    if constexpr (kSplit > 1)
        cluster_sync_all();  // no CTA exits while its peer may still arrive on its barriers
    else
        __syncthreads();
    span_end(p.span);
    if (threadIdx.x == 0 && p.experiment == 5) {
        p.trace[(blockIdx.x * 16 + 15) * 4 + 2] = clock64();
        p.trace[(blockIdx.x * 16 + 14) * 4 + 1] = static_cast<long long>(globaltimer_ns());
    }
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem_base);
    }
}

// =========================================================================================
// CTA-pair variant (cta_group::2): a 2-CTA cluster owns a 256 x BN output tile. CTA c loads
// its own 128 rows of A and its half (BN/2 rows) of B into its own smem; the leader's single
// MMA thread issues M=256 x N=BN x K=16 pair MMAs that read both CTAs' smem, so each SM
// streams half the B operand it would for a 128 x BN tile (operand bytes per MMA cycle
// halve, the L2 -> SM limit of the 1-CTA kernel). Accumulators: 128 lanes x BN columns in
// each CTA's TMEM, double-buffered; each CTA's epilogue drains its own rows.
//   full[s]   leader only, 1 arrival + 2 x stage bytes (both CTAs' TMA count on it)
//   empty[s]  both CTAs, released by the leader's multicast commit
//   tfull[a]  both CTAs, multicast commit after the tile's last k-block
//   tempty[a] leader only, 2 x 128 epilogue arrivals (the peer's arrive remotely)
// =========================================================================================
constexpr int kPairStages = 6;

template <int BN>
constexpr size_t gemm_pair_smem_bytes() {
    return 1024 + static_cast<size_t>(kPairStages) * (128 * kBK * 2 + (BN / 2) * kBK * 2) + 256 +
           kRopeSmemPairs * 8 + kEpiWarps * kEpiStageBytes;
}

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_bf16_tn_pair_kernel(const __grid_constant__ CUtensorMap map_a,
                             const __grid_constant__ CUtensorMap map_b, const GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    constexpr uint32_t kABytes = 128 * kBK * 2;
    constexpr uint32_t kBBytes = (BN / 2) * kBK * 2;
    constexpr uint32_t kTmemCols = 2 * BN <= 256 ? 256 : 512;  // power of two >= 2 x BN
    uint8_t* sA = smem;
    uint8_t* sB = smem + kPairStages * kABytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + kPairStages * kBBytes);
    uint64_t* empty = full + kPairStages;
    uint64_t* tfull = empty + kPairStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const uint32_t s_rope = smem_u32(reinterpret_cast<uint8_t*>(full) + 256);
    const uint32_t s_stage = s_rope + kRopeSmemPairs * 8 + (threadIdx.x / 32 - 4) * kEpiStageBytes;
    const RopeSmem rope_l = p.epi_mode == 2 ? rope_smem_layout(p.rope) : RopeSmem{};

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    pdl_trigger();  // the next kernel may launch; it waits for this grid before its main loop
    span_begin(p.span);
    if (threadIdx.x == 0 && p.experiment == 5) {
        p.trace[(blockIdx.x * 16 + 15) * 4 + 0] = clock64();
        p.trace[(blockIdx.x * 16 + 14) * 4 + 0] = static_cast<long long>(globaltimer_ns());
    }
    const int cta = static_cast<int>(cluster_ctarank());
    const bool leader = cta == 0;
    const int pair = blockIdx.x / 2;
    const int npairs = gridDim.x / 2;
    const int num_tiles = p.num_m_tiles * p.num_n_tiles;  // m tiles of 256 rows
    const int num_kt = p.K / kBK;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&map_a);
        tma_prefetch_desc(&map_b);
        for (int s = 0; s < kPairStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * kEpiWarps);  // one per epilogue warp of both CTAs
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc_pair<kTmemCols>(tmem_slot);
    // everything up to griddepcontrol.wait overlaps the previous kernel's tail: the barriers
    // and the TMEM slot are published cluster-wide, a constant RoPE table is staged, and the
    // producer streams the weight (B) halves of the first stages onto the leader's barriers
    if (p.epi_mode == 2 && p.rope.tab_constant) rope_stage_tables(p.rope, s_rope);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (warp == 0 && lane == 0 && pair < num_tiles) {
        const int n0 = tile_n(p, pair) * BN + cta * (BN / 2);
        for (int kt = 0; kt < p.b_early; ++kt) {
            // the leader arms the stage for both CTAs' A and B bytes; the peer's early B bytes
            // may land first (the transaction count goes transiently negative, and the phase
            // cannot complete before the leader's arrival)
            if (leader) mbar_arrive_expect_tx(&full[kt], 2 * (kABytes + kBBytes));
            tma_load_2d_pair(sB + kt * kBBytes, &map_b, &full[kt], kt * kBK, n0);
        }
    }
    pdl_wait();
    if (p.epi_mode == 2 && !p.rope.tab_constant) {
        rope_stage_tables(p.rope, s_rope);
        __syncthreads();  // the table is CTA-local: the epilogue warps read their own copy
    }
    if (threadIdx.x == 0 && p.experiment == 5) p.trace[(blockIdx.x * 16 + 15) * 4 + 1] = clock64();

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = pair; tile < num_tiles; tile += npairs) {
                const int m0 = tile_m(p, tile) * 256 + cta * 128;
                const int n0 = tile_n(p, tile) * BN + cta * (BN / 2);
                for (int kt = 0; kt < num_kt; ++kt) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    const bool early = tile == pair && kt < p.b_early;
                    if (leader && !early) mbar_arrive_expect_tx(&full[stage], 2 * (kABytes + kBBytes));
                    const int k0 = kt * kBK;
                    tma_load_3d_pair(sA + stage * kABytes, &map_a, &full[stage], k0 % p.k_inner, m0,
                                     k0 / p.k_inner);
                    if (!early) tma_load_2d_pair(sB + stage * kBBytes, &map_b, &full[stage], k0, n0);
                    if (++stage == kPairStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
            // drain: every multicast release of this CTA's stages has landed before exit
            for (int s = 0; s < kPairStages; ++s) {
                mbar_wait(&empty[stage], phase ^ 1);
                if (++stage == kPairStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        const bool issuer = elect_one();
        if (leader) {
            constexpr uint32_t idesc = make_idesc_bf16(256, BN, false, false);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int tile = pair; tile < num_tiles; tile += npairs, ++it) {
                const int acc = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                mbar_wait_cluster(&tempty[acc], aphase ^ 1);
                tc_fence_after();
                if (issuer) trace_mark(p, it, 0);
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kt = 0; kt < num_kt; ++kt) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_addr = smem_u32(sA + stage * kABytes);
                    const uint32_t b_addr = smem_u32(sB + stage * kBBytes);
                    if (issuer) {
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k) {
                            umma_bf16_ss_pair(d_tmem, make_desc_sw128(a_addr + k * 32, 16, 1024),
                                              make_desc_sw128(b_addr + k * 32, 16, 1024), idesc,
                                              (kt | k) != 0);
                        }
                        umma_commit_pair(&empty[stage], 0x3);
                    }
                    __syncwarp();
                    if (++stage == kPairStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (issuer) umma_commit_pair(&tfull[acc], 0x3);
                if (issuer) trace_mark(p, it, 1);
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        const int ew = warp % 4;
        const int half = (warp - 4) / 4;
        int it = 0;
        for (int tile = pair; tile < num_tiles; tile += npairs, ++it) {
            const int acc = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            const int m0 = tile_m(p, tile) * 256 + cta * 128;
            const int n0 = tile_n(p, tile) * BN;
            mbar_wait(&tfull[acc], aphase);
            tc_fence_after();
            if (warp == 4 && lane == 0) trace_mark(p, it, 2);
            const int row = m0 + ew * 32 + lane;
            const uint32_t t_row = tmem_base + acc * BN + (static_cast<uint32_t>(ew * 32) << 16);
            RopeRow rr{};
            if (p.epi_mode == 2 && row < p.M) rr = rope_row(p.rope, rope_l, s_rope, row);
            if (p.experiment == 1 || !p.rope.rotate) rr.valid = false;
#pragma unroll 1
            for (int c = half * (BN / 64); c < (half + 1) * (BN / 64); ++c) {
                uint32_t r[32];
                tmem_ld32(t_row + c * 32, r);
                tmem_ld_wait();
                epilogue_chunk(p, m0 + ew * 32, lane, n0 + c * 32, r, s_stage, rr);
            }
            // the warp's TMEM reads are complete (wait::ld); no global-store ordering is
            // needed, so the remote arrival is relaxed (no per-thread MEMBAR.GPU)
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_leader_relaxed(&tempty[acc]);
            if (warp == 4 && lane == 0) trace_mark(p, it, 3);
        }
    }
    tc_fence_before();
    cluster_sync_all();
    span_end(p.span);
    if (threadIdx.x == 0 && p.experiment == 5) {
        p.trace[(blockIdx.x * 16 + 15) * 4 + 2] = clock64();
        p.trace[(blockIdx.x * 16 + 14) * 4 + 1] = static_cast<long long>(globaltimer_ns());
    }
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_pair<kTmemCols>(tmem_base);
    }
}

template <int BN>
void set_pair_smem_attr() {
    static bool done[64] = {};
    int dev = 0;
    SPX_CUDA(cudaGetDevice(&dev));
    if (!done[dev & 63]) {
        SPX_CUDA(cudaFuncSetAttribute(gemm_bf16_tn_pair_kernel<BN>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(gemm_pair_smem_bytes<BN>())));
        done[dev & 63] = true;
    }
}

template <int BN, bool kRopeSmem = true, int kSplit = 1>
void set_smem_attr() {
    static bool done[64] = {};  // the attribute is per function per device
    int dev = 0;
    SPX_CUDA(cudaGetDevice(&dev));
    if (!done[dev & 63]) {
        SPX_CUDA(cudaFuncSetAttribute(gemm_bf16_tn_kernel<BN, kRopeSmem, kSplit>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(gemm_smem_bytes<BN, kRopeSmem, kSplit>())));
        done[dev & 63] = true;
    }
}

}  // namespace

namespace {
// tuning / test override of the planner: SPX_GEMM_VARIANT=0..4 (index into cands below) at
// load time, or spx_debug_set_gemm_variant at run time; -1 = modelled choice
std::atomic<int> g_forced_variant{[] {
    const char* e = std::getenv("SPX_GEMM_VARIANT");
    return e ? std::atoi(e) : -1;
}()};
}  // namespace

namespace {
long long* g_trace = nullptr;
}
long long* gemm_trace_buffer() {
    if (!g_trace) {
        SPX_CUDA(cudaMalloc(&g_trace, 1024 * 16 * 4 * sizeof(long long)));
        SPX_CUDA(cudaMemset(g_trace, 0, 1024 * 16 * 4 * sizeof(long long)));
    }
    return g_trace;
}

int gemm_forced_variant() { return g_forced_variant.load(std::memory_order_relaxed); }
void gemm_force_variant(int v) { g_forced_variant.store(v, std::memory_order_relaxed); }
int gemm_num_variants() { return 6; }

void gemm_plan(GemmPlan* plan, const GemmOperands& ops, int sm_count) {
    require(ops.M > 0 && ops.N > 0 && ops.K > 0, SPX_ERR_SHAPE, "gemm: empty problem");
    require(ops.K % kBK == 0, SPX_ERR_SHAPE, "gemm: K must be a multiple of 64");
    require(ops.k_inner % kBK == 0 && ops.groups * ops.k_inner == ops.K, SPX_ERR_SHAPE,
            "gemm: K must split into groups of a multiple of 64");
    require(ops.N % 32 == 0, SPX_ERR_SHAPE, "gemm: N must be a multiple of 32");
    require((reinterpret_cast<uintptr_t>(ops.out) & 15) == 0 && ops.out_row_stride % 8 == 0,
            SPX_ERR_ALIGNMENT, "gemm: output must be 16-byte aligned");
    plan->ops = ops;
    // Variant: modelled time = waves x per-SM tile work / efficiency, over
    //   pair (cta_group::2) 256 x {256, 128} tiles and single-CTA 128 x {256, 192, 128} tiles.
    // The single-CTA kernels stream 1.5-2x the operand bytes per MMA cycle (L2 -> SM bound).
    struct Cand { bool pair; int bn; double eff; int split; };
    // efficiencies measured on B200 (tools/kbench.py gemm, K = 1536): pair-256 1358 TFLOP/s
    // at 4680x4608, pair-128 908, single-256 1237, single-128 1077; single-192 estimated
    // between them (its 2-wave fit of the 4680x1536 O-projection is what it is for).
    // Split-K (2-CTA clusters, 128 x 128): half the k-blocks per SM plus the 64 KB partial
    // hand-off through DSMEM. Measured (r02ce): 585 x 8960 x 1536 (the Wan FFN down-projection
    // per rank at P = 8) 23.8 us against 29.6 for the best unsplit tile, but slower at K = 1536
    // (585 x 1536 x 1536: 10.8 vs 9.2 us), where the hand-off and the pipeline fill of the short
    // halves dominate: used from 64 k-blocks (K >= 4096), where the caller allows the changed
    // rounding
    static const Cand cands[] = {{true, 256, 1.0, 1}, {true, 128, 0.65, 1}, {false, 256, 0.88, 1},
                                 {false, 128, 0.72, 1}, {false, 192, 0.85, 1}, {false, 128, 0.9, 2}};
    const int forced = gemm_forced_variant();
    double best = 1e30;
    for (int ci = 0; ci < 6; ++ci) {
        const Cand& c = cands[ci];
        if (ops.N % 32 != 0) continue;
        if (c.split > 1 && (ops.K / kBK < 2 || (forced != ci && (!ops.allow_split_k || ops.K / kBK < 64))))
            continue;
        const int64_t bm = c.pair ? 256 : 128;
        const int64_t tiles = ceil_div(static_cast<int64_t>(ops.M), bm) * ceil_div(ops.N, c.bn);
        const int64_t slots = c.pair || c.split > 1 ? sm_count / 2 : sm_count;
        const double t = static_cast<double>(ceil_div(tiles, slots)) * 128.0 * c.bn / c.eff;
        if ((forced < 0 && t < best) || forced == ci) {
            best = forced == ci ? -1.0 : t;
            plan->pair = c.pair;
            plan->bn = c.bn;
            plan->ksplit = c.split;
        }
    }
    const int bm = plan->pair ? 256 : 128;
    char err[256];
    {
        const uint64_t dims[3] = {static_cast<uint64_t>(ops.k_inner), static_cast<uint64_t>(ops.M),
                                  static_cast<uint64_t>(ops.groups)};
        const uint64_t strides[2] = {static_cast<uint64_t>(ops.a_row_stride) * 2,
                                     static_cast<uint64_t>(ops.a_group_stride) * 2};
        const uint32_t box[3] = {kBK, 128, 1};
        require(make_tma_map_bf16(&plan->map_a, ops.a, 3, dims, strides, box, err, sizeof(err)),
                SPX_ERR_ALIGNMENT, err);
    }
    {
        const uint64_t dims[2] = {static_cast<uint64_t>(ops.K), static_cast<uint64_t>(ops.N)};
        const uint64_t strides[1] = {static_cast<uint64_t>(ops.b_row_stride) * 2};
        const uint32_t box[2] = {kBK, static_cast<uint32_t>(plan->pair ? plan->bn / 2 : plan->bn)};
        require(make_tma_map_bf16(&plan->map_b, ops.b, 2, dims, strides, box, err, sizeof(err)),
                SPX_ERR_ALIGNMENT, err);
    }
    const int64_t tiles = ceil_div(static_cast<int64_t>(ops.M), bm) * ceil_div(ops.N, plan->bn);
    if (plan->pair || plan->ksplit > 1) {
        const int64_t pairs = sm_count / 2;
        plan->grid = 2 * static_cast<int>(tiles < pairs ? tiles : pairs);
    } else {
        plan->grid = static_cast<int>(tiles < sm_count ? tiles : sm_count);
    }
}

bool gemm_rope_fusable(const GemmPlan& plan, const RopeLaunch& rope) {
    const int C = rope.heads * rope.head_dim;
    return rope.norm == 0 && rope.has_kv == 1 && rope.head_dim % 32 == 0 && C % plan.bn == 0 &&
           rope_smem_pairs(rope) <= kRopeSmemPairs &&
           plan.ops.N == 3 * C && plan.ops.M == rope.rows && plan.ops.groups == 1 &&
           rope.rows < (int64_t(1) << 31) && rope.row_offset + rope.rows_per_batch < (int64_t(1) << 31);
}

bool gemm_vpack_fusable(const GemmPlan& plan, const RopeLaunch& rope) {
    const int C = rope.heads * rope.head_dim;
    return rope.has_kv == 1 && rope.head_dim % 32 == 0 && C % plan.bn == 0 && C % 32 == 0 &&
           plan.ops.N == 3 * C && plan.ops.M == rope.rows && plan.ops.groups == 1 &&
           plan.ops.epi_mode == 0 && plan.ops.out_row_stride == 3 * C;
}

void gemm_run(const GemmPlan& plan, cudaStream_t stream, const RopeLaunch* rope) {
    const GemmOperands& o = plan.ops;
    GemmParams p{};
    p.M = o.M;
    p.N = o.N;
    p.K = o.K;
    p.k_inner = o.k_inner;
    p.num_m_tiles = static_cast<int>(ceil_div(o.M, plan.pair ? 256 : kBM));
    p.num_n_tiles = static_cast<int>(ceil_div(o.N, plan.bn));
    // raster: when A is the larger operand (the FFN's second projection: 84 MB of
    // activations against 27.5 MB of weights) the CTAs in flight walk n first, so each A row
    // block is read by its n-tiles at about the same time (once from DRAM) instead of once per
    // wave of m-fastest tiles (ncu: 208 MB DRAM read per launch against 111 MB of operands)
    static const int raster_env = [] {  // SPX_GEMM_RASTER: -1 auto, 0 m fastest, 1 n fastest
        const char* e = std::getenv("SPX_GEMM_RASTER");
        return e ? std::atoi(e) : -1;
    }();
    p.n_fastest = raster_env >= 0 ? raster_env
                                  : (static_cast<int64_t>(o.M) * o.K > static_cast<int64_t>(o.N) * o.K * 2 ? 1 : 0);
    p.out = o.out;
    p.ldo = o.out_row_stride;
    p.epi_mode = o.epi_mode;
    p.residual = o.residual;
    p.ldr = o.residual_row_stride;
    p.gate = o.gate;
    p.bias = o.bias;
    require(o.epi_mode != 1 || o.residual, SPX_ERR_CONFIG, "gemm: residual epilogue without residual");
    require(!o.bias || (reinterpret_cast<uintptr_t>(o.bias) & 15) == 0, SPX_ERR_ALIGNMENT,
            "gemm: bias must be 16-byte aligned");
    if (rope && rope->skip_v) {
        require(gemm_vpack_fusable(plan, *rope), SPX_ERR_UNSUPPORTED,
                "gemm: v-pack epilogue needs 3C outputs of stride 3C, C % BN == 0, D % 32 == 0");
        p.epi_mode = 4;
        p.rope = *rope;
    } else if (rope) {
        require(gemm_rope_fusable(plan, *rope), SPX_ERR_UNSUPPORTED,
                "gemm: rope epilogue needs 3C outputs, C % BN == 0, D % 32 == 0, no QK-norm");
        p.epi_mode = 2;
        p.rope = *rope;
    }
    if (rope) {
        require(rope->heads <= 16 && (rope->head_dim & (rope->head_dim - 1)) == 0, SPX_ERR_UNSUPPORTED,
                "gemm: rope epilogue needs <= 16 heads and a power-of-two head_dim");
        p.head_shift = 0;
        while ((1 << p.head_shift) < rope->head_dim) ++p.head_shift;
        const int hpg = rope->heads / rope->groups;
        for (int h = 0; h < rope->heads; ++h) {
            p.head_group[h] = static_cast<int8_t>(h / hpg);
            p.head_slot[h] = static_cast<int8_t>(h % hpg);
        }
    }
    static const int experiment = [] {
        const char* e = std::getenv("SPX_GEMM_EXPERIMENT");
        return e ? std::atoi(e) : 0;
    }();
    p.experiment = experiment;
    // 5: trace the QKV launches (RoPE epilogue) only; 7: every launch
    if ((experiment == 5 && rope) || experiment == 7) p.trace = gemm_trace_buffer();
    p.experiment = p.trace ? 5 : (experiment == 5 || experiment == 7 ? 0 : experiment);
    p.span = span_slot();
    // early B loads: the weight tiles of the first stages stream in before griddepcontrol.wait
    // (the pair kernel publishes its barriers cluster-wide first, then loads its B halves)
    static const int early_env = [] {  // SPX_GEMM_EARLY_B: 0 off, 1 single-CTA only, 2 all (A/B)
        const char* e = std::getenv("SPX_GEMM_EARLY_B");
        return e ? std::atoi(e) : 2;
    }();
    const bool early_ok = o.b_constant && (plan.pair ? early_env >= 2 : early_env >= 1);
    p.b_early = !early_ok ? 0
                : plan.pair ? std::min(p.K / kBK, kPairStages)
                            : std::min(p.K / kBK, plan.bn == 192 && p.epi_mode != 2 ? 5 : kStages);
    if (plan.ksplit > 1) {
        p.b_early = 0;
        set_smem_attr<128, true, 2>();
        launch_pdl_cluster(gemm_bf16_tn_kernel<128, true, 2>, dim3(plan.grid), dim3(kThreads),
                           gemm_smem_bytes<128, true, 2>(), stream, 2, plan.map_a, plan.map_b, p);
    } else if (plan.pair && plan.bn == 256) {
        set_pair_smem_attr<256>();
        launch_pdl(gemm_bf16_tn_pair_kernel<256>, dim3(plan.grid), dim3(kThreads),
                   gemm_pair_smem_bytes<256>(), stream, plan.map_a, plan.map_b, p);
    } else if (plan.pair) {
        set_pair_smem_attr<128>();
        launch_pdl(gemm_bf16_tn_pair_kernel<128>, dim3(plan.grid), dim3(kThreads),
                   gemm_pair_smem_bytes<128>(), stream, plan.map_a, plan.map_b, p);
    } else if (plan.bn == 192 && p.epi_mode == 2) {
        set_smem_attr<192>();
        launch_pdl(gemm_bf16_tn_kernel<192>, dim3(plan.grid), dim3(kThreads), gemm_smem_bytes<192>(),
                   stream, plan.map_a, plan.map_b, p);
    } else if (plan.bn == 192) {
        set_smem_attr<192, false>();
        launch_pdl(gemm_bf16_tn_kernel<192, false>, dim3(plan.grid), dim3(kThreads),
                   gemm_smem_bytes<192, false>(), stream, plan.map_a, plan.map_b, p);
    } else if (plan.bn == 256) {
        set_smem_attr<256>();
        launch_pdl(gemm_bf16_tn_kernel<256>, dim3(plan.grid), dim3(kThreads), gemm_smem_bytes<256>(),
                   stream, plan.map_a, plan.map_b, p);
    } else {
        set_smem_attr<128>();
        launch_pdl(gemm_bf16_tn_kernel<128>, dim3(plan.grid), dim3(kThreads), gemm_smem_bytes<128>(),
                   stream, plan.map_a, plan.map_b, p);
    }
    SPX_CUDA_LAUNCH();
    count_launch();
}

}  // namespace spx
