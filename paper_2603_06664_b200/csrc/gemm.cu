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

struct GemmParams {
    int M, N, K, k_inner;
    int num_m_tiles, num_n_tiles;
    bf16* out;
    int64_t ldo;
    int epi_mode;
    const bf16* residual;
    int64_t ldr;
    const float* gate;
    RopeLaunch rope;  // epi_mode 2
    int experiment;   // profiling (SPX_GEMM_EXPERIMENT): 1 = rope epilogue without rotation
};

template <int BN>
constexpr size_t gemm_smem_bytes() {
    return 1024 + static_cast<size_t>(kStages) * (kBM * kBK * 2 + BN * kBK * 2) + 256 +
           kRopeSmemPairs * 8;
}


// ---- RoPE band tables staged in smem (epi_mode 2) ----
struct RopeSmem {
    int t_lo, n_t;  // frames [t_lo, t_lo + n_t) of the T band
    int off_h, off_w;
};

__host__ __device__ inline RopeSmem rope_smem_layout(const RopeLaunch& l) {
    RopeSmem r;
    const int64_t first = l.row_offset, last = l.row_offset + l.rows_per_batch - 1;
    r.t_lo = static_cast<int>(l.start_frame + first / l.hw);
    r.n_t = static_cast<int>(last / l.hw - first / l.hw + 1);
    r.off_h = r.n_t * l.pairs[0];
    r.off_w = r.off_h + static_cast<int>(l.hw / l.grid_w) * l.pairs[1];
    return r;
}

__host__ __device__ inline int rope_smem_pairs(const RopeLaunch& l) {
    const RopeSmem r = rope_smem_layout(l);
    return r.off_w + static_cast<int>(l.grid_w) * l.pairs[2];
}

// every thread of the CTA: copy the slice (before the CTA-wide barrier that follows setup)
__device__ __forceinline__ void rope_stage_tables(const RopeLaunch& l, float2* st) {
    const RopeSmem r = rope_smem_layout(l);
    const int nt = r.n_t * l.pairs[0];
    const int total = rope_smem_pairs(l);
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
        float2 v;
        if (i < nt)
            v = __ldg(&l.tab[0][r.t_lo * l.pairs[0] + i]);
        else if (i < r.off_w)
            v = __ldg(&l.tab[1][i - r.off_h]);
        else
            v = __ldg(&l.tab[2][i - r.off_w]);
        st[i] = v;
    }
}

// a token row's three band rows in the staged tables (computed once per row per tile)
struct RopeRow {
    const float2* t;  // T band row of its frame
    const float2* h;  // H band row
    const float2* w;  // W band row
    bool valid;
};

__device__ __forceinline__ RopeRow rope_row(const RopeLaunch& l, const RopeSmem& r,
                                            const float2* st, int row) {
    int t, h, w;
    rope_thw(l, row, t, h, w);
    return {st + (t - r.t_lo) * l.pairs[0], st + r.off_h + h * l.pairs[1],
            st + r.off_w + w * l.pairs[2], true};
}

// epi_mode 2: a 32-column slice of one head of q, k or v for token `row` at (t, h, w):
// q/k pairs (2j, 2j+1) rotate in fp32 (rope.cpp:106-126) before the single bf16 rounding,
// then the slice is stored into its head group's q slab / every KV-ring copy (the pack of
// the fused all-to-all, as K3 does)
__device__ __forceinline__ void rope_pack_chunk(const RopeLaunch& l, const RopeRow& rr, int row,
                                                int col0, float (&f)[32]) {
    const int C = l.heads * l.head_dim;
    const int which = col0 / C;
    const int c = col0 - which * C;
    const int head = c / l.head_dim;
    const int d0 = c - head * l.head_dim;
    const int hpg = l.heads / l.groups;
    const int g = head / hpg;
    const int64_t off =
        static_cast<int64_t>(row) * l.dst_row_stride + (head - g * hpg) * l.head_dim + d0;
    if (which < 2 && rr.valid) {
        const int p0 = l.pairs[0], p01 = l.pairs[0] + l.pairs[1];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int j = d0 / 2 + e;  // warp-uniform band selection
            const float2 cs = j < p0 ? rr.t[j] : (j < p01 ? rr.h[j - p0] : rr.w[j - p01]);
            const float a = f[2 * e], b = f[2 * e + 1];
            f[2 * e] = a * cs.x - b * cs.y;
            f[2 * e + 1] = a * cs.y + b * cs.x;
        }
    }
    uint4 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
        v[q] = make_uint4(pack_bf16x2(f[q * 8 + 0], f[q * 8 + 1]), pack_bf16x2(f[q * 8 + 2], f[q * 8 + 3]),
                          pack_bf16x2(f[q * 8 + 4], f[q * 8 + 5]), pack_bf16x2(f[q * 8 + 6], f[q * 8 + 7]));
    if (which == 0) {
        uint4* d = reinterpret_cast<uint4*>(l.dst.q[g] + off);
#pragma unroll
        for (int q = 0; q < 4; ++q) d[q] = v[q];
    } else {
        for (int cp = 0; cp < l.dst.copies; ++cp) {
            uint4* d = reinterpret_cast<uint4*>((which == 1 ? l.dst.k[g][cp] : l.dst.v[g][cp]) + off);
#pragma unroll
            for (int q = 0; q < 4; ++q) d[q] = v[q];
        }
    }
}

// one 32-column slice of an accumulator row -> (gate, residual | rope + pack) -> bf16 -> global
__device__ __forceinline__ void epilogue_chunk(const GemmParams& p, int row, int col0,
                                               const uint32_t (&r)[32],
                                               const RopeRow& rr = RopeRow{}) {
    if (row >= p.M || col0 >= p.N) return;
    float f[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(r[j]);
    if (p.epi_mode == 2) {
        rope_pack_chunk(p.rope, rr, row, col0, f);
        return;
    }
    if (p.epi_mode == 1) {
        const uint4* res = reinterpret_cast<const uint4*>(p.residual + row * p.ldr + col0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint4 rv = res[q];
            const uint32_t rw[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float2 rr = unpack_bf16x2(rw[e]);
                const int j = q * 8 + e * 2;
                f[j] = rr.x + p.gate[col0 + j] * f[j];
                f[j + 1] = rr.y + p.gate[col0 + j + 1] * f[j + 1];
            }
        }
    }
    uint4* dst = reinterpret_cast<uint4*>(p.out + static_cast<int64_t>(row) * p.ldo + col0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        dst[q] = make_uint4(pack_bf16x2(f[q * 8 + 0], f[q * 8 + 1]),
                            pack_bf16x2(f[q * 8 + 2], f[q * 8 + 3]),
                            pack_bf16x2(f[q * 8 + 4], f[q * 8 + 5]),
                            pack_bf16x2(f[q * 8 + 6], f[q * 8 + 7]));
    }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_b, const GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    constexpr uint32_t kABytes = kBM * kBK * 2;
    constexpr uint32_t kBBytes = BN * kBK * 2;
    constexpr uint32_t kTmemCols = 2 * BN;
    uint8_t* sA = smem;
    uint8_t* sB = smem + kStages * kABytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    float2* s_rope = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(full) + 256);
    const RopeSmem rope_l = p.epi_mode == 2 ? rope_smem_layout(p.rope) : RopeSmem{};

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int num_tiles = p.num_m_tiles * p.num_n_tiles;
    const int num_kt = p.K / kBK;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&map_a);
        tma_prefetch_desc(&map_b);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kEpiWarps * 32);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
    if (p.epi_mode == 2) rope_stage_tables(p.rope, s_rope);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int m0 = (tile % p.num_m_tiles) * kBM;
                const int n0 = (tile / p.num_m_tiles) * BN;
                for (int kt = 0; kt < num_kt; ++kt) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], kABytes + kBBytes);
                    const int k0 = kt * kBK;
                    tma_load_3d(sA + stage * kABytes, &map_a, &full[stage], k0 % p.k_inner, m0,
                                k0 / p.k_inner);
                    tma_load_2d(sB + stage * kBBytes, &map_b, &full[stage], k0, n0);
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
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
                const int acc = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                mbar_wait(&tempty[acc], aphase ^ 1);
                tc_fence_after();
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
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        const int ew = warp % 4;         // TMEM lane quarter this warp may access
        const int half = (warp - 4) / 4;  // which half of the tile's columns
        int it = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
            const int acc = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            const int m0 = (tile % p.num_m_tiles) * kBM;
            const int n0 = (tile / p.num_m_tiles) * BN;
            mbar_wait(&tfull[acc], aphase);
            tc_fence_after();
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
                epilogue_chunk(p, row, n0 + c * 32, r, rr);
            }
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
        }
    }
    __syncthreads();
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
           kRopeSmemPairs * 8;
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
    constexpr uint32_t kTmemCols = 2 * BN;
    uint8_t* sA = smem;
    uint8_t* sB = smem + kPairStages * kABytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + kPairStages * kBBytes);
    uint64_t* empty = full + kPairStages;
    uint64_t* tfull = empty + kPairStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    float2* s_rope = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(full) + 256);
    const RopeSmem rope_l = p.epi_mode == 2 ? rope_smem_layout(p.rope) : RopeSmem{};

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
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
            mbar_init(&tempty[a], 2 * kEpiWarps * 32);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc_pair<kTmemCols>(tmem_slot);
    if (p.epi_mode == 2) rope_stage_tables(p.rope, s_rope);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = pair; tile < num_tiles; tile += npairs) {
                const int m0 = (tile % p.num_m_tiles) * 256 + cta * 128;
                const int n0 = (tile / p.num_m_tiles) * BN + cta * (BN / 2);
                for (int kt = 0; kt < num_kt; ++kt) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * (kABytes + kBBytes));
                    const int k0 = kt * kBK;
                    tma_load_3d_pair(sA + stage * kABytes, &map_a, &full[stage], k0 % p.k_inner, m0,
                                     k0 / p.k_inner);
                    tma_load_2d_pair(sB + stage * kBBytes, &map_b, &full[stage], k0, n0);
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
            const int m0 = (tile % p.num_m_tiles) * 256 + cta * 128;
            const int n0 = (tile / p.num_m_tiles) * BN;
            mbar_wait(&tfull[acc], aphase);
            tc_fence_after();
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
                epilogue_chunk(p, row, n0 + c * 32, r, rr);
            }
            tc_fence_before();
            mbar_arrive_leader(&tempty[acc]);
        }
    }
    tc_fence_before();
    cluster_sync_all();
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

template <int BN>
void set_smem_attr() {
    static bool done[64] = {};  // the attribute is per function per device
    int dev = 0;
    SPX_CUDA(cudaGetDevice(&dev));
    if (!done[dev & 63]) {
        SPX_CUDA(cudaFuncSetAttribute(gemm_bf16_tn_kernel<BN>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(gemm_smem_bytes<BN>())));
        done[dev & 63] = true;
    }
}

}  // namespace

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
    //   pair (cta_group::2) 256 x {256, 128} tiles and single-CTA 128 x {256, 128} tiles.
    // The single-CTA kernels stream 1.5-2x the operand bytes per MMA cycle (L2 -> SM bound).
    struct Cand { bool pair; int bn; double eff; };
    // efficiencies measured on B200 (tools/kbench.py gemm, K = 1536): pair-256 1358 TFLOP/s
    // at 4680x4608, pair-128 908, single-256 1237, single-128 1077
    static const Cand cands[] = {{true, 256, 1.0}, {true, 128, 0.65}, {false, 256, 0.88},
                                 {false, 128, 0.72}};
    static const int forced = [] {  // tuning override: SPX_GEMM_VARIANT=0..3 (index above)
        const char* e = std::getenv("SPX_GEMM_VARIANT");
        return e ? std::atoi(e) : -1;
    }();
    double best = 1e30;
    for (int ci = 0; ci < 4; ++ci) {
        const Cand& c = cands[ci];
        if (ops.N % 32 != 0) continue;
        const int64_t bm = c.pair ? 256 : 128;
        const int64_t tiles = ceil_div(static_cast<int64_t>(ops.M), bm) * ceil_div(ops.N, c.bn);
        const int64_t slots = c.pair ? sm_count / 2 : sm_count;
        const double t = static_cast<double>(ceil_div(tiles, slots)) * 128.0 * c.bn / c.eff;
        if ((forced < 0 && t < best) || forced == ci) {
            best = forced == ci ? -1.0 : t;
            plan->pair = c.pair;
            plan->bn = c.bn;
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
    if (plan->pair) {
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

void gemm_run(const GemmPlan& plan, cudaStream_t stream, const RopeLaunch* rope) {
    const GemmOperands& o = plan.ops;
    GemmParams p{};
    p.M = o.M;
    p.N = o.N;
    p.K = o.K;
    p.k_inner = o.k_inner;
    p.num_m_tiles = static_cast<int>(ceil_div(o.M, plan.pair ? 256 : kBM));
    p.num_n_tiles = static_cast<int>(ceil_div(o.N, plan.bn));
    p.out = o.out;
    p.ldo = o.out_row_stride;
    p.epi_mode = o.epi_mode;
    p.residual = o.residual;
    p.ldr = o.residual_row_stride;
    p.gate = o.gate;
    if (rope) {
        require(gemm_rope_fusable(plan, *rope), SPX_ERR_UNSUPPORTED,
                "gemm: rope epilogue needs 3C outputs, C % BN == 0, D % 32 == 0, no QK-norm");
        p.epi_mode = 2;
        p.rope = *rope;
    }
    static const int experiment = [] {
        const char* e = std::getenv("SPX_GEMM_EXPERIMENT");
        return e ? std::atoi(e) : 0;
    }();
    p.experiment = experiment;
    if (plan.pair && plan.bn == 256) {
        set_pair_smem_attr<256>();
        gemm_bf16_tn_pair_kernel<256><<<plan.grid, kThreads, gemm_pair_smem_bytes<256>(), stream>>>(
            plan.map_a, plan.map_b, p);
    } else if (plan.pair) {
        set_pair_smem_attr<128>();
        gemm_bf16_tn_pair_kernel<128><<<plan.grid, kThreads, gemm_pair_smem_bytes<128>(), stream>>>(
            plan.map_a, plan.map_b, p);
    } else if (plan.bn == 256) {
        set_smem_attr<256>();
        gemm_bf16_tn_kernel<256><<<plan.grid, kThreads, gemm_smem_bytes<256>(), stream>>>(
            plan.map_a, plan.map_b, p);
    } else {
        set_smem_attr<128>();
        gemm_bf16_tn_kernel<128><<<plan.grid, kThreads, gemm_smem_bytes<128>(), stream>>>(
            plan.map_a, plan.map_b, p);
    }
    SPX_CUDA_LAUNCH();
    count_launch();
}

}  // namespace spx
