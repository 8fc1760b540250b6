// gemm_ln.cu -- the Wan-mode output projection fused with the next layer's adaLN input
// (north_star item 4: adaLN-modulation / residual fusion in the projection epilogues):
//
//   x_new = x + gate * (o W_o^T + b)                  the gated residual (gemm.cu epi_mode 1)
//   x_mod = LN(x_new) * mul + add                      K1 of the next layer: mul = 1 + scale,
//                                                      add = shift (adaLN), or weight / bias
//
// A LayerNorm row spans all C = 1536 columns, so a cluster of 3 CTAs owns 128 full rows: CTA c
// of the cluster computes columns [512 c, 512 c + 512) with two N = 256 MMAs per k-step into
// all 512 TMEM columns (one tile per CTA: 3 x ceil(M / 128) CTAs, 111 at the Wan chunk).
//   warp 0      TMA producer: A box 32 x 128, B two boxes 32 x 256 (SWIZZLE_64B: 4 stages of
//               40 KB keep ~160 KB of operands in flight)
//   warp 1      single-thread tcgen05.mma issuer
//   warp 2      TMEM allocator
//   warps 4-11  epilogue, two per TMEM lane quarter (256 columns each):
//     1. the residual tile (128 x 512 bf16) is TMA-loaded into the drained pipeline buffers;
//        x_new = residual + gate (acc + bias) is formed in place, rounded to bf16 (exactly the
//        values the unfused epilogue stores), row sums accumulated
//     2. row means: per-CTA partial sums combined over the cluster through DSMEM; then the
//        squared deviations the same way (two passes, as K1 does), rstd
//     3. x_new TMA-stored; the tile is overwritten in place by x_mod and TMA-stored again
// The K1 launch of the next layer (a one-wave, latency-bound 28.8 MB pass) disappears.
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "common.hpp"
#include "kernels.hpp"
#include "sm100.cuh"
#include "tma.hpp"

namespace spx {

using namespace sm100;

namespace {

constexpr int kLnCluster = 3;
constexpr int kLnCols = 512;                     // columns per CTA
constexpr int kLnC = kLnCluster * kLnCols;       // the model dim this kernel serves
constexpr int kLnBM = 128;
constexpr int kLnBK = 32;                        // SWIZZLE_64B boxes
constexpr int kLnStages = 4;
constexpr uint32_t kLnABytes = kLnBM * kLnBK * 2;        // 8 KB
constexpr uint32_t kLnBBytes = kLnCols * kLnBK * 2;      // 32 KB (two 256-row boxes)
constexpr uint32_t kLnStageBytes = kLnABytes + kLnBBytes;
constexpr uint32_t kLnTileBytes = kLnBM * kLnCols * 2;   // 128 KB: the residual / x_new / x_mod tile
constexpr uint32_t kLnPipeBytes = kLnStages * kLnStageBytes;  // 160 KB
static_assert(kLnTileBytes <= kLnPipeBytes, "the tile reuses the drained pipeline buffers");
constexpr uint32_t kLnOffBar = kLnPipeBytes;
constexpr uint32_t kLnOffStats = kLnOffBar + 128;
constexpr uint32_t kLnOffVec = kLnOffStats + 4 * 128 * 4;  // [4][512] fp32: bias, gate, mul, add
constexpr size_t kLnSmem = 1024 + kLnOffVec + 4 * kLnCols * 4;
constexpr int kLnThreads = 384;

struct LnParams {
    int M, K, k_inner;
    const float* bias;   // [C] or null
    const float* gate;   // [C] or null (1)
    const float* mul;    // [C]: scale (adaLN: multiplier 1 + scale) or weight (affine)
    const float* add;    // [C]: shift or bias
    float one;           // 1 (adaLN) or 0 (affine)
    float eps;
    unsigned long long* span;
    long long* trace;  // SPX_GEMM_EXPERIMENT=8 (profiling): per-CTA phase marks [cta][16]
};

__device__ __forceinline__ void ln_mark(const LnParams& p, int k) {
    if (p.trace && blockIdx.x < 1024) p.trace[blockIdx.x * 64 + k] = clock64();
}

__global__ void __cluster_dims__(kLnCluster, 1, 1) __launch_bounds__(kLnThreads, 1)
    gemm_ln_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_res, const __grid_constant__ CUtensorMap map_out,
                   const __grid_constant__ CUtensorMap map_out2, const LnParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kLnOffBar);  // [kLnStages]
    uint64_t* empty = full + kLnStages;                               // [kLnStages]
    uint64_t* tfull = empty + kLnStages;
    uint64_t* res_full = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(res_full + 1);
    float* st_part = reinterpret_cast<float*>(smem + kLnOffStats);  // [2][128]: the two column halves
    float* st_sum = st_part + 256;                                  // [128]: this CTA's row sums
    float* st_sq = st_sum + 128;                                    // [128]: its squared deviations
    uint8_t* tile = smem;  // [8 boxes][128 rows][128 B] (SWIZZLE_128B), after the main loop
    float* s_vec = reinterpret_cast<float*>(smem + kLnOffVec);  // this CTA's 512 columns of each vector

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t crank = cluster_ctarank();
    const int m0 = static_cast<int>(blockIdx.x / kLnCluster) * kLnBM;
    const int n0 = static_cast<int>(crank) * kLnCols;
    const int num_kt = p.K / kLnBK;
    pdl_trigger();
    span_begin(p.span);
    if (threadIdx.x == 0) ln_mark(p, 0);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&map_a);
        tma_prefetch_desc(&map_b);
        tma_prefetch_desc(&map_res);
        tma_prefetch_desc(&map_out);
        tma_prefetch_desc(&map_out2);
        for (int s = 0; s < kLnStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(res_full, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();  // the A operand (attention output) and the residual were written earlier
    if (threadIdx.x == 0) ln_mark(p, 1);

    if (warp == 0) {
        if (lane == 0) {
            // the residual tile into L2 while the main loop runs (its TMA load after the loop
            // then hits L2)
            for (int b = 0; b < kLnCols / 64; ++b)
                asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(
                                 reinterpret_cast<uint64_t>(&map_res)),
                             "r"(n0 + b * 64), "r"(m0)
                             : "memory");
            for (int kt = 0; kt < num_kt; ++kt) {
                const int s = kt % kLnStages;
                mbar_wait(&empty[s], ((kt / kLnStages) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], kLnStageBytes);
                const int k0 = kt * kLnBK;
                uint8_t* st = smem + s * kLnStageBytes;
                tma_load_3d(st, &map_a, &full[s], k0 % p.k_inner, m0, k0 / p.k_inner);
                tma_load_2d(st + kLnABytes, &map_b, &full[s], k0, n0);
                tma_load_2d(st + kLnABytes + kLnBBytes / 2, &map_b, &full[s], k0, n0 + 256);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        const bool issuer = elect_one();
        constexpr uint32_t idesc = make_idesc_bf16(kLnBM, 256, false, false);
        for (int kt = 0; kt < num_kt; ++kt) {
            const int s = kt % kLnStages;
            mbar_wait(&full[s], (kt / kLnStages) & 1);
            tc_fence_after();
            const uint32_t a = smem_u32(smem + s * kLnStageBytes);
            const uint32_t b = a + kLnABytes;
            if (issuer) {
#pragma unroll
                for (int k = 0; k < kLnBK / 16; ++k) {
                    const uint64_t da = make_desc_sw64(a + k * 32);
                    umma_bf16_ss(tmem_base, da, make_desc_sw64(b + k * 32), idesc, (kt | k) != 0);
                    umma_bf16_ss(tmem_base + 256, da, make_desc_sw64(b + kLnBBytes / 2 + k * 32), idesc,
                                 (kt | k) != 0);
                }
                umma_commit(&empty[s]);
            }
            __syncwarp();
        }
        if (issuer) umma_commit(tfull);
        __syncwarp();
    } else if (warp >= 4) {
        const int ew = warp % 4;          // TMEM lane quarter
        const int h = (warp - 4) / 4;     // column half: CTA columns [256 h, 256 h + 256)
        const int r = ew * 32 + lane;     // row in the tile == TMEM lane
        const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16);
        // the per-column vectors of this CTA's 512 columns into shared memory while the main
        // loop runs: bias, gate (1 when absent), the LN multiplier (one + mul), add
        for (int i = static_cast<int>(threadIdx.x) - 128; i < 4 * (kLnCols / 4); i += 256) {
            const int v = i / (kLnCols / 4), c4 = (i % (kLnCols / 4)) * 4;
            const float* src = v == 0 ? p.bias : v == 1 ? p.gate : v == 2 ? p.mul : p.add;
            float4 x = src ? __ldg(reinterpret_cast<const float4*>(src + n0 + c4))
                           : (v == 1 ? make_float4(1.0f, 1.0f, 1.0f, 1.0f) : make_float4(0.0f, 0.0f, 0.0f, 0.0f));
            if (v == 2) {
                x.x += p.one;
                x.y += p.one;
                x.z += p.one;
                x.w += p.one;
            }
            reinterpret_cast<float4*>(s_vec)[i] = x;
        }
        // row r's 16-byte unit (8 columns) at CTA column col, as the SWIZZLE_128B TMA boxes lay
        // the tile out: box col / 64, row r, unit ((col % 64) / 8) ^ (r % 8)
        auto unit = [&](int col) -> uint4* {
            const int bx = col >> 6, u = (col & 63) >> 3;
            return reinterpret_cast<uint4*>(tile + bx * (kLnBM * 128) + r * 128 + ((u ^ (r & 7)) << 4));
        };
        mbar_wait(tfull, 0);  // the accumulator is complete: every MMA has read its operands
        tc_fence_after();
        if (threadIdx.x == 128) {  // the residual tile (L2-prefetched) into the drained pipeline buffers
            ln_mark(p, 2);
            mbar_arrive_expect_tx(res_full, kLnTileBytes);
#pragma unroll 1
            for (int b = 0; b < kLnCols / 64; ++b)
                tma_load_2d(tile + b * (kLnBM * 128), &map_res, res_full, n0 + b * 64, m0);
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");  // the vectors are staged
        mbar_wait(res_full, 0);
        if (threadIdx.x == 128) ln_mark(p, 3);
        // ---- 1. x_new = residual + gate (acc + bias), bf16, in place; row sums ----
        float s1a = 0.0f, s1b = 0.0f;
#pragma unroll 1
        for (int c = 0; c < 256 / 32; ++c) {
            const int col = h * 256 + c * 32;  // CTA column of the slice
            uint32_t acc[32];
            tmem_ld32(t_row + col, acc);  // in flight while the residual units are read
            uint4 rv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) rv[q] = *unit(col + q * 8);
            tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t rw[4] = {rv[q].x, rv[q].y, rv[q].z, rv[q].w};
                const float4 b0 = *reinterpret_cast<const float4*>(s_vec + col + q * 8);
                const float4 b1 = *reinterpret_cast<const float4*>(s_vec + col + q * 8 + 4);
                const float4 g0 = *reinterpret_cast<const float4*>(s_vec + kLnCols + col + q * 8);
                const float4 g1 = *reinterpret_cast<const float4*>(s_vec + kLnCols + col + q * 8 + 4);
                const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
                uint32_t ow[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 rs = unpack_bf16x2(rw[e]);
                    const int j = q * 8 + e * 2;
                    const float f0 = __uint_as_float(acc[j]) + bb[2 * e];
                    const float f1 = __uint_as_float(acc[j + 1]) + bb[2 * e + 1];
                    ow[e] = pack_bf16x2(rs.x + gg[2 * e] * f0, rs.y + gg[2 * e + 1] * f1);
                    const float2 v = unpack_bf16x2(ow[e]);
                    s1a += v.x;
                    s1b += v.y;
                }
                *unit(col + q * 8) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
            }
        }
        st_part[h * 128 + r] = s1a + s1b;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (h == 0) st_sum[r] = st_part[r] + st_part[128 + r];
        if (threadIdx.x == 128) ln_mark(p, 4);
    }
    // ---- 2. row statistics over the cluster (every thread of the 3 CTAs joins the barriers) ----
    cluster_sync_all();  // #1: every CTA's row sums are in its shared memory
    if (threadIdx.x == 128) ln_mark(p, 5);
    float mean = 0.0f, rstd = 0.0f;
    if (warp >= 4) {
        const int ew = warp % 4, h = (warp - 4) / 4, r = ew * 32 + lane;
        auto unit = [&](int col) -> uint4* {
            const int bx = col >> 6, u = (col & 63) >> 3;
            return reinterpret_cast<uint4*>(tile + bx * (kLnBM * 128) + r * 128 + ((u ^ (r & 7)) << 4));
        };
        float part[kLnCluster];
#pragma unroll
        for (int c = 0; c < kLnCluster; ++c) part[c] = ld_dsmem_f32(peer_smem_addr(st_sum + r, static_cast<uint32_t>(c)));
        mean = (part[0] + part[1] + part[2]) * (1.0f / static_cast<float>(kLnC));
        float s2[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 4
        for (int c = 0; c < 256 / 8; ++c) {
            const uint4 v = *unit(h * 256 + c * 8);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 x = unpack_bf16x2(w[e]);
                const float d0 = x.x - mean, d1 = x.y - mean;
                s2[e] = fmaf(d0, d0, fmaf(d1, d1, s2[e]));
            }
        }
        st_part[h * 128 + r] = (s2[0] + s2[1]) + (s2[2] + s2[3]);
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (h == 0) st_sq[r] = st_part[r] + st_part[128 + r];
    }
    cluster_sync_all();  // #2: every CTA's squared deviations are in its shared memory
    if (threadIdx.x == 128) ln_mark(p, 6);
    if (warp >= 4) {
        const int ew = warp % 4, h = (warp - 4) / 4, r = ew * 32 + lane;
        auto unit = [&](int col) -> uint4* {
            const int bx = col >> 6, u = (col & 63) >> 3;
            return reinterpret_cast<uint4*>(tile + bx * (kLnBM * 128) + r * 128 + ((u ^ (r & 7)) << 4));
        };
        float part[kLnCluster];
#pragma unroll
        for (int c = 0; c < kLnCluster; ++c) part[c] = ld_dsmem_f32(peer_smem_addr(st_sq + r, static_cast<uint32_t>(c)));
        rstd = rsqrtf((part[0] + part[1] + part[2]) * (1.0f / static_cast<float>(kLnC)) + p.eps);
        // ---- 3. x_new out, then x_mod in place and out ----
        fence_proxy_async_smem();  // the generic-proxy tile writes -> the TMA store's reads
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (threadIdx.x == 128) {
#pragma unroll 1
            for (int b = 0; b < kLnCols / 64; ++b) tma_store_2d(&map_out, tile + b * (kLnBM * 128), n0 + b * 64, m0);
            bulk_commit();
            bulk_wait_read_all();  // the tile may be overwritten
            ln_mark(p, 7);
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
#pragma unroll 2
        for (int c = 0; c < 256 / 8; ++c) {
            const int col = h * 256 + c * 8;
            const uint4 v = *unit(col);
            const float4 m0v = *reinterpret_cast<const float4*>(s_vec + 2 * kLnCols + col);
            const float4 m1v = *reinterpret_cast<const float4*>(s_vec + 2 * kLnCols + col + 4);
            const float4 a0v = *reinterpret_cast<const float4*>(s_vec + 3 * kLnCols + col);
            const float4 a1v = *reinterpret_cast<const float4*>(s_vec + 3 * kLnCols + col + 4);
            const float mm[8] = {m0v.x, m0v.y, m0v.z, m0v.w, m1v.x, m1v.y, m1v.z, m1v.w};
            const float aa[8] = {a0v.x, a0v.y, a0v.z, a0v.w, a1v.x, a1v.y, a1v.z, a1v.w};
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 x = unpack_bf16x2(w[e]);
                o[e] = pack_bf16x2(fmaf((x.x - mean) * rstd, mm[2 * e], aa[2 * e]),
                                   fmaf((x.y - mean) * rstd, mm[2 * e + 1], aa[2 * e + 1]));
            }
            *unit(col) = make_uint4(o[0], o[1], o[2], o[3]);
        }
        fence_proxy_async_smem();
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (threadIdx.x == 128) {
#pragma unroll 1
            for (int b = 0; b < kLnCols / 64; ++b) tma_store_2d(&map_out2, tile + b * (kLnBM * 128), n0 + b * 64, m0);
            bulk_commit();
            bulk_wait_all();  // the shared memory stays valid until the stores have read it
            ln_mark(p, 8);
        }
    }
    cluster_sync_all();  // #3: no CTA leaves while a peer may still read its statistics
    if (threadIdx.x == 128) ln_mark(p, 9);
    span_end(p.span);
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

int ln_max_active_clusters() {
    static std::mutex mu;
    static std::map<int, int> cache;
    int dev = 0;
    SPX_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    SPX_CUDA(cudaFuncSetAttribute(gemm_ln_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kLnSmem)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kLnCluster * 64);
    cfg.blockDim = dim3(kLnThreads);
    cfg.dynamicSmemBytes = kLnSmem;
    int n = 0;
    SPX_CUDA(cudaOccupancyMaxActiveClusters(&n, gemm_ln_kernel, &cfg));
    cache[dev] = n;
    return n;
}

}  // namespace

bool gemm_ln_supported(const GemmOperands& ops) {
    return ops.N == kLnC && ops.epi_mode == 1 && ops.residual != nullptr && ops.K % kLnBK == 0 &&
           ops.k_inner % kLnBK == 0 && ops.out_row_stride == kLnC && ops.residual_row_stride == kLnC &&
           (reinterpret_cast<uintptr_t>(ops.out) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(ops.residual) & 15) == 0 &&
           (!ops.bias || (reinterpret_cast<uintptr_t>(ops.bias) & 15) == 0) &&
           (!ops.gate || (reinterpret_cast<uintptr_t>(ops.gate) & 15) == 0);
}

void gemm_ln_plan(GemmLnPlan* plan, const GemmOperands& ops, bf16* out2, const float* mul, const float* add,
                  bool affine, float eps) {
    require(gemm_ln_supported(ops), SPX_ERR_UNSUPPORTED,
            "gemm_ln: N must be 1536 with the residual epilogue and 16-byte aligned buffers");
    require(out2 && mul && add, SPX_ERR_CONFIG, "gemm_ln: null output / modulation");
    require((reinterpret_cast<uintptr_t>(out2) & 15) == 0 && (reinterpret_cast<uintptr_t>(mul) & 15) == 0 &&
                (reinterpret_cast<uintptr_t>(add) & 15) == 0,
            SPX_ERR_ALIGNMENT, "gemm_ln: 16-byte aligned modulation and output");
    plan->ops = ops;
    plan->out2 = out2;
    plan->mul = mul;
    plan->add = add;
    plan->affine = affine;
    plan->eps = eps;
    char err[256];
    {
        const uint64_t dims[3] = {static_cast<uint64_t>(ops.k_inner), static_cast<uint64_t>(ops.M),
                                  static_cast<uint64_t>(ops.groups)};
        const uint64_t strides[2] = {static_cast<uint64_t>(ops.a_row_stride) * 2,
                                     static_cast<uint64_t>(ops.a_group_stride) * 2};
        const uint32_t box[3] = {kLnBK, kLnBM, 1};
        require(make_tma_map_bf16_swizzle(&plan->map_a, ops.a, 3, dims, strides, box, 64, err, sizeof(err)),
                SPX_ERR_ALIGNMENT, err);
    }
    {
        const uint64_t dims[2] = {static_cast<uint64_t>(ops.K), static_cast<uint64_t>(ops.N)};
        const uint64_t strides[1] = {static_cast<uint64_t>(ops.b_row_stride) * 2};
        const uint32_t box[2] = {kLnBK, 256};
        require(make_tma_map_bf16_swizzle(&plan->map_b, ops.b, 2, dims, strides, box, 64, err, sizeof(err)),
                SPX_ERR_ALIGNMENT, err);
    }
    const uint64_t dims[2] = {static_cast<uint64_t>(kLnC), static_cast<uint64_t>(ops.M)};
    const uint64_t strides[1] = {static_cast<uint64_t>(kLnC) * 2};
    const uint32_t box[2] = {64, kLnBM};
    require(make_tma_map_bf16(&plan->map_res, ops.residual, 2, dims, strides, box, err, sizeof(err)),
            SPX_ERR_ALIGNMENT, err);
    require(make_tma_map_bf16(&plan->map_out, ops.out, 2, dims, strides, box, err, sizeof(err)), SPX_ERR_ALIGNMENT,
            err);
    require(make_tma_map_bf16(&plan->map_out2, out2, 2, dims, strides, box, err, sizeof(err)), SPX_ERR_ALIGNMENT,
            err);
    const int64_t tiles = ceil_div(static_cast<int64_t>(ops.M), kLnBM);
    plan->grid = static_cast<int>(tiles) * kLnCluster;
    // every cluster resident at once (a second wave would serialise the whole epilogue), and
    // enough rows to keep at least half the SMs busy: a 128 x 512 tile per CTA is 2.7 x the
    // main loop of the unfused 128 x 192 tiles, which only pays when the grid is full
    // (measured: the Wan chunk's 37 row tiles on 111 SMs; per-rank shapes stay unfused)
    int dev = 0;
    SPX_CUDA(cudaGetDevice(&dev));
    plan->ok = tiles <= ln_max_active_clusters() && 2 * tiles * kLnCluster >= device_sm_count(dev);
}

void gemm_ln_run(const GemmLnPlan& plan, cudaStream_t stream) {
    require(plan.ok, SPX_ERR_UNSUPPORTED, "gemm_ln: not all clusters fit on the device at once");
    const GemmOperands& o = plan.ops;
    LnParams p{};
    p.M = o.M;
    p.K = o.K;
    p.k_inner = o.k_inner;
    p.bias = o.bias;
    p.gate = o.gate;
    p.mul = plan.mul;
    p.add = plan.add;
    p.one = plan.affine ? 0.0f : 1.0f;
    p.eps = plan.eps;
    p.span = span_slot();
    static const bool trace = [] {
        const char* e = std::getenv("SPX_GEMM_EXPERIMENT");
        return e && std::atoi(e) == 8;
    }();
    p.trace = trace ? gemm_trace_buffer() : nullptr;
    static bool done[64] = {};
    int dev = 0;
    SPX_CUDA(cudaGetDevice(&dev));
    if (!done[dev & 63]) {
        SPX_CUDA(cudaFuncSetAttribute(gemm_ln_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kLnSmem)));
        done[dev & 63] = true;
    }
    launch_pdl(gemm_ln_kernel, dim3(static_cast<unsigned>(plan.grid)), dim3(kLnThreads), kLnSmem, stream,
               plan.map_a, plan.map_b, plan.map_res, plan.map_out, plan.map_out2, p);
    SPX_CUDA_LAUNCH();
    count_launch();
}

}  // namespace spx
