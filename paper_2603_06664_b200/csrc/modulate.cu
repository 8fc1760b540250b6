// modulate.cu -- K1: the Wan block's adaLN modulation in front of the QKV projection,
//   x_in = LayerNorm(x) * (1 + scale) + shift          (non-affine LN over the model dim)
// and, with affine = 1, the affine LayerNorm in front of the cross-attention (Wan's norm3),
//   y = LayerNorm(x) * weight + bias                   (scale = weight, shift = bias)
// (a Wan-mode extension with no reference counterpart; the residual + gate after
// the output projection, x += gate * W_o o, is the O-GEMM's epi_mode 1 epilogue).
//
// HBM-bound: one read and one write of the (rows, C) bf16 activation. The rows stream into
// shared memory through the row pipeline (row_pipe.cuh); each lane owns the 16-byte vectors
// v = lane + 32 i of its warp's row; mean and biased variance come from two warp reductions
// over the registers (no second pass over memory).
#include <algorithm>

#include "common.hpp"
#include "kernels.hpp"
#include "row_pipe.cuh"
#include "sm100.cuh"

namespace spx {

using namespace sm100;

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Rows stream through shared memory (row_pipe.cuh: bulk copies of row blocks into a ring of
// stages, one persistent CTA per SM); each consumer warp normalises the rows of its stages from
// shared memory and stores them. shift / (1 + scale) are staged once per CTA.
template <int NV>
__global__ void __launch_bounds__(kPipeThreads, 1)
    ln_modulate_kernel(const bf16* __restrict__ x, bf16* __restrict__ y, int rows, int dim,
                       const float* __restrict__ shift, const float* __restrict__ scale,
                       float eps, int affine, int mod_from_kernel, const RowPipeShape sh) {
    extern __shared__ __align__(16) uint8_t smem_ln[];
    const int nvec = dim / 8;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_ln);
    float4* s_mod = reinterpret_cast<float4*>(smem_ln + 2 * kPipeMaxStages * sizeof(uint64_t));  // [nvec][4]
    uint8_t* ring = reinterpret_cast<uint8_t*>(s_mod + 4 * nvec);
    pdl_trigger();
    if (threadIdx.x == 0) row_pipe_init(bars, sh.stages);
    __syncthreads();
    if (threadIdx.x / 32 == kPipeWarps) {  // producer: x was written by the previous kernel
        pdl_wait();
        row_pipe_produce(reinterpret_cast<const uint8_t*>(x), static_cast<int64_t>(dim) * 2, rows, sh, ring, bars);
        return;
    }
    // constant modulation (uploaded weights) is staged before the PDL wait, overlapping the
    // previous kernel's tail; a per-step modulation written by a kernel (the Wan timestep
    // embedding) only after it. Either way the row reads are already streaming.
    if (mod_from_kernel) pdl_wait();
    const float one = affine ? 0.0f : 1.0f;
    for (int i = threadIdx.x; i < nvec * 4; i += kPipeWarps * 32) {
        const int v = i / 4, q = i % 4;
        const float* srcp = (q < 2 ? shift : scale) + v * 8 + (q & 1) * 4;
        float4 m = __ldg(reinterpret_cast<const float4*>(srcp));
        if (q >= 2) {  // the multiplier: 1 + scale (adaLN) or weight (affine LayerNorm)
            m.x += one;
            m.y += one;
            m.z += one;
            m.w += one;
        }
        s_mod[i] = m;
    }
    row_pipe_consumer_sync();
    if (!mod_from_kernel) pdl_wait();  // y may still be read by the previous kernel
    // two rows per step (a stage holds rb >= 2 rows of a C <= 2048 row): the modulation vectors
    // are read from shared memory once for both; packed f32x2 math, two-pass variance from the
    // registers; y = x a + b with a = rstd (1 + scale), b = shift - mean a
    row_pipe_consume(rows, sh, ring, bars, [&](int r0, int n, const uint8_t* stage, int lane) {
#pragma unroll 1
      for (int ri = 0; ri < n; ri += 2) {
        const bool two = ri + 1 < n;
        const uint4* s0 = reinterpret_cast<const uint4*>(stage + ri * sh.row_bytes);
        const uint4* s1 = reinterpret_cast<const uint4*>(stage + (two ? ri + 1 : ri) * sh.row_bytes);
        uint4 v0[NV], v1[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int c = lane + 32 * i;
            v0[i] = c < nvec ? lds128(s0 + c) : make_uint4(0, 0, 0, 0);
            v1[i] = c < nvec ? lds128(s1 + c) : make_uint4(0, 0, 0, 0);
        }
        float2 a0 = make_float2(0.0f, 0.0f), a1 = a0;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const uint32_t w0[4] = {v0[i].x, v0[i].y, v0[i].z, v0[i].w};
            const uint32_t w1[4] = {v1[i].x, v1[i].y, v1[i].z, v1[i].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                a0 = f2add(a0, make_float2(bf16_lo(w0[e]), bf16_hi(w0[e])));
                a1 = f2add(a1, make_float2(bf16_lo(w1[e]), bf16_hi(w1[e])));
            }
        }
        const float2 mean = make_float2(warp_sum(a0.x + a0.y) / static_cast<float>(dim),
                                         warp_sum(a1.x + a1.y) / static_cast<float>(dim));
        const float2 nm0 = make_float2(-mean.x, -mean.x), nm1 = make_float2(-mean.y, -mean.y);
        float2 q0 = make_float2(0.0f, 0.0f), q1 = q0;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            if (lane + 32 * i >= nvec) continue;
            const uint32_t w0[4] = {v0[i].x, v0[i].y, v0[i].z, v0[i].w};
            const uint32_t w1[4] = {v1[i].x, v1[i].y, v1[i].z, v1[i].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 d0 = f2add(make_float2(bf16_lo(w0[e]), bf16_hi(w0[e])), nm0);
                const float2 d1 = f2add(make_float2(bf16_lo(w1[e]), bf16_hi(w1[e])), nm1);
                q0 = f2fma(d0, d0, q0);
                q1 = f2fma(d1, d1, q1);
            }
        }
        const float rstd0 = rsqrtf(warp_sum(q0.x + q0.y) / static_cast<float>(dim) + eps);
        const float rstd1 = rsqrtf(warp_sum(q1.x + q1.y) / static_cast<float>(dim) + eps);
        const float2 rs0 = make_float2(rstd0, rstd0), rs1 = make_float2(rstd1, rstd1);
        uint4* d0 = reinterpret_cast<uint4*>(y + static_cast<int64_t>(r0 + ri) * dim);
        uint4* d1 = d0 + nvec;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int c = lane + 32 * i;
            if (c >= nvec) continue;
            // s_mod[c]: shift lo, shift hi, multiplier lo, multiplier hi (float4 each)
            const float4 sh0 = s_mod[c * 4], sh1 = s_mod[c * 4 + 1];
            const float4 sc0 = s_mod[c * 4 + 2], sc1 = s_mod[c * 4 + 3];
            const float2 shp[4] = {make_float2(sh0.x, sh0.y), make_float2(sh0.z, sh0.w),
                                   make_float2(sh1.x, sh1.y), make_float2(sh1.z, sh1.w)};
            const float2 scp[4] = {make_float2(sc0.x, sc0.y), make_float2(sc0.z, sc0.w),
                                   make_float2(sc1.x, sc1.y), make_float2(sc1.z, sc1.w)};
            const uint32_t w0[4] = {v0[i].x, v0[i].y, v0[i].z, v0[i].w};
            const uint32_t w1[4] = {v1[i].x, v1[i].y, v1[i].z, v1[i].w};
            uint32_t o0[4], o1[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 m0 = f2mul(scp[e], rs0), m1 = f2mul(scp[e], rs1);
                const float2 b0 = f2fma(nm0, m0, shp[e]), b1 = f2fma(nm1, m1, shp[e]);
                const float2 y0 = f2fma(make_float2(bf16_lo(w0[e]), bf16_hi(w0[e])), m0, b0);
                const float2 y1 = f2fma(make_float2(bf16_lo(w1[e]), bf16_hi(w1[e])), m1, b1);
                o0[e] = pack_bf16x2(y0.x, y0.y);
                o1[e] = pack_bf16x2(y1.x, y1.y);
            }
            stg128(d0 + c, make_uint4(o0[0], o0[1], o0[2], o0[3]));
            if (two) stg128(d1 + c, make_uint4(o1[0], o1[1], o1[2], o1[3]));
        }
      }
    });
}

template <int NV>
void launch_ln(dim3 grid, dim3 block, size_t smem, cudaStream_t s, const bf16* x, bf16* y, int r, int d,
               const float* shift, const float* scale, float eps, int af, int mk, const RowPipeShape& sh) {
    static bool done[64] = {};  // the attribute is per function per device
    int dev = 0;
    SPX_CUDA(cudaGetDevice(&dev));
    if (!done[dev & 63]) {
        SPX_CUDA(cudaFuncSetAttribute(ln_modulate_kernel<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      227 * 1024));
        done[dev & 63] = true;
    }
    launch_pdl(ln_modulate_kernel<NV>, grid, block, smem, s, x, y, r, d, shift, scale, eps, af, mk, sh);
}

}  // namespace

void ln_modulate_run(const bf16* x, bf16* y, int64_t rows, int64_t dim, const float* shift,
                     const float* scale, float eps, cudaStream_t s, bool affine,
                     bool mod_from_kernel) {
    require(rows >= 0 && dim > 0 && dim % 8 == 0 && dim <= 2048, SPX_ERR_SHAPE,
            "layernorm_modulate: dim must be a positive multiple of 8, <= 2048");
    require((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0 &&
                (reinterpret_cast<uintptr_t>(shift) & 15) == 0 &&
                (reinterpret_cast<uintptr_t>(scale) & 15) == 0,
            SPX_ERR_ALIGNMENT, "layernorm_modulate: 16-byte aligned buffers");
    if (rows == 0) return;
    const int nv = static_cast<int>((dim / 8 + 31) / 32);
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        SPX_CUDA(cudaGetDevice(&dev));
        sms = device_sm_count(dev);
    }
    const RowPipeShape sh = row_pipe_shape(rows, static_cast<uint32_t>(dim) * 2u, sms);
    const int64_t nblk = (rows + sh.rb - 1) / sh.rb;
    const dim3 grid(static_cast<unsigned>(std::min<int64_t>(nblk, sms)));
    const dim3 block(kPipeThreads);
    const size_t smem = 2 * kPipeMaxStages * sizeof(uint64_t) + static_cast<size_t>(dim / 8) * 4 * sizeof(float4) +
                        static_cast<size_t>(sh.stages) * sh.rb * sh.row_bytes;
    const int r = static_cast<int>(rows), d = static_cast<int>(dim);
    const int af = affine ? 1 : 0, mk = mod_from_kernel ? 1 : 0;
    switch (nv) {
        case 1: launch_ln<1>(grid, block, smem, s, x, y, r, d, shift, scale, eps, af, mk, sh); break;
        case 2: launch_ln<2>(grid, block, smem, s, x, y, r, d, shift, scale, eps, af, mk, sh); break;
        case 3: launch_ln<3>(grid, block, smem, s, x, y, r, d, shift, scale, eps, af, mk, sh); break;
        case 4: launch_ln<4>(grid, block, smem, s, x, y, r, d, shift, scale, eps, af, mk, sh); break;
        case 5: launch_ln<5>(grid, block, smem, s, x, y, r, d, shift, scale, eps, af, mk, sh); break;
        case 6: launch_ln<6>(grid, block, smem, s, x, y, r, d, shift, scale, eps, af, mk, sh); break;
        case 7: launch_ln<7>(grid, block, smem, s, x, y, r, d, shift, scale, eps, af, mk, sh); break;
        default: launch_ln<8>(grid, block, smem, s, x, y, r, d, shift, scale, eps, af, mk, sh); break;
    }
    SPX_CUDA_LAUNCH();
    count_launch();
}

}  // namespace spx
