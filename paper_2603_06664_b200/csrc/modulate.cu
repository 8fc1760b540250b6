// modulate.cu -- K1: the Wan block's adaLN modulation in front of the QKV projection,
//   x_in = LayerNorm(x) * (1 + scale) + shift          (non-affine LN over the model dim)
// (a Wan-mode extension with no reference counterpart; the residual + gate after
// the output projection, x += gate * W_o o, is the O-GEMM's epi_mode 1 epilogue).
//
// HBM-bound: one read and one write of the (rows, C) bf16 activation. One warp per token
// row; each lane owns the 16-byte vectors v = lane + 32 i of the row, all issued before any
// math; mean and biased variance come from two warp reductions over the registers (no second
// pass over memory); shift / scale are fp32 per column (L1/L2 resident across rows).
#include "common.hpp"
#include "kernels.hpp"
#include "sm100.cuh"

namespace spx {

using namespace sm100;

namespace {

constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int NV>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    ln_modulate_kernel(const bf16* __restrict__ x, bf16* __restrict__ y, int rows, int dim,
                       const float* __restrict__ shift, const float* __restrict__ scale,
                       float eps) {
    const int lane = threadIdx.x % 32;
    const int row = static_cast<int>(blockIdx.x) * kWarpsPerBlock + static_cast<int>(threadIdx.x / 32);
    if (row >= rows) return;
    const int nvec = dim / 8;
    const uint4* src = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(row) * dim);
    uint4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int c = lane + 32 * i;
        v[i] = c < nvec ? __ldg(src + c) : make_uint4(0, 0, 0, 0);
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 f = unpack_bf16x2(w[e]);
            s += f.x + f.y;
        }
    }
    const float mean = warp_sum(s) / static_cast<float>(dim);
    float q = 0.0f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        if (lane + 32 * i >= nvec) continue;
        const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 f = unpack_bf16x2(w[e]);
            q += (f.x - mean) * (f.x - mean) + (f.y - mean) * (f.y - mean);
        }
    }
    const float rstd = rsqrtf(warp_sum(q) / static_cast<float>(dim) + eps);
    uint4* dst = reinterpret_cast<uint4*>(y + static_cast<int64_t>(row) * dim);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int c = lane + 32 * i;
        if (c >= nvec) continue;
        const float4* sh = reinterpret_cast<const float4*>(shift + c * 8);
        const float4* sc = reinterpret_cast<const float4*>(scale + c * 8);
        const float4 sh0 = __ldg(sh), sh1 = __ldg(sh + 1), sc0 = __ldg(sc), sc1 = __ldg(sc + 1);
        const float shv[8] = {sh0.x, sh0.y, sh0.z, sh0.w, sh1.x, sh1.y, sh1.z, sh1.w};
        const float scv[8] = {sc0.x, sc0.y, sc0.z, sc0.w, sc1.x, sc1.y, sc1.z, sc1.w};
        const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
        uint32_t o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 f = unpack_bf16x2(w[e]);
            const float a = (f.x - mean) * rstd * (1.0f + scv[2 * e]) + shv[2 * e];
            const float b = (f.y - mean) * rstd * (1.0f + scv[2 * e + 1]) + shv[2 * e + 1];
            o[e] = pack_bf16x2(a, b);
        }
        dst[c] = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

}  // namespace

void ln_modulate_run(const bf16* x, bf16* y, int64_t rows, int64_t dim, const float* shift,
                     const float* scale, float eps, cudaStream_t s) {
    require(rows >= 0 && dim > 0 && dim % 8 == 0 && dim <= 2048, SPX_ERR_SHAPE,
            "layernorm_modulate: dim must be a positive multiple of 8, <= 2048");
    require((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0 &&
                (reinterpret_cast<uintptr_t>(shift) & 15) == 0 &&
                (reinterpret_cast<uintptr_t>(scale) & 15) == 0,
            SPX_ERR_ALIGNMENT, "layernorm_modulate: 16-byte aligned buffers");
    if (rows == 0) return;
    const int nv = static_cast<int>((dim / 8 + 31) / 32);
    const dim3 grid(static_cast<unsigned>((rows + kWarpsPerBlock - 1) / kWarpsPerBlock));
    const dim3 block(kWarpsPerBlock * 32);
    const int r = static_cast<int>(rows), d = static_cast<int>(dim);
    switch (nv) {
        case 1: ln_modulate_kernel<1><<<grid, block, 0, s>>>(x, y, r, d, shift, scale, eps); break;
        case 2: ln_modulate_kernel<2><<<grid, block, 0, s>>>(x, y, r, d, shift, scale, eps); break;
        case 3: ln_modulate_kernel<3><<<grid, block, 0, s>>>(x, y, r, d, shift, scale, eps); break;
        case 4: ln_modulate_kernel<4><<<grid, block, 0, s>>>(x, y, r, d, shift, scale, eps); break;
        case 5: ln_modulate_kernel<5><<<grid, block, 0, s>>>(x, y, r, d, shift, scale, eps); break;
        case 6: ln_modulate_kernel<6><<<grid, block, 0, s>>>(x, y, r, d, shift, scale, eps); break;
        case 7: ln_modulate_kernel<7><<<grid, block, 0, s>>>(x, y, r, d, shift, scale, eps); break;
        default: ln_modulate_kernel<8><<<grid, block, 0, s>>>(x, y, r, d, shift, scale, eps); break;
    }
    SPX_CUDA_LAUNCH();
    count_launch();
}

}  // namespace spx
