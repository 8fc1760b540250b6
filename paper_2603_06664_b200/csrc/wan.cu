// wan.cu -- the per-step pieces of the full Wan2.1 DiT block (the reference
// model is attention-only, so these are extensions with no reference counterpart,
// restated from Wan2.1's wan/modules/model.py -- the Self-Forcing generator's backbone):
//
//   timestep embedding  e  = W2 SiLU(W1 sinusoidal_256(t) + b1) + b2          (C)
//   time projection     e0 = Wp SiLU(e) + bp                                   (6, C)
//   per-layer modulation mod[l] = modulation_param[l] + e0                     (6, C):
//       shift_msa, scale_msa, gate_msa, shift_mlp, scale_mlp, gate_mlp
//
// They run once per denoise step (M = 1 matrix-vector products over 34 MB of weights: HBM
// bound, a few microseconds); t is read from a device array so that a captured step graph
// replays correctly. Also here: the counter-based normal generator that seeds the Wan-block
// weights on the device (2.8 GB at the Wan2.1-1.3B shape would take seconds on the host).
#include "common.hpp"
#include "kernels.hpp"
#include "sm100.cuh"

namespace spx {

using namespace sm100;

namespace {

// sinusoidal_embedding_1d(dim, t) (Wan2.1): half = dim / 2, f_j = 10000^(-j / half),
// x = [cos(t f_j) | sin(t f_j)], computed in float64 and cast to float32 (as Wan does)
__global__ void sinusoid_kernel(const float* __restrict__ tsteps, int step, int dim,
                                float* __restrict__ out) {
    pdl_trigger();
    pdl_wait();
    const int half = dim / 2;
    const double t = static_cast<double>(tsteps[step]);
    for (int j = threadIdx.x; j < half; j += blockDim.x) {
        const double f = pow(10000.0, -static_cast<double>(j) / static_cast<double>(half));
        double sn, cs;
        sincos(t * f, &sn, &cs);
        out[j] = static_cast<float>(cs);
        out[half + j] = static_cast<float>(sn);
    }
}

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

// y[n] = act_out(sum_k W[n][k] act_in(x[k]) + b[n]); one warp per output row, 16-byte
// weight loads, x staged in shared memory (fp32, K <= 8192)
__global__ void __launch_bounds__(256) gemv_kernel(const bf16* __restrict__ W,
                                                   const float* __restrict__ b,
                                                   const float* __restrict__ x,
                                                   float* __restrict__ y, int N, int K,
                                                   int silu_in, int silu_out) {
    extern __shared__ float s_x[];
    pdl_trigger();
    pdl_wait();
    for (int k = threadIdx.x; k < K; k += blockDim.x) s_x[k] = silu_in ? silu(x[k]) : x[k];
    __syncthreads();
    const int lane = threadIdx.x % 32;
    const int warps = static_cast<int>(gridDim.x) * (blockDim.x / 32);
    for (int n = static_cast<int>(blockIdx.x) * (blockDim.x / 32) + static_cast<int>(threadIdx.x / 32);
         n < N; n += warps) {
        const uint4* row = reinterpret_cast<const uint4*>(W + static_cast<int64_t>(n) * K);
        float acc = 0.0f;
        for (int v = lane; v < K / 8; v += 32) {
            const uint4 w = __ldg(row + v);
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = unpack_bf16x2(ws[e]);
                acc = fmaf(f.x, s_x[8 * v + 2 * e], acc);
                acc = fmaf(f.y, s_x[8 * v + 2 * e + 1], acc);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            const float r = acc + (b ? b[n] : 0.0f);
            y[n] = silu_out ? silu(r) : r;
        }
    }
}

// mod[l][i] = param[l][i] + e0[i % (6 C)] for every layer (i < layers * 6 C)
__global__ void mod_sum_kernel(const float* __restrict__ param, const float* __restrict__ e0,
                               float* __restrict__ mod, int64_t per_layer, int64_t total) {
    pdl_trigger();
    pdl_wait();
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        mod[i] = param[i] + e0[i % per_layer];
}

// counter-based N(0, 1): two splitmix64 draws per element, Box-Muller (cos branch)
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ float normal_at(uint64_t seed, int64_t i) {
    const uint64_t a = splitmix64(seed ^ (static_cast<uint64_t>(i) * 2u));
    const uint64_t b = splitmix64(seed ^ (static_cast<uint64_t>(i) * 2u + 1u));
    const double u1 = (static_cast<double>(a >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
    const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;
    return static_cast<float>(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
}

__global__ void fill_normal_bf16_kernel(bf16* out, int64_t n, uint64_t seed, float scale,
                                        float offset) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = __float2bfloat16_rn(offset + scale * normal_at(seed, i));
}

__global__ void fill_normal_f32_kernel(float* out, int64_t n, uint64_t seed, float scale,
                                       float offset) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = offset + scale * normal_at(seed, i);
}

}  // namespace

void wan_time_embedding_run(const WanTimeEmbed& te, int step, cudaStream_t s) {
    require(te.freq_dim % 16 == 0 && te.freq_dim <= 8192 && te.dim % 8 == 0 && te.dim <= 8192,
            SPX_ERR_SHAPE, "time embedding: freq_dim and dim must be multiples of 16 / 8, <= 8192");
    launch_pdl(sinusoid_kernel, dim3(1), dim3(128), 0, s, te.tsteps, step, te.freq_dim, te.sinus);
    count_launch();
    auto gemv = [&](const bf16* W, const float* b, const float* x, float* y, int N, int K, int si,
                    int so) {
        const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(N, 8), 148 * 4));
        launch_pdl(gemv_kernel, dim3(blocks), dim3(256), static_cast<size_t>(K) * 4, s, W, b, x, y, N, K,
                   si, so);
        count_launch();
    };
    gemv(te.w1, te.b1, te.sinus, te.h1, te.dim, te.freq_dim, 0, 1);  // Linear + SiLU
    gemv(te.w2, te.b2, te.h1, te.e, te.dim, te.dim, 0, 0);           // Linear
    gemv(te.wp, te.bp, te.e, te.e0, 6 * te.dim, te.dim, 1, 0);       // SiLU + Linear
    const int64_t per = 6 * static_cast<int64_t>(te.dim);
    const int64_t total = per * te.layers;
    launch_pdl(mod_sum_kernel, dim3(static_cast<unsigned>(std::min<int64_t>(ceil_div(total, 256), 592))),
               dim3(256), 0, s, te.mod_param, te.e0, te.mod, per, total);
    count_launch();
    SPX_CUDA_LAUNCH();
}

void gemv_run(const bf16* W, const float* b, const float* x, float* y, int N, int K, bool silu_in,
              bool silu_out, cudaStream_t s) {
    require(K % 8 == 0 && K <= 8192 && N >= 1, SPX_ERR_SHAPE, "gemv: K must be a multiple of 8, <= 8192");
    const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(N, 8), 148 * 4));
    launch_pdl(gemv_kernel, dim3(blocks), dim3(256), static_cast<size_t>(K) * 4, s, W, b, x, y, N, K,
               silu_in ? 1 : 0, silu_out ? 1 : 0);
    SPX_CUDA_LAUNCH();
    count_launch();
}

void fill_normal_bf16_run(bf16* out, int64_t n, uint64_t seed, float scale, float offset,
                          cudaStream_t s) {
    if (n <= 0) return;
    fill_normal_bf16_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(n, 256), 148 * 16)), 256, 0,
                              s>>>(out, n, seed, scale, offset);
    SPX_CUDA_LAUNCH();
    count_launch();
}

void fill_normal_f32_run(float* out, int64_t n, uint64_t seed, float scale, float offset,
                         cudaStream_t s) {
    if (n <= 0) return;
    fill_normal_f32_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(n, 256), 148 * 16)), 256, 0,
                             s>>>(out, n, seed, scale, offset);
    SPX_CUDA_LAUNCH();
    count_launch();
}

}  // namespace spx
