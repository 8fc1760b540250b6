// misc.cu -- byte movers for the collectives and the fp32 SIMT debug kernels (Kd).
//
// copy_box: the per-(source, destination) chunk move of all_to_all / fused_all_to_all /
// all_gather (proj/src/collectives.cpp:180-276) as a strided 4-D box copy, templated on the
// element width so fp64 payloads move bit-exactly (the reference's tests are fp64).
//
// naive_*: fp32-accumulating SIMT kernels used only by the tests as the GPU-side oracle at
// shapes the CPU oracle cannot reach in seconds.
#include "common.hpp"
#include "kernels.hpp"
#include "sm100.cuh"

namespace spx {

using namespace sm100;

namespace {

// PEER barrier (see kernels.hpp): one thread per rank.
// signal + wait in one 1-warp launch, chained with PDL: it starts during the previous
// kernel's tail, griddepcontrol.wait makes that kernel's stores (peer stores included)
// complete before the release, and the next kernel's prologue overlaps the spin
__global__ void peer_barrier_kernel(PeerFlags f, uint64_t* my_flags, int world, int my_rank, int slot,
                                    uint64_t timeout_ns, int* error_word) {
    pdl_trigger();
    pdl_wait();
    const int r = threadIdx.x;
    // this slot's epoch lives on the device (after the shared [slots][P] flag words), so that
    // the launch parameters are the same on every call and a captured CUDA graph replays it
    uint64_t* my_epoch = my_flags + kPeerSlots * world + slot;
    uint64_t epoch = 0;
    if (r == 0) epoch = *my_epoch + 1;
    epoch = __shfl_sync(0xffffffffu, epoch, 0);
    if (r < world) {
        uint64_t* dst = f.rank_flags[r] + slot * world + my_rank;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(epoch) : "memory");
    }
    __syncwarp();
    // an earlier barrier of this engine already timed out: do not wait again
    const bool failed = *reinterpret_cast<volatile int*>(error_word) != 0;
    if (r < world && !failed) {
        // bounded spin (the reference raises CollectiveError instead of hanging on a rank that
        // never enters, collectives.cpp:42-52, 88-102): past the deadline the wait gives up,
        // records the missing rank in the host-visible error word and lets the stream drain;
        // the host turns the word into SPX_ERR_COLLECTIVE at the next synchronisation
        const uint64_t* src = my_flags + slot * world + r;
        const uint64_t t0 = globaltimer_ns();
        uint64_t v = 0;
        for (uint32_t it = 0;; ++it) {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(src) : "memory");
            if (v >= epoch) break;
            if ((it & 255u) == 255u && globaltimer_ns() - t0 > timeout_ns) {
                atomicExch(error_word, 1 + r);
                break;
            }
            __nanosleep(64);
        }
    }
    __syncwarp();
    if (r == 0) *my_epoch = epoch;
}


template <typename T>
__global__ void copy_box_kernel(T* __restrict__ dst, const T* __restrict__ src, Box4 box,
                                int64_t total) {
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t rem = idx;
        int64_t so = 0, doff = 0;
#pragma unroll
        for (int a = 3; a >= 0; --a) {
            const int64_t c = rem % box.ext[a];
            rem /= box.ext[a];
            so += c * box.src_str[a];
            doff += c * box.dst_str[a];
        }
        dst[doff] = src[so];
    }
}

struct alignas(16) V16 {
    uint4 v;
};

__global__ void naive_gemm_kernel(const bf16* __restrict__ a, const bf16* __restrict__ b,
                                  float* __restrict__ out, int M, int N, int K) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    const int m = blockIdx.y;
    if (n >= N || m >= M) return;
    float acc = 0.0f;
    for (int k = 0; k < K; ++k)
        acc += __bfloat162float(a[static_cast<int64_t>(m) * K + k]) *
               __bfloat162float(b[static_cast<int64_t>(n) * K + k]);
    out[static_cast<int64_t>(m) * N + n] = acc;
}

// one block per (query row, head); two passes over the keys (max, then weights and values)
__global__ void naive_attention_kernel(const bf16* __restrict__ q, const bf16* __restrict__ k,
                                       const bf16* __restrict__ v, float* __restrict__ out,
                                       int sq, int skv, int heads, int D) {
    extern __shared__ float sh[];
    float* qs = sh;           // D
    float* w = sh + D;        // skv
    __shared__ float red[32];
    const int i = blockIdx.x;
    const int h = blockIdx.y;
    const int b = blockIdx.z;
    const int64_t qoff = ((static_cast<int64_t>(b) * sq + i) * heads + h) * D;
    for (int d = threadIdx.x; d < D; d += blockDim.x) qs[d] = __bfloat162float(q[qoff + d]);
    __syncthreads();
    const float scale = rsqrtf(static_cast<float>(D));
    float mx = -INFINITY;
    for (int t = threadIdx.x; t < skv; t += blockDim.x) {
        const int64_t koff = ((static_cast<int64_t>(b) * skv + t) * heads + h) * D;
        float dot = 0.0f;
        for (int d = 0; d < D; ++d) dot += qs[d] * __bfloat162float(k[koff + d]);
        w[t] = dot * scale;
        mx = fmaxf(mx, dot * scale);
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        float m2 = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : -INFINITY;
        for (int o = 16; o > 0; o >>= 1) m2 = fmaxf(m2, __shfl_xor_sync(0xffffffffu, m2, o));
        if (threadIdx.x == 0) red[0] = m2;
    }
    __syncthreads();
    mx = red[0];
    __syncthreads();
    float z = 0.0f;
    for (int t = threadIdx.x; t < skv; t += blockDim.x) {
        const float e = expf(w[t] - mx);
        w[t] = e;
        z += e;
    }
    for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = z;
    __syncthreads();
    if (threadIdx.x < 32) {
        float z2 = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0f;
        for (int o = 16; o > 0; o >>= 1) z2 += __shfl_xor_sync(0xffffffffu, z2, o);
        if (threadIdx.x == 0) red[0] = z2;
    }
    __syncthreads();
    const float inv = 1.0f / red[0];
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
        float acc = 0.0f;
        for (int t = 0; t < skv; ++t) {
            const int64_t voff = ((static_cast<int64_t>(b) * skv + t) * heads + h) * D;
            acc += w[t] * __bfloat162float(v[voff + d]);
        }
        out[qoff + d] = acc * inv;
    }
}

}  // namespace

void peer_barrier_run(const PeerFlags& f, uint64_t* my_flags, int world, int my_rank, int slot,
                      uint64_t timeout_ns, int* error_word, cudaStream_t s) {
    launch_pdl(peer_barrier_kernel, dim3(1), dim3(32), 0, s, f, my_flags, world, my_rank, slot,
               timeout_ns, error_word);
    count_launch();
}


void copy_box_run(void* dst, const void* src, const Box4& box, int elem_bytes, cudaStream_t s) {
    const int64_t total = box.ext[0] * box.ext[1] * box.ext[2] * box.ext[3];
    if (total == 0) return;
    const int threads = 256;
    const int64_t want = ceil_div(total, threads);
    const unsigned blocks = static_cast<unsigned>(want < 148 * 16 ? want : 148 * 16);
    switch (elem_bytes) {
        case 1:
            copy_box_kernel<uint8_t><<<blocks, threads, 0, s>>>(
                static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), box, total);
            break;
        case 2:
            copy_box_kernel<uint16_t><<<blocks, threads, 0, s>>>(
                static_cast<uint16_t*>(dst), static_cast<const uint16_t*>(src), box, total);
            break;
        case 4:
            copy_box_kernel<uint32_t><<<blocks, threads, 0, s>>>(
                static_cast<uint32_t*>(dst), static_cast<const uint32_t*>(src), box, total);
            break;
        case 8:
            copy_box_kernel<uint64_t><<<blocks, threads, 0, s>>>(
                static_cast<uint64_t*>(dst), static_cast<const uint64_t*>(src), box, total);
            break;
        default:
            fail(SPX_ERR_CONFIG, "byte mover: element width must be 1, 2, 4 or 8");
    }
    SPX_CUDA_LAUNCH();
    count_launch();
}

void naive_gemm_run(const bf16* a, const bf16* b, float* out, int M, int N, int K,
                    cudaStream_t s) {
    dim3 grid(static_cast<unsigned>(ceil_div(N, 128)), static_cast<unsigned>(M));
    naive_gemm_kernel<<<grid, 128, 0, s>>>(a, b, out, M, N, K);
    SPX_CUDA_LAUNCH();
    count_launch();
}

void naive_attention_run(const bf16* q, const bf16* k, const bf16* v, float* out, int batch,
                         int sq, int skv, int heads, int head_dim, cudaStream_t s) {
    const size_t smem = static_cast<size_t>(head_dim + skv) * sizeof(float);
    require(smem <= 200 * 1024, SPX_ERR_UNSUPPORTED, "naive attention: kv too long");
    static bool attr_done[64] = {};
    int dev = 0;
    SPX_CUDA(cudaGetDevice(&dev));
    if (!attr_done[dev & 63]) {
        SPX_CUDA(cudaFuncSetAttribute(naive_attention_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr_done[dev & 63] = true;
    }
    dim3 grid(static_cast<unsigned>(sq), static_cast<unsigned>(heads),
              static_cast<unsigned>(batch));
    naive_attention_kernel<<<grid, 256, smem, s>>>(q, k, v, out, sq, skv, heads, head_dim);
    SPX_CUDA_LAUNCH();
    count_launch();
}

}  // namespace spx
