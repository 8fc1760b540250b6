// rope.cu -- K3: fused [QK-RMSNorm] + Causal-RoPE + bf16 cast + all-to-all pack.
//
// Reference: rotate_rows (proj/src/rope.cpp:78-131) reached through apply_rope_causal_local
// (rope.cpp:145-164): local row i of rank r has global position i_g = r * L/P + i, frame
// t = start_frame + i_g / (H_g W_g), h = (i_g mod H_g W_g) / W_g, w = i_g mod W_g
// (rope.cpp:97-101); pair j < p_T rotates by T[t], then H[h], then W[w], elements (2j, 2j+1)
// as (a, b) -> (a c - b s, a s + b c) (rope.cpp:106-126).
//
// One warp per token row. Each lane owns 16-byte vectors v = lane + 32 i of the C-vector, so
// (for D | 256) its four rotation pairs are the same for every vector it touches: the lane
// loads its cos/sin once per row. q and k are rotated (after the optional RMSNorm over the C
// channels, a Wan-mode extension with no reference counterpart); v is copied. Every vector is
// written straight into the destination slab of its head group (the sequence<->head
// all-to-all's pack step), for every query-split copy of k/v.
#include "common.hpp"
#include "kernels.hpp"
#include "sm100.cuh"

namespace spx {

using namespace sm100;

namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kMaxVecPerLane = 8;  // C <= 2048

__device__ __forceinline__ void rope_position(int64_t i_local, int64_t row_offset, int64_t hw,
                                              int64_t grid_w, int64_t start_frame, int64_t& t,
                                              int64_t& h, int64_t& w) {
    const int64_t ig = row_offset + i_local;
    t = start_frame + ig / hw;
    h = (ig % hw) / grid_w;
    w = ig % grid_w;
}

__device__ __forceinline__ float2 band_cs(const RopeLaunch& l, int j, int64_t t, int64_t h,
                                          int64_t w) {
    if (j < l.pairs[0]) return __ldg(&l.tab[0][t * l.pairs[0] + j]);
    j -= l.pairs[0];
    if (j < l.pairs[1]) return __ldg(&l.tab[1][h * l.pairs[1] + j]);
    j -= l.pairs[1];
    return __ldg(&l.tab[2][w * l.pairs[2] + j]);
}

__device__ __forceinline__ uint4 rotate_vec(uint4 x, const float2 (&cs)[4], float scale,
                                            const uint4* nw) {
    uint32_t in[4] = {x.x, x.y, x.z, x.w};
    uint32_t wv[4] = {0, 0, 0, 0};
    if (nw) {
        const uint4 t = *nw;
        wv[0] = t.x;
        wv[1] = t.y;
        wv[2] = t.z;
        wv[3] = t.w;
    }
    uint32_t out[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        float2 ab = unpack_bf16x2(in[e]);
        if (nw) {
            const float2 g = unpack_bf16x2(wv[e]);
            ab.x = ab.x * scale * g.x;
            ab.y = ab.y * scale * g.y;
        }
        const float c = cs[e].x, s = cs[e].y;
        out[e] = pack_bf16x2(ab.x * c - ab.y * s, ab.x * s + ab.y * c);
    }
    return make_uint4(out[0], out[1], out[2], out[3]);
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    rope_norm_pack_kernel(const RopeLaunch l) {
    const int lane = threadIdx.x % 32;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + threadIdx.x / 32;
    if (row >= l.rows) return;
    const int C = l.heads * l.head_dim;
    const int nvec = C / 8;
    const int hpg = l.heads / l.groups;
    const int64_t i_local = row % l.rows_per_batch;
    int64_t t, h, w;
    rope_position(i_local, l.row_offset, l.hw, l.grid_w, l.start_frame, t, h, w);

    // this lane's four pairs (identical for all of its vectors because D | 256)
    const int e0 = (8 * lane) % l.head_dim;
    float2 cs[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) cs[e] = band_cs(l, e0 / 2 + e, t, h, w);

    const uint4* src = reinterpret_cast<const uint4*>(l.in + row * l.in_row_stride);
    const int ntensor = l.has_kv ? 3 : 1;
#pragma unroll 1
    for (int which = 0; which < ntensor; ++which) {
        const uint4* s = src + which * nvec;
        uint4 x[kMaxVecPerLane];
        float ss = 0.0f;
#pragma unroll
        for (int i = 0; i < kMaxVecPerLane; ++i) {
            const int v = lane + 32 * i;
            if (v < nvec) {
                x[i] = s[v];
                if (l.norm && which < 2) {
                    const uint32_t q[4] = {x[i].x, x[i].y, x[i].z, x[i].w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f = unpack_bf16x2(q[e]);
                        ss += f.x * f.x + f.y * f.y;
                    }
                }
            }
        }
        float scale = 1.0f;
        const uint4* nw_base = nullptr;
        if (l.norm && which < 2) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
            scale = rsqrtf(ss / static_cast<float>(C) + l.norm_eps);
            nw_base = reinterpret_cast<const uint4*>(which == 0 ? l.norm_w_q : l.norm_w_k);
        }
#pragma unroll
        for (int i = 0; i < kMaxVecPerLane; ++i) {
            const int v = lane + 32 * i;
            if (v >= nvec) continue;
            const int head = (8 * v) / l.head_dim;
            const int g = head / hpg;
            const int64_t off = row * l.dst_row_stride + (head - g * hpg) * l.head_dim + e0;
            if (which == 2) {
                for (int c = 0; c < l.dst.copies; ++c)
                    *reinterpret_cast<uint4*>(l.dst.v[g][c] + off) = x[i];
            } else {
                const uint4 y = rotate_vec(x[i], cs, scale, nw_base ? nw_base + v : nullptr);
                if (which == 0) {
                    *reinterpret_cast<uint4*>(l.dst.q[g] + off) = y;
                } else {
                    for (int c = 0; c < l.dst.copies; ++c)
                        *reinterpret_cast<uint4*>(l.dst.k[g][c] + off) = y;
                }
            }
        }
    }
}

__global__ void rope_positions_kernel(int64_t rows, int64_t row_offset, int64_t hw,
                                      int64_t grid_w, int64_t start_frame, int32_t* t32,
                                      int32_t* h32, int32_t* w32) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    int64_t t, h, w;
    rope_position(i, row_offset, hw, grid_w, start_frame, t, h, w);
    t32[i] = static_cast<int32_t>(t);
    h32[i] = static_cast<int32_t>(h);
    w32[i] = static_cast<int32_t>(w);
}

}  // namespace

void rope_run(const RopeLaunch& l, cudaStream_t stream) {
    const int C = l.heads * l.head_dim;
    require(l.head_dim >= 8 && 256 % l.head_dim == 0, SPX_ERR_UNSUPPORTED,
            "rope kernel: head_dim must divide 256 (got " + std::to_string(l.head_dim) + ")");
    require(C % 8 == 0 && C <= 8 * 32 * kMaxVecPerLane, SPX_ERR_UNSUPPORTED,
            "rope kernel: model dim must be a multiple of 8 and <= 2048");
    require(l.groups >= 1 && l.groups <= 8 && l.heads % l.groups == 0, SPX_ERR_PARTITION,
            "rope kernel: heads must split into <= 8 groups");
    require(l.dst.copies >= 1 && l.dst.copies <= 8, SPX_ERR_CONFIG, "rope kernel: 1-8 kv copies");
    if (l.rows == 0) return;
    const unsigned blocks = static_cast<unsigned>(ceil_div(l.rows, kWarpsPerBlock));
    rope_norm_pack_kernel<<<blocks, kWarpsPerBlock * 32, 0, stream>>>(l);
    SPX_CUDA_LAUNCH();
    count_launch();
}

void rope_positions_run(int64_t rows, int64_t row_offset, int64_t hw, int64_t grid_w,
                        int64_t start_frame, int32_t* t, int32_t* h, int32_t* w,
                        cudaStream_t stream) {
    if (rows == 0) return;
    const unsigned blocks = static_cast<unsigned>(ceil_div(rows, 256));
    rope_positions_kernel<<<blocks, 256, 0, stream>>>(rows, row_offset, hw, grid_w, start_frame,
                                                      t, h, w);
    SPX_CUDA_LAUNCH();
    count_launch();
}

}  // namespace spx
