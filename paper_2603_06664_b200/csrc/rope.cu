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
#include <algorithm>

#include "common.hpp"
#include "kernels.hpp"
#include "rope_device.cuh"
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

// NV = 16-byte vectors per lane per tensor (C / 256, rounded up). Every load of the row
// (q, k and v: 3 NV vectors per lane) is issued before any math, so each warp keeps
// 3 x NV x 512 B in flight; the position math is 32-bit.
template <int NV, bool KV, bool NORM>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    rope_norm_pack_kernel(const RopeLaunch l) {
    pdl_trigger();
    pdl_wait();  // qkv was written by the previous kernel (the QKV projection)
    const int lane = threadIdx.x % 32;
    const int row = static_cast<int>(blockIdx.x) * kWarpsPerBlock + static_cast<int>(threadIdx.x / 32);
    const bool live = row < l.rows;  // (q|k|v + norm: no early return, the block stages weights)
    if (!(NORM && KV) && !live) return;
    const int C = l.heads * l.head_dim;
    const int nvec = C / 8;
    const int hpg = l.heads / l.groups;
    const uint4* src = reinterpret_cast<const uint4*>(l.in + static_cast<int64_t>(live ? row : 0) * l.in_row_stride);

    uint4 xq[NV], xk[KV ? NV : 1], xv[KV ? NV : 1];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int v = lane + 32 * i;
        if (live && v < nvec) {
            xq[i] = __ldg(src + v);
            if constexpr (KV) {
                xk[i] = __ldg(src + nvec + v);
                xv[i] = __ldg(src + 2 * nvec + v);
            }
        }
    }
    // q|k|v form: QK-RMSNorm weights staged once per block while the rows are in flight (read
    // after the row reduction: shared-memory latency instead of an L2 round trip on every
    // warp's path; 28.6 -> 23.4 us in the Wan-mode engine). The single-tensor form keeps
    // reading them from L1/L2: its 56 registers keep all 4680 rows of the Wan chunk resident,
    // the staging's extra registers would not (measured slower, 8.3 -> 9.5 us)
    constexpr bool kStage = NORM && KV;
    __shared__ uint4 s_nw[kStage ? 2 : 1][kStage ? kMaxVecPerLane * 32 : 1];
    if constexpr (kStage) {
        for (int i = threadIdx.x; i < nvec; i += blockDim.x) {
            s_nw[0][i] = __ldg(reinterpret_cast<const uint4*>(l.norm_w_q) + i);
            s_nw[1][i] = __ldg(reinterpret_cast<const uint4*>(l.norm_w_k) + i);
        }
        __syncthreads();
    }
    if (!live) return;

    // (t, h, w) of this row (rope.cpp:97-101), 32-bit
    int t, h, w;
    rope_thw(l, row, t, h, w);
    // this lane's four rotation pairs (identical for all of its vectors because D | 256)
    const int e0 = (8 * lane) % l.head_dim;
    float2 cs[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
        cs[e] = l.rotate ? band_cs(l, e0 / 2 + e, t, h, w) : make_float2(1.0f, 0.0f);

    float scale_q = 1.0f, scale_k = 1.0f;
    if constexpr (NORM) {  // QK-RMSNorm over the C channels (Wan mode; no reference counterpart)
        float sq = 0.0f, sk = 0.0f;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            if (lane + 32 * i < nvec) {
                const uint32_t a[4] = {xq[i].x, xq[i].y, xq[i].z, xq[i].w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 fa = unpack_bf16x2(a[e]);
                    sq = fmaf(fa.x, fa.x, fmaf(fa.y, fa.y, sq));
                }
                if constexpr (KV) {
                    const uint32_t b[4] = {xk[i].x, xk[i].y, xk[i].z, xk[i].w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 fb = unpack_bf16x2(b[e]);
                        sk = fmaf(fb.x, fb.x, fmaf(fb.y, fb.y, sk));
                    }
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sq += __shfl_xor_sync(0xffffffffu, sq, o);
            sk += __shfl_xor_sync(0xffffffffu, sk, o);
        }
        scale_q = rsqrtf(sq / static_cast<float>(C) + l.norm_eps);
        scale_k = rsqrtf(sk / static_cast<float>(C) + l.norm_eps);
    }
    const uint4* nwq = !NORM ? nullptr : kStage ? &s_nw[0][0] : reinterpret_cast<const uint4*>(l.norm_w_q);
    const uint4* nwk = !NORM ? nullptr : kStage ? &s_nw[kStage ? 1 : 0][0] : reinterpret_cast<const uint4*>(l.norm_w_k);

#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int v = lane + 32 * i;
        if (v >= nvec) continue;
        const int head = (8 * v) / l.head_dim;
        const int g = head / hpg;
        const int64_t off = static_cast<int64_t>(row) * l.dst_row_stride +
                            (head - g * hpg) * l.head_dim + e0;
        *reinterpret_cast<uint4*>(l.dst.q[g] + off) =
            rotate_vec(xq[i], cs, scale_q, nwq ? nwq + v : nullptr);
        if constexpr (KV) {
            const uint4 yk = rotate_vec(xk[i], cs, scale_k, nwk ? nwk + v : nullptr);
            for (int c = 0; c < l.dst.copies; ++c) {
                *reinterpret_cast<uint4*>(l.dst.k[g][c] + off) = yk;
                *reinterpret_cast<uint4*>(l.dst.v[g][c] + off) = xv[i];
            }
        }
    }
}

__global__ void rope_table_kernel(float2* b0, float2* b1, float2* b2, int r0, int r1, int r2,
                                  int p0, int p1, int p2, double base) {
    const int n0 = r0 * p0, n1 = r1 * p1, n2 = r2 * p2;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n0 + n1 + n2;
         i += gridDim.x * blockDim.x) {
        int k = i, p;
        float2* out;
        if (k < n0) {
            p = p0;
            out = b0;
        } else if (k - n0 < n1) {
            k -= n0;
            p = p1;
            out = b1;
        } else {
            k -= n0 + n1;
            p = p2;
            out = b2;
        }
        const int m = k / p, j = k - m * p;
        // rope.cpp:37-41: freq = base^(-j/p), angle = m * freq
        const double freq = pow(base, -static_cast<double>(j) / static_cast<double>(p));
        double sn, cs;
        sincos(static_cast<double>(m) * freq, &sn, &cs);
        out[k] = make_float2(static_cast<float>(cs), static_cast<float>(sn));
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

template <int NV>
void launch_rope_nv(const RopeLaunch& l, unsigned blocks, cudaStream_t stream) {
    const dim3 b(kWarpsPerBlock * 32);
    if (l.has_kv && l.norm)
        launch_pdl(rope_norm_pack_kernel<NV, true, true>, dim3(blocks), b, 0, stream, l);
    else if (l.has_kv)
        launch_pdl(rope_norm_pack_kernel<NV, true, false>, dim3(blocks), b, 0, stream, l);
    else if (l.norm)
        launch_pdl(rope_norm_pack_kernel<NV, false, true>, dim3(blocks), b, 0, stream, l);
    else
        launch_pdl(rope_norm_pack_kernel<NV, false, false>, dim3(blocks), b, 0, stream, l);
}

void launch_rope(const RopeLaunch& l, int nv, unsigned blocks, cudaStream_t stream) {
    switch (nv) {
        case 1: launch_rope_nv<1>(l, blocks, stream); break;
        case 2: launch_rope_nv<2>(l, blocks, stream); break;
        case 3: launch_rope_nv<3>(l, blocks, stream); break;
        case 4: launch_rope_nv<4>(l, blocks, stream); break;
        case 5: launch_rope_nv<5>(l, blocks, stream); break;
        case 6: launch_rope_nv<6>(l, blocks, stream); break;
        case 7: launch_rope_nv<7>(l, blocks, stream); break;
        default: launch_rope_nv<8>(l, blocks, stream); break;
    }
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
    require(l.rows < (int64_t(1) << 31) && l.row_offset + l.rows_per_batch < (int64_t(1) << 31),
            SPX_ERR_RANGE, "rope kernel: row indices must fit in 32 bits");
    const unsigned blocks = static_cast<unsigned>(ceil_div(l.rows, kWarpsPerBlock));
    launch_rope(l, (C / 8 + 31) / 32, blocks, stream);
    SPX_CUDA_LAUNCH();
    count_launch();
}

void rope_table_run(float2* const band[3], const int rows[3], const int pairs[3], double base,
                    cudaStream_t stream) {
    const int n = rows[0] * pairs[0] + rows[1] * pairs[1] + rows[2] * pairs[2];
    if (n == 0) return;
    rope_table_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(n, 256), 148)), 256, 0, stream>>>(
        band[0], band[1], band[2], rows[0], rows[1], rows[2], pairs[0], pairs[1], pairs[2], base);
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
