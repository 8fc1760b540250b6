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
#include "row_pipe.cuh"
#include "sm100.cuh"

namespace spx {

using namespace sm100;

namespace {

constexpr int kMaxVecPerLane = 8;  // C <= 2048

__device__ __forceinline__ void rope_position(int64_t i_local, int64_t row_offset, int64_t hw,
                                              int64_t grid_w, int64_t start_frame, int64_t& t,
                                              int64_t& h, int64_t& w) {
    const int64_t ig = row_offset + i_local;
    t = start_frame + ig / hw;
    h = (ig % hw) / grid_w;
    w = ig % grid_w;
}

// The lane's four rotation pairs of one row, packed for f32x2 math over pairs (0, 1) and (2, 3):
// c = (c_e, c_e+1), s = (s_e, s_e+1), ns = -s; already multiplied by the row's RMSNorm scale
// (rotation is linear: rope(x g r) = r rope(x g)).
struct RopeCs {
    float2 c[2], s[2], ns[2];
};

// 8 bf16 = rotation pairs (a_e, b_e) = (x[2e], x[2e+1]), e = 0..3 (rope.cpp:106-126:
// (a, b) -> (a c - b s, a s + b c)) in fp32 with one bf16 rounding; NORM: g points at the RMSNorm
// weights of the a elements, then of the b elements (two float4)
template <bool NORM>
__device__ __forceinline__ uint4 rope8(uint4 x, const RopeCs& r, const float4* g) {
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
    float2 a[2], b[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        a[h] = make_float2(bf16_lo(w[2 * h]), bf16_lo(w[2 * h + 1]));
        b[h] = make_float2(bf16_hi(w[2 * h]), bf16_hi(w[2 * h + 1]));
    }
    if constexpr (NORM) {
        const float4 wa = g[0], wb = g[1];
        a[0] = f2mul(a[0], make_float2(wa.x, wa.y));
        a[1] = f2mul(a[1], make_float2(wa.z, wa.w));
        b[0] = f2mul(b[0], make_float2(wb.x, wb.y));
        b[1] = f2mul(b[1], make_float2(wb.z, wb.w));
    }
    uint32_t out[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const float2 oa = f2fma(b[h], r.ns[h], f2mul(a[h], r.c[h]));
        const float2 ob = f2fma(a[h], r.s[h], f2mul(b[h], r.c[h]));
        out[2 * h] = pack_bf16x2(oa.x, ob.x);
        out[2 * h + 1] = pack_bf16x2(oa.y, ob.y);
    }
    return make_uint4(out[0], out[1], out[2], out[3]);
}

__device__ __forceinline__ RopeCs rope_cs(const float2 (&cs)[4], float scale) {
    RopeCs r;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        r.c[h] = make_float2(cs[2 * h].x * scale, cs[2 * h + 1].x * scale);
        r.s[h] = make_float2(cs[2 * h].y * scale, cs[2 * h + 1].y * scale);
        r.ns[h] = make_float2(-r.s[h].x, -r.s[h].y);
    }
    return r;
}

// sum of squares of 8 bf16, two packed accumulators
__device__ __forceinline__ void sumsq8(uint4 x, float2& acc) {
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 v = make_float2(bf16_lo(w[e]), bf16_hi(w[e]));
        acc = f2fma(v, v, acc);
    }
}

// Host-precomputed constants of one K3 launch: fast divisors for the position math (no integer
// division on the device) and the destination pointer table (read from shared memory per store:
// lanes of one warp may write different head groups, which a parameter-space load would
// serialise).
struct RopeAux {
    FastDiv rows_per_batch, hw, grid_w;
    int head_shift;  // log2(head_dim)
};

// NV = 16-byte vectors per lane per tensor (C / 256, rounded up). The rows stream through
// shared memory (row_pipe.cuh: bulk copies into a ring of stages per persistent CTA); each
// consumer warp reduces the QK-RMSNorm sums of its row from shared memory, then re-reads each
// vector, rotates it and stores it straight into its head group's destination slab (the pack of
// the fused all-to-all). Everything that depends only on the lane -- its vectors' head, group and
// slab offset, its four rotation pairs' band and column, the norm weights -- is computed once
// per CTA, so the per-row work is the table lookups, the math and the stores.
template <int NV, bool KV, bool NORM>
__global__ void __launch_bounds__(kPipeThreads, 1)
    rope_norm_pack_kernel(const RopeLaunch l, const RowPipeShape sh, const RopeAux aux,
                          unsigned long long* span) {
    extern __shared__ __align__(16) uint8_t smem_rope[];
    const int C = l.heads * l.head_dim;
    const int nvec = C / 8;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_rope);
    bf16** s_dst = reinterpret_cast<bf16**>(smem_rope + 2 * kPipeMaxStages * sizeof(uint64_t));  // [8][1 + 2 * 8]
    // RMSNorm weights as fp32, per vector: the four a-element weights, then the four b-element
    // weights (q vectors, then k vectors)
    float4* s_nw = reinterpret_cast<float4*>(s_dst + 8 * 17);
    uint8_t* ring = reinterpret_cast<uint8_t*>(s_nw + (NORM ? 4 * nvec : 0));
    pdl_trigger();
    span_begin(span);
    if (threadIdx.x == 0) row_pipe_init(bars, sh.stages);
    __syncthreads();
    if (threadIdx.x / 32 == kPipeWarps) {  // producer: the rows were written by the QKV projection
        pdl_wait();
        row_pipe_produce(reinterpret_cast<const uint8_t*>(l.in), l.in_row_stride * 2, static_cast<int>(l.rows),
                         sh, ring, bars);
        return;
    }
    // consumers: per-CTA constants while the first rows stream in
    for (int i = threadIdx.x; i < 8 * 17; i += kPipeWarps * 32) {
        const int g = i / 17, j = i % 17;
        s_dst[i] = j == 0 ? l.dst.q[g] : (j <= 8 ? l.dst.k[g][j - 1] : l.dst.v[g][j - 9]);
    }
    if constexpr (NORM) {  // constant weights: staged while the previous kernel drains
        for (int i = threadIdx.x; i < (KV ? 2 : 1) * nvec; i += kPipeWarps * 32) {
            const bf16* wsrc = i < nvec ? l.norm_w_q + 8 * i : l.norm_w_k + 8 * (i - nvec);
            const uint4 wv = __ldg(reinterpret_cast<const uint4*>(wsrc));
            s_nw[2 * i] = make_float4(bf16_lo(wv.x), bf16_lo(wv.y), bf16_lo(wv.z), bf16_lo(wv.w));
            s_nw[2 * i + 1] = make_float4(bf16_hi(wv.x), bf16_hi(wv.y), bf16_hi(wv.z), bf16_hi(wv.w));
        }
    }
    const int lane = static_cast<int>(threadIdx.x % 32);
    const int hpg = l.heads / l.groups;
    // per-lane constants: vector i = lane + 32 i lies in head (8 v) >> log2(D), group g, at
    // element offset `off` of its slab row
    int v_off[NV], v_g[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int v = lane + 32 * i;
        const int head = (8 * v) >> aux.head_shift;
        const int g = head / hpg;
        v_g[i] = g;
        v_off[i] = (head - g * hpg) * l.head_dim + ((8 * v) & (l.head_dim - 1));
    }
    // the lane's four rotation pairs (identical for all of its vectors because D | 256):
    // pair j = e0 / 2 + e in band b -> table column, row selected per token by t, h or w
    const int e0 = (8 * lane) & (l.head_dim - 1);
    const float2* tab_e[4];
    int band_e[4], stride_e[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        int j = e0 / 2 + e, b = 0;
        if (j >= l.pairs[0]) {
            j -= l.pairs[0];
            b = 1;
            if (j >= l.pairs[1]) {
                j -= l.pairs[1];
                b = 2;
            }
        }
        band_e[e] = b;
        tab_e[e] = l.tab[b] + j;
        stride_e[e] = l.pairs[b];
    }
    row_pipe_consumer_sync();
    pdl_wait();  // the destinations may still be read by the previous kernels
    row_pipe_consume(static_cast<int>(l.rows), sh, ring, bars, [&](int r0, int n, const uint8_t* stage, int lane_) {
#pragma unroll 1
      for (int ri = 0; ri < n; ++ri) {
        const int row = r0 + ri;
        const uint4* src = reinterpret_cast<const uint4*>(stage + ri * sh.row_bytes);
        uint4 xq[NV], xk[KV ? NV : 1];
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            if (lane_ + 32 * i < nvec) {
                xq[i] = lds128(src + lane_ + 32 * i);
                if constexpr (KV) xk[i] = lds128(src + nvec + lane_ + 32 * i);
            }
        }
        // (t, h, w) of this row (rope.cpp:97-101), 32-bit, fast divisions
        const int i_local = row - static_cast<int>(aux.rows_per_batch.div(static_cast<uint32_t>(row))) *
                                      static_cast<int>(l.rows_per_batch);
        const int ig = static_cast<int>(l.row_offset) + i_local;
        const int tq = static_cast<int>(aux.hw.div(static_cast<uint32_t>(ig)));
        const int rem = ig - tq * static_cast<int>(l.hw);
        const int h = static_cast<int>(aux.grid_w.div(static_cast<uint32_t>(rem)));
        const int pos[3] = {static_cast<int>(l.start_frame) + tq, h, rem - h * static_cast<int>(l.grid_w)};
        float2 cs[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int p = band_e[e] == 0 ? pos[0] : (band_e[e] == 1 ? pos[1] : pos[2]);
            cs[e] = l.rotate ? __ldg(tab_e[e] + p * stride_e[e]) : make_float2(1.0f, 0.0f);
        }
        float scale_q = 1.0f, scale_k = 1.0f;
        if constexpr (NORM) {  // QK-RMSNorm over the C channels (Wan mode; no reference counterpart)
            float2 aq = make_float2(0.0f, 0.0f), ak = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                if (lane_ + 32 * i < nvec) {
                    sumsq8(xq[i], aq);
                    if constexpr (KV) sumsq8(xk[i], ak);
                }
            }
            float sq = aq.x + aq.y, sk = ak.x + ak.y;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                sq += __shfl_xor_sync(0xffffffffu, sq, o);
                if constexpr (KV) sk += __shfl_xor_sync(0xffffffffu, sk, o);
            }
            scale_q = rsqrtf(sq / static_cast<float>(C) + l.norm_eps);
            scale_k = rsqrtf(sk / static_cast<float>(C) + l.norm_eps);
        }
        // q vectors, then k, then v: each tensor's constants and data die before the next
        const int64_t row_off = static_cast<int64_t>(row) * l.dst_row_stride;
        {
            const RopeCs rq = rope_cs(cs, scale_q);
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int v = lane_ + 32 * i;
                if (v >= nvec) continue;
                stg128(s_dst[v_g[i] * 17] + row_off + v_off[i], rope8<NORM>(xq[i], rq, s_nw + 2 * v));
            }
        }
        if constexpr (KV) {
            const RopeCs rk = rope_cs(cs, scale_k);
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int v = lane_ + 32 * i;
                if (v >= nvec) continue;
                const uint4 yk = rope8<NORM>(xk[i], rk, s_nw + 2 * (nvec + v));
                bf16** dg = s_dst + v_g[i] * 17;
#pragma unroll 1
                for (int c = 0; c < l.dst.copies; ++c) stg128(dg[1 + c] + row_off + v_off[i], yk);
            }
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int v = lane_ + 32 * i;
                if (v >= nvec || l.skip_v) continue;  // skip_v: the QKV epilogue packed v
                const uint4 yv = lds128(src + 2 * nvec + v);
                bf16** dg = s_dst + v_g[i] * 17;
#pragma unroll 1
                for (int c = 0; c < l.dst.copies; ++c) stg128(dg[9 + c] + row_off + v_off[i], yv);
            }
        }
      }
    });
    span_end(span);  // (consumer thread 0: profiling only)
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

template <int NV, bool KV, bool NORM>
void launch_rope_k(const RopeLaunch& l, const RowPipeShape& sh, const RopeAux& aux, unsigned ctas,
                   size_t smem, cudaStream_t stream) {
    static bool done[64] = {};  // the attribute is per function per device
    int dev = 0;
    SPX_CUDA(cudaGetDevice(&dev));
    if (!done[dev & 63]) {
        SPX_CUDA(cudaFuncSetAttribute(rope_norm_pack_kernel<NV, KV, NORM>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        done[dev & 63] = true;
    }
    launch_pdl(rope_norm_pack_kernel<NV, KV, NORM>, dim3(ctas), dim3(kPipeThreads), smem, stream, l, sh, aux,
               span_slot());
}

template <int NV>
void launch_rope_nv(const RopeLaunch& l, const RowPipeShape& sh, const RopeAux& aux, unsigned ctas,
                    size_t smem, cudaStream_t stream) {
    if (l.has_kv && l.norm)
        launch_rope_k<NV, true, true>(l, sh, aux, ctas, smem, stream);
    else if (l.has_kv)
        launch_rope_k<NV, true, false>(l, sh, aux, ctas, smem, stream);
    else if (l.norm)
        launch_rope_k<NV, false, true>(l, sh, aux, ctas, smem, stream);
    else
        launch_rope_k<NV, false, false>(l, sh, aux, ctas, smem, stream);
}

void launch_rope(const RopeLaunch& l, int nv, const RowPipeShape& sh, const RopeAux& aux, unsigned ctas,
                 size_t smem, cudaStream_t stream) {
    switch (nv) {
        case 1: launch_rope_nv<1>(l, sh, aux, ctas, smem, stream); break;
        case 2: launch_rope_nv<2>(l, sh, aux, ctas, smem, stream); break;
        case 3: launch_rope_nv<3>(l, sh, aux, ctas, smem, stream); break;
        case 4: launch_rope_nv<4>(l, sh, aux, ctas, smem, stream); break;
        case 5: launch_rope_nv<5>(l, sh, aux, ctas, smem, stream); break;
        case 6: launch_rope_nv<6>(l, sh, aux, ctas, smem, stream); break;
        case 7: launch_rope_nv<7>(l, sh, aux, ctas, smem, stream); break;
        default: launch_rope_nv<8>(l, sh, aux, ctas, smem, stream); break;
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
    require((reinterpret_cast<uintptr_t>(l.in) & 15) == 0 && l.in_row_stride % 8 == 0, SPX_ERR_ALIGNMENT,
            "rope kernel: input rows must be 16-byte aligned");
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        SPX_CUDA(cudaGetDevice(&dev));
        sms = device_sm_count(dev);
    }
    // skip_v: only the q | k part of each 3C input row is streamed
    const uint32_t row_bytes = static_cast<uint32_t>(C) * 2u * (l.has_kv ? (l.skip_v ? 2u : 3u) : 1u);
    const RowPipeShape sh = row_pipe_shape(l.rows, row_bytes, sms);
    const int64_t nblk = ceil_div(l.rows, static_cast<int64_t>(sh.rb));
    const unsigned ctas = static_cast<unsigned>(std::min<int64_t>(nblk, sms));
    const size_t smem = 2 * kPipeMaxStages * sizeof(uint64_t) + 8 * 17 * sizeof(bf16*) +
                        (l.norm ? 2u * static_cast<size_t>(C) * 4u : 0u) +
                        static_cast<size_t>(sh.stages) * sh.rb * row_bytes;
    RopeAux aux{};
    aux.rows_per_batch = FastDiv(static_cast<uint32_t>(l.rows_per_batch));
    aux.hw = FastDiv(static_cast<uint32_t>(l.hw));
    aux.grid_w = FastDiv(static_cast<uint32_t>(l.grid_w));
    aux.head_shift = 0;
    while ((1 << aux.head_shift) < l.head_dim) ++aux.head_shift;
    launch_rope(l, (C / 8 + 31) / 32, sh, aux, ctas, smem, stream);
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
