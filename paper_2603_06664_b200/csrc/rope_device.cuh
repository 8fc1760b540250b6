// rope_device.cuh -- Causal-RoPE device helpers shared by K3 (rope.cu) and the QKV GEMM's
// fused rotate-and-pack epilogue (gemm.cu).
//
// Reference: rotate_rows (proj/src/rope.cpp:78-131): local row i of rank r has global
// position i_g = row_offset + i, frame t = start_frame + i_g / (H_g W_g),
// h = (i_g mod H_g W_g) / W_g, w = i_g mod W_g (rope.cpp:97-101); pair j < p_T rotates by
// T[t], then H[h], then W[w] (rope.cpp:106-126).
#pragma once

#include "kernels.hpp"

namespace spx {

// n / d for 0 <= n < 2^31 by a multiply-high (d >= 1; host-computed magic m and shift s):
// s = ceil(log2 d), m = floor(2^32 (2^s - d) / d) + 1, n / d = (umulhi(n, m) + n) >> s
struct FastDiv {
    uint32_t d = 1, m = 0, s = 0;
    FastDiv() = default;
    __host__ explicit FastDiv(uint32_t divisor) : d(divisor) {
        while ((uint64_t(1) << s) < d) ++s;
        m = static_cast<uint32_t>(((uint64_t(1) << s) - d) * (uint64_t(1) << 32) / d + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> s; }
};

// (cos, sin) of rotation pair j at position (t, h, w): band tables are [pos][pairs_b]
__device__ __forceinline__ float2 band_cs(const RopeLaunch& l, int j, int t, int h, int w) {
    if (j < l.pairs[0]) return __ldg(&l.tab[0][t * l.pairs[0] + j]);
    j -= l.pairs[0];
    if (j < l.pairs[1]) return __ldg(&l.tab[1][h * l.pairs[1] + j]);
    j -= l.pairs[1];
    return __ldg(&l.tab[2][w * l.pairs[2] + j]);
}

// (t, h, w) of local token row `row` (32-bit; rope_run checks the range)
__device__ __forceinline__ void rope_thw(const RopeLaunch& l, int row, int& t, int& h, int& w) {
    const int i_local = row % static_cast<int>(l.rows_per_batch);
    const int ig = static_cast<int>(l.row_offset) + i_local;
    const int hw = static_cast<int>(l.hw), gw = static_cast<int>(l.grid_w);
    const int tq = ig / hw;
    t = static_cast<int>(l.start_frame) + tq;
    const int rem = ig - tq * hw;
    h = rem / gw;
    w = rem - h * gw;
}

// ---- the band-table slice one launch reads, staged in shared memory ----
// frames [t_lo, t_lo + n_t) of the T band (the launch's rows), then the whole H and W bands;
// entries are (cos, sin) pairs, pair-index offsets off_h / off_w
struct RopeSmem {
    int t_lo, n_t;
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

// threads tid = 0 .. nthreads - 1 copy the slice to shared-memory byte address st. All of a
// thread's loads are issued before its first store (the stores' "memory" clobber would
// otherwise serialise one L2 round trip per element).
__device__ __forceinline__ void rope_stage_tables(const RopeLaunch& l, uint32_t st, int tid, int nthreads) {
    const RopeSmem r = rope_smem_layout(l);
    const int nt = r.n_t * l.pairs[0];
    const int total = rope_smem_pairs(l);
    constexpr int kBatch = 8;
    for (int i0 = tid; i0 < total; i0 += kBatch * nthreads) {
        float2 v[kBatch];
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const int i = i0 + b * nthreads;
            v[b] = make_float2(0.0f, 0.0f);
            if (i < nt)
                v[b] = __ldg(&l.tab[0][r.t_lo * l.pairs[0] + i]);
            else if (i < r.off_w)
                v[b] = __ldg(&l.tab[1][i - r.off_h]);
            else if (i < total)
                v[b] = __ldg(&l.tab[2][i - r.off_w]);
        }
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const int i = i0 + b * nthreads;
            if (i < total)
                asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(st + 8u * i), "f"(v[b].x),
                             "f"(v[b].y)
                             : "memory");
        }
    }
}

__device__ __forceinline__ float2 lds_f2(uint32_t addr) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}

}  // namespace spx
