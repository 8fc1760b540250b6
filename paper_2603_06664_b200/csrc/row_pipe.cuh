// row_pipe.cuh -- the streaming skeleton of the HBM-bound row kernels (K3 rope/norm/pack,
// K1 LayerNorm + modulation).
//
// One persistent CTA per SM: a producer warp bulk-copies blocks of `rb` consecutive rows
// (cp.async.bulk, one copy per block when the rows are contiguous) into a deep ring of
// shared-memory stages, completion on an mbarrier's transaction count; the 15 consumer warps take
// the landed stages round-robin, compute from shared memory, store to global and release the
// stage. The ring (~150-190 KB per SM) keeps far more reads in flight than HBM latency x
// bandwidth needs, so the read stream no longer stalls on each warp's load -> reduce -> store
// chain, and the grid is exactly the SM count (no partial second wave).
#pragma once

#include "sm100.cuh"

namespace spx {

using namespace sm100;

constexpr int kPipeWarps = 15;                       // consumer warps (+ the producer: 16 warps, <= 128 registers)
constexpr int kPipeThreads = (kPipeWarps + 1) * 32;  // + the producer warp
constexpr int kPipeMaxStages = 45;                   // a multiple of kPipeWarps
constexpr uint32_t kPipeRingBudget = 192 * 1024;     // shared-memory bytes for the stages

struct RowPipeShape {
    int rb;              // rows per stage (one consumer warp processes a whole stage)
    int stages;          // ring depth (a multiple of kPipeWarps)
    uint32_t row_bytes;  // bytes of one row in shared memory (a multiple of 16)
};

// One row per stage when a row is large (>= 4 KB), else enough rows to make ~4 KB stages; as
// many stages as fit the budget (a multiple of the consumer warps, so stage s always belongs to
// warp s % kPipeWarps). Each SM then keeps up to the whole ring (~150-190 KB) of reads in flight.
inline RowPipeShape row_pipe_shape(int64_t rows, uint32_t row_bytes, int ctas) {
    RowPipeShape s{};
    s.row_bytes = row_bytes;
    int rb = static_cast<int>((4096 + row_bytes - 1) / row_bytes);
    const int64_t per_cta = (rows + ctas - 1) / ctas;  // keep every CTA busy on small inputs
    if (rb > per_cta) rb = static_cast<int>(per_cta < 1 ? 1 : per_cta);
    s.rb = rb;
    int st = static_cast<int>(kPipeRingBudget / (static_cast<uint32_t>(rb) * row_bytes));
    st = st / kPipeWarps * kPipeWarps;
    s.stages = st > kPipeMaxStages ? kPipeMaxStages : (st < kPipeWarps ? kPipeWarps : st);
    return s;
}

__device__ __forceinline__ void bulk_load_g2s(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ uint4 lds128(const void* p) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(smem_u32(p)));
    return v;
}

// packed f32x2 arithmetic (one issue slot for two lanes of math on sm_100)
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3}; mov.b64 rb, {%4, %5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3}; mov.b64 rb, {%4, %5}; mov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3}; mov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
// bf16 pair word -> (lo, hi) as fp32: a shift and a mask
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// 16-byte store to a global address held in a generic pointer (e.g. loaded from shared memory)
__device__ __forceinline__ void stg128(void* p, uint4 v) {
    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// The pipeline, in two halves run by different warps. fn(r0, n, const uint8_t* stage_smem, lane)
// is called by the consumer warp that owns the block of rows [r0, r0 + n) (n <= rb, rows
// row_bytes apart in shared memory). CTA c streams blocks b = c, c + gridDim.x, ... of rb rows;
// its k-th block lands in stage k % stages and is processed by warp k % kPipeWarps, so 15
// stages are computed at a time while the producer keeps the rest of the ring loading. `in`
// rows are `in_stride` bytes apart (one bulk copy per block when equal to row_bytes). bars:
// 2 * kPipeMaxStages uint64_t of shared memory (row_pipe_init, made visible by a CTA barrier
// before either half starts), ring: stages * rb * row_bytes bytes (16-byte aligned).
//
// The producer warp (warp kPipeWarps) starts streaming as soon as the barriers exist (after its
// own griddepcontrol.wait when the rows come from the previous kernel), while the consumer
// warps stage their per-CTA constants; the consumers then sync among themselves only
// (row_pipe_consumer_sync), so the constant staging overlaps the first reads.
__device__ __forceinline__ void row_pipe_produce(const uint8_t* in, int64_t in_stride, int rows,
                                                 const RowPipeShape& sh, uint8_t* ring, uint64_t* bars) {
    uint64_t* full = bars;
    uint64_t* empty = bars + kPipeMaxStages;
    if (threadIdx.x % 32 != 0) return;
    const int nblk = (rows + sh.rb - 1) / sh.rb;
    const uint32_t stage_bytes = static_cast<uint32_t>(sh.rb) * sh.row_bytes;
    int k = 0;
    for (int b = static_cast<int>(blockIdx.x); b < nblk; b += static_cast<int>(gridDim.x), ++k) {
        const int s = k % sh.stages;
        mbar_wait(&empty[s], ((k / sh.stages) & 1) ^ 1);
        const int r0 = b * sh.rb;
        const int n = min(sh.rb, rows - r0);
        uint8_t* dst = ring + s * stage_bytes;
        mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(n) * sh.row_bytes);
        if (in_stride == static_cast<int64_t>(sh.row_bytes)) {
            bulk_load_g2s(dst, in + static_cast<int64_t>(r0) * in_stride, static_cast<uint32_t>(n) * sh.row_bytes,
                          &full[s]);
        } else {
            for (int i = 0; i < n; ++i)
                bulk_load_g2s(dst + i * sh.row_bytes, in + static_cast<int64_t>(r0 + i) * in_stride,
                              sh.row_bytes, &full[s]);
        }
    }
}

// the consumer warps' barrier (named barrier 1; the producer never joins it)
__device__ __forceinline__ void row_pipe_consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kPipeWarps * 32) : "memory");
}

template <class Fn>
__device__ __forceinline__ void row_pipe_consume(int rows, const RowPipeShape& sh, uint8_t* ring,
                                                 uint64_t* bars, Fn&& fn) {
    uint64_t* full = bars;
    uint64_t* empty = bars + kPipeMaxStages;
    const int warp = static_cast<int>(threadIdx.x / 32);
    const int lane = static_cast<int>(threadIdx.x % 32);
    const int nblk = (rows + sh.rb - 1) / sh.rb;
    const uint32_t stage_bytes = static_cast<uint32_t>(sh.rb) * sh.row_bytes;
    int k = warp;
#pragma unroll 1
    for (int b = static_cast<int>(blockIdx.x) + warp * static_cast<int>(gridDim.x); b < nblk;
         b += kPipeWarps * static_cast<int>(gridDim.x), k += kPipeWarps) {
        const int s = k % sh.stages;
        mbar_wait(&full[s], (k / sh.stages) & 1);
        const int r0 = b * sh.rb;
        const int n = min(sh.rb, rows - r0);
        fn(r0, n, ring + s * stage_bytes, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}

// barrier setup of the pipeline (one thread), before the CTA-wide barrier that follows
__device__ __forceinline__ void row_pipe_init(uint64_t* bars, int stages) {
    for (int s = 0; s < stages; ++s) {
        mbar_init(&bars[s], 1);
        mbar_init(&bars[kPipeMaxStages + s], 1);
    }
    fence_mbar_init();
}

}  // namespace spx
