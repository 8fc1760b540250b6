// kernels.hpp -- host launchers for the spx sm_100a kernels (one translation unit each).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace spx {

using bf16 = __nv_bfloat16;

// ---------------------------------------------------------------------------------------
// K2 / K8: tcgen05 GEMM  out[M][N] = A[M][K] * B[N][K]^T  (bf16 in, fp32 TMEM accumulate)
//   A is addressed as a 3-D tensor [G][M][k_inner] (K = G * k_inner): the output all-to-all
//   lands head-group slabs side by side and the A-operand TMA un-interleaves them.
// ---------------------------------------------------------------------------------------
struct GemmOperands {
    const bf16* a = nullptr;
    int64_t a_row_stride = 0;    // elements between consecutive rows of one group slab
    int64_t a_group_stride = 0;  // elements between group slabs
    int groups = 1;
    int k_inner = 0;
    const bf16* b = nullptr;     // [N][K] row-major (K-major)
    int64_t b_row_stride = 0;
    bf16* out = nullptr;
    int64_t out_row_stride = 0;
    int M = 0, N = 0, K = 0;
    // epilogue (acc' = acc + bias[col] when bias != nullptr):
    //   0 -> out = acc'
    //   1 -> out = residual + gate[col] * acc' (adaLN gate + residual; gate == nullptr: 1)
    //   2 -> Causal-RoPE rotate-and-pack (set by gemm_run's rope argument; no bias)
    //   3 -> out = GELU_tanh(acc') (the Wan FFN's first projection)
    // out may alias residual (each element is read, then written, by the same warp)
    int epi_mode = 0;
    const bf16* residual = nullptr;
    int64_t residual_row_stride = 0;
    const float* gate = nullptr;
    const float* bias = nullptr;   // fp32 [N]
    // B is not written by the kernel launched just before (e.g. weights): its first pipeline
    // stages are loaded before griddepcontrol.wait, overlapping the previous kernel's tail
    bool b_constant = false;
    // the planner may split K across a 2-CTA cluster (short-M shapes): the sum of two partial
    // accumulators, so the rounding differs from an unsplit tile (sp_bit_exact turns it off)
    bool allow_split_k = true;
};

struct GemmPlan {
    CUtensorMap map_a;
    CUtensorMap map_b;
    GemmOperands ops;
    int bn = 256;
    bool pair = false;  // cta_group::2 CTA-pair kernel (256-row tiles)
    int ksplit = 1;     // 2: split-K over a 2-CTA cluster (single-CTA 128 x 128 tiles)
    int grid = 0;
};

struct RopeLaunch;
void gemm_plan(GemmPlan* plan, const GemmOperands& ops, int sm_count);
// rope != nullptr (QKV projection only): the epilogue applies Causal-RoPE to the q and k
// columns of the fp32 accumulator and stores q / k / v straight into rope->dst (the K3
// rotate-and-pack without its qkv round trip); requires gemm_rope_fusable()
void gemm_run(const GemmPlan& plan, cudaStream_t stream, const RopeLaunch* rope = nullptr);
bool gemm_rope_fusable(const GemmPlan& plan, const RopeLaunch& rope);
// rope->skip_v: the epilogue packs only the v columns (into rope->dst.v, the KV ring) and stores
// q | k unrotated to the plain output (bias allowed); K3 then normalises and rotates q | k
bool gemm_vpack_fusable(const GemmPlan& plan, const RopeLaunch& rope);

// The residual projection fused with the next LayerNorm + modulation (gemm_ln.cu, Wan mode):
//   out = residual + gate (A B^T + bias);  out2 = LN(out) (one + mul) + add   (one = 1 adaLN,
// 0 affine). Needs N = 1536 (a 3-CTA cluster owns 128 full rows), the residual epilogue and
// 16-byte alignment; ok = false when the clusters do not all fit on the device at once.
struct GemmLnPlan {
    CUtensorMap map_a, map_b, map_res, map_out, map_out2;
    GemmOperands ops;
    bf16* out2 = nullptr;
    const float* mul = nullptr;
    const float* add = nullptr;
    bool affine = false;
    float eps = 1e-6f;
    int grid = 0;
    bool ok = false;
};
bool gemm_ln_supported(const GemmOperands& ops);
void gemm_ln_plan(GemmLnPlan* plan, const GemmOperands& ops, bf16* out2, const float* mul, const float* add,
                  bool affine, float eps);
void gemm_ln_run(const GemmLnPlan& plan, cudaStream_t stream);
// planner override (tests / tuning): -1 = modelled choice, else a tile variant index
int gemm_forced_variant();
void gemm_force_variant(int v);
int gemm_num_variants();
// SPX_GEMM_EXPERIMENT=5: the pair kernel's per-tile clock64 timeline ([cta][16][4], device)
long long* gemm_trace_buffer();

// ---------------------------------------------------------------------------------------
// K6: chunk-causal flash attention, tcgen05/TMEM, TMA-fed.
//   q  : [B][Sq][H][D]    k/v : [B][Skv_rows][H][D] addressed through up to two row
//   segments (the rolling KV ring wraps).  Output rows are scattered to up to 8 destination
//   slabs (the output all-to-all is fused into the epilogue).
// ---------------------------------------------------------------------------------------
struct AttnOperands {
    const bf16* q = nullptr;
    int64_t q_rows = 0;          // rows per batch in q
    const bf16* k = nullptr;
    const bf16* v = nullptr;
    int64_t kv_rows = 0;         // rows per batch in the k/v buffers (ring capacity rows)
    int batch = 1, heads = 0, head_dim = 0;
    int sq = 0;                  // query rows to compute (<= q_rows)
    int seg_start[2] = {0, 0};
    int seg_len[2] = {0, 0};
    int num_segs = 1;
    // output element (b, i, h, d) -> out_base[i / rows_per_chunk] + b * out_batch_stride
    //                                 + (i % rows_per_chunk) * out_row_stride + h * D + d
    bf16* out_base[8] = {};
    int rows_per_chunk = 0;
    int64_t out_row_stride = 0;
    int64_t out_batch_stride = 0;
    // split-KV workspace (zero-initialised once; see attn_workspace_bytes). When the grid of
    // (query tiles x heads) under-fills the SMs, the kv range is split over up to
    // max_splits CTAs per tile, each writing a normalised fp32 partial + its log-sum-exp; the
    // last CTA of a tile to finish merges them (no extra launch).
    void* workspace = nullptr;
    size_t workspace_bytes = 0;
    // optional: byte ranges warmed into L2 while the (tensor-bound) kernel runs, e.g. the
    // weights of the projections that follow (their HBM reads leave the GEMMs' critical path)
    const void* l2_prefetch[2] = {nullptr, nullptr};
    int64_t l2_prefetch_bytes[2] = {0, 0};
    // unsplit layouts run the v3 kernel when they fill at least one wave of the SMs; true: also
    // below that (cfg.sp_bit_exact: every partition of a run must use the same kernel)
    bool prefer_v3 = false;
};

struct AttnPlan {
    CUtensorMap map_q;
    CUtensorMap map_k;
    CUtensorMap map_v;
    AttnOperands ops;
    int max_splits = 1;
};

// kv splits the planner uses for this (query rows, heads) shape on sm_count SMs
int attn_max_splits(const AttnOperands& ops, int sm_count);
// workspace bytes for that many splits (0 when max_splits == 1)
size_t attn_workspace_bytes(const AttnOperands& ops, int max_splits);
void attn_plan(AttnPlan* plan, const AttnOperands& ops, int sm_count);
void attn_set_segments(AttnPlan* plan, const int* seg_start, const int* seg_len, int num_segs);
// split-KV override (tests / tuning): 0 = modelled choice, else the kv splits per query tile
void attn_force_splits(int s);
// the shared-O / early-S attention kernel (v3) for unsplit layouts: 0 never, 1 auto, 2 always
// (SPX_ATTN_V3)
void attn_set_v3(int on);
bool attn_v3_enabled();
void attn_run(const AttnPlan& plan, cudaStream_t stream);

// ---------------------------------------------------------------------------------------
// K3: fused [QK-RMSNorm] + Causal-RoPE + bf16 cast + all-to-all pack.
//   Input rows are the QKV GEMM output [rows][3C] (or a single tensor, see RopeTensorMode);
//   every 16-byte vector of head h goes to destination slab group g = h / heads_per_group.
// ---------------------------------------------------------------------------------------
struct RopeTable;  // device copy, see rope_table.hpp

struct RopeDest {
    bf16* q[8] = {};           // per head group: base of the (rows, H/G, D) q slab
    bf16* k[8][8] = {};        // per head group, per query split copy
    bf16* v[8][8] = {};
    int copies = 1;            // query-split copies of k/v to write (S)
};

struct RopeLaunch {
    const bf16* in = nullptr;        // rows of the input
    int64_t in_row_stride = 0;       // elements
    int64_t rows = 0;                // tokens (local), batch folded
    int64_t rows_per_batch = 0;      // L/P (for the time index)
    int heads = 0, head_dim = 0;
    int groups = 1;                  // head groups (destinations)
    int has_kv = 0;                  // 1: input holds q|k|v, 0: a single tensor rotated into q
    // position math (rope.cpp:97-101): i_g = row_offset + i, t = start + i_g / hw ...
    int64_t row_offset = 0;
    int64_t hw = 0, grid_w = 0, start_frame = 0;
    // table (device, fp32 cos/sin interleaved per band)
    const float2* tab[3] = {};
    int pairs[3] = {0, 0, 0};
    int tab_constant = 0;            // 1: no kernel writes tab (the precomputed table): the
                                     // GEMM epilogue stages it before griddepcontrol.wait
    // optional QK-RMSNorm over the C = H*D channels
    const bf16* norm_w_q = nullptr;
    const bf16* norm_w_k = nullptr;
    float norm_eps = 1e-6f;
    int norm = 0;
    int rotate = 1;                  // 0: pack only (the exchange-first ablation rotates later)
    int skip_v = 0;                  // K3: v was already packed by the QKV GEMM's epilogue
                                     // (gemm_run with this launch): the rows are read as q | k
    RopeDest dst;
    int64_t dst_row_stride = 0;      // elements between rows in a destination slab (H/G * D)
};

void rope_run(const RopeLaunch& l, cudaStream_t stream);
// precompute_frequencies on the device (the use_precomputed_freqs = false ablation recomputes
// a slice every call, sp_attention.cpp:191-195): band b rows [0, rows[b]) x pairs[b] of
// (cos, sin)(m * base^(-j / pairs[b])) in fp64, stored as fp32
void rope_table_run(float2* const band[3], const int rows[3], const int pairs[3], double base,
                    cudaStream_t stream);
// Debug probe: the kernel's own (t, h, w) index math for every local row.
void rope_positions_run(int64_t rows, int64_t row_offset, int64_t hw, int64_t grid_w,
                        int64_t start_frame, int32_t* t, int32_t* h, int32_t* w,
                        cudaStream_t stream);

// ---------------------------------------------------------------------------------------
// Byte movers (all-to-all / all-gather on any axes, any element width) and helpers.
// ---------------------------------------------------------------------------------------
struct Box4 {
    int64_t ext[4];     // extents copied
    int64_t src_str[4]; // element strides of the source
    int64_t dst_str[4];
};
void copy_box_run(void* dst, const void* src, const Box4& box, int elem_bytes, cudaStream_t s);

// K1 (Wan adaLN extension): y = LayerNorm(x) * (1 + scale) + shift, rows x dim bf16,
// shift/scale fp32 [dim] (modulate.cu); affine: y = LayerNorm(x) * scale + shift (Wan's norm3).
// mod_from_kernel: shift/scale are written by an earlier kernel of the stream (read after the
// PDL wait instead of before it)
void ln_modulate_run(const bf16* x, bf16* y, int64_t rows, int64_t dim, const float* shift,
                     const float* scale, float eps, cudaStream_t s, bool affine = false,
                     bool mod_from_kernel = false);

// ---------------------------------------------------------------------------------------
// Wan2.1 block extensions (wan.cu): timestep embedding + per-layer modulation, once per step.
// ---------------------------------------------------------------------------------------
struct WanTimeEmbed {
    const float* tsteps = nullptr;   // [denoise_steps] timesteps (device)
    int freq_dim = 256, dim = 0, layers = 0;
    const bf16* w1 = nullptr;        // [dim][freq_dim]
    const float* b1 = nullptr;
    const bf16* w2 = nullptr;        // [dim][dim]
    const float* b2 = nullptr;
    const bf16* wp = nullptr;        // [6 dim][dim]
    const float* bp = nullptr;
    const float* mod_param = nullptr;  // [layers][6][dim] per-layer modulation parameters
    float* sinus = nullptr;          // scratch [freq_dim]
    float* h1 = nullptr;             // scratch [dim]
    float* e = nullptr;              // [dim]
    float* e0 = nullptr;             // [6 dim]
    float* mod = nullptr;            // out [layers][6][dim] = mod_param + e0
};
void wan_time_embedding_run(const WanTimeEmbed& te, int step, cudaStream_t s);
// y[n] = act(sum_k W[n][k] act(x[k]) + b[n]) (SiLU on input and/or output), fp32 vectors
void gemv_run(const bf16* W, const float* b, const float* x, float* y, int N, int K, bool silu_in,
              bool silu_out, cudaStream_t s);
// counter-based N(offset, scale^2) fill (the Wan-block synthetic weights, seeded on device)
void fill_normal_bf16_run(bf16* out, int64_t n, uint64_t seed, float scale, float offset,
                          cudaStream_t s);
void fill_normal_f32_run(float* out, int64_t n, uint64_t seed, float scale, float offset,
                         cudaStream_t s);

// ---------------------------------------------------------------------------------------
// PEER transport: device-side rank barrier over IPC-mapped flag words. Each rank owns
// flags[kPeerSlots][P] (uint64, epoch values) followed by its private epoch counters
// [kPeerSlots]. After this stream's prior kernels (whose stores may target peer memory):
// epoch = ++counter[slot]; st.release.sys flags[slot][my_rank] = epoch in every rank's array,
// then spin (ld.acquire.sys) until every entry of flags[slot] >= epoch.
// ---------------------------------------------------------------------------------------
constexpr int kPeerSlots = 2;
constexpr int kMaxPeers = 8;
struct PeerFlags {
    uint64_t* rank_flags[kMaxPeers];  // every rank's flag array (this process's mapping)
};
// signal + wait as one PDL-chained 1-warp launch. The wait is bounded: after timeout_ns it
// stores 1 + (the first missing rank) into *error_word (host-mapped) and returns, so a dead or
// diverged peer surfaces as SPX_ERR_COLLECTIVE instead of a hung stream.
void peer_barrier_run(const PeerFlags& f, uint64_t* my_flags, int world, int my_rank, int slot,
                      uint64_t timeout_ns, int* error_word, cudaStream_t s);

// ---------------------------------------------------------------------------------------
// Kd: naive fp32 SIMT reference kernels (GPU oracle at shapes the CPU oracle cannot reach).
// ---------------------------------------------------------------------------------------
void naive_gemm_run(const bf16* a, const bf16* b, float* out, int M, int N, int K,
                    cudaStream_t s);
void naive_attention_run(const bf16* q, const bf16* k, const bf16* v, float* out, int batch,
                         int sq, int skv, int heads, int head_dim, cudaStream_t s);

}  // namespace spx
