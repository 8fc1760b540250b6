/*
 * spx.h -- C ABI of the B200-native Causal-RoPE sequence-parallel self-attention path.
 *
 * This is the drop-in boundary for the hot path of the reference "spattn" engine
 * (/root/reference/proj, namespace spattn). Every entry point cites the reference
 * interface it replaces (file:line under proj/). Conventions:
 *
 *   - plain C types only; tensors are caller-owned DEVICE pointers (bf16 unless stated)
 *     in the reference's row-major (B, S, H, D) layout (proj/include/spattn/tensor.hpp:12-14);
 *   - every call returns spx_status; on failure spx_last_error() holds a message
 *     (thread-local). No C++ exception crosses the ABI;
 *   - "stream" arguments are cudaStream_t passed as void* (NULL = legacy default stream);
 *   - allocation happens only in *_create calls (and spx_world_reserve), never in the
 *     per-layer hot path.
 */
#ifndef SPX_H_
#define SPX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPX_ABI_VERSION 1

/* 1:1 with the reference exception taxonomy (proj/include/spattn/errors.hpp:8-36),
 * plus device/transport failures the CPU reference cannot have. */
typedef enum spx_status {
    SPX_OK = 0,
    SPX_ERR_SHAPE = 1,       /* ShapeError       */
    SPX_ERR_PARTITION = 2,   /* PartitionError   */
    SPX_ERR_CONFIG = 3,      /* ConfigError      */
    SPX_ERR_RANGE = 4,       /* RangeError       */
    SPX_ERR_ALIGNMENT = 5,   /* AlignmentError   */
    SPX_ERR_EMPTY_CACHE = 6, /* EmptyCacheError  */
    SPX_ERR_COLLECTIVE = 7,  /* CollectiveError  */
    SPX_ERR_CUDA = 8,
    SPX_ERR_NCCL = 9,
    SPX_ERR_UNSUPPORTED = 10
} spx_status;

int spx_abi_version(void);
const char* spx_last_error(void);
const char* spx_status_name(int status);
/* number of spx kernels launched by this process so far (bench "gpu_launches" claim) */
int64_t spx_launch_count(void);
/* SM count of a device (host query; used to size persistent grids) */
spx_status spx_device_info(int device, int32_t out[4]); /* sm_count, cc_major, cc_minor, n_devices */

/* ---------------------------------------------------------------------------------------
 * Host RNG exactly as the reference draws its synthetic inputs
 * (Rng / derive_seed / random_tensor: proj/src/tensor.cpp:108-159).
 * ------------------------------------------------------------------------------------- */
uint64_t spx_derive_seed(uint64_t base, uint64_t a, uint64_t b, uint64_t c);
/* N(0,1)/sqrt(head_dim) noise of one block at one denoise step
 * (block_noise, proj/src/generator.cpp:42-46): n = B*L*H*D doubles */
spx_status spx_block_noise(uint64_t seed, int64_t block, int64_t step, int64_t n,
                           int64_t head_dim, double* out);
/* AttentionLayerParams::seeded(model_dim, derive_seed(seed, 0x20, layer))
 * (proj/src/sp_attention.cpp:29-40, generator.cpp:62-67): four [dim][dim] matrices */
spx_status spx_layer_weights(uint64_t seed, int64_t layer, int64_t model_dim, double* wq,
                             double* wk, double* wv, double* wo);
/* host fp64 -> bf16 (round to nearest even), n elements */
spx_status spx_f64_to_bf16(const double* in, uint16_t* out, int64_t n);
/* tensor_checksum (proj/src/report.cpp:264-279): FNV-1a over the fp64 bytes, 16 hex digits +
 * NUL in out[17] (reference-compatible reports of device outputs) */
spx_status spx_checksum_f64(const double* p, int64_t n, char out[17]);

/* ---------------------------------------------------------------------------------------
 * 3-D RoPE table (BandSplit / precompute_frequencies: proj/src/rope.cpp:15-64,
 * proj/include/spattn/rope.hpp:35-99). Built on the host in fp64 (the reference's exact
 * values), uploaded once per device as fp32 (cos, sin) pairs.
 * ------------------------------------------------------------------------------------- */
typedef struct spx_rope_table spx_rope_table;

spx_status spx_band_split_defaults(int64_t head_dim, int64_t out_split[3]);
/* split == NULL -> BandSplit::defaults_for(head_dim) */
spx_status spx_rope_table_create(int64_t max_frames, int64_t max_h, int64_t max_w,
                                 int64_t head_dim, double base, const int64_t* split,
                                 spx_rope_table** out);
void spx_rope_table_destroy(spx_rope_table* table);
/* out: max_frames, max_h, max_w, p_T, p_H, p_W, head_dim */
spx_status spx_rope_table_info(const spx_rope_table* table, int64_t out[7]);
/* band 0 = temporal, 1 = height, 2 = width (RopeFrequencyTable::cos_at/sin_at) */
spx_status spx_rope_table_at(const spx_rope_table* table, int32_t band, int64_t pos,
                             int64_t pair, double* cos_out, double* sin_out);

/* global_time_index (proj/src/rope.cpp:66-70) */
int64_t spx_global_time_index(int64_t i_local, int64_t rank, int64_t local_len, int64_t grid_hw,
                              int64_t start_frame);
/* (t, h, w) of every local row of rank `rank` (rotate_rows index math, rope.cpp:97-101),
 * computed by the SAME device function the fused kernel uses; t/h/w are device int32[L/P] */
spx_status spx_rope_positions(const int64_t grid[3], int64_t start_frame, int64_t rank,
                              int64_t world_size, int32_t* t, int32_t* h, int32_t* w,
                              void* stream);

/* K3: [QK-RMSNorm] + Causal-RoPE + bf16 cast (apply_rope_causal_local, rope.cpp:145-164).
 * x, y: device bf16 (B, L/P, H, D); y may alias x. norm_weight: NULL (reference semantics)
 * or device bf16 [H*D] for the Wan-mode RMSNorm over the model dimension. */
spx_status spx_rope_apply_causal_local(const spx_rope_table* table, const void* x, void* y,
                                       int64_t batch, int64_t local_len, int64_t heads,
                                       int64_t head_dim, const int64_t grid[3],
                                       int64_t start_frame, int64_t rank, int64_t world_size,
                                       const void* norm_weight, float norm_eps, void* stream);
/* apply_rope_global (rope.cpp:135-143): the P = 1 instance over a full block */
spx_status spx_rope_apply_global(const spx_rope_table* table, const void* x, void* y,
                                 int64_t batch, int64_t seq_len, int64_t heads, int64_t head_dim,
                                 const int64_t grid[3], int64_t start_frame, void* stream);

/* ---------------------------------------------------------------------------------------
 * Dense ops
 * ------------------------------------------------------------------------------------- */
/* K2/K8 project_tokens (proj/src/sp_attention.cpp:51-75): y[t,:] = W x[t,:].
 * x (tokens, c_in) bf16, w (c_out, c_in) bf16 row-major, y (tokens, c_out) bf16. */
spx_status spx_project_tokens(const void* x, const void* w, void* y, int64_t tokens,
                              int64_t c_in, int64_t c_out, void* stream);
/* project_tokens with the epilogues of the Wan block (extension): acc' = x W^T (+ bias[c_out]
 * fp32 when bias != NULL); epilogue 0: y = acc', 1: y = residual + gate * acc' (gate fp32
 * [c_out] or NULL = 1; residual (tokens, c_out) bf16, may alias y), 3: y = GELU_tanh(acc') */
spx_status spx_project_tokens_ex(const void* x, const void* w, void* y, int64_t tokens,
                                 int64_t c_in, int64_t c_out, const float* bias, int32_t epilogue,
                                 const void* residual, const float* gate, void* stream);
/* K6 scaled_dot_product_attention (proj/src/tensor.cpp:161-209), no mask.
 * q (B, Sq, H, D), k/v (B, Skv, H, D), o (B, Sq, H, D); bf16, B == 1, D in {64, 128} on the
 * tcgen05 kernel, D in {16, 32} (the reference default / desk shapes) on a SIMT kernel. */
spx_status spx_attention(const void* q, const void* k, const void* v, void* o, int64_t batch,
                         int64_t sq, int64_t skv, int64_t heads, int64_t head_dim, void* stream);

/* ---------------------------------------------------------------------------------------
 * Rolling KV ring (KvCache: proj/include/spattn/kv_cache.hpp:16-50, proj/src/kv_cache.cpp).
 * One device ring of capacity_frames frame slots; frames are appended in generation order,
 * the same block re-denoised overwrites its own slots, a window evicts whole frames from the
 * front. Reads never copy: attention walks the (at most two) chronological segments.
 * ------------------------------------------------------------------------------------- */
typedef struct spx_kv_ring spx_kv_ring;

/* window_frames < 0 -> unlimited; capacity_frames <= 0 -> derived: the window itself, or 64
 * frames when unlimited (an update that would need more than the capacity raises
 * SPX_ERR_RANGE; pass capacity_frames explicitly for longer unlimited caches) */
spx_status spx_kv_ring_create(int device, int64_t tokens_per_frame, int64_t window_frames,
                              int64_t capacity_frames, int64_t heads, int64_t head_dim,
                              spx_kv_ring** out);
void spx_kv_ring_destroy(spx_kv_ring* ring);
/* KvCache::update(block_index, k_block, v_block): k/v device bf16 (1, seq_len, H, D) */
spx_status spx_kv_ring_update(spx_kv_ring* ring, int64_t block_index, const void* k_block,
                              const void* v_block, int64_t seq_len, void* stream);
/* KvCache::read(): chronological copy (debug; the hot path never copies) */
spx_status spx_kv_ring_read(const spx_kv_ring* ring, void* k_out, void* v_out, void* stream);
/* out: cached_frames, seq_len, oldest_block_index (-1 if empty), capacity_frames */
spx_status spx_kv_ring_info(const spx_kv_ring* ring, int64_t out[4]);
/* attention of q (1, sq, H, D) over everything cached, o (1, sq, H, D) */
spx_status spx_kv_ring_attention(const spx_kv_ring* ring, const void* q, void* o, int64_t sq,
                                 void* stream);

/* ---------------------------------------------------------------------------------------
 * Communicator (CommWorld: proj/include/spattn/collectives.hpp:39-113,
 * proj/src/collectives.cpp). Three transports behind one interface:
 *   LOCAL : all ranks live in this process (one stream each; devices may repeat, i.e.
 *           several ranks can share one GPU); chunks move by direct (peer) stores.
 *   NCCL  : one rank per process, grouped ncclSend/ncclRecv over NVLink.
 *   PEER  : one rank per process; the engine's exchange buffers are shared through CUDA
 *           IPC, the producing kernels store straight into the peer's buffers (NVLink P2P,
 *           or the same device) and device-side flags order the ranks (engine only: the
 *           standalone collectives below need LOCAL or NCCL).
 * Buffers passed to the collectives are indexed by LOCAL rank (1 entry for NCCL).
 * ------------------------------------------------------------------------------------- */
typedef struct spx_world spx_world;

typedef struct spx_comm_stats {
    int64_t all_gather;
    int64_t all_to_all;
    int64_t fused_all_to_all;
    int64_t elements_sent;
    int64_t rounds;
} spx_comm_stats; /* CommStats, collectives.hpp:20-33 */

enum { SPX_AXIS_BATCH = 0, SPX_AXIS_SEQ = 1, SPX_AXIS_HEADS = 2, SPX_AXIS_HEAD_DIM = 3 };
enum { SPX_TRANSPORT_LOCAL = 0, SPX_TRANSPORT_NCCL = 1, SPX_TRANSPORT_PEER = 2 };

/* devices == NULL -> every rank on the current device */
spx_status spx_world_create_local(int world_size, const int* devices, spx_world** out);
spx_status spx_nccl_get_unique_id(uint8_t out_id[128]);
/* PEER transport: rank `rank` of `world_size`, one per process, on `device`. An engine made
 * on it exchanges buffer handles once (spx_engine_ipc_export / _import) before running. */
spx_status spx_world_create_peer(int rank, int world_size, int device, spx_world** out);
spx_status spx_world_create_nccl(int rank, int world_size, const uint8_t id[128], int device,
                                 spx_world** out);
void spx_world_destroy(spx_world* world);
/* out: world_size, local_ranks, first_local_rank, transport */
spx_status spx_world_info(const spx_world* world, int32_t out[4]);
spx_status spx_world_stream(const spx_world* world, int local_rank, void** stream_out);
spx_status spx_world_synchronize(spx_world* world);
spx_status spx_world_stats(const spx_world* world, spx_comm_stats* out);
spx_status spx_world_reset_stats(spx_world* world);

/* NCCL transport: size the staging buffer of the standalone collectives up front (bytes;
 * all_to_all needs 2 x P x its per-rank input, fused_all_to_all 6 x P x one tensor's,
 * all_gather P x its input). Without it the first call of a larger size allocates once. */
spx_status spx_world_reserve(spx_world* world, int64_t bytes);
/* all_to_all(rank, x, scatter, gather) (collectives.cpp:203-235); shape = per-rank input
 * (B, S, H, D); elem_bytes in {1,2,4,8}; out holds the per-rank result */
spx_status spx_all_to_all(spx_world* world, void* const* in, void* const* out,
                          const int64_t shape[4], int32_t elem_bytes, int32_t scatter_axis,
                          int32_t gather_axis);
/* fused_all_to_all(rank, q, k, v) (collectives.cpp:237-276): one invocation, one round --
 * on NCCL one group, one message per peer carrying the q, k and v chunks */
spx_status spx_fused_all_to_all(spx_world* world, void* const* q_in, void* const* k_in,
                                void* const* v_in, void* const* q_out, void* const* k_out,
                                void* const* v_out, const int64_t shape[4], int32_t elem_bytes,
                                int32_t scatter_axis, int32_t gather_axis);
/* all_gather(rank, x, dim) (collectives.cpp:180-201) */
spx_status spx_all_gather(spx_world* world, void* const* in, void* const* out,
                          const int64_t shape[4], int32_t elem_bytes, int32_t axis);

/* Partition of P ranks over H heads and a block of L tokens: out = G (head groups),
 * S (query splits), L/P, L/S, H/G. Ulysses (S = 1) whenever H % P == 0. */
spx_status spx_partition(int32_t world_size, int64_t heads, int64_t block_len, int64_t head_dim,
                         int64_t out[5]);
/* The cross-rank transfers one rank posts in one exchange round (which = 0: q/k/v exchange
 * replacing fused_all_to_all, collectives.cpp:237-276; which = 1: output all_to_all,
 * collectives.cpp:203-235), in posting order. Row i of out (6 int64): peer, is_send,
 * buffer id (0 q_send, 1 k_send, 2 v_send, 3 o_send, 4 q_recv, 5 ring_k, 6 ring_v, 7 o_recv),
 * element offset, element count, 0. The NCCL transport executes exactly this list. */
spx_status spx_exchange_plan(int32_t which, int32_t rank, int32_t world_size, int64_t heads,
                             int64_t block_len, int64_t head_dim, int64_t block_base_row,
                             int64_t* out, int64_t max_entries, int64_t* n_entries);

/* ---------------------------------------------------------------------------------------
 * Engine: the optimized Causal-RoPE SP schedule (sp_self_attention_engine, all flags on:
 * proj/src/sp_attention.cpp:197-313) and the block-wise AR driver (generate:
 * proj/src/generator.cpp:50-147) on device.
 *
 *   x_local --K2 QKV GEMM--> qkv --K3 [norm]+Causal-RoPE+pack--> {q, k, v} straight into the
 *   destination ranks' q buffers and KV-ring slots (one fused exchange round)
 *   --K6 attention over the ring--> o straight into the sources' output slabs (one round)
 *   --K8 O GEMM (3-D TMA un-interleaves the head-group slabs)--> y_local
 *
 * Ulysses needs H % P == 0; otherwise P = G * S with G head groups (G | H) and S query
 * splits (the P = 8, H = 12 case runs 4 head groups x 2 query halves).
 * ------------------------------------------------------------------------------------- */
typedef struct spx_engine spx_engine;

/* AblationFlags bits (proj/include/spattn/sp_attention.hpp:36-44) */
#define SPX_ABLATION_FUSED_ALL_TO_ALL 1
#define SPX_ABLATION_LOCAL_ROPE 2
#define SPX_ABLATION_PRECOMPUTED_FREQS 4
#define SPX_ABLATION_ALL 7

typedef struct spx_engine_config {
    int64_t frames, grid_h, grid_w;   /* GridSpec per block (F = tau, H_g, W_g) */
    int64_t num_blocks;
    int64_t layers;
    int64_t denoise_steps;
    int64_t batch;                    /* must be 1 on device */
    int64_t heads;
    int64_t head_dim;
    int64_t window_frames;            /* < 0: unlimited */
    double rope_base;
    int64_t band_split[3];            /* all < 0: BandSplit::defaults_for(head_dim) */
    uint64_t seed;
    int32_t force_start_frame_zero;   /* fault injection (generator.hpp:30-32) */
    int32_t qk_norm;                  /* 0 = reference semantics; 1 = Wan QK-RMSNorm */
    float norm_eps;
    int32_t profile;                  /* 1: CUDA-event stage timing on every call;
                                         2: the attention launch only */
    int32_t fuse_rope_epilogue;       /* 1 (default): Causal-RoPE + pack in the QKV GEMM
                                         epilogue when qk_norm = 0; 0: standalone K3 kernel */
    int32_t ablation;                 /* AblationFlags (sp_attention.hpp:36-44) as bits:
                                         1 use_fused_all_to_all, 2 use_local_rope,
                                         4 use_precomputed_freqs; 7 = optimized (default),
                                         0 = the baseline Alg. 1 schedule */
    int32_t adaln;                    /* 0 = reference semantics; 1 = the Wan block's adaLN
                                         modulation: x_in = LN(x)(1 + scale) + shift before
                                         the QKV projection (K1), x + gate * W_o o in the
                                         O-projection epilogue (extension, no reference
                                         counterpart; per-layer shift/scale/gate) */
    int32_t l2_prefetch;              /* 1: the attention kernel warms the next projections'
                                         weights into L2 (bulk prefetch); 0 (default) since
                                         the weight-tile-early GEMM pipelines made it a net
                                         loss under the power cap */
    /* The full Wan2.1 DiT block (extension; the reference model is attention-only).
     * wan_block = 1 implies adaln = qk_norm = 1 and adds, per layer, biases on every
     * projection, the cross-attention to text_len cached context tokens (affine LayerNorm,
     * QK-RMSNorm, K/V computed once per video by spx_engine_set_context) and the GELU(tanh)
     * FFN dim -> ffn_dim -> dim, each with its residual; the six per-layer modulation vectors
     * come from the timestep embedding of the current denoise step (freq_dim sinusoid, two
     * Linear layers, SiLU, Linear to 6 dim) plus the layer's modulation parameters. */
    int32_t wan_block;
    int64_t ffn_dim;                  /* <= 0: ceil(dim * 35 / 6 / 64) * 64 (8960 at 1536) */
    int64_t text_len;                 /* context tokens (512) */
    int64_t text_dim;                 /* raw context width (4096, the umT5 encoder's) */
    int64_t freq_dim;                 /* sinusoidal timestep embedding width (256) */
    int32_t sp_bit_exact;             /* 1: attention never splits a query tile's kv range over
                                         CTAs, so every partition P = G x S keeps the P = 1
                                         summation order and SP outputs equal P = 1 bit for bit
                                         (the reference's invariant); 0 (default): split-KV
                                         layouts where the per-rank grid under-fills the SMs
                                         (P = 2, 8 at the Wan shape), outputs within bf16
                                         rounding of P = 1 */
} spx_engine_config;

/* GenerationConfig defaults (proj/include/spattn/generator.hpp:14-42) */
void spx_engine_config_defaults(spx_engine_config* cfg);
/* GenerationConfig::validate (proj/src/generator.cpp:7-38) + device constraints */
spx_status spx_engine_config_validate(const spx_engine_config* cfg, int32_t world_size);
spx_status spx_engine_create(spx_world* world, const spx_engine_config* cfg, spx_engine** out);
void spx_engine_destroy(spx_engine* engine);
/* out: G (head groups), S (query splits), L (block len), L/P, heads per group, query rows
 * per rank, kv ring capacity frames, model dim */
spx_status spx_engine_info(const spx_engine* engine, int64_t out[8]);
/* weights from the reference's seeded init, rounded to bf16 (host -> every device) */
spx_status spx_engine_seed_weights(spx_engine* engine);
/* explicit weights: host bf16 [dim][dim] each ([out][in], y = W x) */
spx_status spx_engine_set_layer_weights(spx_engine* engine, int64_t layer, const uint16_t* wq,
                                        const uint16_t* wk, const uint16_t* wv,
                                        const uint16_t* wo);
/* QK-RMSNorm weights (host bf16 [dim] each); only used when cfg.qk_norm = 1 */
/* adaLN modulation of one layer (fp32 [dim] each; used when cfg.adaln = 1). Default: seeded
 * N(0, 1)/sqrt(dim), the Wan modulation-parameter init, from derive_seed(seed, 0x30, layer). */
spx_status spx_engine_set_modulation(spx_engine* engine, int64_t layer, const float* shift,
                                     const float* scale, const float* gate);
spx_status spx_engine_set_norm_weights(spx_engine* engine, int64_t layer, const uint16_t* wq,
                                       const uint16_t* wk);
/* KvCache::update bookkeeping for a block (once per denoise step; every layer's ring gets
 * the same slots) -- generate() calls this itself */
spx_status spx_engine_begin_block(spx_engine* engine, int64_t block_index);
/* start a new video: every layer's KV cache empty (a fresh generate() builds new caches,
 * generator.cpp:69-81); waits for the engine's streams */
spx_status spx_engine_reset_cache(spx_engine* engine);
/* one optimized_sp_self_attention call on every local rank: x_local / y_local are device
 * bf16 (1, L/P, H, D), indexed by local rank; y may not alias x */
spx_status spx_engine_layer(spx_engine* engine, int64_t layer, int64_t block_index,
                            int64_t start_frame, void* const* x_local, void* const* y_local);
/* the whole block (denoise_steps x layers calls). noise_host: bf16 (steps, L, H, D) of the
 * FULL block or NULL (draw it from cfg.seed with the reference RNG); out_host: bf16
 * (L/P, H, D) rows of every local rank in rank order (a full block on a LOCAL world).
 * Host buffers should be pinned for async copies. */
spx_status spx_engine_generate_block(spx_engine* engine, int64_t block, const uint16_t* noise_host,
                                     uint16_t* out_host);
/* device-resident variant for benchmarking: noise_dev[local rank] holds (steps, L/P, H, D),
 * out_dev[local rank] receives (L/P, H, D); asynchronous on the world's streams */
spx_status spx_engine_generate_block_device(spx_engine* engine, int64_t block,
                                            const void* const* noise_dev, void* const* out_dev);
/* streaming generator: n blocks back to back (blocks[i] may repeat -- a block denoised again
 * overwrites its own KV slots); noise_host[i]: bf16 (steps, L, H, D) of the FULL block i,
 * out_host[i]: bf16 rows of the local ranks (rank order). The upload of the next step's noise
 * and the download of the previous block's latent run on their own streams, overlapped with
 * the compute; returns when every latent is on the host. Host buffers must be pinned. */
spx_status spx_engine_generate_stream(spx_engine* engine, const int64_t* blocks, int64_t n,
                                      const uint16_t* const* noise_host, uint16_t* const* out_host);
/* ---- the full Wan2.1 block (cfg.wan_block = 1; extension) ----
 * Per-layer weights (host pointers; [out][in] row-major bf16 matrices, fp32 vectors). The
 * self-attention projections themselves are spx_engine_set_layer_weights, its QK-RMSNorm
 * weights spx_engine_set_norm_weights; this sets everything else of the layer. */
typedef struct spx_wan_layer_weights {
    const float *self_bq, *self_bk, *self_bv, *self_bo;      /* [dim] */
    const float *norm3_w, *norm3_b;                          /* [dim] affine LayerNorm */
    const uint16_t *cross_q, *cross_k, *cross_v, *cross_o;   /* [dim][dim] */
    const float *cross_bq, *cross_bk, *cross_bv, *cross_bo;  /* [dim] */
    const uint16_t *cross_norm_q, *cross_norm_k;             /* [dim] RMSNorm weights */
    const uint16_t* ffn_w1;                                  /* [ffn_dim][dim] */
    const float* ffn_b1;                                     /* [ffn_dim] */
    const uint16_t* ffn_w2;                                  /* [dim][ffn_dim] */
    const float* ffn_b2;                                     /* [dim] */
    const float* modulation;                                 /* [6][dim] */
} spx_wan_layer_weights;
spx_status spx_engine_set_wan_layer(spx_engine* engine, int64_t layer,
                                    const spx_wan_layer_weights* w);
/* the embeddings shared by all layers */
typedef struct spx_wan_embed_weights {
    const uint16_t* time_w1; const float* time_b1;  /* [dim][freq_dim], [dim] */
    const uint16_t* time_w2; const float* time_b2;  /* [dim][dim], [dim] */
    const uint16_t* proj_w;  const float* proj_b;   /* [6 dim][dim], [6 dim] */
    const uint16_t* text_w1; const float* text_b1;  /* [dim][text_dim], [dim] */
    const uint16_t* text_w2; const float* text_b2;  /* [dim][dim], [dim] */
} spx_wan_embed_weights;
spx_status spx_engine_set_wan_embeddings(spx_engine* engine, const spx_wan_embed_weights* w);
/* timesteps of the denoise steps (host fp32 [denoise_steps]; default 1000 -> 250 evenly) */
spx_status spx_engine_set_timesteps(spx_engine* engine, const float* t);
/* a video's text context (host bf16 [text_len][text_dim]): runs the text embedding and every
 * layer's cross-attention K (RMSNorm'd) and V once; they stay cached until the next call */
spx_status spx_engine_set_context(spx_engine* engine, const uint16_t* text);

/* per-step CUDA graphs (default on): the layer calls of a denoise step are captured once per
 * KV-ring state and replayed (one launch per step instead of 3 x layers), on a world with one
 * local rank (PEER, or LOCAL P = 1), the optimized schedule and profiling off; off = every
 * kernel enqueued by the host (SPX_GRAPHS=0 at load time does the same) */
spx_status spx_engine_set_graphs(spx_engine* engine, int32_t on);
/* number of per-step graphs the engine holds (tests) */
spx_status spx_debug_engine_graphs(const spx_engine* engine, int64_t* count);
/* one denoise step of a block (the per-step body of generate, generator.cpp:94-110):
 * KvCache::update of the block, then every layer on x_local[local rank] (device bf16
 * (L/P, H, D)) into y_local[local rank]; asynchronous on the world's streams */
spx_status spx_engine_denoise_step(spx_engine* engine, int64_t block, int64_t step,
                                   const void* const* x_local, void* const* y_local);
/* generate(cfg): every block; out_host: (num_blocks, rows_local, H, D) bf16 */
spx_status spx_engine_generate(spx_engine* engine, uint16_t* out_host);
spx_status spx_engine_synchronize(spx_engine* engine);
/* per-stage device time (ms, summed over calls on local rank 0) in the reference's stage
 * order qkv, rope, gather_or_fused, cache, attention, output_exchange
 * (sp_attention.hpp:92-97); calls = number of profiled layer calls */
spx_status spx_engine_stage_times(spx_engine* engine, double out_ms[6], int64_t* calls);
spx_status spx_engine_reset_stage_times(spx_engine* engine);
/* CUDA-event stage timing for subsequent calls: 0 off, 1 every stage, 2 attention only,
 * 3 attention only on every 8th call (a sample that keeps PDL chaining of the others) */
spx_status spx_engine_set_profile(spx_engine* engine, int32_t on);
spx_status spx_engine_stats(const spx_engine* engine, spx_comm_stats* out);
/* PEER transport: this rank's exchange buffers as CUDA IPC handles (an opaque blob of
 * *bytes <= capacity; query the size with out == NULL). Every rank gathers all blobs in rank
 * order (any host channel: torch.distributed, MPI, a file) and passes them to _import. */
spx_status spx_engine_ipc_export(spx_engine* engine, void* out, int64_t capacity, int64_t* bytes);
spx_status spx_engine_ipc_import(spx_engine* engine, const void* blobs, int64_t bytes_per_rank);

/* verify_stream(cfg, tol) (proj/src/generator.cpp:149-177, generator.hpp:65-83): runs cfg on a
 * LOCAL world of world_size ranks (devices[r], NULL = all on the current device) and the
 * P = 1 optimized path (= the reference pipeline at P = 1, true start frames) with the same
 * seeded weights and noise, and reports per block the max |variant - expected| over the bf16
 * outputs. blocks[] needs num_blocks entries; ledger (optional) = the variant's CommStats. */
typedef struct spx_verify_block {
    int64_t block;
    double max_abs_dev;
    int32_t pass;
} spx_verify_block;
spx_status spx_verify_stream(const spx_engine_config* cfg, int32_t world_size, const int* devices,
                             double tolerance, spx_verify_block* blocks, int64_t max_blocks,
                             int32_t* pass, spx_comm_stats* ledger);

/* ---------------------------------------------------------------------------------------
 * Debug / GPU-oracle kernels (fp32 SIMT; tests only)
 * ------------------------------------------------------------------------------------- */
spx_status spx_debug_naive_gemm(const void* a, const void* b, float* out, int64_t m, int64_t n,
                                int64_t k, void* stream);
/* K1 (Wan adaLN extension) on device buffers: y = LayerNorm(x)(1 + scale) + shift over the
 * last dim; x, y (tokens, dim) bf16; shift, scale fp32 [dim] device pointers. */
spx_status spx_layernorm_modulate(const void* x, void* y, int64_t tokens, int64_t dim,
                                  const float* shift, const float* scale, float eps, void* stream);
/* Force the projection GEMM tile variant for plans made after the call: -1 = the planner's
 * modelled choice; 0 pair 256x256, 1 pair 256x128, 2 single 128x256, 3 single 128x128,
 * 4 single 128x192 (tests and tuning; also SPX_GEMM_VARIANT at load time). */
spx_status spx_debug_set_gemm_variant(int32_t variant);
/* Force the attention kernel's kv splits per query tile (1..8) for plans made after the call;
 * 0 = the planner's wave model (tests and tuning; also SPX_ATTN_SPLITS at load time). */
spx_status spx_debug_set_attn_splits(int32_t splits);
/* attention kernel for unsplit layouts: v3 = one O accumulator shared by both softmax slots,
 * separate P buffers, S(j+1) issued while the softmax works on S(j); v2 = per-slot O with P
 * written over S. 0 = always v2, 1 (default) = v3 when the layout fills >= one wave of SMs (or
 * the run asks for exact SP layouts), 2 = always v3; also SPX_ATTN_V3 at load time */
spx_status spx_debug_set_attn_v3(int32_t on);
/* SPX_SPAN_TRACE=1 only: per traced launch (GEMM, attention, in launch order) the earliest CTA
 * start and the latest CTA end, globaltimer ns: out[2 i], out[2 i + 1] (capacity u64 slots). */
spx_status spx_debug_spans(uint64_t* out, int64_t capacity, int64_t* count);
/* SPX_GEMM_EXPERIMENT=5 only: copy n of the pair GEMM's per-tile clock64 marks of the last
 * launch ([cta][16 tiles][mma start, mma issued, epilogue start, epilogue end]) */
spx_status spx_debug_gemm_trace(int64_t* out, int64_t n);
spx_status spx_debug_naive_attention(const void* q, const void* k, const void* v, float* out,
                                     int64_t batch, int64_t sq, int64_t skv, int64_t heads,
                                     int64_t head_dim, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPX_H_ */
