"""ctypes binding of libspx.so (include/spx.h).

The product path is the C++/CUDA library; this module only loads it and maps its status
codes onto the reference's exception taxonomy (proj/include/spattn/errors.hpp:8-36). There is
no Python fallback: if libspx.so is missing, importing anything that needs it raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_int64, c_uint8, c_uint16, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPX_LIB: an alternative build of the same library (tools/build_variant.sh experiments)
LIB_PATH = os.environ.get("SPX_LIB") or os.path.join(_HERE, "libspx.so")


class SpxError(RuntimeError):
    """Base class; `status` is the spx_status code."""

    status = -1


class ShapeError(SpxError):
    status = 1


class PartitionError(SpxError):
    status = 2


class ConfigError(SpxError):
    status = 3


class RangeError(SpxError):
    status = 4


class AlignmentError(SpxError):
    status = 5


class EmptyCacheError(SpxError):
    status = 6


class CollectiveError(SpxError):
    status = 7


class CudaError(SpxError):
    status = 8


class NcclError(SpxError):
    status = 9


class UnsupportedError(SpxError):
    status = 10


_BY_STATUS = {cls.status: cls for cls in (ShapeError, PartitionError, ConfigError, RangeError,
                                          AlignmentError, EmptyCacheError, CollectiveError,
                                          CudaError, NcclError, UnsupportedError)}


class CommStats(ctypes.Structure):
    """CommStats (proj/include/spattn/collectives.hpp:20-33)."""

    _fields_ = [("all_gather", c_int64), ("all_to_all", c_int64), ("fused_all_to_all", c_int64),
                ("elements_sent", c_int64), ("rounds", c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class EngineConfig(ctypes.Structure):
    """spx_engine_config: GenerationConfig (proj/include/spattn/generator.hpp:14-42) + device knobs."""

    _fields_ = [("frames", c_int64), ("grid_h", c_int64), ("grid_w", c_int64),
                ("num_blocks", c_int64), ("layers", c_int64), ("denoise_steps", c_int64),
                ("batch", c_int64), ("heads", c_int64), ("head_dim", c_int64),
                ("window_frames", c_int64), ("rope_base", c_double),
                ("band_split", c_int64 * 3), ("seed", c_uint64),
                ("force_start_frame_zero", c_int32), ("qk_norm", c_int32),
                ("norm_eps", c_float), ("profile", c_int32),
                ("fuse_rope_epilogue", c_int32), ("ablation", c_int32), ("adaln", c_int32),
                ("l2_prefetch", c_int32), ("wan_block", c_int32), ("ffn_dim", c_int64),
                ("text_len", c_int64), ("text_dim", c_int64), ("freq_dim", c_int64),
                ("sp_bit_exact", c_int32)]


WAN_LAYER_FIELDS = ("self_bq", "self_bk", "self_bv", "self_bo", "norm3_w", "norm3_b", "cross_q",
                    "cross_k", "cross_v", "cross_o", "cross_bq", "cross_bk", "cross_bv", "cross_bo",
                    "cross_norm_q", "cross_norm_k", "ffn_w1", "ffn_b1", "ffn_w2", "ffn_b2",
                    "modulation")
WAN_EMBED_FIELDS = ("time_w1", "time_b1", "time_w2", "time_b2", "proj_w", "proj_b", "text_w1",
                    "text_b1", "text_w2", "text_b2")


class WanLayerWeights(ctypes.Structure):
    """spx_wan_layer_weights (include/spx.h): host pointers, NULL = leave unchanged."""

    _fields_ = [(n, c_void_p) for n in WAN_LAYER_FIELDS]


class WanEmbedWeights(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in WAN_EMBED_FIELDS]


class VerifyBlock(ctypes.Structure):
    """spx_verify_block: VerificationReport::BlockCheck (proj/include/spattn/generator.hpp:68-73)."""

    _fields_ = [("block", c_int64), ("max_abs_dev", c_double), ("pass_", c_int32)]


# (name, restype, argtypes); restype None for void
_SIGS = [
    ("spx_abi_version", c_int, []),
    ("spx_last_error", c_char_p, []),
    ("spx_status_name", c_char_p, [c_int]),
    ("spx_launch_count", c_int64, []),
    ("spx_device_info", c_int, [c_int, POINTER(c_int32)]),
    ("spx_derive_seed", c_uint64, [c_uint64, c_uint64, c_uint64, c_uint64]),
    ("spx_block_noise", c_int, [c_uint64, c_int64, c_int64, c_int64, c_int64, POINTER(c_double)]),
    ("spx_layer_weights", c_int, [c_uint64, c_int64, c_int64, POINTER(c_double), POINTER(c_double),
                                  POINTER(c_double), POINTER(c_double)]),
    ("spx_f64_to_bf16", c_int, [POINTER(c_double), POINTER(c_uint16), c_int64]),
    ("spx_band_split_defaults", c_int, [c_int64, POINTER(c_int64)]),
    ("spx_rope_table_create", c_int, [c_int64, c_int64, c_int64, c_int64, c_double, POINTER(c_int64),
                                      POINTER(c_void_p)]),
    ("spx_rope_table_destroy", None, [c_void_p]),
    ("spx_rope_table_info", c_int, [c_void_p, POINTER(c_int64)]),
    ("spx_rope_table_at", c_int, [c_void_p, c_int32, c_int64, c_int64, POINTER(c_double),
                                  POINTER(c_double)]),
    ("spx_global_time_index", c_int64, [c_int64, c_int64, c_int64, c_int64, c_int64]),
    ("spx_rope_positions", c_int, [POINTER(c_int64), c_int64, c_int64, c_int64, c_void_p, c_void_p,
                                   c_void_p, c_void_p]),
    ("spx_rope_apply_causal_local", c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64,
                                            c_int64, POINTER(c_int64), c_int64, c_int64, c_int64,
                                            c_void_p, c_float, c_void_p]),
    ("spx_rope_apply_global", c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64,
                                      c_int64, POINTER(c_int64), c_int64, c_void_p]),
    ("spx_project_tokens", c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p]),
    ("spx_project_tokens_ex", c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p,
                                      c_int32, c_void_p, c_void_p, c_void_p]),
    ("spx_attention", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64,
                              c_int64, c_int64, c_void_p]),
    ("spx_kv_ring_create", c_int, [c_int, c_int64, c_int64, c_int64, c_int64, c_int64,
                                   POINTER(c_void_p)]),
    ("spx_kv_ring_destroy", None, [c_void_p]),
    ("spx_kv_ring_update", c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_void_p]),
    ("spx_kv_ring_read", c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    ("spx_kv_ring_info", c_int, [c_void_p, POINTER(c_int64)]),
    ("spx_kv_ring_attention", c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    ("spx_world_create_local", c_int, [c_int, POINTER(c_int), POINTER(c_void_p)]),
    ("spx_nccl_get_unique_id", c_int, [POINTER(c_uint8)]),
    ("spx_world_create_nccl", c_int, [c_int, c_int, POINTER(c_uint8), c_int, POINTER(c_void_p)]),
    ("spx_world_destroy", None, [c_void_p]),
    ("spx_world_info", c_int, [c_void_p, POINTER(c_int32)]),
    ("spx_world_stream", c_int, [c_void_p, c_int, POINTER(c_void_p)]),
    ("spx_world_synchronize", c_int, [c_void_p]),
    ("spx_world_stats", c_int, [c_void_p, POINTER(CommStats)]),
    ("spx_world_reset_stats", c_int, [c_void_p]),
    ("spx_world_reserve", c_int, [c_void_p, c_int64]),
    ("spx_all_to_all", c_int, [c_void_p, POINTER(c_void_p), POINTER(c_void_p), POINTER(c_int64),
                               c_int32, c_int32, c_int32]),
    ("spx_fused_all_to_all", c_int, [c_void_p] + [POINTER(c_void_p)] * 6 + [POINTER(c_int64), c_int32,
                                                                           c_int32, c_int32]),
    ("spx_all_gather", c_int, [c_void_p, POINTER(c_void_p), POINTER(c_void_p), POINTER(c_int64),
                               c_int32, c_int32]),
    ("spx_partition", c_int, [c_int32, c_int64, c_int64, c_int64, POINTER(c_int64)]),
    ("spx_exchange_plan", c_int, [c_int32, c_int32, c_int32, c_int64, c_int64, c_int64, c_int64,
                                  POINTER(c_int64), c_int64, POINTER(c_int64)]),
    ("spx_engine_config_defaults", None, [POINTER(EngineConfig)]),
    ("spx_engine_config_validate", c_int, [POINTER(EngineConfig), c_int32]),
    ("spx_engine_create", c_int, [c_void_p, POINTER(EngineConfig), POINTER(c_void_p)]),
    ("spx_engine_destroy", None, [c_void_p]),
    ("spx_engine_info", c_int, [c_void_p, POINTER(c_int64)]),
    ("spx_engine_seed_weights", c_int, [c_void_p]),
    ("spx_engine_set_layer_weights", c_int, [c_void_p, c_int64] + [c_void_p] * 4),
    ("spx_engine_set_norm_weights", c_int, [c_void_p, c_int64, c_void_p, c_void_p]),
    ("spx_engine_begin_block", c_int, [c_void_p, c_int64]),
    ("spx_engine_reset_cache", c_int, [c_void_p]),
    ("spx_engine_layer", c_int, [c_void_p, c_int64, c_int64, c_int64, POINTER(c_void_p),
                                 POINTER(c_void_p)]),
    ("spx_engine_generate_block", c_int, [c_void_p, c_int64, c_void_p, c_void_p]),
    ("spx_engine_generate_block_device", c_int, [c_void_p, c_int64, POINTER(c_void_p), POINTER(c_void_p)]),
    ("spx_engine_generate", c_int, [c_void_p, c_void_p]),
    ("spx_engine_generate_stream", c_int, [c_void_p, POINTER(c_int64), c_int64, POINTER(c_void_p),
                                           POINTER(c_void_p)]),
    ("spx_engine_set_graphs", c_int, [c_void_p, c_int32]),
    ("spx_engine_set_wan_layer", c_int, [c_void_p, c_int64, POINTER(WanLayerWeights)]),
    ("spx_engine_set_wan_embeddings", c_int, [c_void_p, POINTER(WanEmbedWeights)]),
    ("spx_engine_set_timesteps", c_int, [c_void_p, c_void_p]),
    ("spx_engine_set_context", c_int, [c_void_p, c_void_p]),
    ("spx_debug_engine_graphs", c_int, [c_void_p, POINTER(c_int64)]),
    ("spx_engine_denoise_step", c_int, [c_void_p, c_int64, c_int64, POINTER(c_void_p), POINTER(c_void_p)]),
    ("spx_verify_stream", c_int, [POINTER(EngineConfig), c_int32, POINTER(c_int), c_double,
                                  POINTER(VerifyBlock), c_int64, POINTER(c_int32), POINTER(CommStats)]),
    ("spx_engine_synchronize", c_int, [c_void_p]),
    ("spx_engine_stage_times", c_int, [c_void_p, POINTER(c_double), POINTER(c_int64)]),
    ("spx_engine_reset_stage_times", c_int, [c_void_p]),
    ("spx_engine_set_profile", c_int, [c_void_p, c_int32]),
    ("spx_engine_stats", c_int, [c_void_p, POINTER(CommStats)]),
    ("spx_world_create_peer", c_int, [c_int, c_int, c_int, c_void_p]),
    ("spx_checksum_f64", c_int, [c_void_p, c_int64, c_char_p]),
    ("spx_engine_set_modulation", c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    ("spx_layernorm_modulate", c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_float,
                                       c_void_p]),
    ("spx_engine_ipc_export", c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    ("spx_engine_ipc_import", c_int, [c_void_p, c_void_p, c_int64]),
    ("spx_debug_set_gemm_variant", c_int, [c_int32]),
    ("spx_debug_set_attn_splits", c_int, [c_int32]),
    ("spx_debug_set_attn_v3", c_int, [c_int32]),
    ("spx_debug_spans", c_int, [c_void_p, c_int64, c_void_p]),
    ("spx_debug_gemm_trace", c_int, [c_void_p, c_int64]),
    ("spx_debug_naive_gemm", c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p]),
    ("spx_debug_naive_attention", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                                          c_int64, c_int64, c_int64, c_void_p]),
]

EXPORTED = [name for name, _, _ in _SIGS]

_lib = None


def lib():
    """Load libspx.so once; raises if it was not built (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(make -C paper_2603_06664_b200/csrc)")
        handle = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, res, args in _SIGS:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().spx_last_error().decode(errors="replace")
        raise _BY_STATUS.get(status, SpxError)(msg)


def i64_array(values):
    arr = (c_int64 * len(values))(*values)
    return arr


def ptr_array(ptrs):
    return (c_void_p * len(ptrs))(*[c_void_p(int(p)) for p in ptrs])
