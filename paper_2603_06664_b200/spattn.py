"""Python mirror of the reference operator API (namespace spattn, proj/include/spattn/*.hpp)
over the B200 C ABI (include/spx.h, libspx.so).

Same names, argument meaning and error classes as the reference, so a caller -- and the
parity tests -- read like proj/tests. Differences forced by the device:
  * tensors are torch CUDA bf16 tensors in the reference's (B, S, H, D) layout;
  * the reference calls collectives per rank inside CommWorld::run threads; here one call
    moves the buffers of every rank of a LOCAL world (lists indexed by rank);
  * KvCache lives on the device and attention reads it in place (KvCache.attention).
torch is used only to own device memory and streams.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (AlignmentError, CollectiveError, ConfigError, EmptyCacheError, PartitionError,  # noqa: F401
                   RangeError, ShapeError, SpxError, UnsupportedError, check, i64_array, lib, ptr_array)


def _torch():
    import torch

    return torch


def _stream():
    return _torch().cuda.current_stream().cuda_stream


def _bf16(t):
    torch = _torch()
    if not (t.is_cuda and t.dtype == torch.bfloat16 and t.is_contiguous()):
        raise ShapeError("expected a contiguous CUDA bf16 tensor")
    return t


class Axis(enum.IntEnum):
    """Axis (proj/include/spattn/tensor.hpp:16)."""

    Batch = 0
    Seq = 1
    Heads = 2
    HeadDim = 3


@dataclass(frozen=True)
class GridSpec:
    """GridSpec (rope.hpp:13-21): F frames of H_g x W_g tokens, row-major (t, h, w)."""

    frames: int
    height: int
    width: int

    def tokens_per_frame(self) -> int:
        return self.height * self.width

    def seq_len(self) -> int:
        return self.frames * self.height * self.width

    def as_array(self):
        return i64_array([self.frames, self.height, self.width])


@dataclass(frozen=True)
class BandSplit:
    """BandSplit (rope.hpp:35-44)."""

    temporal: int
    height: int
    width: int

    def total(self) -> int:
        return self.temporal + self.height + self.width

    @staticmethod
    def defaults_for(head_dim: int) -> "BandSplit":
        out = i64_array([0, 0, 0])
        check(lib().spx_band_split_defaults(head_dim, out))
        return BandSplit(*out)


class RopeFrequencyTable:
    """RopeFrequencyTable (rope.hpp:52-88): fp64 on the host, fp32 copies per device."""

    def __init__(self, handle):
        self._h = handle
        self._destroy = lib().spx_rope_table_destroy

    def __del__(self):
        # the bound destroy function outlives module teardown at interpreter exit
        if getattr(self, "_h", None):
            (getattr(self, "_destroy", None) or lib().spx_rope_table_destroy)(self._h)
            self._h = None

    def _info(self):
        out = i64_array([0] * 7)
        check(lib().spx_rope_table_info(self._h, out))
        return list(out)

    def max_frames(self):
        return self._info()[0]

    def max_height(self):
        return self._info()[1]

    def max_width(self):
        return self._info()[2]

    def split(self) -> BandSplit:
        return BandSplit(*self._info()[3:6])

    def _at(self, band, pos, pair):
        c = ctypes.c_double()
        s = ctypes.c_double()
        check(lib().spx_rope_table_at(self._h, int(band), pos, pair, ctypes.byref(c), ctypes.byref(s)))
        return c.value, s.value

    def cos_at(self, band, pos, pair):
        return self._at(band, pos, pair)[0]

    def sin_at(self, band, pos, pair):
        return self._at(band, pos, pair)[1]


def precompute_frequencies(max_frames, max_h, max_w, head_dim, base=10000.0,
                           split: Optional[BandSplit] = None) -> RopeFrequencyTable:
    """precompute_frequencies (rope.hpp:90-99, rope.cpp:21-64)."""
    h = ctypes.c_void_p()
    sp = i64_array([split.temporal, split.height, split.width]) if split else None
    check(lib().spx_rope_table_create(max_frames, max_h, max_w, head_dim, base, sp, ctypes.byref(h)))
    return RopeFrequencyTable(h)


def global_time_index(i_local, rank, local_len, grid_hw, start_frame) -> int:
    """global_time_index (rope.cpp:66-70)."""
    return int(lib().spx_global_time_index(i_local, rank, local_len, grid_hw, start_frame))


def rope_positions(grid: GridSpec, start_frame, rank, world_size):
    """(t, h, w) int32 tensors of rank `rank`'s local rows, from the device index path."""
    torch = _torch()
    n = grid.seq_len() // world_size if world_size > 0 else 0
    t = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    h = torch.empty_like(t)
    w = torch.empty_like(t)
    check(lib().spx_rope_positions(grid.as_array(), start_frame, rank, world_size, t.data_ptr(),
                                   h.data_ptr(), w.data_ptr(), _stream()))
    return t[:n], h[:n], w[:n]


def apply_rope_causal_local(x_local, grid: GridSpec, table: RopeFrequencyTable, start_frame, rank,
                            world_size, norm_weight=None, norm_eps=1e-6, out=None):
    """apply_rope_causal_local (rope.hpp:121-123): x_local (B, L/P, H, D) bf16 -> rotated."""
    x = _bf16(x_local)
    B, S, H, D = x.shape
    y = _torch().empty_like(x) if out is None else out
    nw = _bf16(norm_weight).data_ptr() if norm_weight is not None else None
    check(lib().spx_rope_apply_causal_local(table._h, x.data_ptr(), y.data_ptr(), B, S, H, D,
                                            grid.as_array(), start_frame, rank, world_size, nw,
                                            norm_eps, _stream()))
    return y


def apply_rope_global(x, grid: GridSpec, table: RopeFrequencyTable, start_frame, out=None):
    """apply_rope_global (rope.hpp:113-114)."""
    x = _bf16(x)
    B, S, H, D = x.shape
    y = _torch().empty_like(x) if out is None else out
    check(lib().spx_rope_apply_global(table._h, x.data_ptr(), y.data_ptr(), B, S, H, D,
                                      grid.as_array(), start_frame, _stream()))
    return y


def project_tokens(x, w):
    """project_tokens (sp_attention.hpp:34): y[b,s] = W x[b,s]; W (H*D, H*D) bf16 [out][in]."""
    x = _bf16(x)
    w = _bf16(w)
    B, S, H, D = x.shape
    if w.shape[1] != H * D:
        raise ShapeError(f"projection is {w.shape[0]}x{w.shape[1]}, tokens have H*D = {H * D}")
    y = _torch().empty(B, S, w.shape[0] // D, D, dtype=x.dtype, device=x.device)
    check(lib().spx_project_tokens(x.data_ptr(), w.data_ptr(), y.data_ptr(), B * S, H * D, w.shape[0],
                                   _stream()))
    return y


def scaled_dot_product_attention(q, k, v):
    """scaled_dot_product_attention (tensor.hpp:99): no mask, scale 1/sqrt(D)."""
    q, k, v = _bf16(q), _bf16(k), _bf16(v)
    if k.shape != v.shape:
        raise ShapeError(f"k/v shape mismatch: {tuple(k.shape)} vs {tuple(v.shape)}")
    B, Sq, H, D = q.shape
    if k.shape[0] != B or k.shape[2] != H or k.shape[3] != D:
        raise ShapeError("q/kv mismatch on batch, heads or head_dim")
    o = _torch().empty_like(q)
    check(lib().spx_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), B, Sq, k.shape[1], H,
                              D, _stream()))
    return o


class KvCache:
    """KvCache (kv_cache.hpp:16-50) as a device ring of frame slots."""

    def __init__(self, tokens_per_frame, window_frames=None, heads=1, head_dim=2, capacity_frames=0,
                 device=0):
        self._h = ctypes.c_void_p()
        self._destroy = lib().spx_kv_ring_destroy
        self.heads, self.head_dim = heads, head_dim
        self._tpf = tokens_per_frame
        check(lib().spx_kv_ring_create(device, tokens_per_frame, -1 if window_frames is None else window_frames,
                                       capacity_frames, heads, head_dim, ctypes.byref(self._h)))

    def __del__(self):
        # the bound destroy function outlives module teardown at interpreter exit
        if getattr(self, "_h", None):
            (getattr(self, "_destroy", None) or lib().spx_kv_ring_destroy)(self._h)
            self._h = None

    def _info(self):
        out = i64_array([0] * 4)
        check(lib().spx_kv_ring_info(self._h, out))
        return list(out)

    def update(self, block_index, k_block, v_block):
        k, v = _bf16(k_block), _bf16(v_block)
        if k.shape != v.shape:
            raise ShapeError("k/v block shape mismatch")
        if k.shape[2] != self.heads or k.shape[3] != self.head_dim:
            raise ShapeError("block shape incompatible with cached frames")
        check(lib().spx_kv_ring_update(self._h, block_index, k.data_ptr(), v.data_ptr(), k.shape[1], _stream()))

    def read(self):
        torch = _torch()
        n = self.seq_len()
        k = torch.empty(1, max(n, 1), self.heads, self.head_dim, dtype=torch.bfloat16, device="cuda")
        v = torch.empty_like(k)
        check(lib().spx_kv_ring_read(self._h, k.data_ptr(), v.data_ptr(), _stream()))
        return k, v

    def attention(self, q):
        q = _bf16(q)
        o = _torch().empty_like(q)
        check(lib().spx_kv_ring_attention(self._h, q.data_ptr(), o.data_ptr(), q.shape[1], _stream()))
        return o

    def cached_frames(self):
        return self._info()[0]

    def seq_len(self):
        return self._info()[1]

    def empty(self):
        return self.cached_frames() == 0

    def oldest_block_index(self):
        info = self._info()
        if info[0] == 0:
            raise EmptyCacheError("oldest_block_index() on an empty cache")
        return info[2]

    def capacity_frames(self):
        return self._info()[3]


class CommStats(dict):
    pass


class CommWorld:
    """CommWorld (collectives.hpp:39-113): LOCAL transport, every rank in this process.

    devices: per-rank CUDA device ids (default: all ranks share the current device)."""

    def __init__(self, world_size, devices: Optional[Sequence[int]] = None, _handle=None):
        self._destroy = lib().spx_world_destroy
        if _handle is not None:
            self._h = _handle
        else:
            self._h = ctypes.c_void_p()
            devs = (ctypes.c_int * world_size)(*devices) if devices else None
            check(lib().spx_world_create_local(world_size, devs, ctypes.byref(self._h)))
        self._world_size = self.info()[0]

    @classmethod
    def nccl(cls, rank, world_size, unique_id: bytes, device):
        h = ctypes.c_void_p()
        uid = (ctypes.c_uint8 * 128)(*unique_id)
        check(lib().spx_world_create_nccl(rank, world_size, uid, device, ctypes.byref(h)))
        return cls(world_size, _handle=h)

    @classmethod
    def peer(cls, rank, world_size, device):
        """PEER transport (one rank per process): the engine's kernels store into the peers'
        exchange buffers through CUDA IPC mappings; call Engine.connect_peers once."""
        h = ctypes.c_void_p()
        check(lib().spx_world_create_peer(rank, world_size, device, ctypes.byref(h)))
        return cls(world_size, _handle=h)

    @staticmethod
    def nccl_unique_id() -> bytes:
        uid = (ctypes.c_uint8 * 128)()
        check(lib().spx_nccl_get_unique_id(uid))
        return bytes(uid)

    def __del__(self):
        # the bound destroy function outlives module teardown at interpreter exit
        if getattr(self, "_h", None):
            (getattr(self, "_destroy", None) or lib().spx_world_destroy)(self._h)
            self._h = None

    def info(self):
        out = (ctypes.c_int32 * 4)()
        check(lib().spx_world_info(self._h, out))
        return list(out)

    def world_size(self):
        return self._world_size

    def stats(self) -> dict:
        s = _lib.CommStats()
        check(lib().spx_world_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def reset_stats(self):
        check(lib().spx_world_reset_stats(self._h))

    def synchronize(self):
        check(lib().spx_world_synchronize(self._h))

    def _sync_in(self):
        _torch().cuda.synchronize()

    @staticmethod
    def _raw(t):
        if not t.is_cuda or not t.is_contiguous():
            raise ShapeError("expected contiguous CUDA tensors")
        return t.data_ptr()

    def all_to_all(self, xs: List, scatter_dim: Axis, gather_dim: Axis):
        """all_to_all (collectives.cpp:203-235) for every rank: xs[r] is rank r's tensor."""
        torch = _torch()
        P = self._world_size
        shape = list(xs[0].shape)
        out_shape = list(shape)
        if shape[scatter_dim] % P:
            raise PartitionError(f"all_to_all scatter extent {shape[scatter_dim]} not divisible by world size {P}")
        out_shape[scatter_dim] //= P
        out_shape[gather_dim] *= P
        outs = [torch.empty(out_shape, dtype=x.dtype, device=x.device) for x in xs]
        self._sync_in()
        check(lib().spx_all_to_all(self._h, ptr_array([self._raw(x) for x in xs]),
                                   ptr_array([o.data_ptr() for o in outs]), i64_array(shape),
                                   xs[0].element_size(), int(scatter_dim), int(gather_dim)))
        self.synchronize()
        return outs

    def fused_all_to_all(self, qs, ks, vs, scatter_dim=Axis.Heads, gather_dim=Axis.Seq):
        """fused_all_to_all (collectives.cpp:237-276): one invocation, one round."""
        torch = _torch()
        P = self._world_size
        shape = list(qs[0].shape)
        if shape[scatter_dim] % P:
            raise PartitionError(f"fused_all_to_all scatter extent {shape[scatter_dim]} not divisible by world size {P}")
        out_shape = list(shape)
        out_shape[scatter_dim] //= P
        out_shape[gather_dim] *= P
        outs = [[torch.empty(out_shape, dtype=t.dtype, device=t.device) for t in ts] for ts in (qs, ks, vs)]
        self._sync_in()
        arrs = [ptr_array([self._raw(t) for t in ts]) for ts in (qs, ks, vs)]
        oarrs = [ptr_array([t.data_ptr() for t in ts]) for ts in outs]
        check(lib().spx_fused_all_to_all(self._h, *arrs, *oarrs, i64_array(shape), qs[0].element_size(),
                                         int(scatter_dim), int(gather_dim)))
        self.synchronize()
        return outs

    def all_gather(self, xs, dim: Axis):
        """all_gather (collectives.cpp:180-201)."""
        torch = _torch()
        P = self._world_size
        shape = list(xs[0].shape)
        out_shape = list(shape)
        out_shape[dim] *= P
        outs = [torch.empty(out_shape, dtype=x.dtype, device=x.device) for x in xs]
        self._sync_in()
        check(lib().spx_all_gather(self._h, ptr_array([self._raw(x) for x in xs]),
                                   ptr_array([o.data_ptr() for o in outs]), i64_array(shape),
                                   xs[0].element_size(), int(dim)))
        self.synchronize()
        return outs


@dataclass(frozen=True)
class AblationFlags:
    """AblationFlags (sp_attention.hpp:36-44): the optimized schedule is all_on(), the
    baseline Alg. 1 schedule (3 all-gathers, global RoPE, head split) all_off()."""

    use_fused_all_to_all: bool = False
    use_local_rope: bool = False
    use_precomputed_freqs: bool = False

    @staticmethod
    def all_off():
        return AblationFlags()

    @staticmethod
    def all_on():
        return AblationFlags(True, True, True)

    @staticmethod
    def lattice():
        """the 2^3 combinations (tests/acceptance.cpp:269-321)"""
        return [AblationFlags(bool(m & 1), bool(m & 2), bool(m & 4)) for m in range(8)]

    def bits(self) -> int:
        return int(self.use_fused_all_to_all) | int(self.use_local_rope) << 1 | \
            int(self.use_precomputed_freqs) << 2


@dataclass
class GenerationConfig:
    """GenerationConfig (generator.hpp:14-42) with the device knobs of spx_engine_config."""

    grid_per_block: GridSpec = field(default_factory=lambda: GridSpec(3, 4, 4))
    num_blocks: int = 5
    layers: int = 4
    denoise_steps: int = 2
    batch: int = 1
    heads: int = 8
    head_dim: int = 16
    world_size: int = 1
    seed: int = 0
    window_frames: Optional[int] = None
    rope_base: float = 10000.0
    band_split: Optional[BandSplit] = None
    force_start_frame_zero: bool = False
    qk_norm: bool = False
    norm_eps: float = 1e-6
    profile: bool = False
    fuse_rope_epilogue: bool = True  # RoPE + pack in the QKV GEMM epilogue (qk_norm off)
    adaln: bool = False  # Wan adaLN modulation + gated residual (extension, default off)
    l2_prefetch: bool = False  # attention warms the next projections' weights into L2 (opt-in)
    # the full Wan2.1 DiT block (extension): cross-attention, GELU FFN, timestep adaLN
    wan_block: bool = False
    ffn_dim: int = 0          # 0: ceil(dim * 35 / 6 / 64) * 64 (8960 at dim 1536)
    text_len: int = 512
    text_dim: int = 4096
    freq_dim: int = 256
    # attention never splits kv ranges across CTAs: SP outputs == P = 1 bit for bit at every P
    sp_bit_exact: bool = False
    ablation: AblationFlags = field(default_factory=AblationFlags.all_on)

    def block_len(self):
        return self.grid_per_block.seq_len()

    def local_len(self):
        return self.block_len() // self.world_size

    def total_calls(self):
        return self.num_blocks * self.denoise_steps * self.layers

    def to_c(self) -> _lib.EngineConfig:
        c = _lib.EngineConfig()
        lib().spx_engine_config_defaults(ctypes.byref(c))
        g = self.grid_per_block
        c.frames, c.grid_h, c.grid_w = g.frames, g.height, g.width
        c.num_blocks, c.layers, c.denoise_steps = self.num_blocks, self.layers, self.denoise_steps
        c.batch, c.heads, c.head_dim = self.batch, self.heads, self.head_dim
        c.window_frames = -1 if self.window_frames is None else self.window_frames
        c.rope_base = self.rope_base
        if self.band_split is not None:
            c.band_split[0], c.band_split[1], c.band_split[2] = (self.band_split.temporal, self.band_split.height,
                                                                 self.band_split.width)
        c.seed = self.seed
        c.force_start_frame_zero = int(self.force_start_frame_zero)
        c.qk_norm = int(self.qk_norm)
        c.norm_eps = self.norm_eps
        c.profile = int(self.profile)
        c.fuse_rope_epilogue = int(self.fuse_rope_epilogue)
        c.ablation = self.ablation.bits()
        c.adaln = int(self.adaln)
        c.l2_prefetch = int(self.l2_prefetch)
        c.wan_block = int(self.wan_block)
        c.ffn_dim = self.ffn_dim
        c.text_len, c.text_dim, c.freq_dim = self.text_len, self.text_dim, self.freq_dim
        c.sp_bit_exact = int(self.sp_bit_exact)
        return c

    def validate(self):
        """GenerationConfig::validate (generator.cpp:7-38) + device constraints."""
        c = self.to_c()
        check(lib().spx_engine_config_validate(ctypes.byref(c), self.world_size))


STAGES = ("qkv", "rope", "gather_or_fused", "cache", "attention", "output_exchange")


class Engine:
    """The optimized Causal-RoPE SP schedule + generator on device (spx_engine)."""

    def __init__(self, cfg: GenerationConfig, world: Optional[CommWorld] = None, seed_weights=True):
        self.cfg = cfg
        self.world = world if world is not None else CommWorld(cfg.world_size)
        self._c = cfg.to_c()
        self._h = ctypes.c_void_p()
        self._destroy = lib().spx_engine_destroy
        check(lib().spx_engine_create(self.world._h, ctypes.byref(self._c), ctypes.byref(self._h)))
        info = i64_array([0] * 8)
        check(lib().spx_engine_info(self._h, info))
        (self.head_groups, self.query_splits, self.block_len, self.local_len, self.heads_per_group,
         self.query_rows, self.capacity_frames, self.model_dim) = list(info)
        self.local_ranks = self.world.info()[1]
        if seed_weights:
            check(lib().spx_engine_seed_weights(self._h))

    def __del__(self):
        # the bound destroy function outlives module teardown at interpreter exit
        if getattr(self, "_h", None):
            (getattr(self, "_destroy", None) or lib().spx_engine_destroy)(self._h)
            self._h = None

    def ipc_export(self) -> bytes:
        """PEER transport: this rank's exchange-buffer handles (an opaque blob)."""
        n = ctypes.c_int64()
        check(lib().spx_engine_ipc_export(self._h, None, 0, ctypes.byref(n)))
        buf = (ctypes.c_uint8 * n.value)()
        check(lib().spx_engine_ipc_export(self._h, buf, n.value, ctypes.byref(n)))
        return bytes(buf)

    def ipc_import(self, blobs: Sequence[bytes]):
        """PEER transport: map every rank's buffers (blobs of all ranks, in rank order)."""
        per = len(blobs[0])
        if any(len(b) != per for b in blobs):
            raise ShapeError("ipc blobs differ in size")
        joined = b"".join(blobs)
        buf = (ctypes.c_uint8 * len(joined)).from_buffer_copy(joined)
        check(lib().spx_engine_ipc_import(self._h, buf, per))

    def connect_peers(self, all_gather_object):
        """PEER transport: exchange handles through a host all-gather (e.g.
        torch.distributed.all_gather_object) and map them."""
        mine = self.ipc_export()
        blobs = [None] * self.world.world_size()
        all_gather_object(blobs, mine)
        self.ipc_import(blobs)

    def set_modulation(self, layer, shift, scale, gate):
        """adaLN modulation of one layer (cfg.adaln): fp32 [dim] shift, scale, gate."""
        arrs = [np.ascontiguousarray(a, dtype=np.float32).reshape(-1) for a in (shift, scale, gate)]
        check(lib().spx_engine_set_modulation(self._h, layer, *[a.ctypes.data for a in arrs]))

    def set_layer_weights(self, layer, wq, wk, wv, wo):
        """host weights (dim, dim) [out][in]; float arrays are rounded to bf16 (RNE)."""
        self.set_layer_weights_bits(layer, *[float_to_bf16_bits(w) for w in (wq, wk, wv, wo)])

    def set_layer_weights_bits(self, layer, wq, wk, wv, wo):
        arrs = [np.ascontiguousarray(w, dtype=np.uint16) for w in (wq, wk, wv, wo)]
        check(lib().spx_engine_set_layer_weights(self._h, layer, *[a.ctypes.data for a in arrs]))

    def set_norm_weights_bits(self, layer, wq, wk):
        a = np.ascontiguousarray(wq, dtype=np.uint16)
        b = np.ascontiguousarray(wk, dtype=np.uint16)
        check(lib().spx_engine_set_norm_weights(self._h, layer, a.ctypes.data, b.ctypes.data))

    def begin_block(self, block_index):
        check(lib().spx_engine_begin_block(self._h, block_index))

    def reset_cache(self):
        """a new video: empty KV caches (a fresh generate() builds new ones)."""
        check(lib().spx_engine_reset_cache(self._h))

    def optimized_sp_self_attention(self, layer, block_index, start_frame, x_locals):
        """one optimized_sp_self_attention call (sp_attention.hpp:118-130) on every rank."""
        torch = _torch()
        ys = [torch.empty_like(x) for x in x_locals]
        torch.cuda.synchronize()
        check(lib().spx_engine_layer(self._h, layer, block_index, start_frame,
                                     ptr_array([_bf16(x).data_ptr() for x in x_locals]),
                                     ptr_array([y.data_ptr() for y in ys])))
        check(lib().spx_engine_synchronize(self._h))
        return ys

    def generate_block(self, block, noise_bits: Optional[np.ndarray] = None) -> np.ndarray:
        """bf16 bits (rows_local * local_ranks, H, D) of the block output."""
        rows = self.local_len * self.local_ranks
        out = np.empty((rows, self.cfg.heads, self.cfg.head_dim), dtype=np.uint16)
        nz = None
        if noise_bits is not None:
            nz = np.ascontiguousarray(noise_bits, dtype=np.uint16)
            want = self.cfg.denoise_steps * self.cfg.block_len() * self.cfg.heads * self.cfg.head_dim
            if nz.size != want:
                raise ShapeError(f"noise_bits holds {nz.size} values, expected denoise_steps x L x H x D"
                                 f" = {want} (the full block at every step)")
        check(lib().spx_engine_generate_block(self._h, block, nz.ctypes.data if nz is not None else None,
                                              out.ctypes.data))
        return out

    def generate_stream(self, blocks, noise_bits):
        """blocks back to back with host copies overlapped (spx_engine_generate_stream):
        noise_bits[i] (steps, L, H, D) uint16 of block blocks[i]; returns the latents, one
        (rows of the local ranks, H, D) uint16 array per block. Pinned buffers are used."""
        torch = _torch()
        n = len(blocks)
        want = self.cfg.denoise_steps * self.cfg.block_len() * self.cfg.heads * self.cfg.head_dim
        pins = []
        for nb in noise_bits:
            a = np.ascontiguousarray(nb, dtype=np.uint16)
            if a.size != want:
                raise ShapeError(f"noise holds {a.size} values, expected {want}")
            pins.append(torch.from_numpy(a.view(np.int16).reshape(-1)).pin_memory())
        rows = self.local_len * self.local_ranks
        outs = [torch.empty(rows * self.cfg.heads * self.cfg.head_dim, dtype=torch.int16).pin_memory()
                for _ in range(n)]
        check(lib().spx_engine_generate_stream(self._h, i64_array(list(blocks)), n,
                                               ptr_array([p.data_ptr() for p in pins]),
                                               ptr_array([o.data_ptr() for o in outs])))
        return [o.numpy().view(np.uint16).reshape(rows, self.cfg.heads, self.cfg.head_dim) for o in outs]

    # ---- the full Wan2.1 block (cfg.wan_block) ----
    @staticmethod
    def _wan_struct(cls, fields, arrays):
        keep = []
        st = cls()
        for name, a in arrays.items():
            if name not in fields:
                raise ConfigError(f"unknown Wan weight {name!r}")
            if a is None:
                continue
            a = np.asarray(a)
            # matrices / RMSNorm weights are bf16 bits (uint16), everything else fp32
            arr = np.ascontiguousarray(a, dtype=np.uint16 if a.dtype == np.uint16 else np.float32)
            keep.append(arr)
            setattr(st, name, arr.ctypes.data)
        return st, keep

    def set_wan_layer(self, layer, **arrays):
        """spx_engine_set_wan_layer: keyword arrays named as in spx_wan_layer_weights (bf16 bit
        arrays as uint16 for matrices and RMSNorm weights, float arrays for the rest)."""
        st, keep = self._wan_struct(_lib.WanLayerWeights, _lib.WAN_LAYER_FIELDS, arrays)
        check(lib().spx_engine_set_wan_layer(self._h, layer, ctypes.byref(st)))
        del keep

    def set_wan_embeddings(self, **arrays):
        st, keep = self._wan_struct(_lib.WanEmbedWeights, _lib.WAN_EMBED_FIELDS, arrays)
        check(lib().spx_engine_set_wan_embeddings(self._h, ctypes.byref(st)))
        del keep

    def set_timesteps(self, t):
        a = np.ascontiguousarray(t, dtype=np.float32)
        if a.size != self.cfg.denoise_steps:
            raise ShapeError(f"{a.size} timesteps for {self.cfg.denoise_steps} denoise steps")
        check(lib().spx_engine_set_timesteps(self._h, a.ctypes.data))

    def set_context(self, text_bits):
        """a video's text context, bf16 bits (text_len, text_dim)"""
        a = np.ascontiguousarray(text_bits, dtype=np.uint16)
        if a.size != self.cfg.text_len * self.cfg.text_dim:
            raise ShapeError(f"context holds {a.size} values, expected text_len x text_dim")
        check(lib().spx_engine_set_context(self._h, a.ctypes.data))

    def set_graphs(self, on: bool):
        """per-step CUDA graphs (default on) / every kernel enqueued by the host"""
        check(lib().spx_engine_set_graphs(self._h, int(bool(on))))

    def denoise_step(self, block, step, x_locals):
        """one denoise step of `block` (generator.cpp:94-110) on every local rank: x_locals are
        (L/P, H, D) bf16 CUDA tensors (noise), returns the last layer's outputs."""
        torch = _torch()
        ys = [torch.empty_like(x) for x in x_locals]
        torch.cuda.synchronize()
        check(lib().spx_engine_denoise_step(self._h, block, step,
                                            ptr_array([_bf16(x).data_ptr() for x in x_locals]),
                                            ptr_array([y.data_ptr() for y in ys])))
        check(lib().spx_engine_synchronize(self._h))
        return ys

    def generate(self) -> np.ndarray:
        rows = self.local_len * self.local_ranks
        out = np.empty((self.cfg.num_blocks, rows, self.cfg.heads, self.cfg.head_dim), dtype=np.uint16)
        check(lib().spx_engine_generate(self._h, out.ctypes.data))
        return out

    def stage_times(self):
        ms = (ctypes.c_double * 6)()
        calls = ctypes.c_int64()
        check(lib().spx_engine_stage_times(self._h, ms, ctypes.byref(calls)))
        return dict(zip(STAGES, list(ms))), calls.value

    def reset_stage_times(self):
        check(lib().spx_engine_reset_stage_times(self._h))

    def stats(self) -> dict:
        s = _lib.CommStats()
        check(lib().spx_engine_stats(self._h, ctypes.byref(s)))
        return s.as_dict()


@dataclass
class BlockCheck:
    block: int
    max_abs_dev: float
    passed: bool


@dataclass
class VerificationReport:
    """VerificationReport (proj/include/spattn/generator.hpp:66-80)."""

    config: "GenerationConfig"
    tolerance: float
    blocks: list
    ledger: dict
    passed: bool


def verify_stream(cfg: "GenerationConfig", tolerance: float = 1e-10,
                  devices: Optional[Sequence[int]] = None) -> VerificationReport:
    """verify_stream(cfg, tol) (generator.cpp:149-177) on the device: cfg's schedule at
    cfg.world_size ranks (a LOCAL world; devices may repeat) against the P = 1 optimized path
    (the reference pipeline at P = 1, true start frames) on the same seeded weights and noise;
    per-block max |deviation| of the bf16 outputs. The reference's 1e-10 default is met exactly
    by the schedules that keep the P = 1 arithmetic (every partition: bit-identical outputs)."""
    c = cfg.to_c()
    n = cfg.num_blocks
    blocks = (_lib.VerifyBlock * n)()
    ok = ctypes.c_int32()
    st = _lib.CommStats()
    devs = None if devices is None else (ctypes.c_int * len(devices))(*devices)
    check(lib().spx_verify_stream(ctypes.byref(c), cfg.world_size, devs, tolerance, blocks, n,
                                  ctypes.byref(ok), ctypes.byref(st)))
    checks = [BlockCheck(int(b.block), float(b.max_abs_dev), bool(b.pass_)) for b in blocks]
    return VerificationReport(cfg, tolerance, checks, st.as_dict(), bool(ok.value))


def tensor_checksum(x: np.ndarray) -> str:
    """tensor_checksum (report.cpp:264-279) of the values as fp64."""
    d = np.ascontiguousarray(x, dtype=np.float64)
    out = ctypes.create_string_buffer(17)
    check(lib().spx_checksum_f64(d.ctypes.data, d.size, out))
    return out.value.decode()


def generation_result_json(cfg: "GenerationConfig", block_outputs: np.ndarray, stats: dict,
                           stage_us_total: Optional[dict] = None, calls: Optional[int] = None,
                           wall_ms: Optional[float] = None, variant: Optional[str] = None) -> dict:
    """to_json(GenerationResult) (report.cpp:87-175): the reference's report layout for a
    device run, so its report tooling reads GPU runs. block_outputs: (blocks, L, H, D) values
    (bf16 bits or floats); stats: Engine.stats(); element width 2 (bf16).

    variant: the reference PipelineKind name (sp_attention.hpp:46-66). Default: "baseline"
    when every ablation flag is off (the Alg. 1 schedule), else "optimized"; "reference" labels
    a P = 1 run as reference_self_attention (no exchange stage, flags all on). Pinned against
    reports the reference's own report.cpp wrote (tests/golden/reference_reports.json)."""
    out = np.asarray(block_outputs)
    if out.dtype == np.uint16:
        out = bf16_bits_to_float(out)
    bits = cfg.ablation.bits()
    if variant is None:
        variant = "baseline" if bits == 0 else "optimized"
    if variant not in ("reference", "baseline", "optimized"):
        raise ConfigError(f"unknown variant {variant!r}")
    if variant == "reference" and (cfg.world_size != 1 or bits != 7):
        raise ConfigError("the reference variant is the P = 1 path with every flag on")
    ab = {"use_fused_all_to_all": bool(bits & 1), "use_local_rope": bool(bits & 2),
          "use_precomputed_freqs": bool(bits & 4)}
    order = (["qkv", "rope", "gather_or_fused", "cache", "attention", "output_exchange"] if bits & 2
             else ["qkv", "gather_or_fused", "rope", "cache", "attention", "output_exchange"])
    if variant == "reference":  # sp_attention.cpp:317-348: no exchange stage
        order = ["qkv", "rope", "cache", "attention", "output_exchange"]
    g = cfg.grid_per_block
    conf = {"frames_per_block": g.frames, "grid_h": g.height, "grid_w": g.width,
            "num_blocks": cfg.num_blocks, "layers": cfg.layers, "denoise_steps": cfg.denoise_steps,
            "batch": cfg.batch, "heads": cfg.heads, "head_dim": cfg.head_dim,
            "world_size": cfg.world_size, "seed": cfg.seed, "variant": variant, "ablation": ab,
            "element_width_bytes": 2, "rope_base": cfg.rope_base,
            "force_start_frame_zero": cfg.force_start_frame_zero,
            "window_frames": cfg.window_frames}
    blocks = []
    for b in range(out.shape[0]):
        blocks.append({"block": b, "start_frame": 0 if cfg.force_start_frame_zero else b * g.frames,
                       "shape": [1, int(out.shape[1]), cfg.heads, cfg.head_dim],
                       "checksum": tensor_checksum(out[b])})
    ledger = dict(stats)
    if variant == "reference":
        # reference_self_attention calls no collective (sp_attention.cpp:317-348); the P = 1
        # device run moves no data either (its exchange rounds are local no-ops)
        if ledger.get("elements_sent", 0) != 0:
            raise ConfigError("a reference-variant report needs a run that moved no data")
        ledger = {k: 0 for k in ("all_gather", "all_to_all", "fused_all_to_all", "elements_sent",
                                 "rounds")}
    ledger["bytes_sent_at_width"] = ledger["elements_sent"] * 2
    profile = {"calls": calls if calls is not None else cfg.total_calls(),
               "wall_ms": wall_ms, "stage_order": order,
               "stage_us_total": stage_us_total or {k: 0.0 for k in order}, "ledger": ledger}
    return {"config": conf, "blocks": blocks, "profile": profile}


_TIMING_KEYS = ("wall_ms", "wall_ms_all", "mean_stage_us", "stage_us_total", "stage_times_us",
                "total_us", "time_us", "deltas", "speedup_vs_baseline")


def strip_timing_fields(j):
    """strip_timing_fields (report.cpp:246-262): drops every timing key, recursively, in
    place, so two reports compare on their deterministic content. Returns j."""
    if isinstance(j, dict):
        for k in _TIMING_KEYS:
            j.pop(k, None)
        for v in j.values():
            strip_timing_fields(v)
    elif isinstance(j, list):
        for v in j:
            strip_timing_fields(v)
    return j


def bf16_bits_to_float(bits: np.ndarray) -> np.ndarray:
    b = np.asarray(bits, dtype=np.uint16)
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def float_to_bf16_bits(x) -> np.ndarray:
    d = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    out = np.empty(d.size, dtype=np.uint16)
    check(lib().spx_f64_to_bf16(d.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16)), d.size))
    return out.reshape(np.shape(x))


def generate(cfg: GenerationConfig) -> np.ndarray:
    """generate(cfg) (generator.hpp:65): block outputs as float64 (bf16 values), (blocks, L, H, D)."""
    eng = Engine(cfg)
    return bf16_bits_to_float(eng.generate())
