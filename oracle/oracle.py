"""CPU ORACLE -- test infrastructure only (tests/, __graft_entry__.smoke(), bench.py's
cpu_baseline / --impl reference). The product path never imports this module.

Two backends behind one numpy interface:
  * liboracle.so           -- our fp64 restatement of the reference P = 1 path
                              (oracle/spattn_oracle.cpp, every function cites proj/ file:line)
  * _ref/libspattn_ref.so  -- the reference sources themselves, compiled from /root/reference
                              by oracle/Makefile (absent when the tree was not available)
The restatement is pinned bit-exactly against the reference's golden checksums
(tests/test_oracle.py, tests/golden/).
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int64, c_uint64

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspattn_ref.so")

_o = None
_r = None

D_P = POINTER(c_double)
I64_P = POINTER(c_int64)


def build():
    """Compile the oracle (and the reference, when /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ol():
    global _o
    if _o is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = ctypes.CDLL(ORACLE_SO)
        sig = {
            "oracle_derive_seed": (c_uint64, [c_uint64] * 4),
            "oracle_rng_u64": (None, [c_uint64, c_int64, POINTER(c_uint64)]),
            "oracle_rng_normal": (None, [c_uint64, c_int64, D_P]),
            "oracle_round_bf16": (c_double, [c_double]),
            "oracle_block_noise": (None, [c_uint64, c_int64, c_int64, c_int64, c_int64, D_P]),
            "oracle_layer_weights": (None, [c_uint64, c_int64, c_int64, D_P]),
            "oracle_band_split": (None, [c_int64, I64_P]),
            "oracle_table_at": (None, [c_int64, c_int64, c_int64, c_int64, c_double, I64_P, c_int,
                                       c_int64, c_int64, D_P, D_P]),
            "oracle_global_time_index": (c_int64, [c_int64] * 5),
            "oracle_rope_causal_local": (None, [D_P, c_int64, c_int64, c_int64, c_int64, c_int64,
                                                c_int64, c_int64, c_double, I64_P, c_int64, c_int64]),
            "oracle_project": (None, [D_P, D_P, D_P, c_int64, c_int64]),
            "oracle_sdpa": (None, [D_P, D_P, D_P, D_P, c_int64, c_int64, c_int64, c_int64]),
            "oracle_rms_norm": (None, [D_P, D_P, c_int64, c_int64, c_double]),
            "oracle_checksum": (c_uint64, [D_P, c_int64]),
            "oracle_generate": (None, [I64_P, c_uint64, c_double, I64_P, D_P, D_P, D_P, D_P,
                                       c_double, D_P, D_P]),
            "oracle_layernorm_modulate": (None, [D_P, D_P, D_P, D_P, c_int64, c_int64, c_double]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _o = lib
    return _o


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _rl():
    global _r
    if _r is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_SO} not built (no /root/reference here?)")
        lib = ctypes.CDLL(REF_SO)
        lib.ref_generate.restype = c_int
        lib.ref_generate.argtypes = [I64_P, c_uint64, D_P, I64_P]
        lib.ref_sample_call.restype = c_int
        lib.ref_sample_call.argtypes = [I64_P, c_int64, c_int64, c_int64, c_int64, D_P]
        _r = lib
    return _r


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(D_P)


def _i64(vals):
    return (c_int64 * len(vals))(*vals)


# ---- scalar helpers -----------------------------------------------------------------------
def derive_seed(base, a, b=0, c=0) -> int:
    return int(_ol().oracle_derive_seed(base, a, b, c))


def rng_u64(seed, n):
    out = np.empty(n, dtype=np.uint64)
    _ol().oracle_rng_u64(seed, n, out.ctypes.data_as(POINTER(c_uint64)))
    return out


def rng_normal(seed, n):
    out = np.empty(n, dtype=np.float64)
    _ol().oracle_rng_normal(seed, n, _dp(out))
    return out


def round_bf16(x) -> np.ndarray:
    """Round float64 values to the nearest bf16 (ties to even), kept as float64."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    bits = a.view(np.uint64)
    sign = bits & np.uint64(0x8000000000000000)
    mag = bits & np.uint64(0x7FFFFFFFFFFFFFFF)
    lsb = (mag >> np.uint64(45)) & np.uint64(1)
    mag = (mag + np.uint64(0xFFFFFFFFFFF) + lsb) & ~np.uint64((1 << 45) - 1)
    out = (sign | mag).view(np.float64)
    return np.where(a == 0.0, a, out)


def to_bf16_bits(x) -> np.ndarray:
    """bf16 bit patterns (uint16) of values that are already bf16-representable."""
    f = np.ascontiguousarray(round_bf16(x)).astype(np.float32)
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def from_bf16_bits(b) -> np.ndarray:
    b = np.asarray(b, dtype=np.uint16)
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def band_split(D):
    out = (c_int64 * 3)()
    _ol().oracle_band_split(D, out)
    return tuple(out)


def table_at(D, band, pos, pair, base=10000.0, split=None):
    c = c_double()
    s = c_double()
    sp = _i64(split) if split else None
    _ol().oracle_table_at(0, 0, 0, D, base, sp, band, pos, pair, ctypes.byref(c), ctypes.byref(s))
    return c.value, s.value


def global_time_index(i_local, rank, local_len, hw, start):
    return int(_ol().oracle_global_time_index(i_local, rank, local_len, hw, start))


def checksum(a) -> str:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return "%016x" % _ol().oracle_checksum(_dp(a), a.size)


# ---- tensor ops (fp64) ------------------------------------------------------------------
def block_noise(seed, block, step, shape):
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np.float64)
    _ol().oracle_block_noise(seed, block, step, n, shape[-1], _dp(out))
    return out.reshape(shape)


def layer_weights(seed, layer, dim):
    out = np.empty((4, dim, dim), dtype=np.float64)
    _ol().oracle_layer_weights(seed, layer, dim, _dp(out))
    return out


def rope_causal_local(x, grid, start, rank, world, max_frames, base=10000.0, split=None):
    """x: (L/P, H, D) float64 -> rotated copy (rope.cpp:145-164)."""
    x = np.ascontiguousarray(x, dtype=np.float64).copy()
    rows, H, D = x.shape
    sp = _i64(split) if split else None
    _ol().oracle_rope_causal_local(_dp(x), rows, H, D, grid[0], grid[1], grid[2], max_frames, base,
                                   sp, start, rank)
    return x


def project(x, W):
    x = np.ascontiguousarray(x, dtype=np.float64)
    W = np.ascontiguousarray(W, dtype=np.float64)
    tokens = x.shape[0]
    dim = W.shape[0]
    y = np.empty((tokens, dim), dtype=np.float64)
    _ol().oracle_project(_dp(x.reshape(tokens, dim)), _dp(W), _dp(y), tokens, dim)
    return y.reshape(x.shape)


def sdpa(q, k, v):
    """(Sq, H, D), (Skv, H, D), (Skv, H, D) -> (Sq, H, D)"""
    q, k, v = (np.ascontiguousarray(t, dtype=np.float64) for t in (q, k, v))
    out = np.empty_like(q)
    _ol().oracle_sdpa(_dp(q), _dp(k), _dp(v), _dp(out), q.shape[0], k.shape[0], q.shape[1], q.shape[2])
    return out


def rms_norm(x, w=None, eps=1e-6):
    x = np.ascontiguousarray(x, dtype=np.float64).copy()
    tokens = x.shape[0]
    dim = x.size // tokens
    wp = _dp(np.ascontiguousarray(w, dtype=np.float64)) if w is not None else None
    _ol().oracle_rms_norm(_dp(x), wp, tokens, dim, eps)
    return x


def layernorm_modulate(x, shift, scale, eps=1e-6):
    """Wan adaLN modulation (extension, no reference counterpart): LN(x) (1 + scale) + shift."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    tokens = x.shape[0]
    dim = x.size // tokens
    y = np.empty_like(x)
    _ol().oracle_layernorm_modulate(_dp(x), _dp(y), _dp(np.ascontiguousarray(shift, dtype=np.float64)),
                                    _dp(np.ascontiguousarray(scale, dtype=np.float64)), tokens, dim, eps)
    return y


def generate(frames=3, grid_h=4, grid_w=4, num_blocks=5, layers=4, steps=2, heads=8, head_dim=16,
             window=None, force_start_frame_zero=False, seed=0, base=10000.0, split=None,
             weights=None, noise=None, round_inputs=False, qk_norm=False, norm_weights=None,
             norm_eps=1e-6, return_layers=False, modulation=None):
    """generate() with the reference pipeline at P = 1 (generator.cpp:50-147), fp64.

    weights: (layers, 4, dim, dim) or None (seeded); noise: (blocks, steps, L, dim) or None.
    modulation: (layers, 3, dim) [shift | scale | gate] switches on the Wan adaLN extension
    (x_in = LN(x)(1 + scale) + shift before the projections, x += gate * W_o o after).
    Returns (num_blocks, L, H, D) [, per-call outputs (blocks, steps, layers, L, H, D)].
    """
    L = frames * grid_h * grid_w
    dim = heads * head_dim
    cfg = _i64([frames, grid_h, grid_w, num_blocks, layers, steps, heads, head_dim,
                -1 if window is None else window, int(force_start_frame_zero), int(round_inputs),
                int(qk_norm), int(modulation is not None)])
    out = np.empty((num_blocks, L, heads, head_dim), dtype=np.float64)
    lo = None
    if return_layers:
        lo = np.empty((num_blocks, steps, layers, L, heads, head_dim), dtype=np.float64)
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    nz = None if noise is None else np.ascontiguousarray(noise, dtype=np.float64)
    nw = None if norm_weights is None else np.ascontiguousarray(norm_weights, dtype=np.float64)
    md = None if modulation is None else np.ascontiguousarray(modulation, dtype=np.float64)
    _ol().oracle_generate(cfg, seed, base, _i64(split) if split else None,
                          _dp(w) if w is not None else None, _dp(nz) if nz is not None else None,
                          _dp(nw) if nw is not None else None, _dp(md) if md is not None else None,
                          norm_eps, _dp(out),
                          _dp(lo) if lo is not None else None)
    return (out, lo) if return_layers else out


# ---- the reference itself (oracle/_ref) -----------------------------------------------------
VARIANTS = {"reference": 0, "baseline": 1, "optimized": 2}


def ref_generate(frames=3, grid_h=4, grid_w=4, num_blocks=5, layers=4, steps=2, heads=8,
                 head_dim=16, world=1, window=None, variant="reference", ablation=7,
                 force_start_frame_zero=False, seed=0):
    L = frames * grid_h * grid_w
    cfg = _i64([frames, grid_h, grid_w, num_blocks, layers, steps, heads, head_dim, world,
                -1 if window is None else window, VARIANTS[variant], ablation,
                int(force_start_frame_zero)])
    out = np.empty((num_blocks, L, heads, head_dim), dtype=np.float64)
    ledger = (c_int64 * 5)()
    rc = _rl().ref_generate(cfg, seed, _dp(out), ledger)
    if rc != 0:
        raise RuntimeError(f"reference generate failed (code {rc})")
    keys = ("all_gather", "all_to_all", "fused_all_to_all", "elements_sent", "rounds")
    return out, dict(zip(keys, list(ledger)))


REF_REPORT_SO = os.path.join(HERE, "_ref", "libspattn_ref_report.so")


def ref_report_json(frames=3, grid_h=4, grid_w=4, num_blocks=5, layers=4, steps=2, heads=8,
                    head_dim=16, world=1, window=None, variant="reference", ablation=7,
                    force_start_frame_zero=False, seed=0) -> str:
    """The reference's own report of a generate run: to_json(GenerationResult)
    (report.cpp:161-175) with strip_timing_fields (report.cpp:246-262), indent 2, produced by
    the unmodified report.cpp compiled into _ref/libspattn_ref_report.so."""
    lib = ctypes.CDLL(REF_REPORT_SO)
    lib.ref_report_json.restype = c_int
    cfg = _i64([frames, grid_h, grid_w, num_blocks, layers, steps, heads, head_dim, world,
                -1 if window is None else window, VARIANTS[variant], ablation,
                int(force_start_frame_zero)])
    buf = ctypes.create_string_buffer(1 << 20)
    n = c_int64()
    rc = lib.ref_report_json(cfg, ctypes.c_uint64(seed), buf, len(buf), ctypes.byref(n))
    if rc != 0:
        raise RuntimeError(f"reference report failed (code {rc})")
    return buf.value.decode()


def ref_sample_call(frames, grid_h, grid_w, heads, head_dim, kv_frames, tokens, rows, threads):
    """Reference operators timed on a bounded sample of one layer call (seconds, extrapolated)."""
    out = np.zeros(7, dtype=np.float64)
    rc = _rl().ref_sample_call(_i64([frames, grid_h, grid_w, heads, head_dim]), kv_frames, tokens,
                               rows, threads, _dp(out))
    if rc != 0:
        raise RuntimeError("reference sample failed")
    return {"call_s": out[0], "qkv_s": out[1], "rope_s": out[2], "cache_s": out[3],
            "attention_s": out[4], "output_s": out[5], "sample_wall_s": out[6]}
