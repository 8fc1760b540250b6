"""GPU fp64 ORACLE -- test infrastructure only (tests/ and nothing else; the product path never
imports it). A torch float64 restatement of the reference P = 1 path on a CUDA device, for
the Wan-shape configurations the CPU oracle cannot finish (one Wan layer call takes 6 minutes
on the CPU reference):

  reference_self_attention   proj/src/sp_attention.cpp:317-348  (QKV -> global RoPE -> cache
                                                                  -> SDPA -> W_o)
  project_tokens             proj/src/sp_attention.cpp:51-75    (y = W x, W [out][in])
  rotate_rows                proj/src/rope.cpp:78-131            (interleaved pairs, bands T|H|W)
  KvCache::update / read     proj/src/kv_cache.cpp:18-67         (pop same block, append, evict)
  scaled_dot_product_attention proj/src/tensor.cpp:161-209       (max-subtracted softmax, no mask)
  generate                   proj/src/generator.cpp:50-147       (steps do not chain)

plus the Wan-mode extensions the CPU oracle (oracle/spattn_oracle.cpp) restates: QK-RMSNorm
and the adaLN modulation + gated residual.

storage="bf16" is an error MODEL, not a second oracle: the same float64 arithmetic, but every
tensor the device path stores between kernels (the layer input x, q / k after RoPE, v, the
attention output o, the projection output y) is rounded to bf16 there. Its distance to the
float64 result is the error budget that bf16 storage alone implies at a given depth -- the
yardstick for the deep-stack tolerance (a 30-layer chain re-rounds 5 tensors per layer; the
rounding errors random-walk through the stack).

Everything else is float64; the RoPE tables, seeded weights and noise come from the CPU oracle
(liboracle: the reference's own RNG and std::pow / cos / sin), so only the summation order of
the matmuls differs from the CPU oracle. It is pinned to the CPU oracle at the shapes that one
finishes (tests/test_oracle_pin.py: relative difference <= 1e-12).
"""
from __future__ import annotations

import math
from typing import Optional

import numpy as np

from . import oracle


def _torch():
    import torch

    return torch


class RopeRows:
    """cos/sin of every (row, pair) of a block starting at frame `start` (P = 1 positions:
    i_g = i, t = start + i / HW, h = (i mod HW) / W_g, w = i mod W_g; rope.cpp:97-101), built from
    the reference's table values (precompute_frequencies, rope.cpp:21-64)."""

    def __init__(self, grid, max_frames, head_dim, base=10000.0, split=None, device="cuda"):
        torch = _torch()
        F, Hg, Wg = grid
        self.grid = grid
        sp = tuple(split) if split else oracle.band_split(head_dim)
        self.split = sp
        ext = (max_frames, Hg, Wg)
        tabs = []
        for band in range(3):
            c = np.empty((ext[band], sp[band]))
            s = np.empty((ext[band], sp[band]))
            for m in range(ext[band]):
                for j in range(sp[band]):
                    c[m, j], s[m, j] = oracle.table_at(head_dim, band, m, j, base, split)
            tabs.append((torch.from_numpy(c).to(device), torch.from_numpy(s).to(device)))
        self.tabs = tabs
        self.max_frames = max_frames
        self.device = device
        self._cache = {}

    def rows(self, start):
        if start in self._cache:
            return self._cache[start]
        torch = _torch()
        F, Hg, Wg = self.grid
        hw = Hg * Wg
        if start + F > self.max_frames:
            raise ValueError("block frames exceed the table")  # RangeError (rope.cpp:86-94)
        i = torch.arange(F * hw, device=self.device)
        pos = (start + i // hw, (i % hw) // Wg, i % Wg)
        cos = torch.cat([self.tabs[b][0][pos[b]] for b in range(3)], dim=1)
        sin = torch.cat([self.tabs[b][1][pos[b]] for b in range(3)], dim=1)
        self._cache[start] = (cos, sin)
        return cos, sin


def rope(x, cos, sin):
    """x (L, H, D) float64: (a, b) -> (a c - b s, a s + b c) on pairs (2j, 2j+1)."""
    a = x[..., 0::2]
    b = x[..., 1::2]
    c = cos[:, None, :]
    s = sin[:, None, :]
    out = _torch().empty_like(x)
    out[..., 0::2] = a * c - b * s
    out[..., 1::2] = a * s + b * c
    return out


def sdpa(q, k, v, head_chunk=4):
    """q (Sq, H, D), k/v (Skv, H, D) float64 -> (Sq, H, D): softmax(q k^T / sqrt(D)) v, no mask."""
    torch = _torch()
    D = q.shape[-1]
    out = torch.empty_like(q)
    for h0 in range(0, q.shape[1], head_chunk):
        h1 = min(q.shape[1], h0 + head_chunk)
        qh = q[:, h0:h1].transpose(0, 1)
        kh = k[:, h0:h1].transpose(0, 1)
        vh = v[:, h0:h1].transpose(0, 1)
        logits = torch.matmul(qh, kh.transpose(1, 2)) / math.sqrt(D)
        w = torch.softmax(logits, dim=-1)
        del logits
        out[:, h0:h1] = torch.matmul(w, vh).transpose(0, 1)
        del w
    return out


def rms_norm(x, w, eps):
    """x (L, C): x / sqrt(mean(x^2) + eps) * w (the oracle's rms_norm, spattn_oracle.cpp)."""
    torch = _torch()
    r = 1.0 / torch.sqrt((x * x).sum(dim=1, keepdim=True) / x.shape[1] + eps)
    return x * r * (w[None, :] if w is not None else 1.0)


def layernorm(x, eps):
    """non-affine LayerNorm over the last dim (biased variance, eps inside the sqrt)"""
    mean = x.mean(dim=1, keepdim=True)
    var = ((x - mean) ** 2).mean(dim=1, keepdim=True)
    return (x - mean) / _torch().sqrt(var + eps)


def gelu_tanh(x):
    """torch.nn.GELU(approximate="tanh"): 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))"""
    return 0.5 * x * (1.0 + _torch().tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * x ** 3)))


def silu(x):
    return x * _torch().sigmoid(x)


def sinusoidal_embedding(dim, t, device="cpu"):
    """Wan2.1 sinusoidal_embedding_1d(dim, t): [cos(t f_j) | sin(t f_j)], f_j = 10000^(-j/half)"""
    torch = _torch()
    half = dim // 2
    f = torch.pow(torch.tensor(10000.0, dtype=torch.float64, device=device),
                  -torch.arange(half, dtype=torch.float64, device=device) / half)
    a = float(t) * f
    return torch.cat([torch.cos(a), torch.sin(a)])


def layernorm_modulate(x, shift, scale, eps):
    mean = x.mean(dim=1, keepdim=True)
    var = ((x - mean) ** 2).mean(dim=1, keepdim=True)
    return (x - mean) / _torch().sqrt(var + eps) * (1.0 + scale[None, :]) + shift[None, :]


class FrameCache:
    """KvCache (kv_cache.cpp:18-67): frames tagged by block index; update pops the trailing
    frames of the same block, appends the block's frames, evicts from the front while more
    than `window` frames are held; read() is the chronological concatenation."""

    def __init__(self, hw, window=None):
        self.hw = hw
        self.window = window
        self.frames = []  # (block, k (hw, H, D), v)

    def update(self, block, k, v):
        while self.frames and self.frames[-1][0] == block:
            self.frames.pop()
        F = k.shape[0] // self.hw
        for f in range(F):
            sl = slice(f * self.hw, (f + 1) * self.hw)
            self.frames.append((block, k[sl], v[sl]))
        if self.window is not None:
            while len(self.frames) > self.window:
                self.frames.pop(0)

    def read(self):
        torch = _torch()
        return (torch.cat([f[1] for f in self.frames]), torch.cat([f[2] for f in self.frames]))


class ReferenceModel:
    """generate() of the reference P = 1 pipeline (generator.cpp:50-147) in float64 on a GPU.

    weights: (layers, 4, C, C) numpy [q|k|v|o] ([out][in]) or None (the reference's seeded init
    AttentionLayerParams::seeded, derive_seed(seed, 0x20, layer)); round_inputs: round weights
    and noise to bf16 first (the device path's inputs). qk_norm / modulation: the Wan-mode
    extensions (modulation (layers, 3, C) [shift | scale | gate])."""

    def __init__(self, frames, grid_h, grid_w, heads, head_dim, layers, num_blocks, steps,
                 window=None, seed=0, base=10000.0, split=None, weights=None, round_inputs=True,
                 qk_norm=False, norm_weights=None, modulation=None, norm_eps=1e-6,
                 force_start_frame_zero=False, device="cuda", storage="fp64", wan=None):
        torch = _torch()
        self.grid = (frames, grid_h, grid_w)
        self.H, self.D = heads, head_dim
        self.C = heads * head_dim
        self.L = frames * grid_h * grid_w
        self.layers, self.num_blocks, self.steps = layers, num_blocks, steps
        self.window, self.seed = window, seed
        self.round_inputs = round_inputs
        self.device = device
        self.force0 = force_start_frame_zero
        assert storage in ("fp64", "bf16")
        self.storage = storage
        self.table = RopeRows(self.grid, num_blocks * frames, head_dim, base, split, device)
        W = []
        for l in range(layers):
            w = weights[l] if weights is not None else oracle.layer_weights(seed, l, self.C)
            if round_inputs:
                w = oracle.round_bf16(w)
            W.append(torch.from_numpy(np.ascontiguousarray(w, dtype=np.float64)).to(device))
        self.W = W
        self.qk_norm = qk_norm
        self.norm_eps = norm_eps
        self.norm_w = None
        if qk_norm and norm_weights is not None:
            self.norm_w = torch.from_numpy(np.asarray(norm_weights, dtype=np.float64)).to(device)
        self.mod = None
        if modulation is not None:
            self.mod = torch.from_numpy(np.asarray(modulation, dtype=np.float64)).to(device)
        self.wan = None
        if wan is not None:
            self._init_wan(wan)
        self.reset()

    # ---- the full Wan2.1 block (extension; wan/modules/model.py: WanAttentionBlock, the time
    # embedding / projection and the text embedding of WanModel) ----
    def _init_wan(self, wan):
        """wan: dict of numpy arrays -- per layer lists under 'layers' (keys as in
        spx_wan_layer_weights plus norm_q / norm_k for the self-attention RMSNorm), the
        embeddings (spx_wan_embed_weights keys), 'text' (text_len, text_dim) and 'timesteps'.
        Matrices / norm weights must already be bf16 values."""
        torch = _torch()
        dev = self.device
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
        self.wan = {"layers": [{k: T(v) for k, v in lw.items()} for lw in wan["layers"]]}
        for k in ("time_w1", "time_b1", "time_w2", "time_b2", "proj_w", "proj_b", "text_w1",
                  "text_b1", "text_w2", "text_b2"):
            self.wan[k] = T(wan[k])
        self.wan["timesteps"] = [float(t) for t in wan["timesteps"]]
        self.wan["freq_dim"] = self.wan["time_w1"].shape[1]
        E = self.wan
        text = T(wan["text"])
        ctx = self._st(gelu_tanh(self._st(text) @ E["text_w1"].t() + E["text_b1"]))
        ctx = self._st(ctx @ E["text_w2"].t() + E["text_b2"])
        self.ctx_kv = []
        for lw in E["layers"]:
            k = self._st(rms_norm(self._st(ctx @ lw["cross_k"].t() + lw["cross_bk"]), lw["cross_norm_k"],
                                  self.norm_eps))
            v = self._st(ctx @ lw["cross_v"].t() + lw["cross_bv"])
            self.ctx_kv.append((k.reshape(-1, self.H, self.D), v.reshape(-1, self.H, self.D)))

    def wan_modulation(self, step):
        """e0 = W_p SiLU(W_2 SiLU(W_1 sinusoid(t) + b_1) + b_2) + b_p, as (6, C)"""
        E = self.wan
        x = sinusoidal_embedding(E["freq_dim"], E["timesteps"][step], self.device)
        h = silu(E["time_w1"] @ x + E["time_b1"])
        e = E["time_w2"] @ h + E["time_b2"]
        return (E["proj_w"] @ silu(e) + E["proj_b"]).reshape(6, self.C)

    def wan_layer(self, l, block, start, x, e0):
        """WanAttentionBlock.forward on x (L, C) with e = modulation[l] + e0 (6, C)"""
        lw = self.wan["layers"][l]
        L, H, D = self.L, self.H, self.D
        e = lw["modulation"] + e0
        eps = self.norm_eps
        x = self._st(x)
        xin = self._st(layernorm(x, eps) * (1.0 + e[1]) + e[0])
        W = self.W[l]
        q = xin @ W[0].t() + lw["self_bq"]
        k = xin @ W[1].t() + lw["self_bk"]
        v = xin @ W[2].t() + lw["self_bv"]
        q = rms_norm(self._st(q), lw["norm_q"], eps)
        k = rms_norm(self._st(k), lw["norm_k"], eps)
        cos, sin = self.table.rows(start)
        q = self._st(rope(q.reshape(L, H, D), cos, sin))
        k = self._st(rope(k.reshape(L, H, D), cos, sin))
        v = self._st(v)
        cache = self.caches[l]
        cache.update(block, k, v.reshape(L, H, D))
        kk, vv = cache.read()
        o = self._st(sdpa(q, kk, vv).reshape(L, self.C))
        x = self._st(x + e[2] * (o @ W[3].t() + lw["self_bo"]))
        # cross-attention over the cached context (no RoPE)
        xn = self._st(layernorm(x, eps) * lw["norm3_w"] + lw["norm3_b"])
        cq = self._st(xn @ lw["cross_q"].t() + lw["cross_bq"])
        cq = self._st(rms_norm(cq, lw["cross_norm_q"], eps)).reshape(L, H, D)
        kc, vc = self.ctx_kv[l]
        oc = self._st(sdpa(cq, kc, vc).reshape(L, self.C))
        x = self._st(x + oc @ lw["cross_o"].t() + lw["cross_bo"])
        # FFN
        xf = self._st(layernorm(x, eps) * (1.0 + e[4]) + e[3])
        h = self._st(gelu_tanh(xf @ lw["ffn_w1"].t() + lw["ffn_b1"]))
        return self._st(x + e[5] * (h @ lw["ffn_w2"].t() + lw["ffn_b2"]))

    def reset(self):
        hw = self.grid[1] * self.grid[2]
        self.caches = [FrameCache(hw, self.window) for _ in range(self.layers)]

    def noise(self, block, step):
        x = oracle.block_noise(self.seed, block, step, (self.L, self.H, self.D))
        if self.round_inputs:
            x = oracle.round_bf16(x)
        return _torch().from_numpy(x.reshape(self.L, self.C)).to(self.device)

    def _st(self, t):
        """a tensor stored between kernels: bf16 under storage="bf16" (the error model)"""
        if self.storage == "bf16":
            torch = _torch()
            return t.to(torch.bfloat16).to(torch.float64)
        return t

    def layer(self, l, block, start, x):
        """reference_self_attention (sp_attention.cpp:317-348) on x (L, C) float64."""
        W = self.W[l]
        L, H, D = self.L, self.H, self.D
        x = self._st(x)
        xin = x
        if self.mod is not None:
            m = self.mod[l]
            xin = self._st(layernorm_modulate(x, m[0], m[1], self.norm_eps))
        q, k, v = (xin @ W[m].t() for m in range(3))
        if self.qk_norm:
            nq = self.norm_w[l, 0] if self.norm_w is not None else None
            nk = self.norm_w[l, 1] if self.norm_w is not None else None
            q = rms_norm(q, nq, self.norm_eps)
            k = rms_norm(k, nk, self.norm_eps)
        cos, sin = self.table.rows(start)
        q = self._st(rope(q.reshape(L, H, D), cos, sin))
        k = self._st(rope(k.reshape(L, H, D), cos, sin))
        v = self._st(v)
        cache = self.caches[l]
        cache.update(block, k, v.reshape(L, H, D))
        kk, vv = cache.read()
        o = self._st(sdpa(q, kk, vv).reshape(L, self.C))
        y = o @ W[3].t()
        if self.mod is not None:
            return self._st(x + self.mod[l, 2][None, :] * y)
        return self._st(y)

    def block(self, b, noise=None):
        """one block: steps x layers calls (generator.cpp:89-115); noise: optional
        callable(step) -> (L, C) float64 tensor (default: the reference's seeded draws)."""
        start = 0 if self.force0 else b * self.grid[0]
        x = None
        for s in range(self.steps):
            x = noise(s) if noise is not None else self.noise(b, s)
            e0 = self.wan_modulation(s) if self.wan is not None else None
            for l in range(self.layers):
                x = self.wan_layer(l, b, start, x, e0) if e0 is not None else self.layer(l, b, start, x)
        return x

    def generate(self):
        """(num_blocks, L, C) float64 numpy (generate, generator.cpp:50-147)."""
        return np.stack([self.block(b).cpu().numpy() for b in range(self.num_blocks)])
