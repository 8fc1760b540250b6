"""Known-answer tests of the oracle's full Wan2.1 block extension (oracle/gpu_oracle.py, torch
float64 on the CPU). The reference model is attention-only, so these pieces are
pinned by closed forms instead of reference vectors: GELU(tanh) against the erf GELU, the
sinusoidal timestep embedding, a zero-gate / zero-projection block being the identity, and a
one-token context making the cross-attention a broadcast of that token's value."""
import math

import numpy as np
import pytest
import torch

from oracle import gpu_oracle, oracle

import wan_weights

KW = dict(frames=3, grid_h=4, grid_w=4, heads=4, head_dim=16)
C = 64


def test_gelu_tanh_close_to_erf_gelu_and_exact_at_zero():
    x = torch.linspace(-4, 4, 801, dtype=torch.float64)
    erf_gelu = 0.5 * x * (1 + torch.erf(x / math.sqrt(2)))
    assert float((gpu_oracle.gelu_tanh(x) - erf_gelu).abs().max()) < 1e-3
    assert float(gpu_oracle.gelu_tanh(torch.zeros(1, dtype=torch.float64))) == 0.0
    # closed form at x = 1: 0.5 (1 + tanh(sqrt(2/pi) 1.044715))
    v = 0.5 * (1 + math.tanh(math.sqrt(2 / math.pi) * 1.044715))
    assert abs(float(gpu_oracle.gelu_tanh(torch.ones(1, dtype=torch.float64))) - v) < 1e-15


def test_sinusoidal_embedding_closed_form():
    e = gpu_oracle.sinusoidal_embedding(256, 0.0)
    assert torch.equal(e[:128], torch.ones(128, dtype=torch.float64))
    assert torch.equal(e[128:], torch.zeros(128, dtype=torch.float64))
    e = gpu_oracle.sinusoidal_embedding(256, 750.0)
    assert abs(float(e[0]) - math.cos(750.0)) < 1e-15 and abs(float(e[128]) - math.sin(750.0)) < 1e-15
    j = 37
    assert abs(float(e[j]) - math.cos(750.0 * 10000 ** (-j / 128))) < 1e-12


def _model(w_self, wan, **kw):
    return gpu_oracle.ReferenceModel(**KW, layers=len(wan["layers"]), num_blocks=1,
                                     steps=len(wan["timesteps"]), weights=w_self, wan=wan,
                                     qk_norm=True, device="cpu", **kw)


def test_zero_gates_and_projections_make_the_block_the_identity():
    w_self, wan = wan_weights.make(C, 128, 2, 8, 64, 32, 2, seed=1)
    for lw in wan["layers"]:
        lw["modulation"][:] = 0
        lw["cross_o"][:] = 0
        lw["cross_bo"][:] = 0
    for k in ("proj_w", "proj_b"):
        wan[k][:] = 0  # e0 = 0: gate_msa = gate_mlp = 0
    m = _model(w_self, wan)
    x = m.noise(0, 1)
    assert torch.equal(m.block(0), x)


def test_single_context_token_broadcasts_its_value():
    w_self, wan = wan_weights.make(C, 128, 1, 1, 64, 32, 1, seed=2)
    m = _model(w_self, wan)
    lw = m.wan["layers"][0]
    kc, vc = m.ctx_kv[0]
    x = torch.randn(m.L, C, dtype=torch.float64)
    xn = gpu_oracle.layernorm(x, 1e-6) * lw["norm3_w"] + lw["norm3_b"]
    q = gpu_oracle.rms_norm(xn @ lw["cross_q"].t() + lw["cross_bq"], lw["cross_norm_q"], 1e-6)
    o = gpu_oracle.sdpa(q.reshape(m.L, 4, 16), kc, vc).reshape(m.L, C)
    assert torch.allclose(o, vc.reshape(1, C).expand(m.L, C), rtol=0, atol=1e-15)


def test_wan_block_bf16_storage_model_is_close():
    """the storage="bf16" error model stays within bf16 resolution of fp64 for 2 layers"""
    w_self, wan = wan_weights.make(C, 128, 2, 8, 64, 32, 2, seed=3)
    a = _model(w_self, wan).block(0)
    b = _model(w_self, wan, storage="bf16").block(0)
    assert float((a - b).norm() / a.norm()) < 2e-2
