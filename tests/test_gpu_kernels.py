"""GPU numerics of the individual sm_100a kernels against fp32 references of the same op.

K2/K8 GEMM vs torch fp32 matmul, K6 attention vs fp32 softmax attention (torch on the same
bf16 inputs, and the library's own fp32 SIMT kernel at the Wan shape), K3 index math vs the
reference formula (bit-exact). Calls go through the C ABI (libspx.so).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _t():
    import torch

    return torch


def _stream():
    return _t().cuda.current_stream().cuda_stream


def _lib():
    from paper_2603_06664_b200._lib import lib

    return lib()


def _check(status):
    from paper_2603_06664_b200._lib import check

    check(status)


def rel_l2(a, b):
    a = a.double()
    b = b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


@pytest.mark.parametrize("M,K,N", [(192, 256, 768), (300, 256, 256), (4680, 1536, 4608),
                                   (585, 1536, 1536), (1170, 1536, 4608)])
def test_project_tokens_matches_fp32(cuda, M, K, N, parity_log):
    torch = _t()
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    x = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda, generator=g) / math.sqrt(K)).to(torch.bfloat16)
    y = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    _check(_lib().spx_project_tokens(x.data_ptr(), w.data_ptr(), y.data_ptr(), M, K, N, _stream()))
    torch.cuda.synchronize()
    ref = x.float() @ w.float().t()
    # bf16 output rounding: |err| <= 2^-8 |y|; rel-L2 bar 3e-3
    e = rel_l2(y.float(), ref)
    parity_log(rel_l2=e, max_abs_over_max=float((y.float() - ref).abs().max() / ref.abs().max()), bar=3e-3)
    assert e < 3e-3
    assert float((y.float() - ref).abs().max()) <= 2 ** -7 * float(ref.abs().max())


@pytest.mark.parametrize("variant", range(6))
@pytest.mark.parametrize("M,K,N", [(300, 128, 1600), (4680, 1536, 1536), (585, 1536, 4608),
                                   (585, 8960, 1536)])
def test_project_tokens_every_tile_variant(cuda, variant, M, K, N):
    """each tile variant (pair 256x{256,128}, single 128x{256,128,192}, split-K 2 x 128x128) on
    ragged M and an N that no tile width divides, forced through the planner override"""
    torch = _t()
    g = torch.Generator(device="cuda").manual_seed(M + N + variant)
    x = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda, generator=g) / math.sqrt(K)).to(torch.bfloat16)
    y = torch.full((M, N), float("nan"), device=cuda, dtype=torch.bfloat16)
    _check(_lib().spx_debug_set_gemm_variant(variant))
    try:
        _check(_lib().spx_project_tokens(x.data_ptr(), w.data_ptr(), y.data_ptr(), M, K, N,
                                         _stream()))
        torch.cuda.synchronize()
    finally:
        _check(_lib().spx_debug_set_gemm_variant(-1))
    ref = x.float() @ w.float().t()
    assert bool(torch.isfinite(y.float()).all())
    assert rel_l2(y.float(), ref) < 3e-3
    assert float((y.float() - ref).abs().max()) <= 2 ** -7 * float(ref.abs().max())


@pytest.fixture(params=[0, 2], ids=["v2", "v3"])
def attn_kernel(request):
    """run the test with the v2 kernel (per-slot O) and with v3 (shared O, early S) forced"""
    _check(_lib().spx_debug_set_attn_v3(request.param))
    yield request.param
    _check(_lib().spx_debug_set_attn_v3(1))


@pytest.mark.parametrize("sq,skv,H,D", [(192, 192, 4, 64), (300, 450, 2, 64), (256, 640, 3, 128),
                                        (4680, 4680, 12, 128), (1170, 9360, 3, 128), (128, 100, 1, 128),
                                        # 222 tiles: v3's triple layout (whole tile + half of a third
                                        # per CTA, halves merged through DSMEM); 57 tiles: the pair split
                                        (4680, 4680, 6, 128), (4680, 14040, 6, 128), (2340, 4680, 3, 128)])
def test_attention_matches_fp32(cuda, sq, skv, H, D, parity_log, attn_kernel):
    torch = _t()
    g = torch.Generator(device="cuda").manual_seed(sq + skv + H)
    # O(1) logits (well-conditioned softmax), as in the tolerance tier of SURVEY 8c
    q = torch.randn(1, sq, H, D, device=cuda, generator=g).to(torch.bfloat16)
    k = torch.randn(1, skv, H, D, device=cuda, generator=g).to(torch.bfloat16)
    v = torch.randn(1, skv, H, D, device=cuda, generator=g).to(torch.bfloat16)
    o = torch.empty_like(q)
    _check(_lib().spx_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), 1, sq, skv,
                                H, D, _stream()))
    torch.cuda.synchronize()
    qf, kf, vf = (t.float().transpose(1, 2) for t in (q, k, v))
    ref = torch.softmax(qf @ kf.transpose(-1, -2) / math.sqrt(D), dim=-1) @ vf
    ref = ref.transpose(1, 2)
    e = rel_l2(o.float(), ref)
    parity_log(rel_l2=e, bar=5e-3)
    assert e < 5e-3  # SURVEY 8c K6 bar (bf16 P, fp32 O / l, one bf16 output rounding)


def test_attention_matches_simt_kernel(cuda):
    torch = _t()
    sq, skv, H, D = 640, 1560, 2, 128
    g = torch.Generator(device="cuda").manual_seed(3)
    q = torch.randn(1, sq, H, D, device=cuda, generator=g).to(torch.bfloat16)
    k = torch.randn(1, skv, H, D, device=cuda, generator=g).to(torch.bfloat16)
    v = torch.randn(1, skv, H, D, device=cuda, generator=g).to(torch.bfloat16)
    o = torch.empty_like(q)
    ref = torch.empty(1, sq, H, D, device=cuda, dtype=torch.float32)
    _check(_lib().spx_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), 1, sq, skv,
                                H, D, _stream()))
    _check(_lib().spx_debug_naive_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), ref.data_ptr(),
                                            1, sq, skv, H, D, _stream()))
    torch.cuda.synchronize()
    assert rel_l2(o.float(), ref) < 5e-3


@pytest.mark.parametrize("grid,P,start", [((3, 30, 52), 8, 18), ((3, 8, 8), 2, 3), ((3, 4, 4), 4, 0)])
def test_rope_positions_bit_exact(cuda, grid, P, start):
    torch = _t()
    from paper_2603_06664_b200._lib import i64_array

    F, Hg, Wg = grid
    L = F * Hg * Wg
    Lp = L // P
    for r in range(P):
        t = torch.empty(Lp, dtype=torch.int32, device=cuda)
        h = torch.empty_like(t)
        w = torch.empty_like(t)
        _check(_lib().spx_rope_positions(i64_array(grid), start, r, P, t.data_ptr(), h.data_ptr(),
                                         w.data_ptr(), _stream()))
        torch.cuda.synchronize()
        ig = r * Lp + np.arange(Lp)
        np.testing.assert_array_equal(t.cpu().numpy(), start + ig // (Hg * Wg))
        np.testing.assert_array_equal(h.cpu().numpy(), (ig % (Hg * Wg)) // Wg)
        np.testing.assert_array_equal(w.cpu().numpy(), ig % Wg)


@pytest.mark.parametrize("splits", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("sq,skv,H", [(2340, 4680, 3), (300, 2000, 2)])
def test_attention_split_kv_matches_fp32(cuda, splits, sq, skv, H, parity_log):
    """split-KV: fp32 partials staged in smem, bulk-copied out, bulk-loaded back and merged
    lse-weighted by the last CTA of each query tile; every split count (including counts the
    merge has to batch: 8 > 2 partials per batch at D = 128) against fp32 softmax attention."""
    torch = _t()
    D = 128
    g = torch.Generator(device="cuda").manual_seed(splits * 31 + sq)
    q = (torch.randn(1, sq, H, D, device=cuda, generator=g) * 0.5).to(torch.bfloat16)
    k = (torch.randn(1, skv, H, D, device=cuda, generator=g) * 0.5).to(torch.bfloat16)
    v = torch.randn(1, skv, H, D, device=cuda, generator=g).to(torch.bfloat16)
    o = torch.empty_like(q)
    _check(_lib().spx_debug_set_attn_splits(splits))
    try:
        for _ in range(2):  # the second launch runs on re-armed counters
            _check(_lib().spx_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), 1, sq,
                                        skv, H, D, _stream()))
        torch.cuda.synchronize()
    finally:
        _check(_lib().spx_debug_set_attn_splits(0))
    qf, kf, vf = (t.float()[0].transpose(0, 1) for t in (q, k, v))
    ref = torch.softmax(qf @ kf.transpose(1, 2) / math.sqrt(D), dim=-1) @ vf
    e = rel_l2(o.float()[0].transpose(0, 1), ref)
    parity_log(rel_l2=e, bar=5e-3)
    assert e < 5e-3


@pytest.mark.parametrize("skv", [640, 4680])
def test_attention_offset_guard_on_growing_logits(cuda, skv, attn_kernel):
    """The softmax takes its exponent offset from each warpgroup's first kv tile and skips the
    per-tile max afterwards; logits that later jump far above that offset (here by ~500 in
    natural units, > 2^64 after exp) must trip the overflow guard, which redoes the tile with
    its true max and rescales O and l."""
    torch = _t()
    D, H, sq = 128, 2, 256
    g = torch.Generator(device="cuda").manual_seed(skv)
    q = (torch.randn(1, sq, H, D, device=cuda, generator=g) * 0.2 + 2.0).to(torch.bfloat16)
    k = (torch.randn(1, skv, H, D, device=cuda, generator=g) * 0.2).to(torch.bfloat16)
    k[:, 384:] += 5.0  # kv tiles 3.. : q.k / sqrt(D) ~ 113 above tile 0 (exp2 would overflow fp32)
    v = torch.randn(1, skv, H, D, device=cuda, generator=g).to(torch.bfloat16)
    o = torch.empty_like(q)
    _check(_lib().spx_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), 1, sq, skv,
                                H, D, _stream()))
    torch.cuda.synchronize()
    qf, kf, vf = (t.float()[0].transpose(0, 1) for t in (q, k, v))
    ref = torch.softmax(qf @ kf.transpose(1, 2) / math.sqrt(D), dim=-1) @ vf
    got = o.float()[0].transpose(0, 1)
    assert bool(torch.isfinite(got).all())
    assert rel_l2(got, ref) < 5e-3


@pytest.mark.parametrize("epilogue", [0, 1, 3])
@pytest.mark.parametrize("M,K,N", [(585, 1536, 1536), (1170, 8960, 1536), (200, 1024, 4000)])
def test_split_k_epilogues(cuda, epilogue, M, K, N, parity_log):
    """split-K (variant 5: a 2-CTA cluster per 128 x 128 tile, CTA 1's fp32 partial added in
    CTA 0 through DSMEM) with the bias, in-place gated residual and GELU epilogues, persistent
    over more tiles than clusters (1170 x 1536: 120 tiles on 74 clusters) and ragged M / N"""
    torch = _t()
    g = torch.Generator(device="cuda").manual_seed(M + K + N + epilogue)
    x = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda, generator=g) / math.sqrt(K)).to(torch.bfloat16)
    b = torch.randn(N, device=cuda, generator=g) * 0.1
    gate = torch.rand(N, device=cuda, generator=g) + 0.5
    r = torch.randn(M, N, device=cuda, generator=g).to(torch.bfloat16)
    y = r.clone() if epilogue == 1 else torch.full((M, N), float("nan"), device=cuda, dtype=torch.bfloat16)
    _check(_lib().spx_debug_set_gemm_variant(5))
    try:
        _check(_lib().spx_project_tokens_ex(x.data_ptr(), w.data_ptr(), y.data_ptr(), M, K, N, b.data_ptr(),
                                            epilogue, y.data_ptr() if epilogue == 1 else None,
                                            gate.data_ptr() if epilogue == 1 else None, _stream()))
        torch.cuda.synchronize()
    finally:
        _check(_lib().spx_debug_set_gemm_variant(-1))
    acc = x.float() @ w.float().t() + b
    ref = {0: acc, 1: r.float() + gate * acc, 3: torch.nn.functional.gelu(acc, approximate="tanh")}[epilogue]
    e = rel_l2(y.float(), ref)
    parity_log(rel_l2=e, bar=3e-3)
    assert bool(torch.isfinite(y.float()).all())
    assert e < 3e-3
