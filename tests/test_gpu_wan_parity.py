"""Parity at the BASELINE configurations (Wan2.1-1.3B shape: 3 x 30 x 52 tokens per chunk,
H = 12, D = 128, C = 1536) against the GPU fp64 oracle (oracle/gpu_oracle.py, a float64
restatement of the reference P = 1 path pinned to the CPU oracle in tests/test_oracle_pin.py).

  C2  one chunk, 30 layers x 4 denoise steps (the bench workload)
  C3  5 s video: 7 chunks, unlimited KV window (the cache grows to 21 frames = 32,760 keys)
  C5  long video: 24 chunks with a 21-frame rolling window (the ring wraps from chunk 7 on and
      attention walks two segments); 2 layers x 2 steps per chunk (the ring logic is per layer
      and per step; depth only multiplies the run time of the fp64 oracle)
plus sequence-parallel bit identity at H = 12 (P = 2, 4 Ulysses; P = 8 the 4 x 2 head-group x
query-split partition), the attention kernel at 4680 x 32760 x 12 and over a wrapped Wan-scale
ring, and a well-conditioned 2-layer check of the token-discriminating (centred) signal.

Tolerances. Deep stacks: the reference model has no residual or norm and its
N(0, 1/fan_in) weights give logits of std ~ 1/D, so every token collapses toward the block mean
of V; the token-discriminating part is below bf16 resolution (the centred check
therefore uses O(1) logits). Each block's latent is checked
  * at RMS level: | ||device|| / ||fp64|| - 1 | < 1e-2, and
  * element-wise: rel-L2(device, fp64) < 1.5 x rel-L2(bf16-storage model, fp64) + 1e-3, where
    the model is the same fp64 pipeline with every inter-kernel tensor rounded to bf16
    (gpu_oracle storage="bf16"): the error that bf16 storage alone implies at that depth
    (one layer: ~3e-3; 30 layers: ~1.1e-2 -- the per-layer roundings random-walk through the
    chain, so a fixed 1e-2 bar is not a property of the kernels at depth 30).
The measured errors are logged (SPX_PARITY_LOG) and committed as profiles/parity_r02.json.
"""
import math

import numpy as np
import pytest

from oracle import gpu_oracle, oracle

pytestmark = pytest.mark.gpu

WAN = dict(frames=3, grid_h=30, grid_w=52, heads=12, head_dim=128)
L, C = 4680, 1536


def spattn():
    from paper_2603_06664_b200 import spattn as s

    return s


def cfg(num_blocks, layers, steps, world=1, **extra):
    s = spattn()
    return s.GenerationConfig(grid_per_block=s.GridSpec(3, 30, 52), num_blocks=num_blocks,
                              layers=layers, denoise_steps=steps, heads=12, head_dim=128,
                              world_size=world, **extra)


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def centered(x):
    return x - x.mean(axis=0, keepdims=True)


def device_out(eng):
    s = spattn()
    out = s.bf16_bits_to_float(eng.generate())  # (blocks, L, H, D)
    return out.reshape(out.shape[0], L, C)


def free_gpu():
    import gc

    import torch

    gc.collect()
    torch.cuda.empty_cache()


def compare_blocks(got, ref, model, parity_log):
    """got: device latents, ref: fp64 oracle, model: the bf16-storage error model (or None
    for single-layer checks, bar 1e-2)."""
    rows = []
    for b in range(ref.shape[0]):
        e = rel_l2(got[b], ref[b])
        em = rel_l2(model[b], ref[b]) if model is not None else None
        rms = abs(np.linalg.norm(got[b]) / np.linalg.norm(ref[b]) - 1.0)
        rows.append((e, em, rms, float(np.abs(got[b] - ref[b]).max())))
    parity_log(rel_l2_per_block=[r[0] for r in rows],
               bf16_storage_model_rel_l2_per_block=[r[1] for r in rows] if model is not None else None,
               rms_level_dev_per_block=[r[2] for r in rows], max_abs_per_block=[r[3] for r in rows],
               ref_rms=float(np.sqrt(np.mean(ref ** 2))),
               bar="rms-level < 1e-2; rel-L2 < 1.5 x bf16-storage model + 1e-3")
    for b, (e, em, rms, _) in enumerate(rows):
        assert rms < 1e-2, (b, rows)
        assert e < (1.5 * em + 1e-3 if em is not None else 1e-2), (b, rows)


def oracle_pair(**kw):
    """the fp64 oracle and the bf16-storage error model of one configuration"""
    ref = gpu_oracle.ReferenceModel(**WAN, **kw).generate()
    free_gpu()
    model = gpu_oracle.ReferenceModel(**WAN, **kw, storage="bf16").generate()
    free_gpu()
    return ref, model


def test_c2_chunk_30_layers_4_steps_vs_fp64(cuda, parity_log):
    """BASELINE C2 (the bench workload): seeded reference init, reference noise draws."""
    eng = spattn().Engine(cfg(1, 30, 4))
    got = device_out(eng)
    del eng
    free_gpu()
    ref, model = oracle_pair(layers=30, num_blocks=1, steps=4)
    compare_blocks(got, ref, model, parity_log)


def test_c3_video_7_chunks_vs_fp64(cuda, parity_log):
    """BASELINE C3: 7 chunks, unlimited window; chunk 6 attends 21 frames (32,760 keys)."""
    eng = spattn().Engine(cfg(7, 30, 4))
    got = device_out(eng)
    del eng
    free_gpu()
    ref, model = oracle_pair(layers=30, num_blocks=7, steps=4)
    compare_blocks(got, ref, model, parity_log)


@pytest.mark.parametrize("world", [1, 8])
def test_c5_rolling_window_ring_wraps_vs_fp64(cuda, parity_log, world):
    """BASELINE C5 shape: 24 chunks through a 21-frame rolling window (ring capacity 21 frames:
    from chunk 7 on the new block overwrites the oldest slots and attention reads two
    segments). P = 8 runs the 4 x 2 partition, each rank's ring wrapping the same way."""
    eng = spattn().Engine(cfg(24, 2, 2, world=world, window_frames=21))
    assert eng.capacity_frames == 21
    got = device_out(eng)
    del eng
    free_gpu()
    ref, model = oracle_pair(layers=2, num_blocks=24, steps=2, window=21)
    compare_blocks(got, ref, model, parity_log)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c2_sp_bit_identical_to_p1_at_h12(cuda, world, parity_log):
    """The reference's invariant (test_sp_attention.cpp:116-130) at the Wan shape and depth
    (30 layers x 4 steps, 2 chunks): with sp_bit_exact the partitions P = 2, 4 (Ulysses: 6 / 3
    heads per rank) and P = 8 (4 head groups x 2 query halves, which the reference itself
    cannot run: 12 % 8 != 0) produce the P = 1 latents bit for bit."""
    s = spattn()
    base = s.Engine(cfg(2, 30, 4, sp_bit_exact=True)).generate()
    free_gpu()
    got = s.Engine(cfg(2, 30, 4, world=world, sp_bit_exact=True)).generate()
    parity_log(identical=bool(np.array_equal(got, base)), world=world)
    assert np.array_equal(got, base)


@pytest.fixture(scope="module")
def c2_two_chunks_oracle():
    """fp64 oracle and bf16-storage model of C2 over 2 chunks (shared by the SP tests)"""
    return oracle_pair(layers=30, num_blocks=2, steps=4)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c2_sp_default_layout_vs_fp64(cuda, world, parity_log, c2_two_chunks_oracle):
    """The default (fast) layouts: where a rank's (query tile x head) grid under-fills the
    148 SMs (P = 2: 222 tiles, P = 8: 57 tiles) attention splits kv ranges over CTAs, which
    changes the fp32 summation order, so the latents are not bit-identical to P = 1 (north_star
    asks bit-exactness for indices / permutations, a stated bf16 tolerance for activations).
    Each P is held to the same bar as P = 1 against the fp64 oracle. (P = 4 does not split, but
    its single wave of 111 tiles runs the v2 attention kernel while P = 1's three waves run v3:
    also not bit-identical; sp_bit_exact pins one kernel and one layout.)"""
    s = spattn()
    got = device_out(s.Engine(cfg(2, 30, 4, world=world)))
    free_gpu()
    ref, model = c2_two_chunks_oracle
    compare_blocks(got, ref, model, parity_log)
    base = device_out(s.Engine(cfg(2, 30, 4)))
    parity_log(rel_l2_vs_p1=[rel_l2(got[b], base[b]) for b in range(2)],
               identical_to_p1=bool(np.array_equal(got, base)), world=world)


def _scaled_weights(layers, scale_qk, seed):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((layers, 4, C, C)) / math.sqrt(C)
    w[:, 0:2] *= scale_qk  # O(1) logits: the token-discriminating signal is well above bf16
    return oracle.round_bf16(w)


@pytest.mark.parametrize("world", [1, 8])
def test_wan_one_layer_centred_signal(cuda, parity_log, world):
    """1 layer x 1 step over 2 chunks with O(1) logits (W_q, W_k scaled by 16: logit std
    s^2 / D = 2 at D = 128): the centred (per-token) part of the output, not only the block
    mean, matches the fp64 oracle. (With the reference init the logit std is ~1/D and the
    token-discriminating signal is below bf16 resolution; a second layer of
    this residual-free model collapses it again.)"""
    s = spattn()
    w = _scaled_weights(1, 16.0, seed=21)
    eng = s.Engine(cfg(2, 1, 1, world=world), seed_weights=False)
    eng.set_layer_weights_bits(0, *[oracle.to_bf16_bits(w[0, m]) for m in range(4)])
    got = device_out(eng)
    del eng
    free_gpu()
    ref = gpu_oracle.ReferenceModel(**WAN, layers=1, num_blocks=2, steps=1, weights=w).generate()
    e = [rel_l2(got[b], ref[b]) for b in range(2)]
    ec = [rel_l2(centered(got[b]), centered(ref[b])) for b in range(2)]
    cshare = [float(np.linalg.norm(centered(ref[b])) / np.linalg.norm(ref[b])) for b in range(2)]
    parity_log(rel_l2=e, centred_rel_l2=ec, centred_share_of_ref=cshare, bar_rel_l2=1e-2,
               bar_centred=3e-2)
    assert min(cshare) > 0.1  # the check is meaningful: tokens are distinct
    assert max(e) < 1e-2 and max(ec) < 3e-2, (e, ec)


def test_wan_mode_qknorm_adaln_4_layers_vs_fp64(cuda, parity_log):
    """Wan-mode self-attention (QK-RMSNorm + adaLN modulation + gated residual, extensions
    with no reference counterpart) at the Wan shape, 4 layers x 2 steps x 2 chunks. With the
    residual the tokens stay distinct, so the centred signal is compared too."""
    s = spattn()
    w = _scaled_weights(4, 1.0, seed=22)
    rng = np.random.default_rng(23)
    mod = (rng.standard_normal((4, 3, C)) * 0.3).astype(np.float32)
    eng = s.Engine(cfg(2, 4, 2, qk_norm=True, adaln=True), seed_weights=False)
    for l in range(4):
        eng.set_layer_weights_bits(l, *[oracle.to_bf16_bits(w[l, m]) for m in range(4)])
        eng.set_modulation(l, mod[l, 0], mod[l, 1], mod[l, 2])
    got = device_out(eng)
    del eng
    free_gpu()
    ref = gpu_oracle.ReferenceModel(**WAN, layers=4, num_blocks=2, steps=2, weights=w, qk_norm=True,
                                    modulation=mod.astype(np.float64)).generate()
    e = [rel_l2(got[b], ref[b]) for b in range(2)]
    ec = [rel_l2(centered(got[b]), centered(ref[b])) for b in range(2)]
    parity_log(rel_l2=e, centred_rel_l2=ec, bar_rel_l2=1e-2, bar_centred=3e-2)
    assert max(e) < 1e-2 and max(ec) < 3e-2, (e, ec)


def _fp32_attention(q, k, v):
    import torch

    D = q.shape[-1]
    out = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    for h in range(q.shape[2]):
        qh, kh, vh = (t[0, :, h].float() for t in (q, k, v))
        w = torch.softmax((qh @ kh.t()) / math.sqrt(D), dim=-1)
        out[0, :, h] = w @ vh
    return out


def test_attention_at_c3_length_vs_fp32(cuda, parity_log):
    """K6 at the C3/C5 per-call shape: 4680 queries x 32,760 keys x 12 heads (O(1) logits)."""
    import torch

    from paper_2603_06664_b200._lib import check, lib

    g = torch.Generator(device="cuda").manual_seed(7)
    q = torch.randn(1, 4680, 12, 128, device=cuda, generator=g).to(torch.bfloat16)
    k = torch.randn(1, 32760, 12, 128, device=cuda, generator=g).to(torch.bfloat16)
    v = torch.randn(1, 32760, 12, 128, device=cuda, generator=g).to(torch.bfloat16)
    o = torch.empty_like(q)
    check(lib().spx_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), 1, 4680, 32760,
                              12, 128, torch.cuda.current_stream().cuda_stream))
    ref = _fp32_attention(q, k, v)
    torch.cuda.synchronize()
    e = float((o.float() - ref).norm() / ref.norm())
    parity_log(rel_l2=e, bar=5e-3)
    assert e < 5e-3


def test_wrapped_ring_attention_at_wan_scale(cuda, parity_log):
    """The rolling ring at Wan scale: 21-frame window, 10 chunk updates (the ring wraps, the
    cached frames are two segments) -- attention through the ring == fp32 attention over the
    chronological read()."""
    import torch

    s = spattn()
    cache = s.KvCache(1560, 21, heads=12, head_dim=128)
    g = torch.Generator(device="cuda").manual_seed(8)
    for b in range(10):
        k = torch.randn(1, L, 12, 128, device=cuda, generator=g).to(torch.bfloat16)
        v = torch.randn(1, L, 12, 128, device=cuda, generator=g).to(torch.bfloat16)
        cache.update(b, k, v)
    assert cache.cached_frames() == 21 and cache.oldest_block_index() == 3
    q = torch.randn(1, L, 12, 128, device=cuda, generator=g).to(torch.bfloat16)
    o = cache.attention(q)
    kk, vv = cache.read()
    ref = _fp32_attention(q, kk, vv)
    torch.cuda.synchronize()
    e = float((o.float() - ref).norm() / ref.norm())
    parity_log(rel_l2=e, bar=5e-3)
    assert e < 5e-3
