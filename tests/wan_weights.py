"""Synthetic parameters of the full Wan2.1 block for the parity tests (test helper): one numpy
draw shared by the device engine (through spx_engine_set_*) and the fp64 oracle
(oracle/gpu_oracle.py, wan=...). Matrices N(0, 1/fan_in) and RMSNorm weights are bf16 values,
the other vectors fp32 values (what the device stores)."""
import numpy as np

from oracle import oracle

BF16_LAYER = ("cross_q", "cross_k", "cross_v", "cross_o", "cross_norm_q", "cross_norm_k", "ffn_w1",
              "ffn_w2")
BF16_EMBED = ("time_w1", "time_w2", "proj_w", "text_w1", "text_w2")


def make(C, F, layers, text_len, text_dim, freq_dim, steps, seed, gate_scale=1.0):
    rng = np.random.default_rng(seed)
    bf = oracle.round_bf16

    def mat(o, i):
        return bf(rng.standard_normal((o, i)) / np.sqrt(i))

    def vec(n, sc=0.02, off=0.0):
        return (off + sc * rng.standard_normal(n)).astype(np.float32).astype(np.float64)

    def nw(n):
        return bf(1.0 + 0.1 * rng.standard_normal(n))

    w_self = np.stack([np.stack([mat(C, C) for _ in range(4)]) for _ in range(layers)])
    lays = []
    for _ in range(layers):
        mod = vec(6 * C, 1.0 / np.sqrt(C)).reshape(6, C)
        mod[2] *= gate_scale
        mod[5] *= gate_scale
        lays.append(dict(
            self_bq=vec(C), self_bk=vec(C), self_bv=vec(C), self_bo=vec(C),
            norm_q=nw(C), norm_k=nw(C), norm3_w=vec(C, 0.1, 1.0), norm3_b=vec(C),
            cross_q=mat(C, C), cross_k=mat(C, C), cross_v=mat(C, C), cross_o=mat(C, C),
            cross_bq=vec(C), cross_bk=vec(C), cross_bv=vec(C), cross_bo=vec(C),
            cross_norm_q=nw(C), cross_norm_k=nw(C),
            ffn_w1=mat(F, C), ffn_b1=vec(F), ffn_w2=mat(C, F), ffn_b2=vec(C),
            modulation=mod))
    emb = dict(time_w1=mat(C, freq_dim), time_b1=vec(C), time_w2=mat(C, C), time_b2=vec(C),
               proj_w=mat(6 * C, C), proj_b=vec(6 * C), text_w1=mat(C, text_dim), text_b1=vec(C),
               text_w2=mat(C, C), text_b2=vec(C))
    wan = dict(layers=lays, text=bf(rng.standard_normal((text_len, text_dim))),
               timesteps=[1000.0 - 1000.0 * i / steps for i in range(steps)], **emb)
    return w_self, wan


def load(eng, w_self, wan):
    """push the parameters into a device engine (cfg.wan_block = 1)"""
    bits = oracle.to_bf16_bits
    for l, lw in enumerate(wan["layers"]):
        eng.set_layer_weights_bits(l, *[bits(w_self[l, m]) for m in range(4)])
        eng.set_norm_weights_bits(l, bits(lw["norm_q"]), bits(lw["norm_k"]))
        eng.set_wan_layer(l, **{k: (bits(v) if k in BF16_LAYER else np.asarray(v, np.float32))
                                for k, v in lw.items() if k not in ("norm_q", "norm_k")})
    eng.set_wan_embeddings(**{k: (bits(wan[k]) if k in BF16_EMBED else np.asarray(wan[k], np.float32))
                              for k in ("time_w1", "time_b1", "time_w2", "time_b2", "proj_w", "proj_b",
                                        "text_w1", "text_b1", "text_w2", "text_b2")})
    eng.set_timesteps(np.asarray(wan["timesteps"], np.float32))
    eng.set_context(bits(wan["text"]))
