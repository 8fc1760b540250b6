"""Engine stage probe: per-call stage times of the Wan-shape chunk (CUDA events between every
stage, one chunk after warm-up) and the chunk time without stage events. Used to compare
kernel variants selected by environment (SPX_GEMM_EXPERIMENT, SPX_ATTN_KERNEL, ...).

usage: python tools/stage_probe.py [--no-fuse-rope] [--P N] [--chunks K] [--label S]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06664_b200 import spattn  # noqa: E402
from paper_2603_06664_b200._lib import check, lib, ptr_array  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--no-fuse-rope", action="store_true")
    ap.add_argument("--P", type=int, default=1, help="virtual ranks on one device (LOCAL transport)")
    ap.add_argument("--chunks", type=int, default=5)
    ap.add_argument("--label", default="")
    ap.add_argument("--wan", action="store_true", help="Wan mode: QK-RMSNorm + adaLN modulation")
    ap.add_argument("--prefetch", action="store_true", help="L2 weight prefetch in attention (opt-in)")
    args = ap.parse_args()
    F, Hg, Wg, H, D, layers, steps = 3, 30, 52, 12, 128, 30, 4
    L, C = F * Hg * Wg, H * D
    world = spattn.CommWorld(args.P, [0] * args.P)
    cfg = spattn.GenerationConfig(grid_per_block=spattn.GridSpec(F, Hg, Wg), num_blocks=1,
                                  layers=layers, denoise_steps=steps, heads=H, head_dim=D,
                                  world_size=args.P, seed=0, profile=False,
                                  fuse_rope_epilogue=not args.no_fuse_rope, qk_norm=args.wan,
                                  adaln=args.wan, l2_prefetch=args.prefetch)
    eng = spattn.Engine(cfg, world=world)
    Lp = L // args.P
    noise = [torch.randn(steps, Lp, C, device="cuda").mul_(D ** -0.5).to(torch.bfloat16)
             for _ in range(args.P)]
    out = [torch.empty(Lp, C, device="cuda", dtype=torch.bfloat16) for _ in range(args.P)]
    nptr = ptr_array([t.data_ptr() for t in noise])
    optr = ptr_array([t.data_ptr() for t in out])

    def chunk():
        check(lib().spx_engine_generate_block_device(eng._h, 0, nptr, optr))

    for _ in range(3):
        chunk()
    check(lib().spx_engine_synchronize(eng._h))
    torch.cuda.synchronize()
    s = ctypes_stream(world)
    st = torch.cuda.ExternalStream(s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.chunks):
        chunk()
    e1.record(st)
    check(lib().spx_engine_synchronize(eng._h))
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.chunks
    check(lib().spx_engine_reset_stage_times(eng._h))
    check(lib().spx_engine_set_profile(eng._h, 1))
    chunk()
    check(lib().spx_engine_synchronize(eng._h))
    check(lib().spx_engine_set_profile(eng._h, 0))
    stages, calls = eng.stage_times()
    if os.environ.get("SPX_GEMM_EXPERIMENT") in ("5", "7"):  # last traced GEMM launch: tile timeline (7: the O-projection)
        import numpy as np

        tr = np.zeros(1024 * 16 * 4, dtype=np.int64)
        check(lib().spx_debug_gemm_trace(tr.ctypes.data, tr.size))
        tr = tr.reshape(1024, 16, 4)
        g = tr[:, 14, :2]
        live = g[:, 0] > 0
        ent, ex = g[live, 0], g[live, 1]
        print(json.dumps({"ctas": int(live.sum()),
                          "entry_spread_us": round(float(ent.max() - ent.min()) / 1e3, 2),
                          "exit_spread_us": round(float(ex.max() - ex.min()) / 1e3, 2),
                          "span_us": round(float(ex.max() - ent.min()) / 1e3, 2),
                          "entry_us_sorted_pct": [round(float(np.percentile(ent - ent.min(), q)) / 1e3, 2)
                                                  for q in (10, 50, 90, 100)]}))
        for cta in (0, 1, 2, 3, 100, 101):
            # pair kernel: odd CTAs have no MMA marks (relative to their first epilogue);
            # single-CTA kernel: every CTA has all four
            base = tr[cta, 0, 0] if tr[cta, 0, 0] else tr[cta, 0, 2]
            rows = [[round((v - base) / 1965.0, 2) if v else None
                     for v in tr[cta, it]] for it in range(6) if tr[cta, it].any()]
            ent = tr[cta, 15]
            print(json.dumps({"cta": cta, "us_since_first[mma_start,mma_issued,epi_start,epi_end]": rows,
                              "entry_to_prologue_end_us": round((ent[1] - ent[0]) / 1965.0, 2),
                              "prologue_end_to_first_mma_us": round((tr[cta, 0, 0] - ent[1]) / 1965.0, 2)
                              if tr[cta, 0, 0] else None,
                              "entry_to_exit_us": round((ent[2] - ent[0]) / 1965.0, 2)}))
    print(json.dumps({"label": args.label, "P": args.P, "fuse_rope": not args.no_fuse_rope, "wan": args.wan,
                      "env": {k: v for k, v in os.environ.items() if k.startswith("SPX_")},
                      "chunk_ms": round(ms, 3), "frames_per_s": round(3e3 / ms, 2),
                      "stage_us_per_call": {k: round(v / max(calls, 1) * 1e3, 2)
                                            for k, v in stages.items()}}), flush=True)


def ctypes_stream(world):
    import ctypes

    p = ctypes.c_void_p()
    check(lib().spx_world_stream(world._h, 0, ctypes.byref(p)))
    return p.value


if __name__ == "__main__":
    main()
