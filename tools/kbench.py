"""Kernel microbenchmarks through the C ABI (CUDA events on the launching stream, warm,
inputs resident in HBM). Prints one line per case: time, achieved rate, fraction of peak.

usage: python tools/kbench.py [attn|gemm|rope|all] [iters]
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06664_b200._lib import check, lib  # noqa: E402

PEAK_TF = 1590.0   # fallback burst bf16 (B200_PROFILING.md) unless MEASURED_PEAKS.json
PEAK_GBS = 6650.0
try:
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "MEASURED_PEAKS.json")) as f:
        _p = json.load(f)
        PEAK_TF = float(_p.get("bf16_tflops", PEAK_TF))
        PEAK_GBS = float(_p.get("hbm_gbs", PEAK_GBS))
except Exception:
    pass


_STREAM = None


def stream_handle():
    return torch.cuda.current_stream().cuda_stream


def timeit(fn, iters):
    """device time per call: `iters` calls captured in one CUDA graph (host launch cost out)"""
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


ATTN_SHAPES = [(4680, 4680, 12), (4680, 32760, 12), (2340, 4680, 6), (1170, 4680, 3),
               (2340, 4680, 3), (4680, 14040, 12)]
if os.environ.get("KBENCH_ATTN_SHAPES"):  # e.g. "4680x4680x6,4680x4680x3" (per-rank shapes)
    ATTN_SHAPES = [tuple(int(v) for v in t.split("x")) for t in os.environ["KBENCH_ATTN_SHAPES"].split(",")]


def attn(iters):
    for sq, skv, H in ATTN_SHAPES:
        D = 128
        q = (torch.randn(1, sq, H, D, device="cuda") * 0.5).to(torch.bfloat16)
        k = (torch.randn(1, skv, H, D, device="cuda") * 0.5).to(torch.bfloat16)
        v = torch.randn(1, skv, H, D, device="cuda").to(torch.bfloat16)
        o = torch.empty_like(q)
        ms = timeit(lambda: check(lib().spx_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                                      o.data_ptr(), 1, sq, skv, H, D, stream_handle())), iters)
        tf = 4.0 * sq * skv * H * D / (ms * 1e-3) / 1e12
        print(json.dumps({"kernel": "attention", "sq": sq, "skv": skv, "heads": H, "ms": round(ms, 4),
                          "tflops": round(tf, 1), "frac_peak": round(tf / PEAK_TF, 3)}), flush=True)


def gemm(iters):
    shapes = [(4680, 1536, 4608), (4680, 1536, 1536), (2340, 1536, 4608), (1170, 1536, 4608),
              (585, 1536, 4608), (2340, 1536, 1536), (1170, 1536, 1536), (585, 1536, 1536),
              (8192, 8192, 8192)]
    only = os.environ.get("KBENCH_GEMM_SHAPES")  # e.g. "585x1536x4608,1170x1536x1536"
    if only:
        shapes = [tuple(int(v) for v in t.split("x")) for t in only.split(",")]
    for M, K, N in shapes:
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
        y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ms = timeit(lambda: check(lib().spx_project_tokens(x.data_ptr(), w.data_ptr(), y.data_ptr(),
                                                           M, K, N, stream_handle())), iters)
        tf = 2.0 * M * N * K / (ms * 1e-3) / 1e12
        ref_ms = timeit(lambda: torch.matmul(x, w.t()), iters)
        print(json.dumps({"kernel": "gemm", "M": M, "K": K, "N": N, "ms": round(ms, 4),
                          "tflops": round(tf, 1), "frac_peak": round(tf / PEAK_TF, 3),
                          "torch_ms": round(ref_ms, 4)}), flush=True)


def gemm_variants(iters):
    """every tile variant (spx_debug_set_gemm_variant) against the planner's choice and torch"""
    shapes = [(4680, 1536, 4608), (4680, 1536, 1536), (2340, 1536, 4608), (2340, 1536, 1536),
              (1170, 1536, 4608), (1170, 1536, 1536), (585, 1536, 4608), (585, 1536, 1536),
              (585, 1536, 8960), (585, 8960, 1536)]
    only = os.environ.get("KBENCH_GEMM_SHAPES")
    if only:
        shapes = [tuple(int(v) for v in t.split("x")) for t in only.split(",")]
    nv = 0
    while lib().spx_debug_set_gemm_variant(nv) == 0:  # count the planner's variants
        nv += 1
    check(lib().spx_debug_set_gemm_variant(-1))
    for M, K, N in shapes:
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
        y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        row = {"kernel": "gemm_variants", "M": M, "K": K, "N": N}
        for v in list(range(nv)) + [-1]:
            check(lib().spx_debug_set_gemm_variant(v))
            ms = timeit(lambda: check(lib().spx_project_tokens(x.data_ptr(), w.data_ptr(), y.data_ptr(),
                                                               M, K, N, stream_handle())), iters)
            row["auto" if v < 0 else f"v{v}"] = round(ms * 1e3, 2)
        check(lib().spx_debug_set_gemm_variant(-1))
        row["torch_us"] = round(timeit(lambda: torch.matmul(x, w.t()), iters) * 1e3, 2)
        row["auto_frac_peak"] = round(2.0 * M * N * K / (row["auto"] * 1e-6) / 1e12 / PEAK_TF, 3)
        print(json.dumps(row), flush=True)


def gemm_epilogues(iters):
    """the projection epilogues at the Wan shapes: plain, + bias, residual + gate (in place, as
    the engine runs it), GELU"""
    for M, K, N in [(4680, 1536, 1536), (4680, 8960, 1536), (4680, 1536, 8960)]:
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
        y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        res = torch.randn(M, N, device="cuda").to(torch.bfloat16)
        bias = torch.randn(N, device="cuda") * 0.1
        gate = torch.randn(N, device="cuda") * 0.1
        row = {"kernel": "gemm_epilogues", "M": M, "K": K, "N": N}
        cases = {"plain": (None, 0, None, None), "bias": (bias, 0, None, None),
                 "residual_gate": (bias, 1, res, gate), "gelu": (bias, 3, None, None)}
        for name, (b, epi, r, g) in cases.items():
            out = r if r is not None else y
            ms = timeit(lambda: check(lib().spx_project_tokens_ex(
                x.data_ptr(), w.data_ptr(), out.data_ptr(), M, K, N,
                b.data_ptr() if b is not None else None, epi,
                r.data_ptr() if r is not None else None,
                g.data_ptr() if g is not None else None,
                stream_handle())), iters)
            row[name + "_us"] = round(ms * 1e3, 2)
        print(json.dumps(row), flush=True)


def attn_splits(iters):
    """attention at per-rank shapes, each forced kv split count 1..6 against the planner's"""
    for sq, skv, H in ATTN_SHAPES:
        D = 128
        q = (torch.randn(1, sq, H, D, device="cuda") * 0.5).to(torch.bfloat16)
        k = (torch.randn(1, skv, H, D, device="cuda") * 0.5).to(torch.bfloat16)
        v = torch.randn(1, skv, H, D, device="cuda").to(torch.bfloat16)
        o = torch.empty_like(q)
        row = {"kernel": "attn_splits", "sq": sq, "skv": skv, "heads": H}
        for sp in [1, 2, 3, 4, 6, 0]:
            check(lib().spx_debug_set_attn_splits(sp))
            ms = timeit(lambda: check(lib().spx_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                                          o.data_ptr(), 1, sq, skv, H, D, stream_handle())), iters)
            row["auto" if sp == 0 else f"s{sp}"] = round(ms * 1e3, 2)
        check(lib().spx_debug_set_attn_splits(0))
        ideal = 4.0 * sq * skv * H * D / (PEAK_TF * 1e12) * 1e6
        row["auto_frac_peak"] = round(ideal / row["auto"], 3)
        print(json.dumps(row), flush=True)


def rope(iters):
    tab = ctypes.c_void_p()
    split = (ctypes.c_int64 * 3)(22, 21, 21)
    check(lib().spx_rope_table_create(240, 30, 52, 128, 10000.0, split, ctypes.byref(tab)))
    grid = (ctypes.c_int64 * 3)(3, 30, 52)
    for P, norm in [(1, False), (1, True), (8, False)]:
        Lp, H, D = 4680 // P, 12, 128
        x = torch.randn(Lp, H, D, device="cuda").to(torch.bfloat16)
        y = torch.empty_like(x)
        nw = torch.ones(H * D, device="cuda", dtype=torch.bfloat16)
        for start in (0, 18):
            ms = timeit(lambda: check(lib().spx_rope_apply_causal_local(
                tab, x.data_ptr(), y.data_ptr(), 1, Lp, H, D, grid, start, 0, P,
                nw.data_ptr() if norm else None, 1e-6, stream_handle())), iters)
            gbs = 2 * x.numel() * 2 / (ms * 1e-3) / 1e9
            print(json.dumps({"kernel": "rope_single", "P": P, "norm": norm, "start": start,
                              "ms": round(ms, 5), "GBs": round(gbs, 1),
                              "frac_peak": round(gbs / PEAK_GBS, 3)}), flush=True)


def modulate(iters):
    """K1 (Wan adaLN): LayerNorm + modulation, rows x C bf16 -> bf16 (read + write bytes)."""
    for rows in (4680, 585):
        C = 1536
        n = max(2, int(2 * 126 * 2 ** 20 // (2 * rows * C * 2)) + 2)  # rotate past L2
        xs = [torch.randn(rows, C, device="cuda").to(torch.bfloat16) for _ in range(n)]
        ys = [torch.empty_like(xs[0]) for _ in range(n)]
        sh = torch.randn(C, device="cuda") * 0.1
        sc = torch.randn(C, device="cuda") * 0.1
        it = [0]

        def fn():
            i = it[0] % n
            it[0] += 1
            check(lib().spx_layernorm_modulate(xs[i].data_ptr(), ys[i].data_ptr(), rows, C,
                                               sh.data_ptr(), sc.data_ptr(), 1e-6, stream_handle()))
        ms = timeit(fn, iters)
        gbs = 2 * rows * C * 2 / (ms * 1e-3) / 1e9
        print(json.dumps({"kernel": "ln_modulate", "rows": rows, "ms": round(ms, 5), "GBs": round(gbs, 1),
                          "frac_peak": round(gbs / PEAK_GBS, 3), "l2": "cold (rotating buffers)"}), flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which.startswith("attn:"):  # attn:SQxSKVxH
        ATTN_SHAPES[:] = [tuple(int(v) for v in which[5:].split("x"))]
        which = "attn"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    lib()
    if os.environ.get("KBENCH_ATTN_V3"):
        check(lib().spx_debug_set_attn_v3(int(os.environ["KBENCH_ATTN_V3"])))
    _side = torch.cuda.Stream()  # graph capture needs a non-default stream
    torch.cuda.set_stream(_side)
    if which in ("attn", "all"):
        attn(iters)
    if which == "gemmv":
        gemm_variants(iters)
    if which == "gemmepi":
        gemm_epilogues(iters)
    if which == "attnsplit":
        attn_splits(iters)
    if which in ("gemm", "all"):
        gemm(iters)
    if which in ("rope", "all"):
        rope(iters)
    if which in ("modulate", "all"):
        modulate(iters)
