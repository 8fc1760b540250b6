"""Generate tests/golden/reference_golden.json by running the REFERENCE itself.

Runs the unmodified reference sources compiled into oracle/_ref/libspattn_ref.so (see
oracle/Makefile; needs /root/reference at build time) and records checksums and sample
values that pin the oracle restatement (tests/test_oracle.py) and the device path.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402

TINY = dict(frames=3, grid_h=8, grid_w=8, num_blocks=3, layers=2, heads=4, head_dim=64)
DESK = dict(frames=3, grid_h=4, grid_w=4, num_blocks=5, layers=4, steps=2, heads=8, head_dim=16)


def run(**kw):
    out, ledger = oracle.ref_generate(**kw)
    return {
        "checksums": [oracle.checksum(b) for b in out],
        "first": [repr(float(b.reshape(-1)[0])) for b in out],
        "samples": [repr(float(out.reshape(-1)[i])) for i in (0, 1, 17, 1000, out.size - 1)],
        "ledger": ledger,
    }


def main():
    assert oracle.ref_available(), "build oracle/_ref first (make -C oracle)"
    g = {"source": "reference proj/ compiled from /root/reference by oracle/Makefile"}
    g["tiny_steps2_p1"] = run(**TINY, steps=2)
    g["tiny_steps4_p1"] = run(**TINY, steps=4)
    g["tiny_steps2_window3_p1"] = run(**TINY, steps=2, window=3)
    for P in (2, 4):
        g[f"tiny_steps2_opt_p{P}"] = run(**TINY, steps=2, world=P, variant="optimized")
    g["desk_p1"] = run(**DESK)
    for P in (2, 4, 8):
        g[f"desk_opt_p{P}"] = run(**DESK, world=P, variant="optimized")
        g[f"desk_base_p{P}"] = run(**DESK, world=P, variant="baseline")
    g["desk_fault_p2"] = run(**DESK, world=2, variant="optimized", force_start_frame_zero=True)
    g["desk_window6_p2"] = run(**DESK, world=2, variant="optimized", window=6)
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.json"), "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)
    print("wrote", len(g), "entries")
    reports()


# the reference's own run reports (report.cpp to_json(GenerationResult), timing fields
# stripped) for the report-layout parity tests (tests/test_report.py, test_gpu_engine.py)
REPORTS = {
    "tiny_steps2_opt_p2": dict(TINY, steps=2, world=2, variant="optimized"),
    "tiny_steps2_p1_reference": dict(TINY, steps=2),
    "desk_base_p4": dict(DESK, world=4, variant="baseline"),
    "desk_opt_p8_window6": dict(DESK, world=8, variant="optimized", window=6),
    "desk_fault_p2": dict(DESK, world=2, variant="optimized", force_start_frame_zero=True),
    "desk_opt_p2_ablation_5": dict(DESK, world=2, variant="optimized", ablation=5),
}


def reports():
    r = {"source": "reference proj/src/report.cpp to_json(GenerationResult) + strip_timing_fields, "
                   "compiled from /root/reference by oracle/Makefile (_ref/libspattn_ref_report.so)",
         "configs": {k: {kk: vv for kk, vv in v.items()} for k, v in REPORTS.items()}}
    for name, kw in REPORTS.items():
        r[name] = json.loads(oracle.ref_report_json(**kw))
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_reports.json"), "w") as f:
        json.dump(r, f, indent=1, sort_keys=True)
    print("wrote", len(REPORTS), "reports")


if __name__ == "__main__":
    main()
