#!/bin/bash
# A/B of the working tree against ab_libs/libspx_head.so on one box (tools/ab_build.sh first):
# kbench of the given kind and the bench line, alternating B (HEAD) / A (tree) twice.
# usage: tools/gpu_ab.sh <tag> <kbench kind: attn|gemm|rope|gemmepi|...> [bench args]
O=gpurun_out/${1:-ab}; K=${2:-attn}; shift 2
mkdir -p $O
for rep in 1 2; do
  SPX_LIB=$PWD/ab_libs/libspx_head.so timeout 300 python tools/kbench.py $K 20 > $O/kbench_head_$rep.txt 2>&1
  timeout 300 python tools/kbench.py $K 20 > $O/kbench_tree_$rep.txt 2>&1
done
for rep in 1 2; do
  SPX_LIB=$PWD/ab_libs/libspx_head.so timeout 600 python bench.py --no-cpu-baseline --skip-long-video "$@" > $O/bench_head_$rep.json 2> $O/bench_head_$rep.err
  timeout 600 python bench.py --no-cpu-baseline --skip-long-video "$@" > $O/bench_tree_$rep.json 2> $O/bench_tree_$rep.err
done
python3 - $O <<'PY'
import json, sys, glob, os
O = sys.argv[1]
for f in sorted(glob.glob(os.path.join(O, "bench_*.json"))):
    try:
        d = json.load(open(f))
        print(os.path.basename(f), round(d["value"], 2), "e2e", round(d["e2e"]["value"], 2), "attn_us",
              round(d["roofline"]["avg_launch_ms"] * 1e3, 2), "wan", round(d["wan_block"]["latent_frames_per_s"], 2),
              "full", round(d["wan_block_full"]["latent_frames_per_s"], 2), "clk", d["clocks"]["sm_mhz"])
    except Exception as e:
        print(f, "unreadable", e)
PY
