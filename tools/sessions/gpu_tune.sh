#!/bin/bash
# Tuning session on one B200: GEMM tile-variant tests + sweep, attention split sweep at the
# per-rank shapes, the Wan-mode launch list, one bench line. usage: tools/gpu_tune.sh <tag>
set -x
O=gpurun_out/${1:-tune}
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu > $O/pytest_kernels.log 2>&1; echo "rc=$?" >> $O/pytest_kernels.log
timeout 600 python tools/kbench.py gemmv 20 > $O/gemmv.txt 2>&1
KBENCH_ATTN_SHAPES="4680x4680x12,4680x4680x6,4680x4680x3,2340x4680x3,4680x32760x3,2340x32760x3" \
  timeout 600 python tools/kbench.py attnsplit 20 > $O/attnsplit.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_wan.csv \
    python tools/wan_chunk.py wan 30 > $O/launches_wan.log 2>&1
python tools/launch_shares.py $O/launches_wan.csv > $O/launches_wan.md 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
ls -la $O
