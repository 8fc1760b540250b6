#!/bin/bash
# One GPU session: gpu tests, smoke, bench line, ncu launch list of one chunk, ncu full captures
# of the hot kernels (attention, QKV GEMM + RoPE epilogue, O-projection GEMM).
# usage: tools/gpu_full.sh <tag>
set -x
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --profile-only --steps 1 --warmup 1 > $OUT/ncu_launch.log 2>&1
for K in attn_fwd_v2 gemm_bf16_tn_pair gemm_bf16_tn_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 8 -c 1 -o $OUT/prof_$K \
      python bench.py --profile-only --steps 0 --warmup 1 > $OUT/ncu_$K.log 2>&1
done
ls -la $OUT
