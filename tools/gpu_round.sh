#!/bin/bash
# One evidence session on one B200: gpu tests, smoke, the bench line, then the profiling pass
# (tools/gpu_profile_r02.sh). usage: tools/gpu_round.sh <tag> [skip-tests]
set -x
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 1200 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 1500 bash tools/gpu_profile_r02.sh $TAG > $O/profile.log 2>&1
ls -la $O
