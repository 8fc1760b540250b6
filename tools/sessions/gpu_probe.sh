#!/bin/bash
# Probe session on one B200: correctness of the touched kernels, then timelines and kbench.
# usage: tools/gpu_probe.sh <tag>
set -x
O=gpurun_out/${1:-probe}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q -m gpu -k "rope or norm or layernorm or wan_mode or variant or split or attention" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
SPX_ATTN_EXPERIMENT=5 timeout 300 python tools/attn_timeline.py 4680x4680x12 4680x32760x12 4680x4680x3 > $O/attn_timeline.txt 2>&1
SPX_ATTN_EXPERIMENT=5 SPX_ATTN_SPLITS=2 timeout 300 python tools/attn_timeline.py 2340x4680x3 > $O/attn_timeline_s2.txt 2>&1
SPX_ATTN_EXPERIMENT=5 SPX_ATTN_SPLITS=1 timeout 300 python tools/attn_timeline.py 2340x4680x3 >> $O/attn_timeline_s2.txt 2>&1
for v in 1 3 4 7; do
  SPX_GEMM_EXPERIMENT=7 SPX_GEMM_VARIANT=$v timeout 300 python tools/gemm_timeline.py 585x1536x1536 585x1536x4608 4680x1536x1536 > $O/gemm_timeline_v$v.txt 2>&1
done
timeout 300 python tools/kbench.py rope 20 > $O/kbench_rope.txt 2>&1
timeout 300 python -c "
import sys; sys.argv=['kbench','x','20']; sys.path.insert(0,'tools')
import kbench, torch
kbench.lib(); s=torch.cuda.Stream(); torch.cuda.set_stream(s); kbench.modulate(20)" >> $O/kbench_rope.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --skip-long-video > $O/bench.json 2> $O/bench.err
ls -la $O
