#!/bin/bash
# v3 attention: correctness tests + kbench A/B against v2 + ncu of both (one B200)
O=gpurun_out/${1:-r02v}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k "attention" > $O/tests.txt 2>&1; echo rc=$? >> $O/tests.txt
for v in 0 1 0 1; do KBENCH_ATTN_V3=$v python tools/kbench.py attn 20 >> $O/kbench_v$v.txt 2>&1; done
SPX_GRAPHS=0 SPX_ATTN_V3=1 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 9 -c 1 -o $O/attn_v3 python tools/wan_chunk.py ref 2 > $O/ncu_v3.log 2>&1
SPX_GRAPHS=0 SPX_ATTN_V3=0 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 9 -c 1 -o $O/attn_v2 python tools/wan_chunk.py ref 2 > $O/ncu_v2.log 2>&1
for r in attn_v3 attn_v2; do
  ncu -i $O/$r.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum > $O/$r.raw.csv 2>/dev/null
done
tail -3 $O/tests.txt; cat $O/kbench_v*.txt
