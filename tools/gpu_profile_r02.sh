#!/bin/bash
# Round-2 profiling pass on one B200 (run under gpurun): kernel microbenchmarks, the launch
# list of the bench workload, and ncu --set full captures of every hot kernel of the three
# modes. Outputs under gpurun_out/$1/.
set -x
O=gpurun_out/${1:-r02p}
mkdir -p $O
python tools/kbench.py all 20 > $O/kbench.txt 2>&1
KBENCH_GEMM_SHAPES="4680x1536x8960,4680x8960x1536,585x1536x8960,585x8960x1536" python tools/kbench.py gemm 10 >> $O/kbench.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --profile-only --steps 1 --warmup 1 > $O/launches.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_full.csv \
    python tools/wan_chunk.py full 30 > $O/launches_full.log 2>&1
SPX_GRAPHS=0 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 9 -c 1 -o $O/attn python tools/wan_chunk.py ref 2 > $O/ncu_attn.log 2>&1
SPX_GRAPHS=0 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_tn_pair -s 9 -c 1 -o $O/qkv python tools/wan_chunk.py ref 2 > $O/ncu_qkv.log 2>&1
SPX_GRAPHS=0 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_tn_kernel -s 9 -c 1 -o $O/oproj python tools/wan_chunk.py ref 2 > $O/ncu_oproj.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rope_norm_pack -s 10 -c 1 -o $O/k3 python tools/wan_chunk.py wan 2 > $O/ncu_k3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ln_modulate -s 10 -c 1 -o $O/k1 python tools/wan_chunk.py wan 2 > $O/ncu_k1.log 2>&1
ncu --set full --clock-control none -k regex:gemm -s 100 -c 12 -o $O/fullblock_gemms python tools/wan_chunk.py full 2 > $O/ncu_full.log 2>&1
for r in attn qkv oproj k3 k1 fullblock_gemms; do
  ncu -i $O/$r.ncu-rep --page details --csv > $O/$r.details.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed > $O/$r.raw.csv 2>/dev/null
done
ls -la $O
