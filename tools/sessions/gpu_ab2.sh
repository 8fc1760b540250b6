#!/bin/bash
O=gpurun_out/${1:-r02ab}
mkdir -p $O
python tools/graph_ab.py > $O/graph_ab.txt 2>&1
SPX_PDL=0 python tools/graph_ab.py > $O/graph_ab_nopdl.txt 2>&1
export KBENCH_GEMM_SHAPES="4680x8960x1536,4680x1536x1536,4680x1536x8960,4680x1536x4608"
for r in 0 -1 0 -1; do echo "raster $r" >> $O/raster.txt; SPX_GEMM_RASTER=$r python tools/kbench.py gemm 20 >> $O/raster.txt 2>&1; done
cat $O/graph_ab.txt $O/graph_ab_nopdl.txt $O/raster.txt
