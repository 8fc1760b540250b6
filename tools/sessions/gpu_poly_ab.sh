#!/bin/bash
# A/B of the FMA-pipe exp share (SPX_POLY_OF_8) for the v3 attention kernel (kbench attn)
O=gpurun_out/${1:-r02poly}
mkdir -p $O
export KBENCH_ATTN_SHAPES="4680x4680x12,4680x32760x12"
for rep in 1 2; do
  for v in 3 1 2 4 5; do
    if [ $v = 3 ]; then L=""; else L=paper_2603_06664_b200/variants/poly$v.so; fi
    echo "poly $v rep $rep v3" >> $O/ab.txt
    SPX_LIB=$L KBENCH_ATTN_V3=1 python tools/kbench.py attn 20 >> $O/ab.txt 2>&1
  done
done
cat $O/ab.txt
