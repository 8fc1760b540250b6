O=gpurun_out/r02aq; mkdir -p $O
export KBENCH_ATTN_SHAPES="4680x4680x12,4680x32760x12"
for rep in 1 2; do
  for v in base poly0 poly2 slots5; do
    if [ $v = base ]; then L=""; else L=$PWD/paper_2603_06664_b200/variants/$v.so; fi
    echo "$v rep $rep" >> $O/ab.txt
    SPX_LIB=$L timeout 300 python tools/kbench.py attn 20 >> $O/ab.txt 2>&1
  done
done
