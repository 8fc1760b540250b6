O=gpurun_out/r01ak; mkdir -p $O
for i in 1 2 3; do for v in base slots4 slots3 s4pfw; do
  for shp in 4680x4680x12 4680x32760x12 2340x4680x3; do
    echo -n "$v " >> $O/ab.txt; SPX_LIB=paper_2603_06664_b200/variants/$v.so python tools/kbench.py attn:$shp 30 >> $O/ab.txt 2>&1
  done
done; done
cat $O/ab.txt
