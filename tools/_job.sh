O=gpurun_out/r01ao; mkdir -p $O
for i in 1 2 3; do for v in base new; do
  if [ $v = base ]; then L=paper_2603_06664_b200/variants/base.so; else L=""; fi
  for shp in 4680x4680x12 4680x32760x12; do
    echo -n "$v " >> $O/ab.txt; SPX_LIB=$L python tools/kbench.py attn:$shp 30 >> $O/ab.txt 2>&1
  done
done; done
python tools/stage_probe.py --label new >> $O/probe.txt 2>&1
SPX_LIB=paper_2603_06664_b200/variants/base.so python tools/stage_probe.py --label base >> $O/probe.txt 2>&1
cat $O/ab.txt $O/probe.txt
