O=gpurun_out/r01as; mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
for i in 1 2 3; do for v in base new; do
  if [ $v = base ]; then L=paper_2603_06664_b200/variants/base.so; else L=""; fi
  for shp in 4680x4680x12 4680x32760x12 4680x4680x6; do
    echo -n "$v " >> $O/ab.txt; SPX_LIB=$L python tools/kbench.py attn:$shp 30 >> $O/ab.txt 2>&1
  done
done; done
tail -2 $O/pytest_gpu.log
