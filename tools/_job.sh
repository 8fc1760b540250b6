O=gpurun_out/r01ax; mkdir -p $O
timeout 180 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k attention > $O/pytest_k.log 2>&1; echo rc=$? >> $O/pytest_k.log
tail -5 $O/pytest_k.log
if grep -q "rc=0" $O/pytest_k.log; then
for i in 1 2; do for v in base new; do
  if [ $v = base ]; then L=paper_2603_06664_b200/variants/base.so; else L=""; fi
  for shp in 4680x4680x12 4680x32760x12 4680x4680x6 2340x4680x3; do
    echo -n "$v " >> $O/ab.txt; SPX_LIB=$L timeout 60 python tools/kbench.py attn:$shp 30 >> $O/ab.txt 2>&1
  done
done; done
fi
