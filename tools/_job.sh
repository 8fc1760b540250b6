O=gpurun_out/r01au; mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu -k "rope or wan or norm" > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
for i in 1 2; do for v in base new; do
  if [ $v = base ]; then L=paper_2603_06664_b200/variants/base.so; else L=""; fi
  echo "== $v" >> $O/ab.txt; SPX_LIB=$L python tools/kbench.py rope 20 >> $O/ab.txt 2>&1
  SPX_LIB=$L python tools/stage_probe.py --wan --label $v >> $O/ab.txt 2>&1
done; done
tail -2 $O/pytest_gpu.log; cat $O/ab.txt
