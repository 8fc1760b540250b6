O=gpurun_out/r01bd; mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
for i in 1 2; do for v in base new; do
  if [ $v = base ]; then L=paper_2603_06664_b200/variants/base.so; else L=""; fi
  SPX_LIB=$L SPX_GEMM_EXPERIMENT=5 python tools/stage_probe.py --chunks 3 --label $v >> $O/probe.txt 2>&1
done; done
tail -2 $O/pytest_gpu.log; grep -E "label|\"cta\": 0" $O/probe.txt | cut -c1-250
