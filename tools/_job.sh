O=gpurun_out/r01an; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
for shp in 4680x4680x12 4680x4680x6 4680x4680x3 2340x4680x3 2340x32760x3 4680x32760x6 4680x14040x6 4680x32760x12; do
  SPX_ATTN_VERBOSE=1 python tools/kbench.py attn:$shp 20 2>&1 | sort | uniq | grep -v "^$" >> $O/attn.txt
done
tail -2 $O/pytest_gpu.log; cat $O/attn.txt
