O=gpurun_out/r01x; mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
for shp in 4680x4680x12 4680x4680x6 4680x4680x3 2340x4680x3 2340x32760x3 4680x32760x6 4680x32760x12; do
  python tools/kbench.py attn:$shp 20 >> $O/attn_model.txt 2>&1
done
tail -2 $O/pytest_gpu.log; cat $O/attn_model.txt
