O=gpurun_out/r02as; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "attention" > $O/pytest_attn.log 2>&1; echo "rc=$?" >> $O/pytest_attn.log
export KBENCH_ATTN_SHAPES="2340x4680x3,2340x32760x3,4680x4680x12,1170x4680x6"
for rep in 1 2; do
SPX_ATTN_V3_PAIR=0 timeout 300 python tools/kbench.py attn 20 > $O/kb_v2_$rep.txt 2>&1
timeout 300 python tools/kbench.py attn 20 > $O/kb_v3pair_$rep.txt 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_engine.py -x -q -m gpu > $O/pytest_engine.log 2>&1; echo "rc=$?" >> $O/pytest_engine.log
