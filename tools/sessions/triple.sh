O=gpurun_out/r02bh; mkdir -p $O
SPX_PARITY_LOG=$PWD/$O/parity.jsonl timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "attention" > $O/pytest_attn.log 2>&1; echo "rc=$?" >> $O/pytest_attn.log
export KBENCH_ATTN_SHAPES="4680x4680x6,4680x14040x6,4680x32760x6,4680x4680x12"
for rep in 1 2; do
SPX_ATTN_TRIPLE=0 timeout 300 python tools/kbench.py attn 20 >> $O/kb_off.txt 2>&1
timeout 300 python tools/kbench.py attn 20 >> $O/kb_on.txt 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_wan_parity.py -x -q -m gpu > $O/pytest_engine.log 2>&1; echo "rc=$?" >> $O/pytest_engine.log
