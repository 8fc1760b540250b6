O=gpurun_out/r02z; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "attention" > $O/pytest_attn.log 2>&1; echo "rc=$?" >> $O/pytest_attn.log
KBENCH_ATTN_SHAPES="4680x4680x12,4680x4680x6,4680x4680x3,2340x4680x3,4680x32760x3,2340x32760x3,4680x32760x12" timeout 600 python tools/kbench.py attn 20 > $O/kbench_attn.txt 2>&1
KBENCH_ATTN_SHAPES="4680x4680x6,4680x4680x3,2340x4680x3,2340x32760x3" SPX_ATTN_STREAMK=0 timeout 600 python tools/kbench.py attn 20 > $O/kbench_attn_nosk.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_wan_parity.py tests/test_gpu_wan_block.py -x -q -m gpu > $O/pytest_engine.log 2>&1; echo "rc=$?" >> $O/pytest_engine.log
timeout 600 python bench.py --no-cpu-baseline --skip-long-video > $O/bench.json 2> $O/bench.err
