O=gpurun_out/r02w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "attention" > $O/pytest_attn.log 2>&1; echo "rc=$?" >> $O/pytest_attn.log
SPX_ATTN_EXPERIMENT=5 timeout 300 python tools/attn_timeline.py 4680x4680x12 4680x32760x12 > $O/attn_timeline.txt 2>&1
timeout 300 python tools/kbench.py attn 20 > $O/kbench_attn.txt 2>&1
SPX_ATTN_V3_PERSISTENT=0 timeout 300 python tools/kbench.py attn 20 > $O/kbench_attn_nonpersistent.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_wan_parity.py -x -q -m gpu > $O/pytest_engine.log 2>&1; echo "rc=$?" >> $O/pytest_engine.log
timeout 600 python bench.py --no-cpu-baseline --skip-long-video > $O/bench.json 2> $O/bench.err
SPX_ATTN_V3_PERSISTENT=0 timeout 600 python bench.py --no-cpu-baseline --skip-long-video > $O/bench_nonpersistent.json 2> $O/bench_np.err
