O=gpurun_out/r02ax; mkdir -p $O
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 --target-processes all python tools/sanitize_run.py > $O/synccheck.txt 2>&1; echo "rc=$?" >> $O/synccheck.txt
KBENCH_ATTN_SHAPES="4680x4680x12,4680x32760x12,2340x4680x3" timeout 300 python tools/kbench.py attn 20 > $O/kbench.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
