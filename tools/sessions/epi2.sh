O=gpurun_out/r02ae; mkdir -p $O
timeout 300 python tools/kbench.py gemmepi 20 > $O/epi.txt 2>&1
SPX_GEMM_EPI_DIRECT=1 timeout 300 python tools/kbench.py gemmepi 20 > $O/epi_direct.txt 2>&1
SPX_GEMM_EPI_DIRECT=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "project" > $O/pytest_direct.log 2>&1; echo "rc=$?" >> $O/pytest_direct.log
for m in ref; do SPX_GEMM_EXPERIMENT=7 SPX_GRAPHS=0 timeout 300 python tools/oproj_trace.py $m >> $O/oproj_trace.txt 2>&1; done
for m in ref; do SPX_GEMM_EPI_DIRECT=1 SPX_GEMM_EXPERIMENT=7 SPX_GRAPHS=0 timeout 300 python tools/oproj_trace.py $m >> $O/oproj_trace_direct.txt 2>&1; done
timeout 600 python bench.py --no-cpu-baseline --skip-long-video > $O/bench.json 2> $O/bench.err
SPX_GEMM_EPI_DIRECT=1 timeout 600 python bench.py --no-cpu-baseline --skip-long-video > $O/bench_direct.json 2> $O/bench_direct.err
