O=gpurun_out/r02ad; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "project" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/kbench.py gemmepi 20 > $O/epi.txt 2>&1
for m in wan ref; do SPX_GEMM_EXPERIMENT=7 SPX_GRAPHS=0 timeout 300 python tools/oproj_trace.py $m >> $O/oproj_trace.txt 2>&1; done
for m in wan ref; do SPX_PDL=0 SPX_GEMM_EXPERIMENT=7 SPX_GRAPHS=0 timeout 300 python tools/oproj_trace.py $m >> $O/oproj_trace_nopdl.txt 2>&1; done
