O=gpurun_out/r02ab; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "project" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/kbench.py gemmepi 20 > $O/epi_new.txt 2>&1
SPX_LIB=$PWD/ab_libs/libspx_old.so timeout 300 python tools/kbench.py gemmepi 20 > $O/epi_old.txt 2>&1
SPX_SPAN_TRACE=1 SPX_GRAPHS=0 timeout 300 python tools/span_probe.py --wan > $O/span_wan.txt 2>&1
