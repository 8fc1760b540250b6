# Wan mode: v packed by the QKV GEMM epilogue, K3 on q | k only -- parity, then A/B vs HEAD lib
O=gpurun_out/r02cg; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_wan_block.py tests/test_gpu_wan_parity.py tests/test_gpu_kernels.py -x -q -m gpu > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
if grep -q "rc=0" $O/pytest.log; then
for rep in 1 2; do
 SPX_SPAN_TRACE=1 SPX_LIB=$PWD/ab_libs/libspx_head.so timeout 300 python tools/span_probe.py --wan > $O/span_wan_head_$rep.txt 2>&1
 SPX_SPAN_TRACE=1 timeout 300 python tools/span_probe.py --wan > $O/span_wan_tree_$rep.txt 2>&1
done
bash tools/gpu_ab.sh r02cg gemm
fi
