O=gpurun_out/r02bd; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
export KBENCH_GEMM_SHAPES="4680x1536x1536,4680x1536x4608,585x1536x1536,2340x1536x1536"
for rep in 1 2; do
SPX_LIB=$PWD/ab_libs/libspx_head.so timeout 300 python tools/kbench.py gemm 20 >> $O/kb_head.txt 2>&1
timeout 300 python tools/kbench.py gemm 20 >> $O/kb_tree.txt 2>&1
done
for rep in 1 2; do
SPX_LIB=$PWD/ab_libs/libspx_head.so timeout 600 python bench.py --no-cpu-baseline --skip-long-video > $O/bench_head_$rep.json 2> /dev/null
timeout 600 python bench.py --no-cpu-baseline --skip-long-video > $O/bench_tree_$rep.json 2> /dev/null
done
