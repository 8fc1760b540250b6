O=gpurun_out/r02ai; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "attention" > $O/pytest_attn.log 2>&1; echo "rc=$?" >> $O/pytest_attn.log
for sk in 0 2 3 4 6; do echo "skew $sk"; SPX_ATTN_SKEW=$sk KBENCH_ATTN_SHAPES="4680x4680x12,4680x32760x12" timeout 300 python tools/kbench.py attn 20; done > $O/kbench_skew.txt 2>&1
SPX_LIB=$PWD/ab_libs/libspx_head.so KBENCH_ATTN_SHAPES="4680x4680x12,4680x32760x12" timeout 300 python tools/kbench.py attn 20 > $O/kbench_head.txt 2>&1
