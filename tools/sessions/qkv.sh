mkdir -p gpurun_out/r02v
SPX_GEMM_EXPERIMENT=5 SPX_GRAPHS=0 timeout 300 python tools/qkv_trace.py > gpurun_out/r02v/qkv_trace.txt 2>&1
SPX_GEMM_EXPERIMENT=7 SPX_GEMM_VARIANT=0 timeout 300 python tools/gemm_timeline.py 4680x1536x4608 > gpurun_out/r02v/gemm_plain_qkv.txt 2>&1
SPX_GEMM_EXPERIMENT=7 timeout 300 python tools/gemm_timeline.py 4680x1536x1536 >> gpurun_out/r02v/gemm_plain_qkv.txt 2>&1
