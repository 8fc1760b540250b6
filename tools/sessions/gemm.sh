O=gpurun_out/r02x; mkdir -p $O
SPX_PDL=0 SPX_GEMM_EXPERIMENT=7 SPX_GEMM_VARIANT=0 timeout 300 python tools/gemm_timeline.py 4680x1536x4608 > $O/gemm_v0.txt 2>&1
SPX_PDL=0 SPX_GEMM_EXPERIMENT=7 SPX_GEMM_VARIANT=4 timeout 300 python tools/gemm_timeline.py 4680x1536x1536 > $O/gemm_v4.txt 2>&1
SPX_PDL=0 SPX_GEMM_EXPERIMENT=5 SPX_GRAPHS=0 timeout 300 python tools/qkv_trace.py > $O/qkv_trace.txt 2>&1
