O=gpurun_out/r02al; mkdir -p $O
SPX_GEMM_EXPERIMENT=8 SPX_GRAPHS=0 timeout 300 python tools/ln_trace.py > $O/ln_trace.txt 2>&1
SPX_PDL=0 SPX_GEMM_EXPERIMENT=8 SPX_GRAPHS=0 timeout 300 python tools/ln_trace.py >> $O/ln_trace.txt 2>&1
