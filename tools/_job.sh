O=gpurun_out/r01bc; mkdir -p $O
SPX_SPAN_TRACE=1 python tools/span_probe.py > $O/spans.txt 2>&1
grep kernels_per_call $O/spans.txt
