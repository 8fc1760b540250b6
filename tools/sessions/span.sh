O=gpurun_out/r02aa; mkdir -p $O
SPX_SPAN_TRACE=1 SPX_GRAPHS=0 timeout 300 python tools/span_probe.py > $O/span_ref.txt 2>&1
SPX_SPAN_TRACE=1 SPX_GRAPHS=0 timeout 300 python tools/span_probe.py --wan > $O/span_wan.txt 2>&1
