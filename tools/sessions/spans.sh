O=gpurun_out/r02ap; mkdir -p $O
SPX_SPAN_TRACE=1 timeout 300 python tools/chunk_spans.py 10 > $O/chunk_spans.txt 2>&1
nvidia-smi -q -d POWER,CLOCK > $O/smi.txt 2>&1
