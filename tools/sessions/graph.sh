O=gpurun_out/r02ag; mkdir -p $O
SPX_GRAPH_DEBUG=1 timeout 300 python tools/graph_ab.py > $O/graph_ab.txt 2>&1
