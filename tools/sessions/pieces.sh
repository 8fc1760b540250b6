O=gpurun_out/r02bj; mkdir -p $O
SPX_ATTN_EXPERIMENT=5 timeout 300 python tools/attn_pieces.py 4680x4680x6 4680x4680x12 > $O/pieces_triple.txt 2>&1
SPX_ATTN_TRIPLE=0 SPX_ATTN_EXPERIMENT=5 timeout 300 python tools/attn_pieces.py 4680x4680x6 > $O/pieces_persistent.txt 2>&1
