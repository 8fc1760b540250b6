O=gpurun_out/r02bo; mkdir -p $O
export KBENCH_ATTN_SHAPES="2340x4680x3,1170x4680x6,4680x4680x6,4680x4680x12"
for rep in 1 2; do
SPX_LIB=$PWD/ab_libs/libspx_head.so timeout 300 python tools/kbench.py attn 20 >> $O/kb_prev.txt 2>&1
timeout 300 python tools/kbench.py attn 20 >> $O/kb_tree.txt 2>&1
done
