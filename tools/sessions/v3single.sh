O=gpurun_out/r02au; mkdir -p $O
export KBENCH_ATTN_SHAPES="4680x4680x3,4680x4680x6,2340x4680x6,4680x14040x3,4680x32760x3"
for rep in 1 2; do
timeout 300 python tools/kbench.py attn 20 > $O/kb_default_$rep.txt 2>&1
KBENCH_ATTN_V3=2 timeout 300 python tools/kbench.py attn 20 > $O/kb_v3always_$rep.txt 2>&1
done
