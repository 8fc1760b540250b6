O=gpurun_out/r02bf; mkdir -p $O
export KBENCH_ATTN_SHAPES="4680x4680x12,4680x32760x12"
for rep in 1 2; do
  for v in base bx2 bx4 bx8; do
    if [ $v = base ]; then L=""; else L=$PWD/paper_2603_06664_b200/variants/$v.so; fi
    echo "$v rep $rep" >> $O/kb.txt
    SPX_LIB=$L timeout 300 python tools/kbench.py attn 20 >> $O/kb.txt 2>&1
  done
done
for v in base bx2 bx4 bx8; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2603_06664_b200/variants/$v.so; fi
  SPX_LIB=$L SPX_PARITY_LOG=$PWD/$O/parity_$v.jsonl timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "attention_matches_fp32" > $O/pytest_$v.log 2>&1
done
