O=gpurun_out/r02bc; mkdir -p $O
for b in 4096 1024 3072 8192 16384; do
  echo "stage_bytes $b" >> $O/k1.txt
  SPX_ROWPIPE_STAGE_BYTES=$b timeout 300 python -c "
import sys; sys.argv=['kbench','x','20']; sys.path.insert(0,'tools')
import kbench, torch
kbench.lib(); s=torch.cuda.Stream(); torch.cuda.set_stream(s); kbench.modulate(20); kbench.rope(20)" >> $O/k1.txt 2>&1
done
