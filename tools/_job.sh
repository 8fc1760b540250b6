O=gpurun_out/r01p; mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu -k "rope or wan or ablation or sp_ranks" > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
python tools/kbench.py rope 20 > $O/kbench.txt 2>&1
SPX_ROPE_VARIANT=1 python tools/kbench.py rope 20 >> $O/kbench.txt 2>&1
python tools/stage_probe.py --label wan --wan > $O/probe.txt 2>&1
python tools/stage_probe.py --label nofuse --no-fuse-rope >> $O/probe.txt 2>&1
tail -2 $O/pytest_gpu.log; cat $O/kbench.txt $O/probe.txt
