O=gpurun_out/r01j; mkdir -p $O
timeout 600 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
SPX_GEMM_EXPERIMENT=5 python tools/stage_probe.py --chunks 1 > $O/trace_rot.txt 2>&1
python tools/stage_probe.py --label default > $O/probe.txt 2>&1
python tools/stage_probe.py --label nofuse --no-fuse-rope >> $O/probe.txt 2>&1
tail -2 $O/pytest_gpu.log; cat $O/trace_rot.txt $O/probe.txt
