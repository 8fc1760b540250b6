O=gpurun_out/r01r; mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
for i in 1 2; do
python tools/stage_probe.py --label pf >> $O/probe.txt 2>&1
python tools/stage_probe.py --label nopf --no-prefetch >> $O/probe.txt 2>&1
done
tail -2 $O/pytest_gpu.log; cat $O/probe.txt
