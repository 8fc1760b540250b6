O=gpurun_out/r01q; mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
for v in "pdl::" "nopdl:SPX_PDL=0:"; do
  IFS=: read lab envv flag <<< "$v"
  env $envv python tools/stage_probe.py --label $lab $flag >> $O/probe.txt 2>&1
  env $envv python tools/stage_probe.py --label $lab --wan >> $O/probe.txt 2>&1
done
tail -2 $O/pytest_gpu.log; cat $O/probe.txt
