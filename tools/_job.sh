O=gpurun_out/r01k; mkdir -p $O
nvidia-smi -q | grep -i "compute mode" > $O/mode.txt
timeout 900 python -m pytest tests/test_gpu_peer.py -x -q > $O/pytest_peer.log 2>&1; echo rc=$? >> $O/pytest_peer.log
timeout 600 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
tail -30 $O/pytest_peer.log; tail -2 $O/pytest_gpu.log; cat $O/mode.txt
