O=gpurun_out/r01bb; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_peer.py -x -q > $O/pytest_peer.log 2>&1; echo rc=$? >> $O/pytest_peer.log
tail -15 $O/pytest_peer.log
