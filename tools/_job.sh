O=gpurun_out/r01ai; mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --same-device --steps 2 --warmup 1 --skip-long-video --no-cpu-baseline > $O/bench_p2.json 2> $O/bench_p2.err; echo rc=$? >> $O/bench_p2.err
tail -2 $O/pytest_gpu.log; tail -1 $O/bench_p2.err; head -c 400 $O/bench_p2.json
