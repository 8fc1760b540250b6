O=gpurun_out/r01y; mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
timeout 600 python bench.py --skip-long-video --no-cpu-baseline > $O/bench.json 2> $O/bench.err
tail -2 $O/pytest_gpu.log; python -c "
import json;d=json.load(open('$O/bench.json'))
for k in ('value','first_frame_latency_ms','e2e','clocks'): print(k, d.get(k))"
