O=gpurun_out/r01ag; mkdir -p $O
timeout 600 python bench.py --skip-long-video --no-cpu-baseline > $O/bench.json 2> $O/bench.err
python -c "
import json;d=json.load(open('$O/bench.json'))
for k in ('value','first_frame_latency_ms','e2e','clocks','roofline'): print(k, d.get(k))"
