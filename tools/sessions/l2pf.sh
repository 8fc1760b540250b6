O=gpurun_out/r02be; mkdir -p $O
for rep in 1 2; do
SPX_L2_PREFETCH=0 timeout 600 python bench.py --no-cpu-baseline --skip-long-video > $O/bench_off_$rep.json 2> /dev/null
SPX_L2_PREFETCH=1 timeout 600 python bench.py --no-cpu-baseline --skip-long-video > $O/bench_on_$rep.json 2> /dev/null
done
SPX_L2_PREFETCH=1 SPX_SPAN_TRACE=1 SPX_GRAPHS=0 timeout 300 python tools/span_probe.py > $O/span_on.txt 2>&1
SPX_L2_PREFETCH=0 SPX_SPAN_TRACE=1 SPX_GRAPHS=0 timeout 300 python tools/span_probe.py > $O/span_off.txt 2>&1
