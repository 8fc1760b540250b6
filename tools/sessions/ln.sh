O=gpurun_out/r02aj; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_wan_parity.py tests/test_gpu_engine.py -x -q -m gpu -k "wan" > $O/pytest_wan.log 2>&1; echo "rc=$?" >> $O/pytest_wan.log
SPX_SPAN_TRACE=1 SPX_GRAPHS=0 timeout 300 python tools/span_probe.py --wan > $O/span_wan.txt 2>&1
SPX_FUSE_LN=0 SPX_SPAN_TRACE=1 SPX_GRAPHS=0 timeout 300 python tools/span_probe.py --wan > $O/span_wan_nofuse.txt 2>&1
for rep in 1 2; do
SPX_FUSE_LN=0 timeout 600 python bench.py --no-cpu-baseline --skip-long-video > $O/bench_nofuse_$rep.json 2> $O/bench_nofuse_$rep.err
timeout 600 python bench.py --no-cpu-baseline --skip-long-video > $O/bench_fuse_$rep.json 2> $O/bench_fuse_$rep.err
done
