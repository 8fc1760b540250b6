O=gpurun_out/r02ao; mkdir -p $O
for rep in 1 2; do
SPX_FUSE_LN=0 timeout 600 python bench.py --no-cpu-baseline --skip-long-video > $O/bench_nofuse_$rep.json 2> $O/bench_nofuse_$rep.err
timeout 600 python bench.py --no-cpu-baseline --skip-long-video > $O/bench_fuse_$rep.json 2> $O/bench_fuse_$rep.err
done
