# report-parity GPU test + QKV epilogue cost probe (rotation off: SPX_GEMM_EXPERIMENT=1)
O=gpurun_out/r02cc; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q -m gpu -k "report" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for rep in 1 2; do
 SPX_SPAN_TRACE=1 timeout 300 python tools/span_probe.py > $O/span_base_$rep.txt 2>&1
 SPX_SPAN_TRACE=1 SPX_GEMM_EXPERIMENT=1 timeout 300 python tools/span_probe.py > $O/span_norot_$rep.txt 2>&1
done
