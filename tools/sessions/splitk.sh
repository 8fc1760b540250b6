# split-K GEMM: kernel parity first (bounded), then the GPU suite, then per-variant timings
O=gpurun_out/r02ce; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "split_k or every_tile_variant or project_tokens_matches" > $O/pytest_gemm.log 2>&1; echo rc=$? >> $O/pytest_gemm.log
if grep -q "rc=0" $O/pytest_gemm.log; then
  timeout 1200 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
  KBENCH_GEMM_SHAPES="585x1536x1536,1170x1536x1536,585x8960x1536,585x1536x4608,1170x1536x4608,4680x1536x1536" timeout 300 python tools/kbench.py gemmv 20 > $O/gemmv.txt 2>&1
fi
