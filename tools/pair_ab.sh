# CTA-pair stream-K GEMMs: correctness (GEMM tests, greedy PSD identities) and A/B timing
timeout 900 python -m pytest tests/test_gemm_gpu.py -x -q -m gpu > gpurun_out/r02n_pair_tests.log 2>&1; echo gemm_tests=$?; tail -3 gpurun_out/r02n_pair_tests.log
for v in 0 1; do echo "== PSD_GEMM_PAIR=$v"; PSD_GEMM_PAIR=$v timeout 300 python tools/kbench.py --only gemmguM,gemmpf 2>&1; done > gpurun_out/r02n_pair_ab.txt
cat gpurun_out/r02n_pair_ab.txt
