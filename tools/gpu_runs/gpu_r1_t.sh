cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in 0 1 2; do PSD_SILU_MODE=$m timeout 120 python tools/kbench.py --only gemmx > gpurun_out/kbench_silu$m.log 2>&1; done
timeout 300 python -m pytest tests/test_psd_gpu.py -q -k continuous > gpurun_out/pytest_t.log 2>&1
echo done
