cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_verify_gpu.py tests/test_psd_gpu.py tests/test_pair_gpu.py -q -x > gpurun_out/hh_pytest.log 2>&1
timeout 300 python tools/kbench.py --only k1 > gpurun_out/hh_kbench.log 2>&1
timeout 1200 python bench.py --workload cfg3 --no-cpu-baseline --steps 2 --warmup 2 > gpurun_out/hh_bench_cfg3.log 2>&1
echo done
