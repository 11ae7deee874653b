cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_psd_gpu.py -q -x -k "decode_step" > gpurun_out/ii_pytest_decode.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ii_pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/ii_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ii_launches.csv python tools/prof_step.py 24 1 1 > /dev/null 2>&1
echo done
