cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/a_pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1
timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/a_prof_single.log 2>&1
timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/a_prof_dual.log 2>&1
timeout 900 python bench.py > gpurun_out/a_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/a_launches.csv python tools/prof_step.py 24 0 1 > /dev/null 2>&1
echo done
