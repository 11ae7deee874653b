# round-2 closing run: GPU suite, smoke, default bench line, ncu launch list of the bench
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02z_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02z_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02z_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02z_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02z_bench.log > gpurun_out/r02z_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv --log-file gpurun_out/r02z_bench_launches.csv python bench.py --steps 1 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/r02z_bench_ncu.log 2>&1; echo "ncu rc=$?"
python tools/agg_ncu.py gpurun_out/r02z_bench_launches.csv > gpurun_out/r02z_bench_launches_agg.txt 2>&1
head -20 gpurun_out/r02z_bench_launches_agg.txt
