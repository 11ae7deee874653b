set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -m paper_2603_18016_b200.verify_bench --quick --json gpurun_out/verify_quick.json > gpurun_out/verify_quick.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/verify_launches.csv python tools/prof_verify.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify -s 2 -c 4 -o gpurun_out/verify_prof python tools/prof_verify.py > gpurun_out/ncu_full.log 2>&1
echo done
