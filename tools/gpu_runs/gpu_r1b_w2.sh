cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/w_mem.txt
timeout 1500 python bench.py --layout tp --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/w_bench_cfg4.log 2>&1
echo done
