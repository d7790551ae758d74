set -x
nproc; free -g; lscpu | head -20; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_base_bench.log 2>&1; tail -c 3000 gpurun_out/r2_base_bench.log
