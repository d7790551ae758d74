# GPU tests + the default bench line + the reference arm (what the driver runs at round end).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r2}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputest.log 2>&1; tail -5 gpurun_out/${TAG}_gputest.log
( time timeout 900 python bench.py --steps 20 --warmup 5 ) > gpurun_out/${TAG}_bench.log 2>&1; tail -c 4000 gpurun_out/${TAG}_bench.log
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/${TAG}_ref.log 2>&1; tail -c 2000 gpurun_out/${TAG}_ref.log
