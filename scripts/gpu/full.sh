# Full round-end check: GPU tests, smoke, bench line, reference arm.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r2}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputest.log 2>&1; tail -15 gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -5 gpurun_out/${TAG}_smoke.log
( time timeout 900 python bench.py --steps 20 --warmup 5 ) > gpurun_out/${TAG}_bench.log 2>&1; tail -c 4500 gpurun_out/${TAG}_bench.log
