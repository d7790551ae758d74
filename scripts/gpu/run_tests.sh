# GPU tests only (optionally a -k filter): python -m pytest tests -m gpu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r2}; shift
timeout 1500 python -m pytest tests -m gpu -q "$@" > gpurun_out/${TAG}_gputest.log 2>&1; tail -30 gpurun_out/${TAG}_gputest.log
