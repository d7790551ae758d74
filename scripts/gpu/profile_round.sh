# Launch list of one eager cfg2 step + full ncu captures of the dominant kernels (profiling only; the
# numbers ncu prints are serialised / cold-cache: compare shares, not absolutes).
#   bash scripts/gpu/profile_round.sh TAG
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-r2}
R="--nvtx --nvtx-include steps/ --clock-control none"
timeout 600 ncu $R --metrics gpu__time_duration.sum --csv --log-file gpurun_out/${TAG}_launches.csv \
  python scripts/profile_step.py cfg2 1 > gpurun_out/${TAG}_launch_stdout.log 2>&1
# draft layer-0 gate|up GEMV (the dominant kernel family), verify layer-0 tree attention, verify layer-0 gate|up GEMM
timeout 600 ncu $R --set full --import-source on -k regex:gemv_kernel --launch-skip 2 -c 1 -o gpurun_out/${TAG}_gemv_gu -f \
  python scripts/profile_step.py cfg2 1 > /dev/null 2>&1
timeout 600 ncu $R --set full --import-source on -k regex:attn_tree --launch-skip 0 -c 1 -o gpurun_out/${TAG}_attn_tree -f \
  python scripts/profile_step.py cfg2 1 > /dev/null 2>&1
timeout 600 ncu $R --set full --import-source on -k regex:gemm_bf16_tc --launch-skip 2 -c 1 -o gpurun_out/${TAG}_gemm_gu -f \
  python scripts/profile_step.py cfg2 1 > /dev/null 2>&1
timeout 600 ncu $R --set full --import-source on -k regex:attn_dec --launch-skip 16 -c 1 -o gpurun_out/${TAG}_attn_dec -f \
  python scripts/profile_step.py cfg2 1 > /dev/null 2>&1
ls -la gpurun_out/${TAG}_*
