# DRAM bytes of every row-block GEMV launch of one cfg2 draft pass (ncu metrics pass).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:gemv_kernel \
    --launch-skip 455 --launch-count 65 --csv --log-file gpurun_out/gemv_traffic_ncu.csv \
    python scripts/draft_pass_once.py > gpurun_out/gemv_traffic_stdout.log 2>&1
tail -2 gpurun_out/gemv_traffic_stdout.log | cut -c1-300
