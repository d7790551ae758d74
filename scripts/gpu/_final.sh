cd $GRAFT_REPO_ROOT
bash scripts/gpu/full.sh r2zb
( timeout 900 python bench.py --workload cfg4 --steps 8 --warmup 3 --no-cpu-baseline --aal-steps 0 --no-ar-baseline ) > gpurun_out/r2zb_bench_cfg4.log 2>&1; grep '^{"metric"' gpurun_out/r2zb_bench_cfg4.log | head -c 300; echo
( timeout 1200 python bench.py --workload cfg5 --steps 6 --warmup 3 --no-cpu-baseline --aal-steps 0 --no-ar-baseline ) > gpurun_out/r2zb_bench_cfg5.log 2>&1; grep '^{"metric"' gpurun_out/r2zb_bench_cfg5.log | head -c 300; echo
( timeout 900 python bench.py --impl reference --steps 20 --warmup 3 ) > gpurun_out/r2zb_bench_reference.log 2>&1; tail -c 600 gpurun_out/r2zb_bench_reference.log; echo
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "steps/" --csv --log-file gpurun_out/r2zb_cfg4_launches.csv python scripts/profile_step.py cfg4 1 > /dev/null 2>&1; wc -l gpurun_out/r2zb_cfg4_launches.csv
