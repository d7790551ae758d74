cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_e2e.py -q -x -k "accept or sample" > gpurun_out/acc1.log 2>&1; tail -15 gpurun_out/acc1.log | cut -c1-300
( timeout 900 python bench.py --workload cfg4 --steps 8 --warmup 3 --no-cpu-baseline --aal-steps 0 --no-ar-baseline ) > gpurun_out/acc_bench_cfg4.log 2>&1; grep '^{"metric"' gpurun_out/acc_bench_cfg4.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['stage_us'], d['config'].get('aal'))"
