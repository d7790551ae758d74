cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash scripts/gpu/run_tests.sh r2i -k "two_lane or continuous"
for i in 1 2; do
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-ar-baseline > gpurun_out/ovl_off_$i.log 2>&1
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-ar-baseline --overlap-compaction > gpurun_out/ovl_on_$i.log 2>&1
done
for f in gpurun_out/ovl_*.log; do echo $f; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['p50_step_ms'], d['value'], d['launches_per_step'])"; done
