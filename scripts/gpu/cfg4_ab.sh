# cfg4 plan A/B (bench lines per variant) + cfg5 line.  bash scripts/gpu/cfg4_ab.sh TAG
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-ab}
A="--workload cfg4 --steps 8 --warmup 3 --no-cpu-baseline --aal-steps 0 --no-ar-baseline"
i=0
for v in "" "--plan fused_layout_gemm=1" "--plan tree_attn=0" "--plan fused_layout_gemm=1 --plan tree_attn=0"; do
  timeout 600 python bench.py $A $v > gpurun_out/${TAG}_cfg4_$i.log 2>&1
  echo "variant $i [$v]: $(grep '^{"metric' gpurun_out/${TAG}_cfg4_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(d["ms_per_step"], d["value"], d["config"]["aal"], d["stage_us"])')"
  i=$((i+1))
done
