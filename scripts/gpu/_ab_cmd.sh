cd $GRAFT_REPO_ROOT
for r in 1 2; do
echo "cfg4 draft: $(timeout 900 python scripts/cfg_plan_ab.py cfg4 draft 'tree_attn=0' 'tree_attn=0,attn_kvsplit=2' 'tree_attn=0,attn_kvsplit=4' 'tree_attn=0,attn_kvsplit=2,attn_stages=8' 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:v['min'] for k,v in d.items()})")"
done
