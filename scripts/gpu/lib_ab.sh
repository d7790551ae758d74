# Same-box A/B of two libygg builds (paper_2512_23858_b200/ab_prev/libygg.so = the previous build):
# the graph-replayed draft pass and verify forward, interleaved.   bash scripts/gpu/lib_ab.sh [rounds]
cd $GRAFT_REPO_ROOT
for r in $(seq ${1:-2}); do
  for lib in "" "paper_2512_23858_b200/ab_prev/libygg.so"; do
    echo "lib=${lib:-current}: $(YGG_LIB_PATH=$lib timeout 300 python scripts/attn_ab.py 2>/dev/null | tail -1 | cut -c1-200)"
  done
done
