# sweep the unit-width caps of the fused FFN (experiment; rebuilds the library per setting)
cd $GRAFT_REPO_ROOT
for f in ${@:-"-DSERE_MW_GU_MAX=1 -DSERE_MW_DN_MAX=1"}; do
  echo "== flags: $f"
  SERE_NVCC_FLAGS="$(echo $f | tr ',' ' ')" python -c "from paper_2602_07616_b200 import build; build.build(force=True)"
  timeout 120 python scripts/debug_ffn.py --layers 3 2>&1 | grep "^layer" | cut -c1-120
  timeout 120 python scripts/debug_ffn.py --layers 2 --mode topk 2>&1 | grep "^layer" | cut -c1-120
done
