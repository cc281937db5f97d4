# same-box A/B of compile-time variants on the full C4 step (kernel times + wall span)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for f in "$@"; do
  SERE_NVCC_FLAGS="$(echo $f | tr ',' ' ')" python -c "from paper_2602_07616_b200 import build; build.build(force=True)"
  echo "== [$rep] $f: $(timeout 200 python scripts/kernel_times.py --layers 24 --pdl 0 2>&1 | grep -E 'wall span|combine|route|align|permute' | tr -s ' ' | cut -c1-60 | tr '\n' '|')"
done
done
