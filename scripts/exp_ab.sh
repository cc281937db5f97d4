# A/B sweep of compile-time variants on the SAME box (rebuilds per setting); args: flag sets (commas = spaces)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for f in "$@"; do
  SERE_NVCC_FLAGS="$(echo $f | tr ',' ' ')" python -c "from paper_2602_07616_b200 import build; build.build(force=True)"
  echo "== [$rep] $f: $(timeout 200 python scripts/kernel_times.py --layers 24 --pdl 0 2>&1 | grep -E 'wall span|moe_ffn' | tr -s ' ' | tr '\n' ' ')"
done
done
