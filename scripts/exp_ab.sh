# A/B sweep of compile-time variants on the SAME box (rebuilds per setting); args: flag sets (commas = spaces)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for f in "$@"; do
  SERE_NVCC_FLAGS="$(echo $f | tr ',' ' ')" python -c "from paper_2602_07616_b200 import build; build.build(force=True)"
  echo "== [$rep] $f: $(timeout 200 python scripts/ffn_replay.py sere 2>&1 | tail -1) | $(timeout 200 python scripts/ffn_replay.py topk 2>&1 | tail -1)"
done
done
