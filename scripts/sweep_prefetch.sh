# prefetch budget / mode sweep on one box (C4 bench line per setting; CPU baseline skipped)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for cfg in "0 32 0" "32 32 0" "64 32 0" "96 32 0" "64 64 0" "64 32 1" "96 48 1"; do
  set -- $cfg
  echo "== [$rep] mb=$1 ctas=$2 whole=$3 $(timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 3 --prefetch-mb $1 --prefetch-ctas $2 --prefetch-whole $3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["topk"]["value"], d["roofline"]["stage_us_per_layer_avg"], d["roofline"]["frac"])')"
done
done
