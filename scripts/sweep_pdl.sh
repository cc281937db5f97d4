# PDL bit-mask sweep on one box (C4 bench line per setting): 1 align, 2 permute, 4 FFN, 8 combine, 16 RMSNorm
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for m in 0 4 6 2 1 8 15 31; do
  echo "== [$rep] pdl=$m $(timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 3 --pdl $m 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["topk"]["value"], d["roofline"]["stage_us_per_layer_avg"])')"
done
done
