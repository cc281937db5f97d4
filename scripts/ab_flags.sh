# same-box A/B of compile-time variants: args = flag sets (commas = spaces); bench lines for C4 and C2
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for f in "$@"; do
  SERE_NVCC_FLAGS="$(echo $f | tr ',' ' ')" python -c "from paper_2602_07616_b200 import build; build.build(force=True)"
  for a in "" "--workload c2"; do
    echo "== [$rep] $f $a: $(timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 $a 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["topk"]["value"], d["roofline"]["frac"], d["topk"]["stages"]["ffn_frac"])')"
  done
done
done
python -c "from paper_2602_07616_b200 import build; build.build(force=True)"
