# same-box A/B of compile-time variants on the C4 bench line: bash scripts/ab_build.sh "-DX=1" "-DX=2" ...
# (a variant of "base" = no extra flags); BENCH_ARGS are passed to bench.py
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
i=0
for f in "$@"; do
  i=$((i+1))
  [ "$f" = "base" ] && f=""
  SERE_NVCC_FLAGS="$f" python -c "from paper_2602_07616_b200 import build; build.build(force=True)" > /dev/null
  timeout 300 python bench.py --no-cpu-baseline --steps 20 ${BENCH_ARGS} > gpurun_out/ab_b_$i.json 2>/dev/null
  python - "$i" "$rep" "$f" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ab_b_{sys.argv[1]}.json").read().strip().splitlines()[-1])
st = d["roofline"]["stage_us_per_layer_avg"]
print(f"[{sys.argv[2]}] {sys.argv[3] or 'base':<28}: sere {d['value']:.0f}  topk {d['topk']['value']:.0f}  e2e {d['e2e']['value']:.0f}  "
      f"ratio {d['sere']['speedup_vs_topk']:.3f}  ffn_kernel_frac {d['roofline']['frac']:.3f}  stages " +
      " ".join(f"{k}={v:.1f}" for k, v in st.items()))
PY
done
done
python -c "from paper_2602_07616_b200 import build; build.build(force=True)" > /dev/null
