# same-box A/B of sere_set_l2 scratch policies on the C4 bench line (value, top-k, e2e, FFN frac)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "from paper_2602_07616_b200 import build; build.build()" > /dev/null
for rep in 1 2; do
for v in "$@"; do
  timeout 300 python bench.py --no-cpu-baseline --steps 20 --l2 $v ${BENCH_ARGS} > gpurun_out/ab_l2_$v.json 2>/dev/null
  python - "$v" "$rep" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ab_l2_{sys.argv[1]}.json").read().strip().splitlines()[-1])
st = d["roofline"]["stage_us_per_layer_avg"]
print(f"[{sys.argv[2]}] l2={sys.argv[1]:>3}: sere {d['value']:.0f}  topk {d['topk']['value']:.0f}  e2e {d['e2e']['value']:.0f}  "
      f"ratio {d['sere']['speedup_vs_topk']:.3f}  ffn_kernel_frac {d['roofline']['frac']:.3f}  stages " +
      " ".join(f"{k}={v:.1f}" for k, v in st.items()))
PY
done
done
