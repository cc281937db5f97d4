# same-box A/B of csrc file sets: bash scripts/ab_dirs.sh <dir with .cu/.cuh files>...   (bench line + CUPTI chain)
cd $GRAFT_REPO_ROOT
mkdir -p /tmp/ab_orig; cp paper_2602_07616_b200/csrc/* /tmp/ab_orig/
for rep in 1 2; do
for d in "$@"; do
  cp /tmp/ab_orig/* paper_2602_07616_b200/csrc/; cp $d/* paper_2602_07616_b200/csrc/
  python -c "from paper_2602_07616_b200 import build; build.build(force=True)" > /dev/null
  timeout 300 python bench.py --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$rep] $d bench', d['value'], d['topk']['value'], d['roofline']['frac'], d['e2e']['value'])"
  echo "    $(timeout 200 python scripts/kernel_times.py --layers 48 2>&1 | grep -E "${KPAT:-wall span|align_kernel |ffn_kernel |gap before sere::(reroute|moe)}" | tr -s ' ' | cut -c1-60 | tr '\n' '|')"
done
done
cp /tmp/ab_orig/* paper_2602_07616_b200/csrc/
python -c "from paper_2602_07616_b200 import build; build.build(force=True)" > /dev/null
