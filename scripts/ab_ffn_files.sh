# same-box A/B of whole-file variants of the FFN kernel: kernel-only replay (scripts/ffn_replay.py) + bench line
# bash scripts/ab_ffn_files.sh <variant.cu>...   (BENCH=1 adds the C4 bench line)
cd $GRAFT_REPO_ROOT
tgt=paper_2602_07616_b200/csrc/grouped_ffn.cu
cp $tgt /tmp/ab_orig.cu
for rep in 1 2; do
for f in "$@"; do
  cp $f $tgt
  python -c "from paper_2602_07616_b200 import build; build.build(force=True)" > /dev/null
  echo "[$rep] $f: $(timeout 200 python scripts/ffn_replay.py sere ${DBG:-0} 2>&1 | grep ffn | cut -c1-60 | tr '\n' '|')"
  if [ -n "$BENCH" ]; then
    timeout 300 python bench.py --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('    bench', d['value'], d['topk']['value'], d['roofline']['frac'], d['e2e']['value'])"
  fi
done
done
cp /tmp/ab_orig.cu $tgt
python -c "from paper_2602_07616_b200 import build; build.build(force=True)" > /dev/null
