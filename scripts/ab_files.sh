# same-box A/B of whole-file variants: bash scripts/ab_files.sh <target.cu> <variant.cu>... (kernel_times per variant)
cd $GRAFT_REPO_ROOT
tgt=$1; shift
cp $tgt /tmp/ab_orig.cu
for rep in 1 2; do
for f in "$@"; do
  cp $f $tgt
  python -c "from paper_2602_07616_b200 import build; build.build(force=True)" > /dev/null
  echo "[$rep] $f: $(timeout 200 python scripts/kernel_times.py --layers 48 2>&1 | grep -E "${KPAT:-wall span|align_kernel |permute_kernel |gap before sere::(reroute|permute)}" | tr -s ' ' | cut -c1-70 | tr '\n' '|')"
done
done
cp /tmp/ab_orig.cu $tgt
python -c "from paper_2602_07616_b200 import build; build.build(force=True)" > /dev/null
