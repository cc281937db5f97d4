# per-config bench lines (BASELINE configs[1..3] + C4 variants), one full JSON line each, CPU baseline skipped
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
OUT=gpurun_out/r02_bench_configs.jsonl; rm -f $OUT
run() { timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 "$@" 2>/dev/null | tail -1 >> $OUT; }
for sim in uniform clustered; do
  for T in 64 128 256; do run --workload c1 --T $T --sim $sim; done
  run --workload c3 --sim $sim
  for S in 1 2; do for rho in 0 0.3 0.5 0.7 0.9 1.0; do run --workload c2 --retain $S --threshold $rho --sim $sim; done; done
done
run --workload c2 --beta 0
run --workload c4 --sim clustered
run --workload c4 --retain 2
wc -l $OUT
