# per-config layer benchmarks (BASELINE configs[1..3]) + the C4 headline, one JSON line each
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for wl in c1 c2 c3; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline --steps 50 --warmup 5 2>/dev/null | tail -1 >> gpurun_out/bench_configs.jsonl
done
timeout 600 python bench.py --workload c2 --beta 0 --no-cpu-baseline --steps 50 --warmup 5 2>/dev/null | tail -1 >> gpurun_out/bench_configs.jsonl
timeout 600 python bench.py --workload c4 --sim clustered --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/bench_configs.jsonl
