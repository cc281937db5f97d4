# one GPU pass: -m gpu tests (parity log), smoke, default bench line
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
rm -f gpurun_out/parity.txt
SERE_PARITY_LOG=gpurun_out/parity.txt timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS} 2>&1 | tail -40 > gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
[ -n "$NO_BENCH" ] || timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
for f in gpurun_out/gpu_tests.log gpurun_out/smoke.log gpurun_out/bench.err; do echo "== $f"; tail -n 15 $f; done
cat gpurun_out/bench.json
