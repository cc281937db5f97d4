set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --layers 4 > gpurun_out/launches.log 2>&1
ncu --query-metrics 2>/dev/null | grep -i -E "tensor|tcgen|tmem|utc|pipe_tc|_tc_" > gpurun_out/ncu_tc_metrics.txt
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:moe_ffn -c 2 -o gpurun_out/prof_ffn python scripts/profile_step.py --layers 2 > gpurun_out/prof.log 2>&1
for f in gpurun_out/*.log; do echo == $f; tail -n 5 $f; done; cat gpurun_out/bench.json
