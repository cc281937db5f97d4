# one GPU pass for a profiles/ refresh: -m gpu tests (parity log), smoke, bench line, CUPTI per-kernel
# chain view, ncu launch list of a 4-layer step, one ncu --set full capture of moe_ffn_kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "from paper_2602_07616_b200 import build; build.build()" > /dev/null
rm -f gpurun_out/parity.txt
SERE_PARITY_LOG=gpurun_out/parity.txt timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python scripts/kernel_times.py --layers 48 > gpurun_out/kt.txt 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --layers 4 > gpurun_out/launches.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:moe_ffn -s 1 -c 2 -o gpurun_out/prof_ffn python scripts/profile_step.py --layers 4 > gpurun_out/prof.log 2>&1
for f in gpurun_out/gpu_tests.log gpurun_out/smoke.log gpurun_out/bench.err gpurun_out/prof.log; do echo "== $f"; tail -n 4 $f; done
tail -16 gpurun_out/kt.txt
cat gpurun_out/bench.json
