# ncu --set full with source for the latency-bound kernels of a C4 layer (one launch each)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in reroute_align route_tc combine permute; do
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/prof_$k python scripts/profile_step.py --layers 1 > gpurun_out/prof_$k.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
