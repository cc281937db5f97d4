cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/kernel_times.py --layers 48 --mode sere > gpurun_out/kt_sere.log 2>&1
timeout 300 python scripts/kernel_times.py --layers 48 --mode topk > gpurun_out/kt_topk.log 2>&1
timeout 300 python scripts/kernel_times.py --layers 48 --mode sere --T 128 > gpurun_out/kt_sere128.log 2>&1
timeout 120 python scripts/debug_align.py > gpurun_out/align.log 2>&1
timeout 120 python scripts/debug_align.py --T 128 >> gpurun_out/align.log 2>&1
cat gpurun_out/kt_*.log gpurun_out/align.log
