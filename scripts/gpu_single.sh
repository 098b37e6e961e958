set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "single_launch or fused_select" > gpurun_out/t_single.log 2>&1; echo "rc=$?" >> gpurun_out/t_single.log
tail -5 gpurun_out/t_single.log
for b in 1 4 8; do timeout 300 python scripts/ab_schedules.py --batch $b --reps 5 --steps 50; done > gpurun_out/ab.log 2>&1
timeout 300 python scripts/ab_schedules.py --config cfg4 --batch 16 --reps 3 --steps 20 >> gpurun_out/ab.log 2>&1
timeout 300 python scripts/ab_schedules.py --config cfg3 --batch 4 --reps 3 --steps 20 >> gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
