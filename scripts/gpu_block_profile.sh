timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv python scripts/prof_step.py --config cfg2 --batch 8 --steps 3 --block-size 128 > gpurun_out/blk_launches.csv 2>/dev/null
timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:"step_mma_kernel" -c 1 -o /tmp/blk_single python scripts/prof_step.py --config cfg2 --batch 8 --steps 1 --block-size 128 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/blk_single.ncu-rep --json gpurun_out/ncu_blk_single.json > gpurun_out/ncu_blk_single.txt 2>&1
cat gpurun_out/ncu_blk_single.txt | head -16
