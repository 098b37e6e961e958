# Source-line stall attribution of the fused selects inside the single-launch kernel (cfg2 B=1)
timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:"step_mma_kernel" -c 1 -o /tmp/single_b1 python scripts/prof_step.py --config cfg2 --batch 1 --steps 1 --schedule single > /dev/null 2>&1
python scripts/ncu_lines.py /tmp/single_b1.ncu-rep step 400 | grep -E "samples|select.cuh" | head -45
