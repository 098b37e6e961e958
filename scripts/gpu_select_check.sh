mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
python scripts/select_diag.py cfg2 32768 2048 1 32 2>&1 | head -9
python scripts/select_diag.py cfg2 32768 2048 4 32 2>&1 | head -9
for nt in 256 512 1024; do echo "NT=$nt"; HYLRA_SELECT_THREADS=$nt python scripts/select_diag.py cfg2 32768 2048 1 32 2>&1 | sed -n 5,8p; done
SWEEP_N=8192 SWEEP_K=512 SWEEP_B=1,8 SWEEP_WAVES=2,4,8 SWEEP_TILES=4,8,16,32 python scripts/split_sweep.py > gpurun_out/split_8k.txt 2>&1; cat gpurun_out/split_8k.txt | cut -c1-600
