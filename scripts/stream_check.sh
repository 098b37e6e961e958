# persistent (stream) vs split-K grid attention kernels: tests + launch times
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for st in 1 0; do echo "HYLRA_STREAM=$st"; HYLRA_STREAM=$st python scripts/split_sweep.py --worker; done
for st in 1 0; do echo "HYLRA_STREAM=$st cfg3"; HYLRA_STREAM=$st SWEEP_N=131072 SWEEP_K=4096 SWEEP_B=4 python scripts/split_sweep.py --worker; done
