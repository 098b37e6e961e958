mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
for B in 1 4 8; do python scripts/select_diag.py cfg2 32768 2048 $B 32 2>&1 | head -9; done
python scripts/select_diag.py cfg3 131072 4096 4 32 2>&1 | head -9
timeout 600 python bench.py --no-extra --no-cpu > gpurun_out/bench_quick.json 2>/dev/null
timeout 600 python bench.py --no-extra --no-cpu --batch 1 > gpurun_out/bench_quick_b1.json 2>/dev/null
python - <<'PY'
import json
for f in ("gpurun_out/bench_quick.json", "gpurun_out/bench_quick_b1.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], d["ms_per_step"], json.dumps(d["kernels"])[:300])
PY
