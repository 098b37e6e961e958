# quick GPU check: kernel tests + short bench main line (no extras, no CPU leg)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-extra --no-cpu ${BENCH_ARGS} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?" >> gpurun_out/bench_quick.err
tail -5 gpurun_out/pytest_gpu.log; tail -5 gpurun_out/bench_quick.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_quick.json").read().strip().splitlines()[-1])
for k in ("value", "ms_per_step", "kernels", "e2e", "schedules", "clocks"):
    print(k, json.dumps(d.get(k))[:700])
PY
