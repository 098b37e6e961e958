# quick GPU check: kernel tests + short bench main line (no extras, no CPU leg)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-extra --no-cpu ${BENCH_ARGS} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?" >> gpurun_out/bench_quick.err
tail -5 gpurun_out/pytest_gpu.log; tail -c 3000 gpurun_out/bench_quick.json; tail -5 gpurun_out/bench_quick.err
