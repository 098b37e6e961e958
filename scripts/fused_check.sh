mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for b in 8 1 4; do
  timeout 600 python bench.py --no-extra --no-cpu --batch $b --steps 30 > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
print('B=$b', round(d['ms_per_step'],4), {k: round(v['ms_per_step'],4) for k,v in d['schedules'].items()})" || tail -5 gpurun_out/b.err
done
