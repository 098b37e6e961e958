# Round profile bundle (one GPU): full bench line, reference arm, ncu launch list of the
# bench command, ncu --set full captures of the FULL / SELECT / REUSE kernels at cfg2 B=8.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu \
  > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"attn_mma_kernel|topk_select" -c 3 -o gpurun_out/step_cfg2_b8 \
  python scripts/prof_step.py --config cfg2 --batch 8 --steps 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none \
  -k regex:"attn_mma_kernel|topk_select" -c 3 -o gpurun_out/step_cfg2_b1 \
  python scripts/prof_step.py --config cfg2 --batch 1 --steps 1 > gpurun_out/ncu_full_b1.log 2>&1; echo "ncu full b1 rc=$?"
ls -la gpurun_out
