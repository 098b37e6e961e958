# Round profile bundle (one GPU): full bench line, reference arm, ncu launch list of the
# bench command, ncu --set full captures of the headline step (single launch), of the
# fusedsel schedule's FULL / SELECT / REUSE kernels at cfg2 B=8, of the B=1 fused3 step
# (FULL, shared-memory-resident select, REUSE) and of the layer-sequential schedule's first
# layers at B=1 (one-layer FULL, its select, one-layer REUSE). Reports are summarised ON the
# box (gpurun brings back <= 64 MiB); only the headline capture travels back as .ncu-rep.
#   bash scripts/gpu_profile.sh [--captures-only] [round tag, default r02]
set -x
TAG=${2:-r02}
mkdir -p gpurun_out
if [ "$1" != "--captures-only" ]; then
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu \
  > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
fi
cap() {  # name, kernel regex, count, prof_step args...
  local name=$1 kre=$2 cnt=$3; shift 3
  timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"$kre" -c $cnt \
    -o /tmp/$name python scripts/prof_step.py "$@" > gpurun_out/ncu_$name.log 2>&1
  echo "ncu $name rc=$?"
  python scripts/ncu_summary.py /tmp/$name.ncu-rep --json gpurun_out/${TAG}_ncu_$name.json > gpurun_out/${TAG}_ncu_$name.txt 2>&1
  python scripts/ncu_lines.py /tmp/$name.ncu-rep "$kre" 40 > gpurun_out/${TAG}_ncu_${name}_lines.txt 2>&1
}
cap single_cfg2_b8 "step_mma_kernel" 1 --config cfg2 --batch 8 --steps 1 --schedule single
cp /tmp/single_cfg2_b8.ncu-rep gpurun_out/
cap fusedsel_cfg2_b8 "attn_mma_kernel|topk_select" 3 --config cfg2 --batch 8 --steps 1 --schedule fusedsel
cap fused3_cfg2_b1 "attn_mma_kernel|rowsel|topk_select" 3 --config cfg2 --batch 1 --steps 1 --schedule fused3
cap seq_cfg2_b1 "attn_mma_kernel|rowsel" 4 --config cfg2 --batch 1 --steps 1 --schedule sequential
cap dual_cfg2_b1 "attn_mma_kernel|rowsel" 5 --config cfg2 --batch 1 --steps 1 --schedule dual
ls -la gpurun_out
