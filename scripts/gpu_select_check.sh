# select changes: exactness tests, per-phase timings at the fused width and the widest, schedules
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash scripts/select_width.sh 2>&1 | grep -E "==|N=|B pass|C\+D|E window|A sample|launch time" 
python scripts/determinism.py --reps 3
for b in 1 4 8; do python scripts/ab_schedules.py --batch $b --reps 4 --steps 40; done
for b in 1 4; do python scripts/ab_schedules.py --config cfg3 --batch $b --reps 3 --steps 10; done
python scripts/ab_schedules.py --config cfg4 --batch 8 --reps 3 --steps 10
