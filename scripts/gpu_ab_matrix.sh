# schedule A/B over batch sizes and configs (graph replays, interleaved repetitions)
for b in 1 2 4 8 16; do timeout 300 python scripts/ab_schedules.py --batch $b --reps 4 --steps 30; done
for b in 1 2 4; do timeout 300 python scripts/ab_schedules.py --config cfg3 --batch $b --reps 3 --steps 10; done
for b in 4 8 16; do timeout 300 python scripts/ab_schedules.py --config cfg4 --batch $b --reps 3 --steps 10; done
