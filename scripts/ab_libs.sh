# A/B of library builds (HYLRA_LIB) on the schedule matrix points given as "config:batch"
# usage: bash scripts/ab_libs.sh "cfg2:16 cfg2:1 cfg3:1" build/libA.so build/libB.so ...
pts=$1; shift
for pt in $pts; do
  c=${pt%%:*}; b=${pt##*:}
  for lib in "$@"; do
    echo "== $lib $c B=$b"
    HYLRA_LIB=$PWD/$lib timeout 300 python scripts/ab_schedules.py --config $c --batch $b --reps 3 --steps 15 | tail -1
  done
done
