# A/B of library builds (HYLRA_LIB) on the schedule matrix points given as "config:batch"
# usage: bash scripts/ab_libs.sh "cfg2:16 cfg2:1 cfg3:1" build/libA.so build/libB.so ...
# a point may carry extra ab_schedules.py flags after a comma: "cfg2:32,--context=131072,--layers=8"
pts=$1; shift
for pt in $pts; do
  extra=""
  if [[ "$pt" == *,* ]]; then extra=$(echo "${pt#*,}" | tr ',' ' '); pt=${pt%%,*}; fi
  c=${pt%%:*}; b=${pt##*:}
  for lib in "$@"; do
    echo "== $lib $c B=$b"
    HYLRA_LIB=$PWD/$lib timeout 300 python scripts/ab_schedules.py --config $c --batch $b --reps 3 --steps 15 $extra | tail -1
  done
done
