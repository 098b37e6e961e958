for b in 1 8; do
  echo default; python scripts/full_layer_sweep.py cfg2 $b
  for wm in "1 4" "2 4" "3 4" "4 2" "2 8" "6 2"; do
    set -- $wm
    echo "waves=$1 min_tiles=$2"; HYLRA_FULL_WAVES=$1 HYLRA_FULL_MIN_TILES=$2 python scripts/full_layer_sweep.py cfg2 $b
  done
done
