for cfgb in "cfg2 1" "cfg2 4"; do
  echo "default"; python scripts/reuse_sweep.py $cfgb
  for wm in "1 8" "2 8" "2 4" "3 8" "4 8" "2 16" "6 8"; do
    set -- $wm
    echo "waves=$1 min_tiles=$2"; HYLRA_REUSE_WAVES=$1 HYLRA_REUSE_MIN_TILES=$2 python scripts/reuse_sweep.py $cfgb
  done
done
