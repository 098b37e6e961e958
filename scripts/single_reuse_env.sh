# single-launch vs fused3 at small batch under REUSE split overrides (HYLRA_REUSE_WAVES /
# HYLRA_REUSE_MIN_TILES replace the REUSE rule of choose_splits for every launch)
echo default; python scripts/schedules.py cfg2:1,2
for wm in "2 8" "3 8" "4 4" "2 16" "6 4"; do
  set -- $wm
  echo "reuse waves=$1 min_tiles=$2"; HYLRA_REUSE_WAVES=$1 HYLRA_REUSE_MIN_TILES=$2 python scripts/schedules.py cfg2:1,2
done
