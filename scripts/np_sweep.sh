# REUSE producer-warp count: swap the built library variants (libhylra_np{1,4}.so built with
# -DHYLRA_GATHER_PRODUCERS) against the default (2) and time the REUSE launch
cp paper_2602_00777_b200/libhylra.so /tmp/libhylra_np2.so
for np in ${NP_ORDER:-2 1 4 2 1}; do
  cp /tmp/libhylra_np$np.so paper_2602_00777_b200/libhylra.so 2>/dev/null || cp paper_2602_00777_b200/libhylra_np$np.so paper_2602_00777_b200/libhylra.so
  echo "producers=$np"; SWEEP_B=1,8 python scripts/split_sweep.py --worker
done
cp /tmp/libhylra_np2.so paper_2602_00777_b200/libhylra.so
