# gather probe GB/s vs CTAs per SM (each CTA: 8 warps x 32 lanes x 16 x 16 B = 64 KB in flight)
for sm in 0 8000 20000 40000 60000 100000; do echo "smem=$sm"; HYLRA_PROBE_SMEM=$sm python scripts/gather_probe.py --batch 8 | grep "splits/pair=8"; done
