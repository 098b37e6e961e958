for c in 0 3 4 5 6 8; do echo "CPREFETCH=$c"; HYLRA_REUSE_CPREFETCH=$c SWEEP_B=1,8 python scripts/split_sweep.py --worker; done
