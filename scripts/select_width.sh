for nt in 128 1024; do for N in 32768 131072; do echo "== NT=$nt"; HYLRA_SELECT_THREADS=$nt python scripts/select_diag.py cfg2 $N $((N/16)) 1 32 2>&1 | head -9; done; done
