for n in 8 16 32 64; do for cp in 0 1; do echo "CP=$cp $(WRMG_SWEEP_CP=$cp timeout 120 python tools/time_sweep.py $n 2>&1 | tail -1)" >> gpurun_out/sweep_cp.txt; done; done
