for R in 4 3 5; do for T in 2 1 3 4; do echo "R=$R CTAS=$T $(WRMG_MAC3_R=$R WRMG_MAC_CTAS=$T timeout 120 python tools/time_residual.py 2>&1 | tail -1)" >> gpurun_out/res_sweep.txt; done; done
