for n in 64 32; do for T in 2 1 3 4 6; do echo "CTAS=$T $(WRMG_MAC_CTAS=$T timeout 120 python tools/time_residual.py $n 2>&1 | tail -1)" >> gpurun_out/res_l4.txt; done; done
