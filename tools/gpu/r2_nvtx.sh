python tools/time_sweep_kernel.py 16 > /dev/null 2>&1
ncu --nvtx --nvtx-include "wrmg_smooth/sweep_L2/" --metrics gpu__time_duration.sum -c 2 python tools/time_sweep_kernel.py 16 > gpurun_out/nvtx_ncu.txt 2>&1
ncu --nvtx --nvtx-include "wrmg_smooth/" --metrics gpu__time_duration.sum -c 3 python tools/time_sweep_kernel.py 16 > gpurun_out/nvtx_ncu2.txt 2>&1
cat gpurun_out/nvtx_ncu.txt | grep -v "^n=" | head -40
grep -E "k_|NVTX" gpurun_out/nvtx_ncu2.txt | head
