timeout 600 python bench.py --config C5 --steps 2 --c5-n 512 > gpurun_out/r2_c5a.json 2>&1
WRMG_MAC_K2_SPLIT=0 timeout 600 python bench.py --config C5 --steps 2 --c5-n 512 > gpurun_out/r2_c5b.json 2>&1
python tools/prof_c2_kernels.py > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:"k_krylov" -c 4 -o /tmp/krylov -f python tools/prof_c2_kernels.py > /dev/null 2>&1; python tools/ncu_summary.py report /tmp/krylov.ncu-rep > gpurun_out/r2_krylov_ncu.txt
