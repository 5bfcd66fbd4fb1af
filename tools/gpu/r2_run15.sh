timeout 900 python -m pytest tests/test_gpu_strips.py tests/test_gpu_paper_heat.py -x -q -p no:cacheprovider > gpurun_out/r2_t15.log 2>&1; echo rc=$? >> gpurun_out/r2_t15.log
timeout 600 python bench.py --config C5 --steps 2 --c5-n 512 > gpurun_out/r2_c5s.json 2> gpurun_out/r2_c5s.err
WRMG_MAC_K2=16 timeout 600 python bench.py --config C5 --steps 2 --c5-n 512 > gpurun_out/r2_c5s16.json 2> gpurun_out/r2_c5s16.err
