timeout 600 python -m pytest tests/test_gpu_host_api.py -x -q -p no:cacheprovider > gpurun_out/r2_t33.log 2>&1; echo rc=$? >> gpurun_out/r2_t33.log
timeout 600 python bench.py --config C5 --steps 2 --c5-n 512 > gpurun_out/r2_c5st.json 2>&1
