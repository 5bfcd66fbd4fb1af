timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "transfers or vcycle" > gpurun_out/r2_t24.log 2>&1; echo rc=$? >> gpurun_out/r2_t24.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b24.json 2> gpurun_out/r2_b24.err
