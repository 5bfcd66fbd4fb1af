timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "transfers or vcycle" > gpurun_out/i_test.log 2>&1; echo rc=$? >> gpurun_out/i_test.log
python bench.py --no-cpu-baseline > gpurun_out/i_c2.json 2> gpurun_out/i_c2.err
