timeout 300 python tools/time_sweep_kernel.py 128 64 32 16 8 2>&1 | tail -5 > gpurun_out/v2_time.txt
cat gpurun_out/v2_time.txt
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/v2_tests.txt
cat gpurun_out/v2_tests.txt
python bench.py > gpurun_out/v2_c2.json 2> gpurun_out/v2_c2.err
python tools/bench_view.py gpurun_out/v2_c2.json 2>/dev/null | head -30 || tail -c 1500 gpurun_out/v2_c2.json
