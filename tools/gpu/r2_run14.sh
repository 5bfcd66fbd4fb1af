timeout 900 python bench.py --config C4 --steps 1 --warmup 1 > gpurun_out/r2_c4.json 2> gpurun_out/r2_c4.err; echo rc=$? >> gpurun_out/r2_c4.err
timeout 600 python bench.py --config C3 --steps 3 > gpurun_out/r2_c3.json 2> gpurun_out/r2_c3.err
timeout 900 python bench.py --config C5 --steps 2 > gpurun_out/r2_c5.json 2> gpurun_out/r2_c5.err
