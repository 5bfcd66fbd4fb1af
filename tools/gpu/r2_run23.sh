python tools/prof_ns_factor.py > /dev/null 2>&1
timeout 600 python bench.py --config C3 --steps 1 > gpurun_out/r2_c3wp4.json 2> gpurun_out/r2_c3wp4.err
