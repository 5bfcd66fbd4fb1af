# Round-end measurement (run from the repo root on the GPU box): C2/C3/C4/C5 bench lines,
# the C2 timed-region launch list and ncu --set full summaries of the top kernels.
python bench.py > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err
python bench.py --config C3 --steps 3 > gpurun_out/f_c3.json 2> gpurun_out/f_c3.err
python bench.py --config C4 --steps 1 --warmup 3 > gpurun_out/f_c4.json 2> gpurun_out/f_c4.err
python bench.py --config C5 --steps 2 > gpurun_out/f_c5.json 2> gpurun_out/f_c5.err
timeout 1500 python bench.py --config C4 --c4-n 128 --steps 1 --warmup 3 > gpurun_out/f_c4full.json 2> gpurun_out/f_c4full.err
S=$(python -c "import json;d=json.loads(open('gpurun_out/f_c2.json').read().strip().splitlines()[-1]);print(d['launches_before_timed'], d['gpu_launches'])")
set -- $S
python bench.py --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s $1 -c $2 --csv --log-file gpurun_out/f_c2_launches.csv python bench.py --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/f_c2_launches.csv > gpurun_out/f_c2_launches.txt
# finest-level launches of the C2 hot kernels (short driver: residual x3, sweeps, FGMRES)
python tools/prof_c2_kernels.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_residual_mac|k_sweep_sym|k_sweep_kron_mma|k_krylov" -c 8 -o /tmp/f_c2_full -f python tools/prof_c2_kernels.py > /dev/null 2>&1
python tools/ncu_summary.py report /tmp/f_c2_full.ncu-rep > gpurun_out/f_c2_ncu.txt
# C3: the NS block inversion (short driver), the finest-level NS sweep and residual of the bench
python tools/prof_ns_factor.py > /dev/null 2>&1 && \
ncu --set full --clock-control none -k regex:"k_ns_factor" -c 1 -o /tmp/f_c3_factor -f python tools/prof_ns_factor.py > /dev/null 2>&1
python tools/prof_ns_factor_c4.py > /dev/null 2>&1 && \
ncu --set full --clock-control none -k regex:"k_ns_factor" -c 1 -o /tmp/f_c4_factor -f python tools/prof_ns_factor_c4.py > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"k_ns_sweep" -c 1 -o /tmp/f_c3_sweep -f python bench.py --config C3 --steps 1 --warmup 0 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"k_ns_residual" -c 1 -o /tmp/f_c3_resid -f python bench.py --config C3 --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_summary.py report /tmp/f_c3_factor.ncu-rep /tmp/f_c3_sweep.ncu-rep /tmp/f_c3_resid.ncu-rep > gpurun_out/f_c3_ncu.txt
python tools/ncu_summary.py report /tmp/f_c4_factor.ncu-rep > gpurun_out/f_c4_ncu.txt
ls gpurun_out/f_*
cp /tmp/f_c2_full.ncu-rep gpurun_out/ 2>/dev/null; ls -la gpurun_out/
