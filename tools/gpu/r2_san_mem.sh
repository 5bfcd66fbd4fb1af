python tools/sanitize_driver.py > gpurun_out/r2_san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_driver.py > gpurun_out/r2_san_memcheck.log 2>&1
echo "exit $?" >> gpurun_out/r2_san_memcheck.log
