WRMG_GUARD=1 timeout 900 python tools/guard_check.py > gpurun_out/r2_guard.log 2>&1; echo rc=$? >> gpurun_out/r2_guard.log
bash tools/final_profiles.sh
