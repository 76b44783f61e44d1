export PYTHONDONTWRITEBYTECODE=1
timeout 900 python tools/full_schedule.py config2 2 none > gpurun_out/full_config2.log 2>&1; echo rc=$? >> gpurun_out/full_config2.log
timeout 600 python tools/full_schedule.py config1 3 none > gpurun_out/full_config1.log 2>&1; echo rc=$? >> gpurun_out/full_config1.log
