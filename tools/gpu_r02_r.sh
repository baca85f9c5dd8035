export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python tools/time_configs.py c3 24 > gpurun_out/r02r_c3.jsonl 2>&1
timeout 1200 python tools/time_configs.py c3 32 >> gpurun_out/r02r_c3.jsonl 2>&1
