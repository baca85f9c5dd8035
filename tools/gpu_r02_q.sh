export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 2400 python tools/time_configs.py bem 17 18 > gpurun_out/r02q_bem_large.jsonl 2>&1
