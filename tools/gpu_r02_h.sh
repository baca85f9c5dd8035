export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python tools/diag_updlog.py C2 256 dd > gpurun_out/r02h_updlog_c2.log 2>&1
