# ncu evidence for round 1 (run under gpurun from the repo root; one GPU)
set -e
python bench.py --N 128 --warmup 3 --steps 1 --cpu-N 32 > gpurun_out/plain_N128.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_N128.csv \
    python bench.py --N 128 --warmup 3 --steps 1 --cpu-N 32 > gpurun_out/ncu_launches.log 2>&1
python tools/time_matvec.py 512 factor > gpurun_out/plain_mv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_matvec -s 30 -c 3 -o gpurun_out/prof_matvec \
    python tools/time_matvec.py 512 factor > gpurun_out/ncu_mv.log 2>&1
python tools/time_factor.py 64 > gpurun_out/plain_f64.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_exec_cluster -s 40 -c 1 -o gpurun_out/prof_exec \
    python tools/time_factor.py 64 > gpurun_out/ncu_exec.log 2>&1
