# ncu evidence for round 2 (run under gpurun from the repo root; one GPU; each command has run
# plain first)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
# launch list of the bench command (per-launch duration, cold/serialised)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --warmup 3 --steps 1 --cpu-budget 2 > gpurun_out/ncu_launches_bench.log 2>&1
# full capture of the matvec kernels of the C2 factor L (two products after warm-up: the A and A^T
# products launch 106 nearfield kernels first, then the packing kernel and 3 warm-up products of L)
ncu --set full --clock-control none --import-source on -k "regex:k_m(atvec|v_)" -s 125 -c 12 -o gpurun_out/prof_matvec_L \
    python tools/time_matvec.py 512 factor > gpurun_out/ncu_mv_L.log 2>&1
# full capture of one long executor launch inside the C2 factorization (traffic)
ncu --set full --clock-control none --import-source on -k regex:k_exec_cluster -s 10 -c 1 -o gpurun_out/prof_exec \
    python tools/time_factor.py 512 > gpurun_out/ncu_exec.log 2>&1
