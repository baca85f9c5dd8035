export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -x -q -k "blockwise or dd_tree" --durations=10 ) > gpurun_out/r02b_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02b_pytest.log
python tools/mv_parts.py 512 > gpurun_out/r02b_mv_parts.jsonl 2>&1
python tools/time_configs.py table1 7 8 9 > gpurun_out/r02b_table1.jsonl 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_m(atvec|v_)" -s 120 -c 8 -o gpurun_out/prof_matvec_L \
    python tools/time_matvec.py 512 factor > gpurun_out/ncu_mv_L.log 2>&1
