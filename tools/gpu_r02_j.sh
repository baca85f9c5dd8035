export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -q -k "bem or dd_tree or blockwise" --durations=10 ) > gpurun_out/r02j_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02j_pytest.log
python tools/time_configs.py table1dd 7 8 9 10 > gpurun_out/r02j_table1_dd.jsonl 2>&1
python tools/time_configs.py c2dd 9 > gpurun_out/r02j_c2_dd.jsonl 2>&1
python tools/time_configs.py bem 11 13 15 > gpurun_out/r02j_bem.jsonl 2>&1
python tools/time_configs.py table1 10 > gpurun_out/r02j_table1_l10.jsonl 2>&1
timeout 2400 python tools/time_configs.py c4 1024 1e-2 1e-4 1e-6 > gpurun_out/r02j_c4.jsonl 2>&1
