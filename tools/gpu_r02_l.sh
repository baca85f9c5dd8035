export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 1200 python -m pytest tests -m gpu -q -k "matvec or addmul or test_cholesky_parity and C2-64 or dd_tree and C2-64 or lr_parity or bem" ) > gpurun_out/r02l_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02l_pytest.log
python tools/time_matvec.py 512 factor > gpurun_out/r02l_matvec.json 2>&1
python tools/time_configs.py bem 11 13 15 > gpurun_out/r02l_bem.jsonl 2>&1
