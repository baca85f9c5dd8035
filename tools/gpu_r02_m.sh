export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 1200 python -m pytest tests -m gpu -q -k "matvec or lr_parity or addmul" ) > gpurun_out/r02m_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02m_pytest.log
python tools/time_matvec.py 512 factor > gpurun_out/r02m_matvec.json 2>&1
python tools/time_configs.py bem 11 13 15 16 > gpurun_out/r02m_bem.jsonl 2>&1
