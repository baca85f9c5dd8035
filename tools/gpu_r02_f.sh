export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 1200 python -m pytest tests -m gpu -x -q -k "matvec or addmul or test_cholesky_parity and C2-64 or dd_tree and C2-64" ) > gpurun_out/r02f_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02f_pytest.log
python tools/mv_parts.py 512 > gpurun_out/r02f_mv_parts.jsonl 2>&1
