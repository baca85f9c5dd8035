export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 1200 python -m pytest tests -m gpu -x -q -k "matvec or addmul or test_cholesky_parity and not C3-24 and not C2-256 or lr_parity or dd_tree and C2-64" --durations=5 ) > gpurun_out/r02d_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02d_pytest.log
python tools/mv_parts.py 512 > gpurun_out/r02d_mv_parts.jsonl 2>&1
python tools/diag_updlog.py C2 256 dd > gpurun_out/r02d_updlog.log 2>&1
python tools/diag_blockwise.py > gpurun_out/r02d_diag_blockwise.log 2>&1
