export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python tools/diag_blockwise.py > gpurun_out/r02c_diag_blockwise.log 2>&1
( time timeout 2400 python -m pytest tests -m gpu -q -k "blockwise or dd_tree" --durations=10 ) > gpurun_out/r02c_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02c_pytest.log
