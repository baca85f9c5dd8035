export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 3400 python -m pytest tests -m gpu -x -q ) > gpurun_out/r02z_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02z_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02z_smoke.log 2>&1
( time python bench.py ) > gpurun_out/r02z_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/r02z_bench.log
