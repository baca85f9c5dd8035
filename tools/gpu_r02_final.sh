export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 3400 python -m pytest tests -m gpu -q --durations=15 ) > gpurun_out/r02f_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02f_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1
( time python bench.py --steps 3 --warmup 3 ) > gpurun_out/r02f_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/r02f_bench.log
python tools/time_matvec.py 512 factor > gpurun_out/r02f_matvec.json 2>&1
bash tools/prof_r02.sh
