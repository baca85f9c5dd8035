export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 3000 python -m pytest tests -m gpu -q --durations=15 ) > gpurun_out/r02i_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02i_pytest.log
( time python bench.py --steps 2 --warmup 3 ) > gpurun_out/r02i_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/r02i_bench.log
python tools/time_matvec.py 512 factor > gpurun_out/r02i_matvec.json 2>&1
bash tools/prof_r02.sh
python tools/time_configs.py c1 10000 > gpurun_out/r02i_c1.jsonl 2>&1
