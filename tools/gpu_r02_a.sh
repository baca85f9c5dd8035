# round-2 GPU evidence, one gpurun call: parity tests, bench, then ncu (each plain first)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/r02_gpu.txt
( time timeout 3000 python -m pytest tests -m gpu -x -q --durations=15 ) > gpurun_out/r02_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02_pytest.log
( time python bench.py --steps 2 --warmup 3 ) > gpurun_out/r02_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/r02_bench.log
python tools/time_matvec.py 512 factor > gpurun_out/r02_matvec.json 2>&1
bash tools/prof_r02.sh
ls -la gpurun_out
