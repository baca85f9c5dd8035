export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 1200 python -m pytest tests -m gpu -q -k "matvec or addmul or test_cholesky_parity and C2-64 or dd_tree and C2-64 or lr_parity or bem" ) > gpurun_out/r02o_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02o_pytest.log
python tools/mv_parts.py 512 > gpurun_out/r02o_mv_parts.jsonl 2>&1
H2_MV_DBG=1 python tools/time_matvec.py 512 factor 2>&1 | grep MV_DBG | tail -2 > gpurun_out/r02o_mvdbg_full.log
python tools/time_matvec.py 1024 factor > gpurun_out/r02o_matvec_1024.json 2>&1
