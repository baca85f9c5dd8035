export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
( time timeout 1200 python -m pytest tests -m gpu -x -q -k "matvec or addmul or test_cholesky_parity and C2-64 or lr_parity or dd_tree and C2-64" --durations=5 ) > gpurun_out/r02e_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02e_pytest.log
python tools/mv_parts.py 512 > gpurun_out/r02e_mv_parts.jsonl 2>&1
for g in 1 3 4; do H2_MV_NEARGRID=$g python tools/time_matvec.py 512 factor >> gpurun_out/r02e_neargrid.jsonl 2>&1; done
python tools/diag_updlog.py C3 12 dd > gpurun_out/r02e_updlog_c3.log 2>&1
python tools/diag_updlog.py C2 256 dd > gpurun_out/r02e_updlog_c2.log 2>&1
