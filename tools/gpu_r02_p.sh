export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for v in "" "H2_MV_PRIO=equal" "H2_MV_ORDER=near_first" "H2_MV_PRIO=equal H2_MV_ORDER=near_first"; do
  echo "variant: [$v]" >> gpurun_out/r02p_order.log
  env $v python tools/time_matvec.py 512 factor >> gpurun_out/r02p_order.log 2>&1
done
H2_MV_DBG=1 python tools/time_matvec.py 512 factor 2>&1 | grep MV_DBG | tail -2 > gpurun_out/r02p_mvdbg_full.log
