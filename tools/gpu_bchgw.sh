# k_bchgw (warp-private pipelined basis change): parity in a subprocess per configuration, then
# same-box A/B of the standalone basis change on the C4 meshes (GB/s at 16 B/DoF).
set -u
mkdir -p gpurun_out/bw
for mode in 0 1 2 3; do
  DG_BCHG=5 DG_BCHGW_MODE=$mode DG_BCHGW_GRID=2 timeout 600 python tests/_bchg_check.py > gpurun_out/bw/check_m${mode}_g2.log 2>&1; echo "check mode=$mode grid=2 rc=$?"
done
DG_BCHG=5 timeout 600 python tests/_bchg_check.py > gpurun_out/bw/check_full.log 2>&1; echo "check full grid rc=$?"
tail -3 gpurun_out/bw/check_*.log
for rep in 1 2; do
  for cfg in "DG_BCHG=1" "DG_BCHG=4" "DG_BCHG=5 DG_BCHGW_MODE=0" "DG_BCHG=5 DG_BCHGW_MODE=1" "DG_BCHG=5 DG_BCHGW_MODE=2" "DG_BCHG=5 DG_BCHGW_MODE=3" "DG_BCHG=5 DG_BCHGW_BPS=2" "DG_BCHG=5 DG_BCHGW_BPS=3"; do
    echo -n "$cfg: " >> gpurun_out/bw/ab.log
    env $cfg python tools/bchg_ab.py >> gpurun_out/bw/ab.log 2>&1
  done
done
cat gpurun_out/bw/ab.log
