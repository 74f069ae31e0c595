# k_bchgp (plane mode of k_bchgw, DG_BCHGW_MODE 4 / 6): parity, then same-box A/B against the defaults
set -u
mkdir -p gpurun_out/bp
for mode in 4 6; do
  DG_BCHG=5 DG_BCHGW_MODE=$mode DG_BCHGW_GRID=2 timeout 600 python tests/_bchg_check.py > gpurun_out/bp/check_m${mode}_g2.log 2>&1; echo "check mode=$mode grid=2 rc=$?"
  DG_BCHG=5 DG_BCHGW_MODE=$mode timeout 600 python tests/_bchg_check.py > gpurun_out/bp/check_m${mode}.log 2>&1; echo "check mode=$mode rc=$?"
done
tail -n 3 gpurun_out/bp/check_*.log
for rep in 1 2; do
  for cfg in "DG_BCHG=0" "DG_BCHG=5 DG_BCHGW_MODE=4" "DG_BCHG=5 DG_BCHGW_MODE=6" "DG_BCHG=5 DG_BCHGW_MODE=6 DG_BCHGW_BPS=3" "DG_BCHG=5 DG_BCHGW_MODE=6 DG_BCHGW_BPS=2"; do
    echo -n "$cfg: " >> gpurun_out/bp/ab.log
    env $cfg python tools/bchg_ab.py >> gpurun_out/bp/ab.log 2>&1
  done
done
cat gpurun_out/bp/ab.log
