# fp32 basis change A/B (k_bchg vs the k_bchgw.cu kernels) and the n = 9 line-mode blocks-per-SM sweep
set -u
mkdir -p gpurun_out/bm
for cfg in "DG_BCHG=1" "DG_BCHG=5" "DG_BCHG=5 DG_BCHGW_MODE=6" "DG_BCHG=5 DG_BCHGW_MODE=4 DG_BCHGW_BPS=1" "DG_BCHG=5 DG_BCHGW_MODE=0"; do
  echo -n "$cfg: " >> gpurun_out/bm/f32.log; env $cfg python tools/bchg_ab.py --f32 >> gpurun_out/bm/f32.log 2>&1
done
cat gpurun_out/bm/f32.log
for cfg in "DG_BCHGW_MODE=3 DG_BCHGW_BPS=1" "DG_BCHGW_MODE=3 DG_BCHGW_BPS=2" "DG_BCHGW_MODE=3 DG_BCHGW_BPS=3" "DG_BCHGW_MODE=1 DG_BCHGW_BPS=1" "DG_BCHGW_MODE=1 DG_BCHGW_BPS=2"; do
  echo -n "$cfg: " >> gpurun_out/bm/n9.log; env DG_BCHG=5 $cfg python tools/bchg_ab.py >> gpurun_out/bm/n9.log 2>&1
done
cat gpurun_out/bm/n9.log
