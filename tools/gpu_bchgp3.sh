# vectorised plane mode: parity (modes 4, 6), then A/B of base (C4 = 8, C6 = 5) and bpC (C4 = 16, C6 = 10)
set -u
mkdir -p gpurun_out/bp3
for mode in 4 6; do
  DG_BCHG=5 DG_BCHGW_MODE=$mode DG_BCHGW_GRID=2 timeout 600 python tests/_bchg_check.py > gpurun_out/bp3/check_m${mode}_g2.log 2>&1; echo "check mode=$mode grid=2 rc=$? $(tail -n 1 gpurun_out/bp3/check_m${mode}_g2.log)"
  DG_BCHG=5 DG_BCHGW_MODE=$mode timeout 600 python tests/_bchg_check.py > gpurun_out/bp3/check_m${mode}.log 2>&1; echo "check mode=$mode rc=$? $(tail -n 1 gpurun_out/bp3/check_m${mode}.log)"
done
cp paper_1907_08492_b200/libdg_b200.so /tmp/libdg_base.so
for lib in base bpC; do
  if [ $lib = base ]; then cp /tmp/libdg_base.so paper_1907_08492_b200/libdg_b200.so; else cp variants/libdg_$lib.so paper_1907_08492_b200/libdg_b200.so; fi
  for mode in 4 6; do
    for bps in 1 2 4; do
      echo -n "$lib mode=$mode bps=$bps: " >> gpurun_out/bp3/ab.log
      DG_BCHG=5 DG_BCHGW_MODE=$mode DG_BCHGW_BPS=$bps python tools/bchg_ab.py >> gpurun_out/bp3/ab.log 2>&1
    done
  done
done
cp /tmp/libdg_base.so paper_1907_08492_b200/libdg_b200.so
cat gpurun_out/bp3/ab.log
