# plane-mode tuning sweep: libs (base, bpA = larger tiles at n = 2..5, bpB = 2 warps per block) x mode x blocks per SM
set -u
mkdir -p gpurun_out/bp2
cp paper_1907_08492_b200/libdg_b200.so /tmp/libdg_base.so
for lib in base bpA bpB; do
  if [ $lib = base ]; then cp /tmp/libdg_base.so paper_1907_08492_b200/libdg_b200.so; else cp variants/libdg_$lib.so paper_1907_08492_b200/libdg_b200.so; fi
  for mode in 4 6; do
    for bps in 1 2 3 4 6 8; do
      echo -n "$lib mode=$mode bps=$bps: " >> gpurun_out/bp2/ab.log
      DG_BCHG=5 DG_BCHGW_MODE=$mode DG_BCHGW_BPS=$bps python tools/bchg_ab.py >> gpurun_out/bp2/ab.log 2>&1
    done
  done
done
cp /tmp/libdg_base.so paper_1907_08492_b200/libdg_b200.so
cat gpurun_out/bp2/ab.log
