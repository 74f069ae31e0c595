DG_K5=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_kron5<\(int\)6" -s 2 -c 1 -o /tmp/prof_k5 \
  python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/ncu_k5.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_k5.ncu-rep --page raw --csv > gpurun_out/k5_raw.csv 2>&1
ncu -i /tmp/prof_k5.ncu-rep --page source --csv --print-source sass > gpurun_out/k5_src.csv 2>&1
