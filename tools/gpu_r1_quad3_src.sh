set -u
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_quad3<\(int\)6, \(int\)2, \(int\)2, \(int\)0" -s 2 -c 1 -o /tmp/prof_q3 \
  python bench.py --steps 1 --warmup 0 --quick --workload c3 > gpurun_out/ncu_q3.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_q3.ncu-rep --page raw --csv > gpurun_out/q3_raw.csv 2>&1
ncu -i /tmp/prof_q3.ncu-rep --page source --csv --print-source sass > gpurun_out/q3_src.csv 2>&1
ncu -i /tmp/prof_q3.ncu-rep --page source --csv --print-source cuda > gpurun_out/q3_cuda.csv 2>&1
