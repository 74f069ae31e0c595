set -u
for n in 5 7; do
  p=$((n-1))
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:k_kron4<\(int\)$n, \(int\)2, \(int\)1" -s 2 -c 1 -o /tmp/prof_cheby_n$n \
    python bench.py --steps 1 --warmup 0 --quick --degrees $p > gpurun_out/ncu_cheby_n$n.log 2>&1; echo "ncu $n rc=$?"
  ncu -i /tmp/prof_cheby_n$n.ncu-rep --page raw --csv > gpurun_out/cheby_n${n}_raw.csv 2>&1
  ncu -i /tmp/prof_cheby_n$n.ncu-rep --page source --csv --print-source sass > gpurun_out/cheby_n${n}_src.csv 2>&1
done
