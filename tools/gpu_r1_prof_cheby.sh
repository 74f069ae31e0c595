timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_kron4<\(int\)6, \(int\)2, \(int\)1' -s 1 -c 1 -o gpurun_out/prof_k4f_cheby python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/ncu_k4f.log 2>&1
echo "ncu rc=$?"
