timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:k_kron4<\(int\)6, \(int\)2, \(int\)1' -s 1 -c 1 -o gpurun_out/prof_k4_cheby_p5 python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/ncu_fa.log 2>&1
echo "ncu apply rc=$?"
