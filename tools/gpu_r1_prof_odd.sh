timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_kron4<\(int\)7, \(int\)2, \(int\)[01]' -s 1 -c 2 -o gpurun_out/prof_k4_p6 python bench.py --steps 1 --warmup 0 --quick --degrees 6 > gpurun_out/ncu_p6.log 2>&1
echo "ncu p6 rc=$?"
