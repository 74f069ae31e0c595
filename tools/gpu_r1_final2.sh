timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:k_kron4<\(int\)6, \(int\)2, \(int\)0' -s 2 -c 1 -o gpurun_out/prof_k4_apply_p5 python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/ncu_fa.log 2>&1
echo "ncu apply rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:k_kron4 --csv python bench.py --steps 1 --warmup 0 --quick > gpurun_out/traffic_ncu2.csv 2> gpurun_out/traffic_ncu2.err
echo "ncu traffic rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 2 --warmup 1 --quick > gpurun_out/launches2.log 2>&1
echo "ncu launches rc=$?"
ls -la gpurun_out/*.ncu-rep
