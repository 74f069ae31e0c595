timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_final5.log 2>&1
echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke5.log 2>&1
echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_c4_final5.json 2> gpurun_out/bench_c4_final5.err
echo "c4 rc=$?"
for w in c2 c3 c5; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload $w > gpurun_out/bench_${w}_final5.json 2> gpurun_out/bench_${w}_final5.err
echo "$w rc=$?"
done
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:k_kron4 --csv python bench.py --steps 1 --warmup 0 --quick > gpurun_out/traffic_ncu5.csv 2> gpurun_out/traffic_ncu5.err
echo "traffic rc=$?"
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:k_kron4<\(int\)6, \(int\)2, \(int\)1' -s 1 -c 1 --import-source on -o /tmp/prof_k4_cheby_p5_final5 python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/ncu_f5.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_k4_cheby_p5_final5.ncu-rep --page raw --csv > gpurun_out/cheby_p5_final5_raw.csv 2>&1
ncu -i /tmp/prof_k4_cheby_p5_final5.ncu-rep --page source --csv --print-source sass > gpurun_out/cheby_p5_final5_src.csv 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --steps 2 --warmup 1 --quick > gpurun_out/launches_final5.csv 2> gpurun_out/launches_final5.err
echo "launches rc=$?"
