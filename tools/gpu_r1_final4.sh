timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_final4.log 2>&1
echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke4.log 2>&1
echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_c4_final4.json 2> gpurun_out/bench_c4_final4.err
echo "c4 rc=$?"
for w in c2 c3 c5; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload $w > gpurun_out/bench_${w}_final4.json 2> gpurun_out/bench_${w}_final4.err
echo "$w rc=$?"
done
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:k_kron4 --csv python bench.py --steps 1 --warmup 0 --quick > gpurun_out/traffic_ncu4.csv 2> gpurun_out/traffic_ncu4.err
echo "traffic rc=$?"
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:k_kron4<\(int\)6, \(int\)2, \(int\)1' -s 1 -c 1 -o gpurun_out/prof_k4_cheby_p5_final python bench.py --steps 1 --warmup 0 --quick --degrees 5 > gpurun_out/ncu_f4.log 2>&1
echo "ncu rc=$?"
