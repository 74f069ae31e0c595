set -x
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo "bench rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:k_kron4 --csv python bench.py --steps 1 --warmup 0 --quick > gpurun_out/traffic_ncu.csv 2> gpurun_out/traffic_ncu.err
echo "ncu traffic rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --quick > gpurun_out/launches.log 2>&1
echo "ncu launches rc=$?"
