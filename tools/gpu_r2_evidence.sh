# Round-2 evidence on one B200: bench line, reference arm, launch list, DRAM traffic per launch,
# ncu --set full summaries of the dominant kernels (CSV exports; the .ncu-rep files stay on the box).
set -u
mkdir -p gpurun_out/ev /tmp/ev
python bench.py > gpurun_out/ev/bench_c4.json 2> gpurun_out/ev/bench_c4.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/bench_reference.json 2> gpurun_out/ev/bench_reference.err; echo "ref rc=$?"
python bench.py --steps 2 --warmup 1 --quick > gpurun_out/ev/quick_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/ev/launches.csv \
    python bench.py --steps 2 --warmup 1 --quick > gpurun_out/ev/launches.log 2>&1; echo "launches rc=$?"
python bench.py --steps 1 --warmup 0 --quick > gpurun_out/ev/traffic_plain.json 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --kernel-name-base demangled \
    -k regex:k_kron --csv python bench.py --steps 1 --warmup 0 --quick > gpurun_out/ev/traffic_ncu.csv 2> gpurun_out/ev/traffic.err; echo "traffic rc=$?"
bash tools/ncu_capture.sh ev/cheby_p5 k_kron4 2 1 python tools/prof_driver.py 5 cheby 2
bash tools/ncu_capture.sh ev/cheby_p4 k_kron4 2 1 python tools/prof_driver.py 4 cheby 2
bash tools/ncu_capture.sh ev/apply_p4 k_kron4 1 1 python tools/prof_driver.py 4 apply 2
bash tools/ncu_capture.sh ev/apply_p6 k_kron4 1 1 python tools/prof_driver.py 6 apply 2
bash tools/ncu_capture.sh ev/apply_p2 k_kron6 1 1 python tools/prof_driver.py 2 apply 2
ls -la gpurun_out/ev
