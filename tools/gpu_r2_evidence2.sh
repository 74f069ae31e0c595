# Round-2 evidence on one B200 after the k_kron3c change: full GPU tests, smoke, bench line,
# reference arm, launch list, DRAM traffic per launch, ncu --set full of k_kron3c and k_kron4.
set -u
mkdir -p gpurun_out/ev2 /tmp/ev2
python -m pytest tests -m gpu -q > gpurun_out/ev2/gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ev2/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev2/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/ev2/bench_c4.json 2> gpurun_out/ev2/bench_c4.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev2/bench_reference.json 2> gpurun_out/ev2/bench_reference.err; echo "ref rc=$?"
python bench.py --steps 2 --warmup 1 --quick > gpurun_out/ev2/quick_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/ev2/launches.csv \
    python bench.py --steps 2 --warmup 1 --quick > gpurun_out/ev2/launches.log 2>&1; echo "launches rc=$?"
python bench.py --steps 1 --warmup 0 --quick > gpurun_out/ev2/traffic_plain.json 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --kernel-name-base demangled \
    -k regex:k_kron --csv python bench.py --steps 1 --warmup 0 --quick > gpurun_out/ev2/traffic_ncu.csv 2> gpurun_out/ev2/traffic.err; echo "traffic rc=$?"
bash tools/ncu_capture.sh ev2/k3c_cheby_p2 k_kron3c 2 1 python tools/prof_driver.py 2 cheby 2
bash tools/ncu_capture.sh ev2/k3c_apply_p2 k_kron3c 1 1 python tools/prof_driver.py 2 apply 2
bash tools/ncu_capture.sh ev2/cheby_p5 k_kron4 2 1 python tools/prof_driver.py 5 cheby 2
for n in k3c_cheby_p2 k3c_apply_p2 cheby_p5; do
  zcat gpurun_out/ev2/${n}_src.csv.gz > /tmp/${n}_src.csv
  python tools/ncu_segments.py /tmp/${n}_src.csv > gpurun_out/ev2/${n}_segments.txt 2>&1
  p=$(echo $n | sed 's/.*_p//'); nd=$(python -c "from synthetic import c4_spec; print(c4_spec($p).n_dofs)")
  python tools/ncu_sass_mix.py /tmp/${n}_src.csv $nd > gpurun_out/ev2/${n}_mix.txt 2>&1
done
ls -la gpurun_out/ev2
