timeout 900 python bench.py > gpurun_out/bench_c4_full3.json 2> gpurun_out/bench_c4_full3.err
echo "c4 rc=$?"
for w in c3 c5; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload $w > gpurun_out/bench_${w}_full3.json 2> gpurun_out/bench_${w}_full3.err
echo "$w rc=$?"
done
