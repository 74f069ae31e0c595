timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_full2.log 2>&1
echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/bench_c4_full2.json 2> gpurun_out/bench_c4_full2.err
echo "c4 rc=$?"
for w in c2 c3 c5; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload $w > gpurun_out/bench_${w}_full2.json 2> gpurun_out/bench_${w}_full2.err
echo "$w rc=$?"
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1
echo "smoke rc=$?"
