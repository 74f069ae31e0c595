set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
timeout 600 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo "c4 rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload c3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo "c3 rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"
