timeout 900 python -m pytest tests/test_gpu_quadrature.py -x -q > gpurun_out/pytest_q3a.log 2>&1
echo "pytest rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --workload c3 > gpurun_out/bench_q3a.json 2> gpurun_out/bench_q3a.err
echo "bench rc=$?"
