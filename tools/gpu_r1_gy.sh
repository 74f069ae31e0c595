timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_gy.log 2>&1
echo "pytest rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_gy.json 2> gpurun_out/bench_gy.err
echo done
